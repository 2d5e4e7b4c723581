#!/bin/bash
# ncu full sets: packed empty bottles level 4, streaming carpet level 4 (two CTAs, compacted gathers).  tools/gpu_prof_b.sh tag
tag=${1:-x}
python tools/profile_step.py --fractal empty-bottles --level 11 --packed --tile-level 4 --steps 2 > gpurun_out/pb4_plain_${tag}.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_step_packed -s 1 -c 1 -o gpurun_out/prof_packed_bottles4_${tag} \
    python tools/profile_step.py --fractal empty-bottles --level 11 --packed --tile-level 4 --steps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step_stream -s 1 -c 1 -o gpurun_out/prof_stream_carpet2_${tag} \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --steps 2 > /dev/null 2>&1
echo done

#!/bin/bash
# ncu full set of the streaming carpet step (default plan).  tools/gpu_prof_sc.sh tag
tag=${1:-x}
python tools/profile_step.py --fractal sierpinski-carpet --level 10 --steps 2 > gpurun_out/sc_plain_${tag}.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_step_stream -s 1 -c 1 -o gpurun_out/prof_stream_carpet_${tag} \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --steps 2 > /dev/null 2>&1
echo done

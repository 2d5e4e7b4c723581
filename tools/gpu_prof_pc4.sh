#!/bin/bash
# ncu of the packed carpet step at level 4 (compacted gathers).  tools/gpu_prof_pc4.sh tag
tag=${1:-x}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
python tools/profile_step.py --fractal sierpinski-carpet --level 10 --packed --tile-level 4 --steps 2 > gpurun_out/pc4_plain_${tag}.log 2>&1 || exit 1
ncu --metrics $M --clock-control none -k regex:k_step_packed -s 1 -c 1 --csv --log-file gpurun_out/traffic_packed_carpet4_${tag}.csv \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --packed --tile-level 4 --steps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step_packed -s 1 -c 1 -o gpurun_out/prof_packed_carpet4_${tag} \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --packed --tile-level 4 --steps 2 > /dev/null 2>&1
echo done

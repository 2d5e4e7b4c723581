#!/bin/bash
# ncu full set of the headline byte step (k_step_tile) at r=20, and its DRAM traffic at r=22.  tools/gpu_prof_tile.sh tag
tag=${1:-x}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
python tools/profile_step.py --level 20 --steps 2 > gpurun_out/tile_plain_${tag}.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_step_tile -s 1 -c 1 -o gpurun_out/prof_tile_r20_${tag} \
    python tools/profile_step.py --level 20 --steps 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step_tile -s 1 -c 1 --csv --log-file gpurun_out/traffic_tile_r22_${tag}.csv \
    python tools/profile_step.py --level 22 --steps 2 > /dev/null 2>&1
echo done

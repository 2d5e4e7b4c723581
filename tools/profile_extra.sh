#!/bin/bash
# Round profile evidence for the NEXT-row kernels (run under gpurun, 1 GPU).  Writes gpurun_out/.
# Numbers printed under ncu are never bench values.
set -x
tag=${1:-r1b}
# 1. every launch of a short full bench run (all legs) with its device time (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 3 --warmup 1 --no-e2e > gpurun_out/launches_${tag}.log 2>&1
# 2. DRAM bytes of one packed step at r=22 (g=7) and one heat step at r=21 (single-pass metrics)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_step_packed -s 2 -c 1 --csv --log-file gpurun_out/traffic_packed_${tag}.csv \
    python tools/profile_step.py --level 22 --packed --tile-level 7 --steps 3 > gpurun_out/traffic_packed_${tag}.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_heat_step -s 2 -c 1 --csv --log-file gpurun_out/traffic_heat_${tag}.csv \
    python tools/heat_timing.py sierpinski-triangle 21 > gpurun_out/traffic_heat_${tag}.log 2>&1
# 3. full section sets: heat r=20, LUT and MMA nu maps
ncu --set full --clock-control none --import-source on -k regex:k_heat_step -s 1 -c 1 -o gpurun_out/prof_heat_${tag} \
    python tools/heat_timing.py sierpinski-triangle 20 > gpurun_out/prof_heat_${tag}.log 2>&1
ncu --set full --clock-control none -k regex:k_map_nu -s 3 -c 2 -o gpurun_out/prof_map_${tag} \
    python tools/map_timing.py sierpinski-triangle 22 25 > gpurun_out/prof_map_${tag}.log 2>&1
echo done

#!/bin/bash
# Round-2 profile evidence (run under gpurun, 1 GPU).  Writes gpurun_out/.  Numbers printed under ncu
# are never bench values.
set -x
tag=${1:-r2}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
# 1. every launch of a short bench run with every leg (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 3 --warmup 3 --no-e2e --reps 1 --bb-runs 1 \
    > gpurun_out/launches_${tag}.log 2>&1
# 2. DRAM bytes per launch: byte step r=22 (bench), streaming step (configs[3]), BB r=16, packed r=22
ncu --metrics $M --clock-control none -k regex:k_step_tile -s 1 -c 1 --csv --log-file gpurun_out/traffic_tile_r22_${tag}.csv \
    python tools/profile_step.py --level 22 --steps 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step_stream -s 1 -c 1 --csv --log-file gpurun_out/traffic_stream_carpet_${tag}.csv \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --steps 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step_stream -s 1 -c 1 --csv --log-file gpurun_out/traffic_stream_bottles_${tag}.csv \
    python tools/profile_step.py --fractal empty-bottles --level 11 --steps 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_bb_step_bits -s 1 -c 1 --csv --log-file gpurun_out/traffic_bb16_${tag}.csv \
    python tools/profile_step.py --level 16 --bb --steps 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step_packed -s 1 -c 1 --csv --log-file gpurun_out/traffic_packed_r22_${tag}.csv \
    python tools/profile_step.py --level 22 --packed --tile-level 7 --steps 2 > /dev/null 2>&1
# 3. full section sets
ncu --set full --clock-control none --import-source on -k regex:k_step_stream -s 1 -c 1 -o gpurun_out/prof_stream_carpet_${tag} \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --steps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step_stream -s 1 -c 1 -o gpurun_out/prof_stream_bottles_${tag} \
    python tools/profile_step.py --fractal empty-bottles --level 11 --steps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bb_step_bits -s 1 -c 1 -o gpurun_out/prof_bb16_${tag} \
    python tools/profile_step.py --level 16 --bb --steps 2 > /dev/null 2>&1
echo done

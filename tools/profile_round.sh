#!/bin/bash
# Round profile evidence (run under gpurun, 1 GPU).  Writes gpurun_out/{launches,traffic}_*.csv and a
# full ncu report of the tile kernel at r=20.  Numbers printed under ncu are never bench values.
set -x
tag=${1:-r1}
# 1. every launch of a short bench run with its device time (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/launches_${tag}.log 2>&1
# 2. DRAM bytes of one tile-kernel launch at the bench workload (r=22; single-pass metrics, no replay)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_step_tile -s 1 -c 1 --csv --log-file gpurun_out/traffic_${tag}.csv \
    python bench.py --steps 2 --warmup 1 --no-extras > gpurun_out/traffic_${tag}.log 2>&1
# 3. full section set of the tile kernel at r=20 (3.5 GB buffers, replayable)
ncu --set full --clock-control none --import-source on -k regex:k_step_tile -s 1 -c 1 \
    -o gpurun_out/prof_${tag}_r20 python tools/profile_step.py --level 20 > gpurun_out/prof_${tag}.log 2>&1
# 4. BB baseline and literal per-cell kernels at r=16 for comparison
ncu --set full --clock-control none -k regex:k_bb_step16 -s 1 -c 1 -o gpurun_out/prof_${tag}_bb16 \
    python tools/profile_step.py --level 16 --bb > gpurun_out/prof_${tag}_bb.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:k_step_naive -s 1 -c 1 --csv --log-file gpurun_out/naive_${tag}.csv \
    python tools/profile_step.py --level 18 --naive --steps 2 > gpurun_out/naive_${tag}.log 2>&1
echo done

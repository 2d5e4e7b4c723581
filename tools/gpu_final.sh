#!/bin/bash
# Round-end evidence (1 GPU): every GPU test, smoke, the bench line, the ncu launch list of a short
# bench run, DRAM traffic of the changed kernels.  tools/gpu_final.sh tag
tag=${1:-x}
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_${tag}.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo "bench rc=$?"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
ncu --metrics $M --clock-control none -k regex:k_step_packed -s 1 -c 1 --csv --log-file gpurun_out/traffic_packed_carpet4_${tag}.csv \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --packed --tile-level 4 --steps 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step_stream -s 1 -c 1 --csv --log-file gpurun_out/traffic_stream_carpet_${tag}.csv \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --steps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --reps 1 --bb-runs 1 > gpurun_out/launches_${tag}.log 2>&1
echo done

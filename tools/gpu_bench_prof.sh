#!/bin/bash
# bench line + ncu evidence for the round-2 kernels (1 GPU).  tools/gpu_bench_prof.sh tag
tag=${1:-x}
timeout 1200 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo "bench rc=$?"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
ncu --metrics $M --clock-control none -k regex:k_step_packed -s 1 -c 1 --csv --log-file gpurun_out/traffic_packed_r22_${tag}.csv \
    python tools/profile_step.py --level 22 --packed --tile-level 7 --steps 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step_stream -s 1 -c 1 --csv --log-file gpurun_out/traffic_stream_carpet_${tag}.csv \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --steps 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step_stream -s 1 -c 1 --csv --log-file gpurun_out/traffic_stream_bottles_${tag}.csv \
    python tools/profile_step.py --fractal empty-bottles --level 11 --steps 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step_packed -s 1 -c 1 --csv --log-file gpurun_out/traffic_packed_carpet_${tag}.csv \
    python tools/profile_step.py --fractal sierpinski-carpet --level 10 --packed --tile-level 3 --steps 2 > /dev/null 2>&1
for k in "packed22 k_step_packed --level 22 --packed --tile-level 7" "stream_carpet k_step_stream --fractal sierpinski-carpet --level 10" \
         "stream_bottles k_step_stream --fractal empty-bottles --level 11" "packed_carpet k_step_packed --fractal sierpinski-carpet --level 10 --packed --tile-level 3"; do
  set -- $k; name=$1; kern=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$kern -s 1 -c 1 -o gpurun_out/prof_${name}_${tag} \
      python tools/profile_step.py "$@" --steps 2 > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --reps 1 --bb-runs 1 > gpurun_out/launches_${tag}.log 2>&1
echo done

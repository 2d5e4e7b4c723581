#!/bin/bash
# Full evidence run under gpurun (1 GPU): GPU tests, bench, compute-sanitizer.  tools/gpu_full.sh tag
tag=${1:-x}
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_${tag}.log 2>&1; echo "pytest rc=$?"
timeout 1200 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo "bench rc=$?"
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_${t}_${tag}.log 2>&1; echo "$t rc=$?"
done

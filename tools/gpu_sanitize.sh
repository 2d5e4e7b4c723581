#!/bin/bash
# compute-sanitizer on tools/sanitize_run.py (1 GPU): tools/gpu_sanitize.sh tag
tag=${1:-x}
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_${t}_${tag}.log 2>&1; echo "$t rc=$?"
done

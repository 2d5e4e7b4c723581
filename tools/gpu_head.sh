#!/bin/bash
# HEAD check under gpurun (1 GPU): GPU tests, default bench, ncu launch list.  tools/gpu_head.sh tag
tag=${1:-x}
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_${tag}.log 2>&1; echo "pytest rc=$?"
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo "bench rc=$?"

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r2b.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo "bench rc=$?"
timeout 1200 bash tools/profile_round2.sh r2b > gpurun_out/profile_r2b.log 2>&1; echo "prof rc=$?"

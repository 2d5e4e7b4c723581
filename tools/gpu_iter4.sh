#!/bin/bash
# packed link-heavy iteration: compacted-gather parity + timings.  tools/gpu_iter4.sh tag
tag=${1:-x}
out=gpurun_out/iter_${tag}.log
{
timeout 300 python tools/fractal_timing.py sierpinski-carpet 10 3,4 packed 2>&1 | tail -2
SQZ_PACKED_THREADS=256 timeout 300 python tools/fractal_timing.py sierpinski-carpet 10 4 packed 2>&1 | tail -1
timeout 300 python tools/fractal_timing.py full-square 12 5,6 packed 2>&1 | tail -2
timeout 300 python tools/fractal_timing.py empty-bottles 11 4 packed 2>&1 | tail -1
timeout 300 python tools/fractal_timing.py sierpinski-triangle 22 7 packed 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_packed.py -x -q -p no:cacheprovider -k "compacted or sharded_packed or config3" 2>&1 | tail -5
} > $out 2>&1

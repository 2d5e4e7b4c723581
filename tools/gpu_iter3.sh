#!/bin/bash
# packed-step iteration: parity + timings.  tools/gpu_iter3.sh tag
tag=${1:-x}
out=gpurun_out/iter_${tag}.log
{
timeout 900 python -m pytest tests/test_gpu_packed.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 300 python tools/fractal_timing.py sierpinski-triangle 22 7 packed 2>&1 | tail -1
timeout 300 python tools/fractal_timing.py sierpinski-carpet 10 3,4 packed 2>&1 | tail -2
timeout 300 python tools/fractal_timing.py empty-bottles 11 3,4 packed 2>&1 | tail -2
timeout 300 python tools/fractal_timing.py vicsek 12 0 packed 2>&1 | tail -1
} > $out 2>&1

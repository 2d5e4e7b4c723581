#!/bin/bash
# A/B (abtest/libA.so vs libB.so) on the packed carpet/full square (compacted gathers), then the packed tests.
tag=${1:-x}
bash tools/ab.sh ${tag}_carpet4 python tools/fractal_timing.py sierpinski-carpet 10 4 packed
bash tools/ab.sh ${tag}_square6 python tools/fractal_timing.py full-square 13 6 packed
timeout 1500 python -m pytest tests/test_gpu_packed.py -x -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/ab_${tag}_tests.log

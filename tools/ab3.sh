#!/bin/bash
# A/B of the packed step on link-heavy fractals + packed parity with B
tag=$1
bash tools/ab.sh ${tag}_pcarpet python tools/fractal_timing.py sierpinski-carpet 10 3 packed
bash tools/ab.sh ${tag}_pbottles python tools/fractal_timing.py empty-bottles 11 4 packed
bash tools/ab.sh ${tag}_psier python tools/fractal_timing.py sierpinski-triangle 22 7 packed
SQZ_LIB=abtest/libB.so timeout 1200 python -m pytest tests/test_gpu_packed.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/ab_${tag}_tests.log

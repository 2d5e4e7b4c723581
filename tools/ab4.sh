#!/bin/bash
# A/B on the link-heavy configs (bytes + packed) + stream/packed parity with B
tag=$1
bash tools/ab.sh ${tag}_carpet python tools/fractal_timing.py sierpinski-carpet 10 0 bytes
bash tools/ab.sh ${tag}_pcarpet python tools/fractal_timing.py sierpinski-carpet 10 3 packed
bash tools/ab.sh ${tag}_pbottles python tools/fractal_timing.py empty-bottles 11 4 packed
SQZ_LIB=abtest/libB.so timeout 1200 python -m pytest tests/test_gpu_packed.py tests/test_gpu_stream.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/ab_${tag}_tests.log

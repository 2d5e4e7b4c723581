#!/bin/bash
# A/B of abtest/libA.so vs abtest/libB.so on the configs[3] byte steps + stream parity with B
tag=$1
bash tools/ab.sh ${tag}_carpet python tools/fractal_timing.py sierpinski-carpet 10 0 bytes
bash tools/ab.sh ${tag}_bottles python tools/fractal_timing.py empty-bottles 11 0 bytes
SQZ_LIB=abtest/libB.so timeout 900 python -m pytest tests/test_gpu_stream.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/ab_${tag}_tests.log

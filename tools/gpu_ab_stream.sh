#!/bin/bash
# A/B of two builds (abtest/libA.so, abtest/libB.so) on the streaming step.  tools/gpu_ab_stream.sh tag
tag=${1:-x}
bash tools/ab.sh ${tag}_carpet python tools/fractal_timing.py sierpinski-carpet 10 0 bytes
bash tools/ab.sh ${tag}_bottles python tools/fractal_timing.py empty-bottles 11 0 bytes
bash tools/ab.sh ${tag}_square python tools/fractal_timing.py full-square 13 6 bytes
bash tools/ab.sh ${tag}_vicsek python tools/fractal_timing.py vicsek 13 0 bytes
timeout 1500 python -m pytest tests/test_gpu_stream.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/ab_${tag}_tests.log
SQZ_STREAM_COMPACT=0 bash tools/ab.sh ${tag}_carpet1cta python tools/fractal_timing.py sierpinski-carpet 10 0 bytes

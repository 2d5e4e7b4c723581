#!/bin/bash
# A/B of two builds on the streaming step, then the streaming and packed tests.  tools/gpu_ab_stream2.sh tag
tag=${1:-x}
bash tools/ab.sh ${tag}_carpet python tools/fractal_timing.py sierpinski-carpet 10 0 bytes
bash tools/ab.sh ${tag}_bottles python tools/fractal_timing.py empty-bottles 11 0 bytes
bash tools/ab.sh ${tag}_vicsek python tools/fractal_timing.py vicsek 13 0 bytes
bash tools/ab.sh ${tag}_sier8 python tools/fractal_timing.py sierpinski-triangle 20 8 bytes
timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_packed.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/ab_${tag}_tests.log

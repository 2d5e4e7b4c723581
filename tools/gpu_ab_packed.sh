#!/bin/bash
# A/B of two builds (abtest/libA.so, abtest/libB.so) on the packed link-item fractals.  tools/gpu_ab_packed.sh tag
tag=${1:-x}
bash tools/ab.sh ${tag}_carpet4 python tools/fractal_timing.py sierpinski-carpet 10 4 packed
bash tools/ab.sh ${tag}_carpet3 python tools/fractal_timing.py sierpinski-carpet 10 3 packed
bash tools/ab.sh ${tag}_bottles4 python tools/fractal_timing.py empty-bottles 11 4 packed
bash tools/ab.sh ${tag}_vicsek5 python tools/fractal_timing.py vicsek 13 5 packed
timeout 1500 python -m pytest tests/test_gpu_packed.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/ab_${tag}_tests.log

#!/bin/bash
# A/B/C of three builds on the packed link-item fractals, then the packed tests.  tools/gpu_abc_packed.sh tag
tag=${1:-x}
bash tools/abc.sh ${tag}_carpet4 python tools/fractal_timing.py sierpinski-carpet 10 4 packed
bash tools/abc.sh ${tag}_bottles4 python tools/fractal_timing.py empty-bottles 11 4 packed
bash tools/abc.sh ${tag}_vicsek5 python tools/fractal_timing.py vicsek 13 5 packed
timeout 1500 python -m pytest tests/test_gpu_packed.py -x -q -p no:cacheprovider 2>&1 | tail -2 > gpurun_out/ab_${tag}_tests.log

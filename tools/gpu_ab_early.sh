#!/bin/bash
# A/B: streaming step with the compacted, parity-split gathers issued before the links barrier
# (libB) against the [32][E] buffer (libA); then the streaming tests.  tools/gpu_ab_early.sh tag
tag=${1:-x}
bash tools/ab.sh ${tag}_carpet python tools/fractal_timing.py sierpinski-carpet 10 0 bytes
bash tools/ab.sh ${tag}_square python tools/fractal_timing.py full-square 13 6 bytes
bash tools/ab.sh ${tag}_bottles python tools/fractal_timing.py empty-bottles 11 0 bytes
timeout 1500 python -m pytest tests/test_gpu_stream.py -x -q -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/ab_${tag}_tests.log

#!/bin/bash
# A/B: the packed step with compacted gathers + dynamic link items forced on every link-item context
# (libB with SQZ_PACKED_COMPACT=1) against the default (libA).  tools/gpu_ab_compact.sh tag
tag=${1:-x}
export SQZ_PACKED_COMPACT=1
bash tools/ab.sh ${tag}_bottles4 python tools/fractal_timing.py empty-bottles 11 4 packed
bash tools/ab.sh ${tag}_carpet3 python tools/fractal_timing.py sierpinski-carpet 10 3 packed
bash tools/ab.sh ${tag}_vicsek5 python tools/fractal_timing.py vicsek 13 5 packed
bash tools/ab.sh ${tag}_carpet4 python tools/fractal_timing.py sierpinski-carpet 10 4 packed
timeout 1500 python -m pytest tests/test_gpu_packed.py -x -q -p no:cacheprovider -k "step_vs_oracle or rules or sharded or config3" 2>&1 | tail -3 > gpurun_out/ab_${tag}_tests.log

#!/bin/bash
# packed step A/B: link-free blocks before the chunk barrier (SQZ_PACKED_EARLY=1, default) vs after (0),
# interleaved; then the packed tests.  tools/gpu_iter5.sh tag
tag=${1:-x}
out=gpurun_out/iter_${tag}.log
{
for rep in 1 2; do
for e in 0 1; do
  echo "EARLY=$e"
  SQZ_PACKED_EARLY=$e timeout 300 python tools/fractal_timing.py sierpinski-carpet 10 3,4 packed 2>&1 | tail -2
  SQZ_PACKED_EARLY=$e timeout 300 python tools/fractal_timing.py empty-bottles 11 3,4 packed 2>&1 | tail -2
  SQZ_PACKED_EARLY=$e timeout 300 python tools/fractal_timing.py vicsek 13 5 packed 2>&1 | tail -1
done
done
timeout 300 python tools/fractal_timing.py sierpinski-triangle 22 7 packed 2>&1 | tail -1
timeout 2000 python -m pytest tests/test_gpu_packed.py -x -q -p no:cacheprovider 2>&1 | tail -3
} > $out 2>&1

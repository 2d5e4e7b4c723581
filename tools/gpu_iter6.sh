#!/bin/bash
# streaming step A/B: compacted gathers at two CTAs per SM (default) vs [32][E] at one (SQZ_STREAM_COMPACT=0),
# interleaved; then the streaming-step tests.  tools/gpu_iter6.sh tag
tag=${1:-x}
out=gpurun_out/iter_${tag}.log
{
for rep in 1 2; do
for e in 0 1; do
  echo "COMPACT=$e"
  SQZ_STREAM_COMPACT=$e timeout 300 python tools/fractal_timing.py sierpinski-carpet 10 0 bytes 2>&1 | tail -1
  SQZ_STREAM_COMPACT=$e timeout 300 python tools/fractal_timing.py full-square 13 6 bytes 2>&1 | tail -1
done
done
timeout 300 python tools/fractal_timing.py empty-bottles 11 0 bytes 2>&1 | tail -1
SQZ_DEBUG=1 timeout 300 python tools/fractal_timing.py sierpinski-carpet 10 0 bytes 2>&1 | grep "sqz:" | head -2
timeout 2000 python -m pytest tests/test_gpu_stream.py -x -q -p no:cacheprovider 2>&1 | tail -3
} > $out 2>&1

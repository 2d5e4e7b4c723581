#!/bin/bash
# Iteration run under gpurun (1 GPU): stream/packed parity + timings.  Writes gpurun_out/iter_$1.log
tag=${1:-x}
out=gpurun_out/iter_${tag}.log
{
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_random_fractals.py -x -q -p no:cacheprovider 2>&1 | tail -15
for fr in "sierpinski-carpet 10" "empty-bottles 11"; do
  timeout 300 python tools/fractal_timing.py $fr 0 bytes 2>&1 | tail -3
  SQZ_STREAM_CTAS=1 timeout 300 python tools/fractal_timing.py $fr 0 bytes 2>&1 | tail -3
done
timeout 300 python tools/packed_timing.py sierpinski-triangle 22 7 2>&1 | tail -2
SQZ_PACKED_THREADS=384 timeout 300 python tools/packed_timing.py sierpinski-triangle 22 7 2>&1 | tail -2
} > $out 2>&1
echo done

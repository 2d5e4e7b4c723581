#!/bin/bash
tag=${1:-x}
out=gpurun_out/iter_${tag}.log
{
for v in "" "SQZ_STREAM_RB1=1"; do
  env $v timeout 300 python tools/fractal_timing.py empty-bottles 11 0 bytes 2>&1 | tail -1 | sed "s/^/[$v] /"
  env $v timeout 300 python tools/fractal_timing.py vicsek 12 0 bytes 2>&1 | tail -1 | sed "s/^/[$v] /"
done
} > $out 2>&1

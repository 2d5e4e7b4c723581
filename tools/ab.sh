#!/bin/bash
# A/B timing of two library builds (abtest/libA.so, abtest/libB.so), interleaved: tools/ab.sh tag cmd...
tag=$1; shift
out=gpurun_out/ab_${tag}.log
: > $out
for rep in 1 2 3; do
  for v in A B; do
    SQZ_LIB=abtest/lib$v.so timeout 300 "$@" 2>&1 | tail -1 | sed "s/^/[$v] /" >> $out
  done
done

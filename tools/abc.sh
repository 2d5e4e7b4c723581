#!/bin/bash
# A/B/C timing of three library builds (abtest/lib{A,B,C}.so), interleaved: tools/abc.sh tag cmd...
tag=$1; shift
out=gpurun_out/ab_${tag}.log
: > $out
for rep in 1 2 3; do
  for v in A B C; do
    SQZ_LIB=abtest/lib$v.so timeout 300 "$@" 2>&1 | tail -1 | sed "s/^/[$v] /" >> $out
  done
done

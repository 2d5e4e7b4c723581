#!/bin/bash
# one ncu --set full capture of a step kernel: tools/gpu_prof1.sh tag kernel-regex profile_step-args...
tag=$1; kern=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$kern -s 1 -c 1 -o gpurun_out/prof_${tag} \
    python tools/profile_step.py "$@" > gpurun_out/prof_${tag}.log 2>&1
echo done

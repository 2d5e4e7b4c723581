mkdir -p gpurun_out; rm -f gpurun_out/pk_time.log
timeout 600 python -m pytest tests/test_gpu_packed.py -x -q > gpurun_out/pk_test.log 2>&1; echo test=$? >> gpurun_out/pk_test.log
for g in 6 7; do timeout 120 python tools/packed_timing.py sierpinski-triangle 20,22 $g 2>&1 >> gpurun_out/pk_time.log; done
ncu --set full --clock-control none --import-source on -k regex:k_step_packed -s 1 -c 1 -o gpurun_out/prof_pk10 python tools/profile_step.py --level 20 --packed --tile-level 7 > gpurun_out/prof_pk10.log 2>&1

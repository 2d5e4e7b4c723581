mkdir -p gpurun_out; rm -f gpurun_out/heat_time.log
timeout 900 python -m pytest tests/test_gpu_heat.py -x -q > gpurun_out/heat_test.log 2>&1; echo test=$? >> gpurun_out/heat_test.log
for g in 6 7; do timeout 200 python tools/heat_timing.py sierpinski-triangle 20,21 $g >> gpurun_out/heat_time.log 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:k_heat_step -s 1 -c 1 -o gpurun_out/prof_heat2 python tools/heat_timing.py sierpinski-triangle 19 > gpurun_out/prof_heat2.log 2>&1

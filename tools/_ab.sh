mkdir -p gpurun_out
: > gpurun_out/heat_ab.txt
for rep in 1 2 3; do
SQZ_LIB=abtest/base.so timeout 300 python tools/heat_timing.py sierpinski-triangle 20,21 2>&1 | sed 's/^/base /' >> gpurun_out/heat_ab.txt
timeout 300 python tools/heat_timing.py sierpinski-triangle 20,21 2>&1 | sed 's/^/new  /' >> gpurun_out/heat_ab.txt
SQZ_LIB=abtest/base.so timeout 300 python tools/heat_timing.py vicsek 12 2>&1 | sed 's/^/base /' >> gpurun_out/heat_ab.txt
timeout 300 python tools/heat_timing.py vicsek 12 2>&1 | sed 's/^/new  /' >> gpurun_out/heat_ab.txt
done

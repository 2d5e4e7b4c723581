mkdir -p gpurun_out
for h in peer collective; do
SQZ_DIST_BACKEND=gloo SQZ_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --halo $h --steps 5 --warmup 3 > gpurun_out/bench_n2_$h.json 2> gpurun_out/bench_n2_$h.err; echo $h rc=$?
done

set -u
O=gpurun_out
T=${TAG:-r2g}
MCMP2_BENCH_TRACE=1 MCMP2_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 8 --warmup 3 --strong-total-steps 400 --ttt cfg5-10 --no-cpu-baseline > $O/${T}_bench_2rank.json 2> $O/${T}_bench_2rank.err

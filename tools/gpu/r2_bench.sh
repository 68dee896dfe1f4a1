set -u
O=gpurun_out
T=${TAG:-r2f}
timeout 900 python bench.py > $O/${T}_bench_cfg4.json 2> $O/${T}_bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err
MCMP2_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 8 --warmup 3 --strong-total-steps 400 --ttt cfg5-10 --no-cpu-baseline > $O/${T}_bench_2rank.json 2> $O/${T}_bench_2rank.err

# The torchrun entry points on a 1-GPU box (run under gpurun from the repo root):
#  * bench.py as 2 ranks over gloo sharing the GPU (the N > 1 code path: strong split, max over
#    ranks, interval merge) -- not a scaling number;
#  * `python -m paper_2203_05632_b200.distributed CONFIG` / `resume CHECKPOINT` over NCCL with one
#    rank, against `mcmp2 run` on the same config (reports and checkpoint files must be identical).
set -u
O=gpurun_out
T=${TAG:-r2x}
MCMP2_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline \
  --strong-total-steps 400 --ttt "" > $O/${T}_bench_2rank_gloo_1gpu.json 2> $O/${T}_bench_2rank_gloo_1gpu.err
D=$(mktemp -d)
paper_2203_05632_b200/lib/mcmp2 generate cfg2 --output $D > /dev/null
grep -v "^steps\|^workers\|^checkpoint\|^trace" $D/cfg2.conf > $D/base.conf
printf "steps 600\nworkers 3\ncheckpoint-interval 100\ncheckpoint $D/a.ck\ntrace $D/a.trace\n" | cat $D/base.conf - > $D/a.conf
printf "steps 600\nworkers 3\ncheckpoint-interval 100\ncheckpoint $D/b.ck\ntrace $D/b.trace\n" | cat $D/base.conf - > $D/b.conf
paper_2203_05632_b200/lib/mcmp2 run --config $D/a.conf > $D/a.report 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 \
  -m paper_2203_05632_b200.distributed $D/b.conf > $D/b.report 2> $D/b.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 \
  -m paper_2203_05632_b200.distributed resume $D/b.ck > $D/b2.report 2> $D/b2.err
{
  echo "== mcmp2 run"; cat $D/a.report
  echo "== torchrun distributed"; cat $D/b.report
  echo "== torchrun distributed resume (of the finished run)"; cat $D/b2.report
  # (NCCL prints its version line on stdout)
  echo "== reports equal: $(grep -v "^NCCL version" $D/b.report | cmp -s $D/a.report - && echo yes || echo NO); resume report equal: $(grep -v "^NCCL version" $D/b2.report | cmp -s $D/a.report - && echo yes || echo NO)"
  echo "== checkpoints equal but for the path lines: $(diff <(grep -v "^checkpoint \|^trace " $D/a.ck) <(grep -v "^checkpoint \|^trace " $D/b.ck) > /dev/null && echo yes || echo NO)"
  echo "== traces equal: $(cmp -s $D/a.trace $D/b.trace && echo yes || echo NO)"
  tail -n 3 $D/b.err; tail -n 3 $D/b2.err
} > $O/${T}_dist_cli.log 2>&1
tail -30 $O/${T}_dist_cli.log; tail -c 600 $O/${T}_bench_2rank_gloo_1gpu.json; tail -5 $O/${T}_bench_2rank_gloo_1gpu.err

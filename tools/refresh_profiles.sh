#!/usr/bin/env bash
# Re-measures everything profiles/ is built from, on the GPU box (run under gpurun):
#   bench lines cfg1..cfg4, the ncu launch list of a short cfg4 bench run, and one
#   `ncu --set full` capture of each kernel at cfg4 (tools/ncu_summary.py TAG reads them back).
# usage: gpurun --timeout 1800 -- 'bash tools/refresh_profiles.sh r01k'
set -u
TAG=${1:-r03}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/${TAG}_smi.txt 2>&1
python bench.py > $OUT/${TAG}_bench_cfg4.json 2> $OUT/${TAG}_bench_cfg4.err
for c in cfg1 cfg2 cfg3; do
  python bench.py --config $c --steps 200 --no-cpu-baseline > $OUT/${TAG}_bench_$c.json 2> $OUT/${TAG}_bench_$c.err
done
# several reference workers per GPU as one batched handle
python bench.py --config cfg1 --ensembles 1184 --steps 200 --no-cpu-baseline > $OUT/${TAG}_bench_cfg1_batched.json 2> $OUT/${TAG}_bench_cfg1_batched.err
python bench.py --config cfg2 --ensembles 16 --steps 200 --no-cpu-baseline > $OUT/${TAG}_bench_cfg2_batched.json 2> $OUT/${TAG}_bench_cfg2_batched.err
python tools/batch_scan.py cfg1 --nens 1,16,64,148,296,592,1184 --out $OUT/${TAG}_batch_cfg1.json > /dev/null 2>&1
python tools/batch_scan.py cfg2 --nens 1,4,8,16,32 --out $OUT/${TAG}_batch_cfg2.json > /dev/null 2>&1
# launch list of the bench command itself (cold-cache, serialised per-launch times)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches_cfg4.csv \
  python bench.py --steps 3 --warmup 3 --burnin 20 --no-cpu-baseline > $OUT/${TAG}_ncu_launches.log 2>&1
# one steady-state launch of each kernel, full set
for k in oz_vgemm_kernel pair_kr_kernel oz_slice_kernel mo_kernel chi_kernel walk_kernel; do
  skip=1
  [ $k = walk_kernel ] && skip=22   # past init + 20 burn-in sweeps: a production sweep
  ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -f \
    -o $OUT/prof_${TAG}_$k python tools/prof_step.py cfg4 3 20 > $OUT/${TAG}_ncu_$k.log 2>&1
done
ls -la $OUT | tail -20

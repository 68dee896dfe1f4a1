set -u
O=gpurun_out
timeout 300 python bench.py > $O/r2_bench_cfg4.json 2> $O/r2_bench_cfg4.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches_cfg4.csv \
  python bench.py --steps 3 --warmup 3 --burnin 20 --no-cpu-baseline > $O/r2_ncu_launches.log 2>&1
for k in oz_vgemm_kernel pair_kr_kernel oz_slice_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f \
    -o $O/prof_r2_$k python tools/prof_step.py cfg4 3 20 > $O/r2_ncu_$k.log 2>&1
done
ls -la $O | tail

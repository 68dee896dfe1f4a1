# One GPU validation pass (run with gpurun from the repo root): the GPU suite, smoke, the bench
# lines (cfg4 with strong_run and time_to_target, cfg3, the reference arm), the full-length guard
# chain and guard cost at cfg4, the cfg5 sweep, the
# kernel launch list, the k-step truncation scan and ncu captures of the V-GEMM, the slice kernel, the O pass
# and the MO transform, all into gpurun_out/.
#   gpurun --timeout 5400 -- 'TAG=r2x bash tools/gpu/validate.sh'
set -u
O=gpurun_out
T=${TAG:-r2x}
timeout 2400 python -m pytest tests -m gpu -q > $O/${T}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1
timeout 900 python bench.py > $O/${T}_bench_cfg4.json 2> $O/${T}_bench_cfg4.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err
for c in cfg3; do timeout 600 python bench.py --config $c --strong-total-steps 0 --ttt "" > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err; done
timeout 900 python tools/guard_chain.py cfg4 20000 2e-10 > $O/${T}_guard_chain_cfg4_20000.json 2> $O/${T}_guard_chain.err
timeout 600 python tools/guard_cost.py cfg4 256 2e-10 1e-10 > $O/${T}_guard_cost_cfg4.json 2>&1
timeout 1500 python tools/sweep_cfg5.py --max-seconds 60 --out $O/${T}_sweep_cfg5.json > $O/${T}_sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches_cfg4.csv \
  python bench.py --steps 4 --warmup 3 --burnin 100 --no-cpu-baseline --strong-total-steps 0 --ttt "" > $O/${T}_ncu_launches.log 2>&1
timeout 300 python tools/trunc_scan.py cfg4 2048 > $O/${T}_trunc_scan_cfg4.json 2> $O/${T}_trunc_scan.err
for k in oz_vgemm_kernel oz_slice_kernel pair_kr_kernel mo_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -f \
    -o $O/prof_${T}_$k python tools/prof_step.py cfg4 6 20 > $O/${T}_ncu_$k.log 2>&1
done
ls -la $O | tail -5

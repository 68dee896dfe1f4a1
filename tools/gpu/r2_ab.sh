set -u
O=gpurun_out
T=${TAG:-r2n}
for v in lib; do
  MCMP2_LIBDIR=paper_2203_05632_b200/$v timeout 600 python tools/guard_cost.py cfg4 256 2e-10 1e-10 > $O/${T}_cost_$v.json 2> $O/${T}_cost_$v.err
done
timeout 900 python -m pytest tests/test_gpu_guard.py -x -q > $O/${T}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest.log

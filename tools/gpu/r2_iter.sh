set -u
O=gpurun_out
T=${TAG:-r2w}
timeout 900 python -m pytest tests/test_gpu_guard.py tests/test_gpu_oz.py -x -q > $O/${T}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest.log
timeout 600 python tools/guard_cost.py cfg4 256 2e-10 1e-10 1e-300 > $O/${T}_cost.json 2> $O/${T}_cost.err

set -u
O=gpurun_out
T=${TAG:-r2c}
timeout 1800 python -m pytest tests -m gpu -q > $O/${T}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest_gpu.log
timeout 300 python bench.py > $O/${T}_bench_cfg4.json 2> $O/${T}_bench_cfg4.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1

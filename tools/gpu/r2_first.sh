set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/r2a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r2a_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/r2a_pytest_gpu.log
timeout 300 python bench.py > $O/r2a_bench_cfg4.json 2> $O/r2a_bench_cfg4.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2a_smoke.log 2>&1

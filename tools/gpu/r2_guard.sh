set -u
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_guard.py tests/test_gpu_oz.py -q > $O/r2d_pytest_guard.log 2>&1; echo "pytest exit $?" >> $O/r2d_pytest_guard.log
timeout 300 python bench.py > $O/r2d_bench_cfg4.json 2> $O/r2d_bench_cfg4.err

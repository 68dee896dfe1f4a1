set -u
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_guard.py -q > $O/r2b_pytest_guard.log 2>&1; echo "pytest exit $?" >> $O/r2b_pytest_guard.log

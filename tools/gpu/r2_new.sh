set -u
O=gpurun_out
T=${TAG:-r2o}
timeout 900 python -m pytest tests/test_gpu_reference.py tests/test_gpu_kramers_tol.py -q > $O/${T}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest.log

set -u
O=gpurun_out
timeout 600 python tools/guard_cost.py cfg4 256 3e-10 1e-10 3e-11 > $O/r2e_guard_cost_cfg4.json 2> $O/r2e_guard_cost_cfg4.err

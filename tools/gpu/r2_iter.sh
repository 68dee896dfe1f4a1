set -u
O=gpurun_out
T=${TAG:-r2y}
MCMP2_GUARD_TOL=1e-300 timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz_vgemm_kernel -s 5 -c 1 -f -o $O/${T}_refine python tools/prof_step.py cfg4 6 20 > $O/${T}_ncu_refine.log 2>&1

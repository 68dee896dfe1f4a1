set -u
O=gpurun_out
T=${TAG:-r2h}
# main V-GEMM (steady-state launches), then the refinement pass (forced with a tiny tolerance)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz_vgemm_kernel -s 4 -c 2 -f \
  -o $O/${T}_vgemm python tools/prof_step.py cfg4 6 20 > $O/${T}_ncu_vgemm.log 2>&1
MCMP2_GUARD_TOL=1e-300 timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz_vgemm_kernel -s 5 -c 1 -f \
  -o $O/${T}_refine python tools/prof_step.py cfg4 6 20 > $O/${T}_ncu_refine.log 2>&1
ls -la $O | tail -5

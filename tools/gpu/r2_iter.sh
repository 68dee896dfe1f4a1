set -u
O=gpurun_out
T=${TAG:-r3a}
for v in lib lib_NC; do
  MCMP2_LIBDIR=paper_2203_05632_b200/$v timeout 600 python tools/guard_cost.py cfg4 128 1e-300 > $O/${T}_cost_$v.json 2> $O/${T}_cost_$v.err
done

# quick GPU pass: the INT8-path tests, smoke and one cfg4 bench line
#   gpurun --timeout 1500 -- 'TAG=q1 bash tools/gpu/quick.sh'
set -u
O=gpurun_out
T=${TAG:-q}
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -q ${PYTEST_ARGS:--x} -k "${PYTEST_K:-}" > $O/${T}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest.log
tail -${PYTEST_TAIL:-15} $O/${T}_pytest.log
[ -n "${NO_BENCH:-}" ] && exit 0
timeout 600 python bench.py ${BENCH_ARGS:-} > $O/${T}_bench_cfg4.json 2> $O/${T}_bench_cfg4.err
tail -3 $O/${T}_bench_cfg4.err
python - <<PY
import json
d=json.loads(open("$O/${T}_bench_cfg4.json").read().strip().splitlines()[-1])
print({k:d.get(k) for k in ("value","ms_per_step")}, d.get("e2e",{}).get("value"), d.get("roofline",{}).get("achieved"), d.get("guard"))
PY

"""A full-length production chain on the guarded INT8 path, the bare INT8 path and the DMMA path
from one post-burn-in state (the walk does not depend on the estimates, so the three see the same
walkers and tau): per-step errors against DMMA of the value and the direct/exchange sums, the
guard's decisions, and the condition-aware errors (|error| / (sum |terms| / C(m,2))).
usage: python tools/guard_chain.py [cfg4] [steps] [tol] > out.json"""
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
tol = float(sys.argv[3]) if len(sys.argv) > 3 else 2e-10
m = {"cfg3": 512, "cfg4": 2048}.get(cfg, 8192)
F = {n: i for i, n in enumerate(DeviceWalker.STEP_EX_FIELDS)}
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    dw = DeviceWalker(System(sp, conf.read_text()), max_walkers=m)
    dw.init_ensemble(m, seed=23)
    dw.burn_in(1000)
    st = dw.get_ensemble()
    runs = {}
    for label, int8, t in (("guarded", 1, tol), ("raw", 1, 1e300), ("dmma", 0, tol)):
        dw.set_ensemble(st)
        dw.int8_v(int8)
        dw.guard(t)
        runs[label] = dw.advance_ex(steps)
g, r, dm = runs["guarded"], runs["raw"], runs["dmma"]
npairs = 0.5 * m * (m - 1)
rel = lambda a, b: np.abs(a - b) / np.maximum(np.abs(b), 1e-300)  # noqa: E731
out = {"config": cfg, "m": m, "steps": steps, "guard_tol": tol,
       "refined": int((g[:, F["fallback"]] == 1).sum()), "dmma": int((g[:, F["fallback"]] == 2).sum())}
for k, lab in ((0, "value"), (2, "direct"), (4, "exchange")):
    eg, er = rel(g[:, k], dm[:, k]), rel(r[:, k], dm[:, k])
    absum = (r[:, F["abs_direct"]] + r[:, F["abs_exchange"]]) / npairs if k == 0 else r[:, F["abs_" + lab]]
    out[lab] = {"guarded_max_rel": float(eg.max()), "guarded_steps_over_1e-10": int((eg > 1e-10).sum()),
                "guarded_p99_rel": float(np.percentile(eg, 99)), "raw_max_rel": float(er.max()),
                "raw_steps_over_1e-10": int((er > 1e-10).sum()),
                "raw_max_condition_aware": float((np.abs(r[:, k] - dm[:, k]) / absum).max()),
                "guarded_max_condition_aware": float((np.abs(g[:, k] - dm[:, k]) / absum).max())}
for k, e in ((2, "est_err_direct"), (4, "est_err_exchange")):
    err = np.abs(r[:, k] - dm[:, k])
    ratio = r[:, F[e]] / np.maximum(err, 1e-300)
    out[e] = {"min_est_over_err": float(ratio.min()), "median_est_over_err": float(np.median(ratio)),
              "steps_err_above_est": int((err > r[:, F[e]]).sum())}
print(json.dumps(out, indent=1))

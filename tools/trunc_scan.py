"""Energy-ordered k-step truncation of the INT8 V-GEMM against tau: one ensemble state replayed at
a ladder of tau values (and at the chain's own tau draws), with the fraction of k-steps issued
and the V-GEMM / slice / O-pass times per launch, truncation on and off.
usage: python tools/trunc_scan.py [cfg4] [m]  -> JSON on stdout"""
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
reps = 5
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    dw = DeviceWalker(System(sp, conf.read_text()), max_walkers=m)
    dw.init_ensemble(m, seed=1, stream=0)
    dw.burn_in(200)
    dw.advance(2)
    w = dw.get_ensemble().walkers[:, :8][None]
    rows = []
    for tau in (1e-4, 1e-3, 0.01, 0.03, 0.1, 0.2, 0.4, 0.7, 1.0, 1.5, 2.5, 4.0):
        row = {"tau": tau}
        for mode in (1, 0):
            dw.int8_truncation(mode)
            dw.replay(w, np.array([tau]))
            dw.profile(True, True)
            e0, full = dw.int8_ksteps()
            for _ in range(reps):
                dw.replay(w, np.array([tau]))
            e1, _ = dw.int8_ksteps()
            p = dw.profile(False, False)["int8_v"]
            tag = "trunc" if mode else "full"
            row[tag] = {"ksteps_frac": (e1 - e0) / (reps * full), "vgemm_ms": p["vgemm_ms"] / p["steps"],
                        "slice_ms": p["slice_ms"] / p["steps"], "pair_kr_ms": p["pair_kr_ms"] / p["steps"]}
        rows.append(row)
    # the chain's own draws: tau ~ Exp(lambda), weights.cpp:103-111
    dw.int8_truncation(1)
    e0, full = dw.int8_ksteps()
    n = 512
    dw.advance(n)
    e1, _ = dw.int8_ksteps()
    print(json.dumps({"config": cfg, "m": m, "ladder": rows, "chain": {"steps": n, "ksteps_frac_mean": (e1 - e0) / (n * full)}}, indent=1))

"""Cost of the INT8 path's accuracy guard at one config: device ms/step (CUDA events on the
handle's stream, graph-replayed advance, L2 not flushed) for the guard off, estimate only
(tol 1e300: stats, f store and the two guarded launches that exit at once), a list of
tolerances, and the DMMA pair stage; plus the per-kernel split of one profiled pass.
usage: python tools/guard_cost.py [cfg4] [steps] [tol ...]"""
import json
import sys
import tempfile
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402

WALKERS = {"cfg3": 512, "cfg4": 2048}
WALKERS.update({f"cfg5-{n}": 8192 for n in (2, 10, 18, 36, 54, 86)})
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 256
tols = [float(x) for x in sys.argv[3:]] or [3e-10, 1e-10, 3e-11]
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    m = WALKERS[cfg]
    dw = DeviceWalker(System(sp, conf.read_text()), max_walkers=m)
    dw.init_ensemble(m, seed=1, stream=0)
    dw.burn_in(200)
    st = dw.get_ensemble()
    s = torch.cuda.ExternalStream(dw.stream_ptr)
    out = {"config": cfg, "m": m, "steps": steps}

    def timed(label, int8, tol):
        dw.set_ensemble(st)
        dw.int8_v(int8)
        dw.guard(tol)
        dw.advance(64, keep_on_device=True)  # warm-up and graph capture
        dw.set_ensemble(st)
        dw.guard_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dw.synchronize()
        e0.record(s)
        dw.advance(steps, keep_on_device=True)
        e1.record(s)
        e1.synchronize()
        out[label] = {"ms_per_step": e0.elapsed_time(e1) / steps, **dw.guard_stats()}

    timed("guard_off", 1, 0.0)
    timed("estimate_only", 1, 1e300)
    for t in tols:
        timed(f"tol_{t:.0e}", 1, t)
    timed("dmma", 0, 0.0)
    # per-kernel split (events around each launch): estimate-only and the default tolerance
    for label, tol in (("split_guard_off", 0.0), ("split_estimate_only", 1e300), ("split_default", tols[0])):
        dw.set_ensemble(st)
        dw.int8_v(1)
        dw.guard(tol)
        dw.profile(True, True)
        dw.advance(32)
        out[label] = dw.profile(False, True)
    print(json.dumps(out, indent=1, default=float))

"""Profiling driver: a few production steps of one config on cuda:0 (for ncu / sanitizer).
usage: python tools/prof_step.py [cfg4] [steps] [burnin]; MCMP2_GUARD_TOL sets the INT8 path's
guard tolerance (e.g. 1e-300 forces the refinement and DMMA launches)."""
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402

WALKERS = {"cfg1": 16, "cfg2": 128, "cfg3": 512, "cfg4": 2048}
WALKERS.update({f"cfg5-{n}": 8192 for n in (2, 10, 18, 36, 54, 86)})
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
burn = int(sys.argv[3]) if len(sys.argv) > 3 else 20
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    m = WALKERS[cfg]
    dw = DeviceWalker(System(sp, conf.read_text()), max_walkers=m)
    if os.environ.get("MCMP2_GUARD_TOL"):
        dw.guard(float(os.environ["MCMP2_GUARD_TOL"]))
    dw.init_ensemble(m, seed=1, stream=0)
    dw.burn_in(burn)
    v, im = dw.advance(steps)
    print(cfg, "values", v)

"""Pair-kernel device time per launch for one config (profiling pass), for kernel-variant
experiments: MCMP2_LIBDIR=<variant lib dir> python tools/pair_time.py cfg4 [general|physical]"""
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402

W = {"cfg1": 16, "cfg2": 128, "cfg3": 512, "cfg4": 2048}
W.update({f"cfg5-{n}": 8192 for n in (2, 10, 18, 36, 54, 86)})
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    dw = DeviceWalker(System(sp, conf.read_text()), max_walkers=W[cfg])
    dw.init_ensemble(W[cfg], seed=1)
    mode = sys.argv[2] if len(sys.argv) > 2 else ""
    if mode == "physical":
        dw = DeviceWalker(System(sp, conf.read_text() + "estimator physical\n"), max_walkers=W[cfg])
        dw.init_ensemble(W[cfg], seed=1)
    if mode:  # general kernel (Kramers path off), optionally with the physical epilogue
        dw.kramers(0)
    dw.burn_in(20)
    dw.advance(2, keep_on_device=True)
    dw.profile(True, True)
    dw.advance(6, keep_on_device=True)
    p = dw.profile(False, True)
    print(os.environ.get("MCMP2_LIBDIR", "lib"), cfg, mode, "pair ms", round(p["ms"]["pair"] / p["launches"]["pair"], 4),
          "spinor ms", round(p["ms"]["spinor"] / p["launches"]["spinor"], 4),
          "walk ms", round(p["ms"]["walk"] / max(p["launches"]["walk"], 1), 4))

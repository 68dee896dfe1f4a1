"""Profiling driver for the physical-estimator pair kernel: cfg4, Kramers path, a few steps.
usage: python tools/prof_phys.py [cfg4] [steps]"""
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    dw = DeviceWalker(System(sp, conf.read_text() + "estimator physical\n"), max_walkers=2048)
    dw.init_ensemble(2048, seed=1)
    dw.burn_in(20)
    print(dw.advance(steps)[0])

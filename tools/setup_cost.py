"""Setup phases of one worker at a config (the serial part of the strong-scaling job): SPINOR-TEXT
load, device handle creation, init_ensemble + burn-in, graph capture, first interval.
usage: python tools/setup_cost.py [cfg4] [burnin]"""
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
burn = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
m = {"cfg3": 512, "cfg4": 2048}.get(cfg, 8192)
out = {"config": cfg, "m": m, "burnin": burn}
with tempfile.TemporaryDirectory() as d:
    t = time.perf_counter()
    sp, conf = generate_config(cfg, d)
    out["generate_s"] = time.perf_counter() - t
    import torch
    torch.cuda.init()
    for rep in range(2):
        t0 = time.perf_counter()
        s = System(sp, conf.read_text())
        t1 = time.perf_counter()
        dw = DeviceWalker(s, max_walkers=m)
        t2 = time.perf_counter()
        dw.init_ensemble(m, seed=1)
        dw.burn_in(burn)
        dw.synchronize()
        t3 = time.perf_counter()
        dw.prepare()
        dw.synchronize()
        t4 = time.perf_counter()
        dw.advance(32)
        t5 = time.perf_counter()
        out[f"rep{rep}"] = {"system_load_s": t1 - t0, "create_s": t2 - t1, "init_burnin_s": t3 - t2,
                            "graph_capture_s": t4 - t3, "first_32_steps_s": t5 - t4}
        dw.close()
print(json.dumps(out, indent=1))

"""A/B of the slice kernel's overlap with the O pass (mcmp2dev_oz_overlap): ms per step of
advance() through the captured graphs, series vs overlapped, alternating.
usage: python tools/overlap_ab.py [cfg4] [m] [steps]"""
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 256
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    dw = DeviceWalker(System(sp, conf.read_text()), max_walkers=m)
    dw.init_ensemble(m, seed=1, stream=0)
    dw.burn_in(200)
    state = dw.get_ensemble()   # every timed run advances the same steps (same tau draws)
    out = {"config": cfg, "m": m, "steps": steps, "series_ms": [], "overlap_ms": []}
    for rep in range(3):
        for mode, key in ((0, "series_ms"), (1, "overlap_ms")):
            dw.int8_overlap(mode)
            dw.set_ensemble(state)
            dw.advance(64)
            dw.synchronize()
            t0 = time.perf_counter()
            dw.advance(steps)
            dw.synchronize()
            out[key].append((time.perf_counter() - t0) * 1e3 / steps)
    print(json.dumps(out))

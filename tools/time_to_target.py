"""Wall time to a relative statistical error target through the C++ host Engine (BASELINE
metric, second half): `mcmp2 run` semantics with target-rel-err (driver.cpp:401-412), the stop
rule checked every `interval` steps. usage: python tools/time_to_target.py cfg2 [0.01] [interval]"""
import json
import re
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import generate_config, walker  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
target = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
interval = int(sys.argv[3]) if len(sys.argv) > 3 else 200
with tempfile.TemporaryDirectory() as d:
    sp, conf = generate_config(cfg, d)
    text = re.sub(r"steps \d+\n", "", conf.read_text()) + f"target-rel-err {target}\ncheckpoint-interval {interval}\n"
    t0 = time.perf_counter()
    rep = walker.run_config_text(text)
    wall = time.perf_counter() - t0
    e = float(re.search(r"E2\s+=\s+(\S+)", rep).group(1))
    s = float(re.search(r"sigma_bar\s+=\s+(\S+)", rep).group(1))
    n = int(re.search(r"steps\s+=\s+(\d+)", rep).group(1))
    print(json.dumps({"config": cfg, "target_rel_err": target, "seconds": wall, "steps": n, "E2": e,
                      "sigma_bar": s, "rel_err": s / abs(e), "includes": "spinor load, device setup, burn-in"}))

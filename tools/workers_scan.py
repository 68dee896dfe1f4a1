"""Production throughput of W reference workers sharing one GPU (the run config's `workers`
key: one ensemble, one std::thread and one device handle/stream per worker, driver.cpp:423-438)
through the C++ host Engine. The rate is taken from two step budgets, so setup and burn-in
cancel: samples/s = C(m,2) (S2 - S1) / (t(S2) - t(S1)).

usage: python tools/workers_scan.py cfg1 [--workers 1,4,16,64] [--steps 2000,6000] [--out f.json]
"""
import argparse
import json
import re
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import generate_config, walker  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--workers", default="1,4,16,64")
    ap.add_argument("--steps", default="2000,6000", help="per-worker step budgets S1,S2")
    ap.add_argument("--burnin", type=int, default=100)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    s1, s2 = map(int, args.steps.split(","))
    rows = []
    with tempfile.TemporaryDirectory() as d:
        sp, conf = generate_config(args.config, d)
        base = re.sub(r"(steps|target-rel-err|checkpoint-interval|workers|burnin) \S+\n", "", conf.read_text())
        m = int(re.search(r"walkers (\d+)", base).group(1))
        for w in map(int, args.workers.split(",")):
            t = {}
            walker.run_config_text(base + f"workers {w}\nburnin {args.burnin}\nsteps {s1 * w}\n"
                                   f"checkpoint-interval {s1}\n")  # warm-up (context, graphs, caches)
            for s in (s1, s2):
                text = base + f"workers {w}\nburnin {args.burnin}\nsteps {s * w}\ncheckpoint-interval {s}\n"
                t0 = time.perf_counter()
                rep = walker.run_config_text(text)
                t[s] = time.perf_counter() - t0
            rate = m * (m - 1) // 2 * (s2 - s1) * w / (t[s2] - t[s1])
            e2 = float(re.search(r"E2\s+=\s+(\S+)", rep).group(1))
            row = {"config": args.config, "walkers": m, "workers": w, "steps_per_worker": [s1, s2],
                   "seconds": [t[s1], t[s2]], "samples_per_s": rate, "E2_last": e2}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()

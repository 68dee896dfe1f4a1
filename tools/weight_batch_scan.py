"""Tail diagnostics of the sampling weight g with many independent ensembles (batched handle):
for each candidate `weight` line, R repeats of (nens ensembles x steps) give R merged estimates
E2 +- sigma_bar (ensemble means, independent by construction); consistent candidates agree
across repeats within a few sigma_bar, heavy-tailed ones do not. The largest per-ensemble
|mean - median| in units of the median absolute deviation shows the outliers directly.

Candidates 'f2 a k': z1 = a x (smallest basis exponent), z2 = k x z1, mass fractions 1-f2, f2
(c_k = f_k z_k^{3/4}).  usage: python tools/weight_batch_scan.py cfg1 --m 16 --nens 512 --steps 1000
"""
import argparse
import json
import re
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--nens", type=int, default=512)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--grid", default="0.25 2 10;0.1 2 30;0.25 1 10;0.1 1 100;0.05 2 300")
    ap.add_argument("--physical", action="store_true", help="opt-in physical estimator")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    rows = []
    with tempfile.TemporaryDirectory() as d:
        sp, conf = generate_config(args.config, d)
        text = conf.read_text() + ("estimator physical\n" if args.physical else "")
        el, cur = re.search(r"weight (\S+) (.*)\n", text).groups()
        zmin = min(float(z) for z in re.findall(r"; 1 ; (\S+) 1", sp.read_text()))
        cands = [("current", cur)]
        for g in args.grid.split(";"):
            f2, a, k = map(float, g.split())
            z1, z2 = a * zmin, k * a * zmin
            cands.append((g, f"{(1 - f2) * z1 ** 0.75:.6g} {z1:.6g} {f2 * z2 ** 0.75:.6g} {z2:.6g}"))
        for name, wl in cands:
            t = re.sub(r"weight .*\n", f"weight {el} {wl}\n", text)
            dw = DeviceWalker(System(sp, t), max_walkers=args.nens * args.m)
            reps = []
            for r in range(args.repeats):
                dw.init_batch(args.nens, args.m, seed=100 + r, stream0=0)
                if "step-size" in t:
                    dw.set_sigma_step(0.3)
                    dw.burn_in(500, adapt=False)
                else:
                    dw.burn_in(500, adapt=True)
                v, _ = dw.advance(args.steps)          # [steps][nens]
                means = v.mean(axis=0)
                e2 = float(means.mean())
                sb = float(means.std(ddof=1) / np.sqrt(len(means)))
                med = np.median(means)
                mad = float(np.median(np.abs(means - med))) or 1e-300
                reps.append({"E2": e2, "sigma_bar": sb, "max_dev_over_mad": float(np.max(np.abs(means - med)) / mad)})
            dw.close()
            e = np.array([x["E2"] for x in reps])
            s = np.array([x["sigma_bar"] for x in reps])
            spread = float(np.max(np.abs(e - e.mean())) / np.sqrt(np.mean(s ** 2)))
            row = {"config": args.config, "cand": name, "weight": wl, "repeats": reps,
                   "spread_over_sigma": spread, "rms_sigma_bar": float(np.sqrt(np.mean(s ** 2)))}
            rows.append(row)
            print(json.dumps({"cand": name, "E2": [round(x, 5) for x in e], "sb": [float(f"{x:.2e}") for x in s],
                              "maxdev/mad": [round(x["max_dev_over_mad"]) for x in reps],
                              "spread/sigma": round(spread, 2)}), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()

"""Statistical efficiency of the sampling weight g (the `weight El c1 z1 c2 z2` run-config line,
weights.cpp:57-99) on the synthetic spinor sets: for each candidate weight the device walker
loop runs `--steps` production steps after burn-in and reports E2, sigma_bar (blocking, block
100, estimator.cpp:77-121) and the variance per step, sigma_bar^2 x steps, whose inverse is the
statistical efficiency at fixed m. E2 does not depend on g (importance sampling is unbiased),
so the runs also cross-check each other.

Candidates are given as mass fractions: `f2 z1 z2` -> c_k = f_k (z_k)^{3/4} with f1 = 1 - f2,
i.e. primitive k carries the fraction f_k of the integral of g.

usage: python tools/weight_scan.py cfg2 [--walkers 128] [--steps 20000] [--grid ...]
"""
import argparse
import json
import re
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402


def blocking(v, nb=100):
    k = len(v) // nb
    b = v[: k * nb].reshape(k, nb).mean(axis=1)
    mean = v.mean()
    sig = np.sqrt(np.sum((b - mean) ** 2) / k)
    return mean, sig / np.sqrt(k), b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--walkers", type=int, default=0)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--burnin", type=int, default=1000)
    ap.add_argument("--grid", default="", help="semicolon list of 'f2 z1 z2'")
    ap.add_argument("--rel", action="store_true",
                    help="grid entries 'f2 a k' mean z1 = a x (smallest basis exponent), z2 = k x z1")
    ap.add_argument("--seeds", default="11")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    rows = []
    with tempfile.TemporaryDirectory() as d:
        sp, conf = generate_config(args.config, d)
        text = conf.read_text()
        el, cur = re.search(r"weight (\S+) (.*)\n", text).groups()
        m = args.walkers or int(re.search(r"walkers (\d+)", text).group(1))
        cands = [("current", cur)]
        grid = args.grid or ";".join(f"{f2} {z1} {z2}" for z1 in (0.3, 1.0) for z2 in (3.0, 30.0, 300.0, 3000.0)
                                     for f2 in (0.1, 0.3, 0.6))
        zmin = min(float(z) for z in re.findall(r"; 1 ; (\S+) 1", sp.read_text()))
        for g in grid.split(";"):
            f2, z1, z2 = map(float, g.split())
            if args.rel:
                z1, z2 = z1 * zmin, z2 * z1 * zmin
            c1, c2 = (1 - f2) * z1 ** 0.75, f2 * z2 ** 0.75
            cands.append((g, f"{c1:.6g} {z1:.6g} {c2:.6g} {z2:.6g}"))
        for (name, wl), seed in [(c, s) for c in cands for s in map(int, args.seeds.split(","))]:
            t = re.sub(r"weight .*\n", f"weight {el} {wl}\n", text)
            t0 = time.perf_counter()
            dw = DeviceWalker(System(sp, t), max_walkers=m)
            dw.init_ensemble(m, seed=seed)
            if "step-size" in t:
                dw.burn_in(args.burnin, adapt=False)
            else:
                dw.burn_in(args.burnin, adapt=True)
            st = dw.get_ensemble()
            v, _ = dw.advance(args.steps)
            st2 = dw.get_ensemble()
            dw.close()
            mean, sb, b = blocking(v)
            half = len(v) // 2
            _, sb1, _ = blocking(v[:half])
            _, sb2, _ = blocking(v[half:])
            acc = (st2.accepted - st.accepted) / max(st2.proposed - st.proposed, 1)
            row = {"cand": name, "seed": seed, "weight": wl, "E2": mean, "sigma_bar": sb, "var_per_step": sb ** 2 * len(v),
                   "sigma_bar_halves": [sb1, sb2], "acceptance": acc, "sigma_step": st.sigma_step,
                   "max_block_dev": float(np.max(np.abs(b - mean)) / (sb * np.sqrt(len(b)))),
                   "steps_to_1pct": (sb / (0.01 * abs(mean))) ** 2 * len(v), "seconds": time.perf_counter() - t0}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps({"config": args.config, "walkers": m, "steps": args.steps,
                                              "rows": rows}, indent=1))


if __name__ == "__main__":
    main()

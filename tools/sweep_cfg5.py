"""BASELINE config 5: size sweep over single-centre atoms (n_elec 2..86, basis ~ n_elec,
8192 walker pairs per GPU), wall time to 1% relative statistical error.

For each n_elec: generate the synthetic SPINOR-TEXT (host/generate.cpp, cfg5-N), run the
device walker loop through the C++ host Engine with `target-rel-err 0.01` (stop rule
driver.cpp:401-412, checked every `checkpoint-interval` steps), and report steps, wall time,
samples/s and E2 +- sigma_bar. Runs that would exceed --max-seconds are measured for a fixed
step budget instead and the time to 1% is extrapolated as t * (sigma_bar / 0.01 |E2|)^2
(marked "extrapolated").

`--configs cfg1,cfg2,...` runs the named configurations instead (their own walker counts unless
--walkers is given). The target run goes through the `mcmp2` CLI under a wall-clock timeout; a
run that times out is reported with its extrapolation and "timed_out".

usage: python tools/sweep_cfg5.py [--walkers 8192] [--max-seconds 120] [--out results.json]
"""
import argparse
import json
import re
import subprocess
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import generate_config, walker  # noqa: E402


def parse(rep):
    v = float(re.search(r"E2\s+=\s+(\S+)", rep).group(1))
    s = float(re.search(r"sigma_bar\s+=\s+(\S+)", rep).group(1))
    n = int(re.search(r"steps\s+=\s+(\d+)", rep).group(1))
    return v, s, n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--walkers", type=int, default=0, help="0: 8192 for cfg5-N, the config's own otherwise")
    ap.add_argument("--configs", default="")
    ap.add_argument("--sizes", default="2,10,18,36,54,86")
    ap.add_argument("--probe-steps", type=int, default=200)
    ap.add_argument("--max-seconds", type=float, default=120.0)
    ap.add_argument("--timeout", type=float, default=300.0)
    ap.add_argument("--workers", type=int, default=1,
                    help="reference workers (one GPU: batched ensembles in one handle when m allows)")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    rows = []
    with tempfile.TemporaryDirectory() as d:
        names = args.configs.split(",") if args.configs else [f"cfg5-{x}" for x in args.sizes.split(",")]
        for name in names:
            sp, conf = generate_config(name, d)
            base = re.sub(r"(steps|target-rel-err|checkpoint-interval) \S+\n", "", conf.read_text())
            walkers = args.walkers or (8192 if name.startswith("cfg5") else 0)
            if walkers:
                base = re.sub(r"walkers \d+", f"walkers {walkers}", base)
            walkers = int(re.search(r"walkers (\d+)", base).group(1))
            base = re.sub(r"workers \d+\n", "", base) + f"workers {args.workers}\n"
            # probe: fixed budget, gives samples/s and the variance
            t0 = time.perf_counter()
            rep = walker.run_config_text(base + f"steps {args.probe_steps * args.workers}\n"
                                         f"checkpoint-interval {args.probe_steps}\n")
            t_probe = time.perf_counter() - t0
            e, s, steps = parse(rep)
            pairs = walkers * (walkers - 1) // 2
            rate = steps * pairs / t_probe
            est_steps = steps * (s / (0.01 * abs(e))) ** 2 if e else float("inf")
            est_time = t_probe * est_steps / steps
            row = {"config": name, "walkers": walkers, "workers": args.workers, "probe_steps": steps, "probe_seconds": t_probe,
                   "samples_per_s_incl_setup": rate, "E2_probe": e, "sigma_bar_probe": s,
                   "steps_to_1pct_est": est_steps, "seconds_to_1pct_est": est_time}
            if est_time <= args.max_seconds:
                cf = Path(d) / f"{name}.target.conf"
                cf.write_text(base + "target-rel-err 0.01\ncheckpoint-interval 100\n")
                cli = Path(__file__).resolve().parent.parent / "paper_2203_05632_b200" / "lib" / "mcmp2"
                t0 = time.perf_counter()
                try:
                    rep = subprocess.run([str(cli), "run", "--config", str(cf)], capture_output=True, text=True,
                                         check=True, timeout=args.timeout).stdout
                except subprocess.TimeoutExpired:
                    row.update({"measured": False, "timed_out": args.timeout, "seconds_to_1pct": est_time,
                                "note": f"target run exceeded {args.timeout:.0f} s; probe extrapolation"})
                else:
                    wall = time.perf_counter() - t0
                    e, s, steps = parse(rep)
                    row.update({"measured": True, "seconds_to_1pct": wall, "steps_to_1pct": steps, "E2": e,
                                "sigma_bar": s, "rel_err": s / abs(e)})
            else:
                row.update({"measured": False, "seconds_to_1pct": est_time, "note": "extrapolated from the probe"})
            print(json.dumps(row), flush=True)
            rows.append(row)
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()

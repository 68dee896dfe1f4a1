"""Throughput of batched ensembles (nens reference workers in one handle, mcmp2dev_init_batch):
samples/s = nens x C(m,2) x steps / wall time of advance(steps) with every step's values copied
to the host (graph path, chunks of 32 steps). Also the pair kernel's share from the profiling
pass. usage: python tools/batch_scan.py cfg1 [--nens 1,16,148,592] [--steps 640]"""
import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2203_05632_b200 import DeviceWalker, System, generate_config  # noqa: E402

M = {"cfg1": 16, "cfg2": 128, "cfg3": 512}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--nens", default="1,16,148,592")
    ap.add_argument("--steps", type=int, default=640)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    m = M[args.config]
    rows = []
    with tempfile.TemporaryDirectory() as d:
        sp, conf = generate_config(args.config, d)
        text = conf.read_text()
        sysd = System(sp, text)
        for ne in map(int, args.nens.split(",")):
            dw = DeviceWalker(sysd, max_walkers=max(ne * m, 16))
            dw.init_batch(ne, m, seed=1, stream0=0)
            if "step-size" in text:
                dw.set_sigma_step(0.3)
                dw.burn_in(100, adapt=False)
            else:
                dw.burn_in(100, adapt=True)
            dw.advance(64)  # warm-up + graph capture
            t0 = time.perf_counter()
            v, _ = dw.advance(args.steps)
            t = time.perf_counter() - t0
            dw.profile(True, True)
            dw.advance(4)
            prof = dw.profile(False, True)
            samples = ne * m * (m - 1) // 2 * args.steps
            row = {"config": args.config, "walkers": m, "nens": ne, "steps": args.steps, "seconds": t,
                   "samples_per_s": samples / t, "us_per_step": 1e6 * t / args.steps,
                   "pair_ms": prof["ms"]["pair"] / prof["launches"]["pair"],
                   "spinor_ms": prof["ms"]["spinor"] / prof["launches"]["spinor"],
                   "walk_ms": prof["ms"]["walk"] / prof["launches"]["walk"]}
            rows.append(row)
            print(json.dumps(row), flush=True)
            dw.close()
    if args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()

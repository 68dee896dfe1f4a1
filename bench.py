#!/usr/bin/env python
"""Benchmark of the MC-MP2 walker loop (BASELINE.json metric: walker-pair x tau samples/s, and
time to 1% relative error).

One step = one pass of the hot path over one ensemble: Metropolis sweep of m walker pairs,
tau draw, spinor values + MO transform at 2m points, O/V Green's-function blocks and the
fused direct/exchange integrand over all C(m,2) walker pairs, block reduction
(reference driver.cpp:440-450). samples/step = C(m,2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]
                  [--scaling strong|weak] [--strong-total-steps S] [--ttt cfg5-10,cfg5-2]

N > 1 runs under torchrun, one process per GPU; each rank is one reference worker (its own
ensemble, Philox stream = rank, driver.cpp:354-356). --scaling strong (default): the K timed
steps are the run's total, split over the ranks with worker_share (driver.cpp:307-309);
weak: K steps per rank. Beside the timed steps the line carries
  strong_run:     the north_star strong-scaling job -- a fixed total step budget of the config
                  (2 x 10^4 at cfg4) split with worker_share over the ranks, wall time from
                  handle creation (init + burn-in included) to the merged estimate, max over ranks;
  time_to_target: wall time to sigma_bar/|E| <= 1% through the Engine stop rule
                  (driver.cpp:401-412) on the cfg5 sweep members named by --ttt, all ranks
                  merging at every checkpoint interval, with the CPU counterpart extrapolated.
`--impl reference` times the CPU restatement of the reference path (oracle/, the reference
itself needs Eigen3 and cannot be built here) on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "MC-MP2 walker-pair x tau samples/sec"
UNIT = "samples/s"
WALKERS = {"cfg1": 16, "cfg2": 128, "cfg3": 512, "cfg4": 2048}
WALKERS.update({f"cfg5-{n}": 8192 for n in (2, 10, 18, 36, 54, 86)})
WORKLOAD = {
    "cfg1": "2e atom, 4c, 12s L + 36p S, n_occ 2, n_vir 22, m 16",
    "cfg2": "10e atom, 4c, 14s9p L (R 274), n_occ 10, n_vir 72, m 128",
    "cfg3": "18e diatomic, 4c, 17s12p4d+6s2p L (R 556), n_occ 18, n_vir 152, m 512",
    "cfg4": "54e heavy diatomic, 4c, 24s20p14d+6s2p L (R 1056), n_occ 54, n_vir 278, m 2048/GPU",
}
WORKLOAD.update({f"cfg5-{n}": f"size sweep: {n}e atom, 4c, even-tempered s/p/d/f, m 8192/GPU" for n in (2, 10, 18, 36, 54, 86)})
STRONG_TOTAL = {"cfg1": 2000, "cfg2": 10000, "cfg3": 10000, "cfg4": 20000}  # BASELINE configs' step budgets
DTYPE = ("f64/c128 (reference arithmetic); the V blocks (~90% of the pair FLOPs) as Ozaki sums of exact int8 "
         "products on tcgen05 (six slices of balanced radix-256 digits per FP64 operand, 21 slice products) with a "
         "per-step error guard: steps whose estimated error exceeds 2e-10 of their sums get a 7th-slice refinement "
         "or an FP64 DMMA recompute")
MCMP2_CLI = ROOT / "paper_2203_05632_b200" / "lib" / "mcmp2"


def generate_inputs(cfg: str, directory: Path) -> tuple[Path, Path]:
    """The config's SPINOR-TEXT and run config, written by the C++ CLI in a child process
    (`mcmp2 generate`), so the reference arm's process maps no product library."""
    directory.mkdir(parents=True, exist_ok=True)
    subprocess.run([str(MCMP2_CLI), "generate", cfg, "--output", str(directory)], check=True,
                   stdout=subprocess.DEVNULL)
    return directory / f"{cfg}.spinor", directory / f"{cfg}.conf"


def worker_share(total: int, workers: int, index: int) -> int:  # driver.cpp:307-309
    return total // workers + (1 if index < total % workers else 0)


class NvmlClocks:
    """SM clock and clock-event reasons polled every 5 ms via NVML while the timed region runs."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, local_rank: int):
        import pynvml
        import torch
        self.nv = pynvml
        pynvml.nvmlInit()
        p = torch.cuda.get_device_properties(local_rank)
        bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            r = get_reasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
            time.sleep(0.005)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()

    def summary(self):
        mx = self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": mx,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "NVML, 5 ms polling"}


def clocks_sampler(path: Path):
    """nvidia-smi clocks + throttle reasons every 200 ms during the timed region."""
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        f = open(path, "w")
        return subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "200"],
                                stdout=f, stderr=subprocess.DEVNULL), f
    except (OSError, FileNotFoundError):
        return None, None


def clocks_summary(path: Path, index: int):
    rows = []
    try:
        for line in path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9 and parts[0] == str(index):
                rows.append(parts)
    except OSError:
        return None
    if not rows:
        return None
    sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
    reasons = set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for r in rows:
        for n, v in zip(names, r[5:9]):
            if v.lower().startswith("active"):
                reasons.add(n)
    return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][2]),
            "reasons": sorted(reasons), "samples": len(rows)}


# dense tcgen05 INT8 rate measured on this pool's B200 (tools/umma_rate.cu: M128 N256 K32 kind::i8
# MMAs from shared memory, one issuing thread per SM, 4570 TOPS; nominal dense INT8/FP8 4.5 POPS,
# B200_PROFILING.md). The kernel's own bound is shared-memory bandwidth: per k-step (32 of K') of a
# 128 x 80 tile the 9 merged MMAs read 36 KB of A and 52.5 KB of B slices and the ring's fills write
# 39.9 KB, 128.4 KB against 128 B/clk/SM -> 1003 cycles for 21 x 2 x 128 x 80 x 32 ops = 3993 TOPS per GPU.
INT8_PEAK = 4570.0
INT8_SMEM_BOUND = 148 * 1.965e9 * (21 * 2 * 128 * 80 * 32) / ((36864 + 53760 + 39936) / 128) / 1e12
INT8_PEAK_SOURCE = ("measured: tools/umma_rate.cu tcgen05.mma kind::i8 M128 N256 K32, 4570 TOPS (nominal dense 4500; "
                    "profiles/r03_umma_rate.txt)")


def peaks():
    fp64 = json.loads((ROOT / "MEASURED_FP64.json").read_text())
    return fp64["dmma_tflops"], "MEASURED_FP64.json dmma_tflops (mma.sync m8n8k4 f64 loop on this pool's B200)"


# bounded CPU samples: a step restricted to walker rows [0, r) of the pair loop (the Metropolis
# sweep and the spinor values always cover all 2m points), at three row counts
SAMPLE_ROWS = {"cfg3": (8, 32, 128), "cfg4": (4, 16, 64)}
SAMPLE_ROWS.update({f"cfg5-{n}": (4, 32, 128) for n in (2, 10, 18, 36, 54, 86)})


def cpu_steps(orc, cfg: str, m: int, nsteps: int, threads: int, seed0: int = 1) -> list:
    """nsteps timed steps of the CPU restatement (oracle/, one std::thread worker per core as
    driver.cpp:423-438, each on its own ensemble): step k runs the full pair loop (cfg1/cfg2) or
    rows [0, r_k) with r_k cycling over SAMPLE_ROWS[cfg]. Returns [(rows, seconds, samples/worker)]."""
    step_size = 0.3 if cfg == "cfg1" else 0.0
    rows = SAMPLE_ROWS.get(cfg, (m,))
    out = []
    for k in range(nsteps):
        r = rows[k % len(rows)]
        sec, samples = orc.cpu_baseline(seed=seed0 + k, m=m, rows=r, burn=5, step_size=step_size, steps=1,
                                        threads=threads)
        out.append((r, sec, samples / threads))
    return out


def cpu_full_step(pts: list, npairs: int) -> dict:
    """Per-worker time of a full C(m,2) step from the sampled steps: least squares of
    t = t0 + c n (t0 the O(m) part, c per pair sample) when rows were restricted (extrapolated),
    else the mean measured step."""
    import numpy as np
    n = np.array([p[2] for p in pts])
    t = np.array([p[1] for p in pts])
    if len(set(np.round(n))) < 2:
        return {"t_full": float(t.mean()), "extrapolated": False}
    A = np.stack([np.ones_like(n), n], 1)
    (t0, c), *_ = np.linalg.lstsq(A, t, rcond=None)
    resid = t - A @ np.array([t0, c])
    return {"t_full": float(t0 + c * npairs), "extrapolated": True, "t0_s": float(t0), "us_per_sample": float(c * 1e6),
            "fit_residual_rel": float(np.sqrt(np.mean(resid ** 2)) / t.mean()),
            "rows": sorted({int(p[0]) for p in pts})}


def cpu_leg(cfg: str, spinor: Path, conf_text: str, nsteps: int) -> dict:
    """cpu_baseline of our arm (rank 0, N = 1): the CPU restatement (kind 'port') on all host cores."""
    import oracle_py
    threads = os.cpu_count() or 1
    orc = oracle_py.OracleSystem(spinor, conf_text)
    m = WALKERS[cfg]
    npairs = m * (m - 1) // 2
    pts = cpu_steps(orc, cfg, m, nsteps, threads)
    fit = cpu_full_step(pts, npairs)
    secs = sum(p[1] for p in pts)
    sample = (f"{threads} workers (std::thread, driver.cpp:423-438) x {len(pts)} step(s) of m={m}"
              + (f" at walker rows {fit['rows']} of the pair loop ({secs:.1f} s); full-step rate extrapolated by a "
                 f"least-squares fit t = t0 + c n (t0 {fit['t0_s']:.2f} s, {fit['us_per_sample']:.2f} us/sample per worker, "
                 f"residual {100 * fit['fit_residual_rel']:.1f}%)" if fit["extrapolated"] else f", full steps ({secs:.1f} s)"))
    return {"value": threads * npairs / fit["t_full"], "unit": UNIT, "cores": threads, "kind": "port",
            "sample": sample, "t_full_step_s": fit["t_full"], "fit": fit}


def interval_merge(vals, first_index: int, dist):
    """The checkpoint-interval merge of the multi-GPU driver (distributed.py): each worker's
    (steps, mean, sigma_bar) summary (one per ensemble; vals is [steps] or [steps][ensembles]) is
    all-gathered (NCCL under torchrun) and merged by step-count weighting (driver.cpp:183-196) --
    the only collective of the walker loop."""
    import numpy as np
    from paper_2203_05632_b200.distributed import Summary, merge_estimates, torch_all_gather
    v2 = np.asarray(vals).reshape(len(vals), -1)
    nb = 100 if len(v2) >= 200 else max(1, len(v2) // 2)
    k = len(v2) // nb
    mine = []
    for e in range(v2.shape[1]):
        col = v2[:, e]
        blocks = col[: k * nb].reshape(k, nb).mean(axis=1)
        mean = float(np.mean(col))
        sb = float(np.sqrt(np.sum((blocks - mean) ** 2) / k) / np.sqrt(k)) if k > 0 else 0.0
        mine.append(Summary(first_index + e, len(col), mean, sb, 0.0, 0.0, k).as_array())
    mine = np.stack(mine)
    gathered = torch_all_gather(dist)(mine) if dist else [mine]
    parts = [Summary.from_array(a) for g in gathered for a in g]
    value, sigma_bar, total = merge_estimates(sorted(parts, key=lambda s: s.index))
    return {"E2": value, "sigma_bar": sigma_bar, "steps": total, "workers": len(parts)}


def reference_arm(args, cfg: str) -> None:
    """--impl reference (rank 0): the CPU restatement of the reference path on all host cores, K
    timed bounded steps (plus W untimed) of the same workload; only oracle/ libraries are mapped."""
    import oracle_py
    tmp = Path(tempfile.mkdtemp(prefix="mcmp2_ref_"))
    spinor, conf = generate_inputs(cfg, tmp)
    conf_text = conf.read_text()
    m = WALKERS[cfg]
    npairs = m * (m - 1) // 2
    threads = os.cpu_count() or 1
    orc = oracle_py.OracleSystem(spinor, conf_text)
    if args.warmup:
        cpu_steps(orc, cfg, m, args.warmup, threads, seed0=1000)
    t0 = time.perf_counter()
    pts = cpu_steps(orc, cfg, m, args.steps, threads)
    wall = time.perf_counter() - t0
    fit = cpu_full_step(pts, npairs)
    value = threads * npairs / fit["t_full"]
    secs = sum(p[1] for p in pts)
    sample = (f"{threads} workers (std::thread, driver.cpp:423-438), each one ensemble of m={m}; {len(pts)} timed steps"
              + (f" restricted to walker rows {fit['rows']} of the pair loop (cycled); full-step rate from a least-squares "
                 f"fit t = t0 + c n over the timed steps (t0 {fit['t0_s']:.2f} s, {fit['us_per_sample']:.2f} us/sample per "
                 f"worker, residual {100 * fit['fit_residual_rel']:.1f}%), extrapolated to C(m,2) = {npairs} samples"
                 if fit["extrapolated"] else " of the full pair loop"))
    # the reference's own code, compiled here against the stand-in dense header (oracle/_ref):
    # its per-core rate on replayed sub-ensembles beside the port's, for context (its dense algebra
    # runs on oracle/eigen_subset, not Eigen, so it is not the timed arm)
    ref_build = None
    try:
        import ref_py
        if ref_py.available():
            rs = ref_py.RefSystem(spinor, conf_text)
            tr = orc.trajectory(seed=3, stream=0, m=64, burn=5, nsteps=1)
            pts = []
            for msub in (32, 64):
                w = tr["walkers"][0][:msub]
                t1 = time.perf_counter()
                rs.replay(w[None], tr["tau"][:1], pair_sums=False)
                pts.append((msub, time.perf_counter() - t1))
            (m1, ta), (m2, tb) = pts
            pa, pb = m1 * (m1 - 1) / 2, m2 * (m2 - 1) / 2
            c = (tb - ta) / (pb - pa)  # s per pair sample, one core
            ref_build = {"samples_per_s_per_core": 1.0 / c, "cores": threads, "value": threads / c,
                         "port_samples_per_s_per_core": value / threads,
                         "note": "oracle/_ref/libref_mcmp2.so (the reference's estimator/greens/model sources) "
                                 "on replayed sub-ensembles of 32 and 64 walkers, one core, pair cost by "
                                 "difference; dense algebra on the stand-in oracle/eigen_subset header"}
    except Exception as e:  # context only: never fails the arm
        ref_build = {"error": str(e)}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / len(pts),  # what was timed: the sampled steps
            "timed_region_s": wall,
            "full_step_ms_extrapolated": 1e3 * fit["t_full"] if fit["extrapolated"] else None,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64/c128",
            "data": "synthetic (seeded SPINOR-TEXT from `mcmp2 generate`, host/generate.cpp)",
            "config": {"workload": f"{cfg}: {WORKLOAD[cfg]}", "walkers_per_worker": m,
                       "estimator": "literal (reference estimator.cpp:26-32)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "fit": fit, "reference_build": ref_build,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def trace(msg: str) -> None:
    """progress markers on stderr (MCMP2_BENCH_TRACE=1), rank-tagged"""
    if os.environ.get("MCMP2_BENCH_TRACE"):
        print(f"[bench r{os.environ.get('RANK', '0')} {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def run_config_text(cfg: str, spinor: Path, conf_text: str, extra: str) -> str:
    """A reference run config (driver.cpp:65-121) for the generated system: the generator's
    weight lines plus the run-control keys of `extra`."""
    keep = "".join(l + "\n" for l in conf_text.splitlines() if l.split()[:1] in (["weight"], ["step-size"]))
    return f"spinors {spinor}\n" + keep + extra


def engine_job(text: str, rank: int, world: int, dev: int, dist, max_intervals: int | None = None) -> dict:
    """One fixed job through the host Engine's per-rank group (include/mcmp2host.h mcmp2h_group:
    System load, device handle, init_ensemble + burn-in at creation) and the distributed driver's
    interval merges (distributed.py drive_group, driver.cpp:376-420); wall time from a barrier
    before the creation to the merged estimate, max over ranks."""
    import torch
    from paper_2203_05632_b200 import distributed as D
    rc = D.parse_run_config(text)
    first, count = D.rank_workers(rc["workers"], world, rank)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    group = D.HostGroup(text, first, count, dev)
    rep = D.drive_group(group, rc["workers"], rc["steps"], rc["target"], rc["interval"],
                        D.torch_all_gather(dist) if dist else (lambda a: [a]), max_intervals=max_intervals)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    group.close()
    return {"seconds": wall, "report": rep}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4", choices=sorted(WALKERS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--burnin", type=int, default=1000)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the K timed steps are the run's total, split over the ranks (worker_share); "
                         "weak: K steps per rank")
    ap.add_argument("--strong-total-steps", type=int, default=None,
                    help="step budget of the strong_run job (default: the BASELINE config's, 2e4 at cfg4; 0 skips)")
    ap.add_argument("--ttt", default="cfg5-10,cfg5-2",
                    help="cfg5 members timed to 1%% relative error (comma list; empty skips)")
    ap.add_argument("--target-rel-err", type=float, default=0.01)
    ap.add_argument("--ttt-max-steps", type=int, default=12000,
                    help="cap on a time_to_target run's total steps (all workers); a capped run reports "
                         "stopped_on_target false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--series", action="store_true",
                    help="A/B only: oz_slice_kernel in series with the O pass instead of beside it "
                         "(mcmp2dev_oz_overlap 0)")
    ap.add_argument("--dmma", action="store_true", help="A/B only: the all-DMMA pair stage (mcmp2dev_pair_path 0)")
    ap.add_argument("--whole-ksteps", action="store_true",
                    help="A/B: the INT8 V-GEMM skips only whole empty k-steps, not the leading zero slices "
                         "of the partly empty ones (mcmp2dev_oz_truncation 2)")
    ap.add_argument("--full-k", action="store_true",
                    help="A/B only: every k-step of K' in the V-GEMM (mcmp2dev_oz_truncation 0)")
    ap.add_argument("--ensembles", type=int, default=1,
                    help="reference workers per GPU, batched in one handle (mcmp2dev_init_batch); each is an "
                         "independent ensemble of the config's walker count on Philox stream rank*E + e")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = args.config
    m = WALKERS[cfg]

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, cfg)
        return

    from paper_2203_05632_b200 import generate_config

    tmp = Path(tempfile.mkdtemp(prefix=f"mcmp2_bench_r{rank}_"))
    spinor, conf = generate_config(cfg, tmp)
    conf_text = conf.read_text()
    ens = max(1, args.ensembles)
    samples_per_step = ens * (m * (m - 1) // 2)
    strong = args.scaling == "strong"
    my_steps = worker_share(args.steps, world, rank) if strong else args.steps
    total_steps = args.steps if strong else args.steps * world
    config = {"workload": f"{cfg}: {WORKLOAD[cfg]}" + (f" x {ens} ensembles per GPU" if ens > 1 else ""),
              "walkers_per_gpu": ens * m, "ensembles_per_gpu": ens, "samples_per_step_per_gpu": samples_per_step,
              "estimator": "literal (reference estimator.cpp:26-32)", "rng": "reference Philox stream per worker",
              "timed_steps": f"{total_steps} in total" + (f", split over {world} ranks by worker_share (driver.cpp:307-309)"
                                                         if strong and world > 1 else "")}

    import numpy as np
    import torch

    dev = local % torch.cuda.device_count()  # == local on a real node; lets a 1-GPU box host a 2-rank check
    torch.cuda.set_device(dev)
    dist = None
    backend = os.environ.get("MCMP2_DIST_BACKEND", "nccl")
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)

    def reduce_max(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    from paper_2203_05632_b200 import DeviceWalker, System

    sysd = System(spinor, conf_text)
    dw = DeviceWalker(sysd, device=dev, max_walkers=ens * m)
    if args.series:
        dw.int8_overlap(0)
    if args.full_k:
        dw.int8_truncation(0)
    if args.whole_ksteps:
        dw.int8_truncation(2)
    if args.dmma:
        dw.int8_v(0)
    if ens > 1:
        dw.init_batch(ens, m, seed=1, stream0=rank * ens)
    else:
        dw.init_ensemble(m, seed=1, stream=rank)
    if cfg == "cfg1":
        dw.set_sigma_step(0.3)
        dw.burn_in(args.burnin, adapt=False)
    else:
        dw.burn_in(args.burnin, adapt=True)
    stream = torch.cuda.ExternalStream(dw.stream_ptr, device=torch.device("cuda", dev))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")

    trace("setup done")
    # warm-up
    dw.advance(args.warmup, keep_on_device=True)
    dw.synchronize()
    if ens == 1:
        dw.guard_stats()  # counters from here on

    # ---- timed region: this rank's steps, device time per step on the handle's stream, L2 flushed ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(my_steps)]
    try:
        clk = NvmlClocks(dev)
    except Exception:  # NVML unavailable: fall back to nvidia-smi sampling
        clk = None
    smi, smi_f = clocks_sampler(tmp / "clocks.csv") if (rank == 0 and clk is None) else (None, None)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    if clk:
        clk.__enter__()
    for k in range(my_steps):
        with torch.cuda.stream(stream):
            flush.zero_()
            ev[k][0].record(stream)
        dw.advance(1, keep_on_device=True)
        with torch.cuda.stream(stream):
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    if dist:
        dist.barrier()
    if smi:
        time.sleep(0.25)
        smi.terminate()
        smi_f.close()
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    t_ms = sum(ms_steps)
    t_max = reduce_max(t_ms)
    value = samples_per_step * total_steps / (t_max / 1e3)

    trace("timed region done")
    # ---- per-kernel device time (profiling pass, events around each launch) ----
    ks_timed = dw.int8_ksteps()
    dw.profile(enable=True, reset=True)
    nprof = max(2, min(args.steps, 5))
    dw.advance(nprof, keep_on_device=True)
    prof = dw.profile(enable=False, reset=True)
    ks_prof = dw.int8_ksteps()
    # ---- the same steps with every k-step of K' issued (the truncation is exact; this is the
    # untruncated kernel's time for the record, outside the timed region) ----
    full_k_ms = None
    if ens == 1 and dw.int8_v() and dw.int8_truncation() and not args.full_k:
        dw.int8_truncation(0)
        nfk = max(3, min(args.steps, 10))
        evf = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nfk)]
        dw.advance(1, keep_on_device=True)
        for k in range(nfk):
            with torch.cuda.stream(stream):
                flush.zero_()
                evf[k][0].record(stream)
            dw.advance(1, keep_on_device=True)
            with torch.cuda.stream(stream):
                evf[k][1].record(stream)
        torch.cuda.synchronize()
        full_k_ms = sum(a.elapsed_time(b) for a, b in evf) / nfk
        dw.int8_truncation(2 if args.whole_ksteps else 1)
    work = dw.work()
    pair_ms = prof["ms"]["pair"] / prof["launches"]["pair"]
    step_ms_prof = prof["ms"]["total"] / prof["launches"]["total"]
    peak, peak_src = peaks()
    achieved = work["pair_flop"] / (pair_ms / 1e3) / 1e12
    kramers = dw.kramers()
    kernel_name = "pair_kr_kernel (DMMA m8n8k4 f64, Kramers-restricted)" if kramers else "pair_kernel (DMMA m8n8k4 f64)"
    oz = prof.get("int8_v", {})
    int8_path = oz.get("steps", 0) > 0  # V blocks on the INT8 tensor cores (pair_oz.cu)

    def traffic_of(kernel):  # dram bytes per launch from the committed ncu --set full capture
        tf = ROOT / "profiles" / f"traffic_{cfg}_{kernel}.json"
        return json.loads(tf.read_text()).get("dram_bytes_per_launch") if tf.exists() else None
    traffic = traffic_of("pair_kr_kernel" if kramers else "pair_kernel")

    trace("profile done")
    # ---- e2e through the C ABI: one checkpoint interval of this rank's steps with host buffers ----
    dw.prepare()  # graph capture is setup (as in the host Engine after burn-in), not step time
    import paper_2203_05632_b200.distributed  # noqa: F401  (module import is setup, not step time)
    st = dw.get_ensembles() if ens > 1 else dw.get_ensemble()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    (dw.set_ensembles if ens > 1 else dw.set_ensemble)(st)   # H2D walker state (resume)
    vals, ims = dw.advance(my_steps)                         # every step's (value, imag) D2H
    st2 = dw.get_ensembles() if ens > 1 else dw.get_ensemble()  # D2H walker state (checkpoint)
    merged = interval_merge(vals, rank * ens, dist)  # per-worker summaries -> one estimate (driver.cpp:183-196)
    e2e_s = time.perf_counter() - t0
    e2e_value = samples_per_step * total_steps / reduce_max(e2e_s)
    state_bytes = ens * (m * 9 * 8 + 64)
    h2d = state_bytes / max(my_steps, 1)
    d2h = 16 * ens + state_bytes / max(my_steps, 1)
    guard = dw.guard_stats() if ens == 1 else None
    dw.close()
    del flush

    trace("e2e done")
    # ---- strong_run: the fixed total budget of the config split over the ranks, setup included ----
    strong_run = None
    budget = STRONG_TOTAL.get(cfg, 0) if args.strong_total_steps is None else args.strong_total_steps
    if budget > 0 and ens == 1:
        text = run_config_text(cfg, spinor, conf_text,
                               f"steps {budget}\nwalkers {m}\nworkers {world}\nseed 1\nburnin {args.burnin}\n"
                               f"checkpoint-interval {budget}\n")
        job = engine_job(text, rank, world, dev, dist)
        secs = reduce_max(job["seconds"])
        rep = job["report"]
        strong_run = {"steps_total": budget, "workers": world, "seconds": secs,
                      "value": samples_per_step * budget / secs, "unit": UNIT,
                      "includes": "System load, device handle, init_ensemble + burn-in "
                                  f"{args.burnin}, production, merge (max over ranks, wall clock)",
                      "E2": rep["value"], "sigma_bar": rep["sigma_bar"]}

    trace("strong_run done")
    # ---- time to target: sigma_bar/|E| <= target through the stop rule, cfg5 members ----
    ttt = []
    for name in [x for x in args.ttt.split(",") if x]:
        sp5, conf5 = generate_config(name, tmp)
        c5 = conf5.read_text()
        m5 = WALKERS[name]
        text = run_config_text(name, sp5, c5, f"target-rel-err {args.target_rel_err}\nwalkers {m5}\nworkers {world}\n"
                                              f"seed 1\nburnin {args.burnin}\ncheckpoint-interval 100\n")
        interval = 100
        job = engine_job(text, rank, world, dev, dist, max_intervals=-(-args.ttt_max_steps // (interval * world)))
        secs = reduce_max(job["seconds"])
        rep = job["report"]
        trace(f"ttt {name}: {rep['total_steps']} steps, {secs:.1f} s, on target {rep['stopped_on_target']}")
        entry = {"config": name, "workload": WORKLOAD[name], "target_rel_err": args.target_rel_err, "seconds": secs,
                 "steps": rep["total_steps"], "stopped_on_target": rep["stopped_on_target"], "E2": rep["value"],
                 "sigma_bar": rep["sigma_bar"], "rel_err": rep["sigma_bar"] / abs(rep["value"]) if rep["value"] else None,
                 "checkpoint_interval": interval, "workers": world, "max_steps": args.ttt_max_steps,
                 "includes": f"System load, device handle, init + burn-in {args.burnin}, production to the stop rule"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            import oracle_py
            threads = os.cpu_count() or 1
            fit = cpu_full_step(cpu_steps(oracle_py.OracleSystem(sp5, c5), name, m5, 3, threads), m5 * (m5 - 1) // 2)
            per_worker = -(-rep["total_steps"] // threads)
            entry["cpu_extrapolated"] = {
                "seconds": per_worker * fit["t_full"], "cores": threads, "kind": "port",
                "basis": f"the device run's {rep['total_steps']} steps spread over {threads} CPU workers "
                         f"({per_worker} steps each) x the extrapolated full-step time {fit['t_full']:.2f} s per worker "
                         f"(bounded samples at rows {fit.get('rows')}, fit residual "
                         f"{100 * fit.get('fit_residual_rel', 0):.1f}%); burn-in not counted"}
        ttt.append(entry)

    trace("ttt done")
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    fp64_view = {"kernel": kernel_name, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                 "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                 "achieved_basis": "algorithmic: C(m,2) x F_pair, F_pair = 8 nc^2 (2 n_occ + 4 n_vir) + 32 nc^2 "
                                   "(SURVEY 8d, 8 FLOP per complex MAC of the reference's full 4x4 blocks) over the "
                                   "pair stage's device time",
                 "executed_dmma_flop_per_launch": work["pair_dmma_flop_executed"],
                 "kramers_path": kramers,
                 "pair_flop_per_launch": work["pair_flop"], "pair_ms_per_launch": pair_ms,
                 "pair_share_of_step": prof["ms"]["pair"] / prof["ms"]["total"],
                 "spinor_ms_per_launch": prof["ms"]["spinor"] / prof["launches"]["spinor"],
                 "walk_ms_per_launch": prof["ms"]["walk"] / prof["launches"]["walk"],
                 "step_ms_profiled": step_ms_prof}
    if int8_path:
        n = oz["steps"]
        vg_ms, sl_ms, kr_ms, gd_ms = oz["vgemm_ms"] / n, oz["slice_ms"] / n, oz["pair_kr_ms"] / n, oz["guard_ms"] / n
        # k-steps the V-GEMM issued (energy-ordered truncation, exact) over those of the full K' loop:
        # in the profiling pass (the launches vg_ms times) and over the run so far (warm-up + timed steps)
        ks_frac = (ks_prof[0] - ks_timed[0]) / (n * ks_prof[1]) if ks_prof[1] else 1.0
        ks_frac_run = ks_timed[0] / ((args.warmup + my_steps) * ks_timed[1]) if ks_timed[1] and my_steps else None
        a8_full = oz["vgemm_int8_ops"] / (vg_ms / 1e3) / 1e12
        a8 = a8_full * ks_frac
        equiv = {k: v for k, v in fp64_view.items() if k not in ("frac", "peak", "peak_source")}
        equiv.update(kernel="pair stage: oz_slice_kernel + pair_kr_kernel (O blocks, DMMA) + oz_vgemm_kernel (V "
                            "blocks, INT8, contraction fused) + the guard's refinement / DMMA launches",
                     dmma_peak=peak, ratio_to_dmma_peak=achieved / peak,
                     note="throughput-equivalent, not a roofline fraction: the reference's FP64 operation count over "
                          "the pair stage's time; the kernels do fewer FP64 operations (V blocks as exact int8 "
                          "products, O blocks with 3M complex products on the Kramers alpha rows)")
        roofline = {
            "bound": "tensor", "kernel": "oz_vgemm_kernel (tcgen05.mma kind::i8: the V blocks as 6-slice Ozaki "
                                         "sums of exact int8 products, pair_oz.cu)",
            "achieved": a8, "peak": INT8_PEAK, "unit": "TFLOP/s", "frac": a8 / INT8_PEAK,
            "traffic": traffic_of("oz_vgemm_kernel"),
            "op_basis": "executed int8 tensor ops (2 per MAC): 2 x 128 x 80 x 32 per slice product issued (the "
                        "device counter of mcmp2dev_oz_ksteps over the profiled launches; 21 products per whole "
                        "k-step, fewer in a partly empty one)",
            "peak_source": INT8_PEAK_SOURCE,
            "ksteps_frac": ks_frac, "ksteps_frac_run": ks_frac_run,
            "ksteps_note": "K' follows the virtual energies; k-steps whose digits are all zero at this step's tau "
                           "(exp(-eps tau / 2) below the last slice) are skipped, and so are the slice products of "
                           "the partly empty k-steps whose A or B slice is all zero there (leading digits), "
                           "bit-identical to the full loop (tests/test_gpu_oz.py); ksteps_frac = slice products "
                           "issued / full over the profiled launches, "
                           "ksteps_frac_run over warm-up + timed steps",
            "full_k_ms_per_step": full_k_ms,
            "full_k_samples_per_s": samples_per_step / (full_k_ms / 1e3) if full_k_ms else None,
            "full_k_note": "device time per step of this rank with the truncation switched off "
                           "(mcmp2dev_oz_truncation 0), measured after the timed region over a few steps",
            "full_loop_equivalent": a8_full, "full_loop_equivalent_note": "the full K' loop's int8 ops over the same "
                                                                          "time (what an untruncated kernel would need)",
            "smem_bound": INT8_SMEM_BOUND, "frac_of_smem_bound": a8 / INT8_SMEM_BOUND,
            "smem_bound_note": "the kernel's binding resource is shared-memory bandwidth (128 B/clk/SM): per k-step "
                               "of a 128 x 80 tile the 9 merged MMAs read 36 + 52.5 KB of slices and the ring's "
                               "fills write 39.9 KB",
            "vgemm_ms_per_launch": vg_ms, "slice_ms_per_launch": sl_ms, "pair_kr_ms_per_launch": kr_ms,
            "guard_ms_per_step": gd_ms,
            "vgemm_share_of_step": vg_ms / step_ms_prof,
            "pair_stage_throughput_equivalent": equiv}
    else:
        roofline = dict(fp64_view, bound="tensor",
                        executed_tflops=work["pair_dmma_flop_executed"] / (pair_ms / 1e3) / 1e12,
                        executed_frac=work["pair_dmma_flop_executed"] / (pair_ms / 1e3) / 1e12 / peak,
                        why_frac_above_1="the kernel issues fewer DMMA FLOPs than the algorithmic count: complex "
                                         "products as 3 real products (3M) and, for exact Kramers pairs, only the "
                                         "alpha rows of each 4x4 block (pair_kr.cu); executed_frac is the tensor-pipe "
                                         "utilisation" if kramers else "3M complex products (3 real per complex)")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / max(my_steps, 1), "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": DTYPE if int8_path else "f64/c128",
        "data": "synthetic (seeded SPINOR-TEXT from host/generate.cpp; no public dataset)",
        "config": dict(config, parallelism=f"{world * ens} independent workers ({ens} per GPU)",
                       l2="flushed between timed steps (256 MiB write on the handle's stream)"),
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "mcmp2dev_set_ensemble + mcmp2dev_advance(K, host values) + mcmp2dev_get_ensemble"
                        " + interval merge (all_gather of per-rank summaries, merge_estimates)",
                "merged": merged},
        # per step: walk_kernel, chi_kernel, mo_kernel, then the pair stage: INT8 path oz_slice_kernel,
        # pair_kr_kernel_pw4 (O), oz_vgemm_kernel, the guard's refinement and DMMA launches (both exit at
        # once unless the step failed its check); DMMA path one pair kernel
        "gpu_launches": (8 if int8_path else 4) * my_steps,
        "step_values_checksum": float(np.sum(vals)),
    }
    # which pair stage ran, and why not the INT8 V path when it did not (n_vir > 512, spinors not
    # Kramers-paired within 1e-12, batched ensembles or m below ~180: mcmp2dev.cu oz_active)
    if int8_path:
        line["pair_path"] = "INT8 V blocks (tcgen05 kind::i8, 6-slice radix-256 Ozaki, guarded, energy-ordered k-step truncation) + DMMA O blocks"
    else:
        why = []
        if not kramers:
            why.append(f"spinor set not Kramers-paired within 1e-12 (deviation {dw.kramers_deviation():.3g})")
        if sysd.n_vir > 512:
            why.append(f"n_vir {sysd.n_vir} > 512")
        if sysd.n_vir <= 16:
            why.append(f"n_vir {sysd.n_vir} <= 16: one k-step of K', the DMMA kernel is faster")
        if ens > 1:
            why.append("batched ensembles")
        line["pair_path"] = "DMMA only (INT8 V path inactive: " + ("; ".join(why) or "ensemble below the INT8 tiling size") + ")"
    if guard is not None:
        line["guard"] = dict(guard, note="INT8 steps checked / refined (7th slice) / recomputed on DMMA over the "
                                         "e2e interval; max_est_rel = largest estimated relative error of a kept step")
    if strong_run:
        line["strong_run"] = strong_run
    if ttt:
        line["time_to_target"] = ttt
    cl = clk.summary() if clk else clocks_summary(tmp / "clocks.csv", dev)
    if cl:
        line["clocks"] = cl
    if world == 1 and not args.no_cpu_baseline:
        leg = cpu_leg(cfg, spinor, conf_text, nsteps=3)
        line["cpu_baseline"] = {k: leg[k] for k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

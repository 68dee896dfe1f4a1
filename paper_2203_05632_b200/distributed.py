"""One process per GPU; the run's reference workers are split over the ranks and merged over
torch.distributed.

The reference runs `workers` independent ensembles as std::threads in one process
(driver.cpp:423-438) with Philox stream = worker index (driver.cpp:354-356), splits a step
budget with worker_share (driver.cpp:307-309), and at every checkpoint interval merges the
per-worker estimates by step-count weighting (driver.cpp:183-196) for the target-error stop
rule (driver.cpp:401-412). Here each rank (torchrun, one GPU each) hosts a contiguous range of
the workers (at least one; a range of several shares one batched device handle when the walker
count allows it), and the interval merge is one all_gather of the workers' 7-double summaries --
the only collective; the walker loop itself has no communication. Launch:

  torchrun --nproc-per-node N -m paper_2203_05632_b200.distributed CONFIG_FILE
"""
from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass

import numpy as np

from . import native
from .native import check_host, dptr


@dataclass
class Summary:  # WorkerSummary (driver.hpp:46-53) + the accumulator's block count
    index: int
    steps: int
    mean: float
    sigma_bar: float
    acceptance: float
    imag_ratio: float
    nblocks: int

    def as_array(self):
        return np.array([self.index, self.steps, self.mean, self.sigma_bar, self.acceptance, self.imag_ratio,
                         self.nblocks], dtype=np.float64)

    @staticmethod
    def from_array(a):
        return Summary(int(a[0]), int(a[1]), float(a[2]), float(a[3]), float(a[4]), float(a[5]), int(a[6]))


class HostWorker:
    """A C++ DeviceWorker (host/driver.cpp) on one GPU: init_ensemble + burn_in at creation."""

    def __init__(self, config_text: str, index: int, device: int):
        h = native.host()
        self._w = h.mcmp2h_worker_create(config_text.encode(), index, device)
        if not self._w:
            raise native.Mcmp2Error(h.mcmp2h_last_error().decode())
        self.index = index

    def advance(self, nsteps: int) -> None:
        if nsteps > 0:
            check_host(native.host().mcmp2h_worker_advance(self._w, nsteps, None, None))

    def summary(self) -> Summary:
        o = np.zeros(10)
        check_host(native.host().mcmp2h_worker_stats(self._w, dptr(o)))
        return Summary(self.index, int(o[0]), o[3], o[4], o[8], o[9], int(o[7]))

    def close(self):
        if getattr(self, "_w", None):
            native.host().mcmp2h_worker_free(self._w)
            self._w = None

    def __del__(self):
        self.close()


def worker_share(total: int, workers: int, index: int) -> int:  # driver.cpp:307-309
    return total // workers + (1 if index < total % workers else 0)


def merge_estimates(parts: list[Summary]) -> tuple[float, float, int]:
    """driver.cpp:183-196 through the host library (same arithmetic as the C++ Engine)."""
    arr = np.ascontiguousarray([[p.steps, p.mean, p.sigma_bar] for p in parts], dtype=np.float64)
    out = np.empty(3)
    h = native.host()
    h.mcmp2h_merge_estimates.argtypes = [C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double)]
    check_host(h.mcmp2h_merge_estimates(dptr(arr), len(parts), dptr(out)))
    return float(out[0]), float(out[1]), int(out[2])


def parse_run_config(text: str) -> dict:
    """The run-control keys the driver needs (full validation is the host's parse_config_text)."""
    buf = C.create_string_buffer(1 << 14)
    check_host(native.host().mcmp2h_parse_config(text.encode(), buf, len(buf)))
    cfg = {}
    for line in buf.value.decode().splitlines():
        k, _, v = line.partition(" ")
        cfg[k] = v
    return {"steps": int(cfg["steps"]) if "steps" in cfg else None,
            "target": float(cfg["target-rel-err"]) if "target-rel-err" in cfg else None,
            "interval": int(cfg["checkpoint-interval"]), "workers": int(cfg.get("workers", "1")),
            "checkpoint": cfg.get("checkpoint"), "trace": cfg.get("trace")}


def require_no_files(rc: dict) -> None:
    """The multi-process driver merges estimates only; the checkpoint (driver.cpp:218-305) and
    trace files of the reference Engine hold every worker's record in one file written by one
    process, which this driver does not assemble. A run that asks for them is refused rather
    than silently run without them: use the single-process Engine (`mcmp2 run`, one device
    handle per worker) for checkpointed or traced runs."""
    for key in ("checkpoint", "trace"):
        if rc.get(key):
            raise ValueError(f"distributed driver: '{key}' is not supported across ranks "
                             "(run the config with the single-process Engine, `mcmp2 run`)")


class HostGroup:
    """The reference workers [first, first + count) this rank hosts on its GPU (host/capi.cpp,
    mcmp2h_group): one batched device handle when the walker count allows it
    (include/mcmp2dev.h, batched ensembles), else one handle each; init + burn-in at creation."""

    def __init__(self, config_text: str, first: int, count: int, device: int):
        h = native.host()
        self._g = h.mcmp2h_group_create(config_text.encode(), first, count, device)
        if not self._g:
            raise native.Mcmp2Error(h.mcmp2h_last_error().decode())
        self.first, self.count = first, count

    def advance(self, nsteps) -> None:
        arr = (C.c_longlong * self.count)(*[int(max(n, 0)) for n in nsteps])
        check_host(native.host().mcmp2h_group_advance(self._g, arr))

    def summaries(self) -> list[Summary]:
        out = []
        for k in range(self.count):
            o = np.zeros(10)
            check_host(native.host().mcmp2h_group_stats(self._g, k, dptr(o)))
            out.append(Summary(self.first + k, int(o[0]), o[3], o[4], o[8], o[9], int(o[7])))
        return out

    def close(self):
        if getattr(self, "_g", None):
            native.host().mcmp2h_group_free(self._g)
            self._g = None

    def __del__(self):
        self.close()


class _OneWorker:
    """A single worker (advance(n), summary()) seen as a group of one."""

    def __init__(self, worker, index: int):
        self.w, self.first, self.count = worker, index, 1

    def advance(self, nsteps) -> None:
        self.w.advance(nsteps[0])

    def summaries(self) -> list[Summary]:
        return [self.w.summary()]


def rank_workers(total: int, world: int, rank: int) -> tuple[int, int]:
    """Workers of this rank: a contiguous range of the run's `workers`, split as worker_share
    splits steps (driver.cpp:307-309). Every rank needs at least one worker: fewer workers than
    ranks would change the Philox streams and step shares of the run (its config hash names the
    worker count), so that is an error, not a silent increase."""
    if total < world:
        raise ValueError(f"distributed driver: workers {total} < world size {world} "
                         "(set `workers` to at least the number of ranks)")
    first = sum(worker_share(total, world, r) for r in range(rank))
    return first, worker_share(total, world, rank)


def drive_group(group, total_workers: int, steps: int | None, target: float | None, interval: int, all_gather,
                max_intervals: int | None = None) -> dict:
    """Engine::drive (driver.cpp:376-420) over all ranks' workers: every interval each worker
    advances its share, the summaries of all workers are gathered (one all_gather; ranks hold
    different worker counts, so the rows are padded with index -1) and the stop rule is
    evaluated identically on every rank."""
    intervals = 0
    on_target = False
    done = [0] * group.count
    while True:
        idx = range(group.first, group.first + group.count)
        chunk = [interval if steps is None else min(interval, worker_share(steps, total_workers, i) - d)
                 for i, d in zip(idx, done)]
        group.advance(chunk)
        done = [d + max(c, 0) for d, c in zip(done, chunk)]
        intervals += 1
        local = np.stack([s.as_array() for s in group.summaries()])
        pad = np.full((total_workers - len(local), local.shape[1]), -1.0) if total_workers > len(local) else None
        send = np.concatenate([local, pad]) if pad is not None else local
        parts = [Summary.from_array(a) for g in all_gather(send) for a in np.atleast_2d(g) if a[0] >= 0]
        parts.sort(key=lambda p: p.index)
        if steps is not None:
            if all(p.steps >= worker_share(steps, total_workers, p.index) for p in parts):
                break
        elif all(p.nblocks > 0 for p in parts):
            value, sigma_bar, _ = merge_estimates(parts)
            if sigma_bar > 0 and value != 0 and sigma_bar / abs(value) <= target:
                on_target = True
                break
        if max_intervals is not None and intervals >= max_intervals:
            break
    value, sigma_bar, total = merge_estimates(parts)
    return {"value": value, "sigma_bar": sigma_bar, "total_steps": total, "stopped_on_target": on_target,
            "workers": parts, "intervals": intervals}


def drive(worker, rank: int, world: int, steps: int | None, target: float | None, interval: int,
          all_gather, max_intervals: int | None = None) -> dict:
    """One worker per rank (worker index = rank): drive_group with groups of one."""
    return drive_group(_OneWorker(worker, rank), world, steps, target, interval, all_gather, max_intervals)


def format_report(rep: dict) -> str:  # driver.cpp:523-539
    lines = [f"E2        = {rep['value']:.17g} hartree", f"sigma_bar = {rep['sigma_bar']:.17g} hartree",
             f"steps     = {rep['total_steps']}"]
    if rep["stopped_on_target"]:
        lines.append("stopped on target relative uncertainty")
    for w in rep["workers"]:
        lines.append(f"worker {w.index}: steps {w.steps}, I {w.mean:.17g}, sigma_bar {w.sigma_bar:.17g}, "
                     f"acceptance {w.acceptance:.3f}, imag ratio {w.imag_ratio:.2e}")
    return "\n".join(lines) + "\n"


def torch_all_gather(dist):
    import torch

    def gather(a: np.ndarray):
        t = torch.from_numpy(a)
        if dist.get_backend() == "nccl":
            t = t.cuda()
        out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(out, t)
        return [o.cpu().numpy() for o in out]
    return gather


def main(argv=None):
    import os

    import torch
    import torch.distributed as dist

    argv = sys.argv[1:] if argv is None else argv
    text = open(argv[0]).read()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rc = parse_run_config(text)
    require_no_files(rc)
    first, count = rank_workers(rc["workers"], world, rank)
    group = HostGroup(text, first, count, local)
    rep = drive_group(group, rc["workers"], rc["steps"], rc["target"], rc["interval"],
                      torch_all_gather(dist))
    if rank == 0:
        sys.stdout.write(format_report(rep))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

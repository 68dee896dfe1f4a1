"""One process per GPU; the run's reference workers are split over the ranks and merged over
torch.distributed.

The reference runs `workers` independent ensembles as std::threads in one process
(driver.cpp:423-438) with Philox stream = worker index (driver.cpp:354-356), splits a step
budget with worker_share (driver.cpp:307-309), and at every checkpoint interval merges the
per-worker estimates by step-count weighting (driver.cpp:183-196) for the target-error stop
rule (driver.cpp:401-412). Here each rank (torchrun, one GPU each) hosts a contiguous range of
the workers (at least one; a range of several shares one batched device handle when the walker
count allows it), and the interval merge is one all_gather of the workers' 7-double summaries --
the only collective of the stop rule; the walker loop itself has no communication. A config that
names a `checkpoint` or `trace` file gets them as the reference Engine writes them
(driver.cpp:218-251, 311-334): every interval each rank sends its workers' checkpoint records and
trace lines to rank 0 (a second all_gather, of bytes), which writes the one file holding every
worker's record, byte-identical to the single-process Engine's, so `resume` here, `mcmp2 resume`
and `mcmp2 merge` all read it. Launch:

  torchrun --nproc-per-node N -m paper_2203_05632_b200.distributed CONFIG_FILE
  torchrun --nproc-per-node N -m paper_2203_05632_b200.distributed resume CHECKPOINT_FILE
"""
from __future__ import annotations

import ctypes as C
import os
import struct
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


def _sized_text(call, *args) -> bytes:
    """A text-returning host call of the (buf, cap, need) shape (include/mcmp2host.h)."""
    need = C.c_long(0)
    check_host(call(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    check_host(call(*args, buf, need.value, C.byref(need)))
    return buf.value


def gather_bytes(all_gather, blob: bytes) -> list[bytes]:
    """Every rank's byte string on every rank: the lengths, then the padded bytes."""
    lens = [int(a[0]) for a in all_gather(np.array([len(blob)], dtype=np.int64))]
    send = np.zeros(max(max(lens), 1), dtype=np.uint8)
    send[:len(blob)] = np.frombuffer(blob, dtype=np.uint8)
    return [bytes(np.asarray(a, dtype=np.uint8)[:n]) for a, n in zip(all_gather(send), lens)]


def _pack(items: list[bytes]) -> bytes:
    return struct.pack("<q", len(items)) + b"".join(struct.pack("<q", len(x)) + x for x in items)


def _unpack(blob: bytes) -> list[bytes]:
    (n,), at, out = struct.unpack_from("<q", blob, 0), 8, []
    for _ in range(n):
        (k,) = struct.unpack_from("<q", blob, at)
        out.append(blob[at + 8:at + 8 + k])
        at += 8 + k
    return out


def _replace_file(path: str, data: bytes) -> None:
    with open(path + ".tmp", "wb") as f:
        f.write(data)
    os.replace(path + ".tmp", path)


class RunFiles:
    """The Engine's per-interval files for workers spread over ranks. The checkpoint
    (driver.cpp:218-251: written to <path>.tmp, then renamed) is the header plus every worker's
    record in worker order; the trace (driver.cpp:311-334) is one <trace>.w<k> file per worker
    rewritten every interval and joined in worker order when the run ends. Ranks hold
    contiguous ascending worker ranges (rank_workers), so rank order is worker order. Rank 0
    writes; the other ranks only send."""

    def __init__(self, config_text: str, rc: dict, rank: int, all_gather):
        self.checkpoint, self.trace = rc.get("checkpoint"), rc.get("trace")
        self.rank, self.all_gather, self.nworkers = rank, all_gather, rc["workers"]
        self.header = b""
        if self.checkpoint and rank == 0:
            self.header = _sized_text(native.host().mcmp2h_checkpoint_header, config_text.encode(), self.nworkers)

    def __bool__(self):
        return bool(self.checkpoint or self.trace)

    def write_interval(self, group) -> None:
        if not self:
            return
        records = group.records() if self.checkpoint else []
        traces = group.traces() if self.trace else []
        idx = [struct.pack("<q", group.first + k) for k in range(group.count)]
        parts = [_unpack(b) for b in gather_bytes(self.all_gather, _pack(idx + records + traces))]
        if self.rank != 0:
            return
        workers, recs, trs = [], [], []
        for p in parts:
            n = len(p) // (1 + bool(self.checkpoint) + bool(self.trace))
            workers += [struct.unpack("<q", x)[0] for x in p[:n]]
            if self.checkpoint:
                recs += p[n:2 * n]
            trs += p[len(p) - n:] if self.trace else []
        if workers != list(range(self.nworkers)):
            raise native.Mcmp2Error(f"distributed driver: gathered workers {workers}, expected 0..{self.nworkers - 1}")
        if self.checkpoint:
            _replace_file(self.checkpoint, self.header + b"".join(recs))
        for k, t in zip(workers, trs):
            _replace_file(f"{self.trace}.w{k}", t)

    def finish(self) -> None:  # join_traces, driver.cpp:323-334
        if not self.trace or self.rank != 0:
            return
        with open(self.trace, "wb") as out:
            for k in range(self.nworkers):
                if os.path.exists(f"{self.trace}.w{k}"):
                    out.write(open(f"{self.trace}.w{k}", "rb").read())
        for k in range(self.nworkers):
            if os.path.exists(f"{self.trace}.w{k}"):
                os.remove(f"{self.trace}.w{k}")


def checkpoint_run_config(path: str) -> tuple[str, dict]:
    """The config stored in a checkpoint after the hash check of resume (driver.cpp:482-491);
    the run continues with the saved workers (driver.cpp:349: restored.size())."""
    buf = C.create_string_buffer(1 << 14)
    nw = C.c_int(0)
    check_host(native.host().mcmp2h_checkpoint_config(str(path).encode(), buf, len(buf), C.byref(nw)))
    text = buf.value.decode()
    rc = parse_run_config(text)
    rc["workers"] = nw.value
    return text, rc


class HostGroup:
    """The reference workers [first, first + count) this rank hosts on its GPU (host/capi.cpp,
    mcmp2h_group): one batched device handle when the walker count allows it
    (include/mcmp2dev.h, batched ensembles), else one handle each; init + burn-in at creation."""

    def __init__(self, config_text: str, first: int, count: int, device: int, resume_from: str | None = None):
        h = native.host()
        if resume_from is None:
            self._g = h.mcmp2h_group_create(config_text.encode(), first, count, device)
        else:  # workers restored from their checkpoint records (driver.cpp:360-373)
            self._g = h.mcmp2h_group_resume(str(resume_from).encode(), first, count, device)
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

    def records(self) -> list[bytes]:
        return [_sized_text(native.host().mcmp2h_group_record, self._g, k) for k in range(self.count)]

    def traces(self) -> list[bytes]:
        return [_sized_text(native.host().mcmp2h_group_trace, self._g, k) for k in range(self.count)]

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
                max_intervals: int | None = None, files: "RunFiles | None" = None) -> dict:
    """Engine::drive (driver.cpp:376-420) over all ranks' workers: every interval each worker
    advances its share, the summaries of all workers are gathered (one all_gather; ranks hold
    different worker counts, so the rows are padded with index -1) and the stop rule is
    evaluated identically on every rank. `files` writes the interval's checkpoint and traces
    before the stop rule, as the Engine does; `max_intervals` is its abort hook
    (RunHooks::abort_after_intervals). Resumed workers carry their step counts in."""
    intervals = 0
    on_target = False
    done = [s.steps for s in group.summaries()]
    while True:
        idx = range(group.first, group.first + group.count)
        chunk = [interval if steps is None else min(interval, worker_share(steps, total_workers, i) - d)
                 for i, d in zip(idx, done)]
        group.advance(chunk)
        done = [d + max(c, 0) for d, c in zip(done, chunk)]
        intervals += 1
        if files:
            files.write_interval(group)
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
            value, sigma_bar, total = merge_estimates(parts)
            return {"value": value, "sigma_bar": sigma_bar, "total_steps": total, "stopped_on_target": False,
                    "workers": parts, "intervals": intervals}
    if files:
        files.finish()
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
    import torch
    import torch.distributed as dist

    argv = sys.argv[1:] if argv is None else argv
    resume_from = argv[1] if argv[0] == "resume" else None
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if resume_from is None:
        text = open(argv[0]).read()
        rc = parse_run_config(text)
    else:
        text, rc = checkpoint_run_config(resume_from)
    first, count = rank_workers(rc["workers"], world, rank)
    group = HostGroup(text, first, count, local, resume_from)
    gather = torch_all_gather(dist)
    rep = drive_group(group, rc["workers"], rc["steps"], rc["target"], rc["interval"], gather,
                      files=RunFiles(text, rc, rank, gather))
    if rank == 0:
        sys.stdout.write(format_report(rep))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

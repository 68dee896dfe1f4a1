"""CPU, gloo world size 2: the multi-process driver (paper_2203_05632_b200/distributed.py).

Each rank drives a stand-in worker that replays the oracle's chain for worker index = rank
(same Philox stream as the device worker would use), so the gathered merge, the step-budget
split and the target-error stop rule can be checked against the oracle's own multi-worker
Engine (std::threads, driver.cpp:376-438) on CPU."""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_py
from paper_2203_05632_b200 import distributed as D


class Blocking:  # estimator.cpp:81-105, for the stand-in only
    def __init__(self, nb):
        self.nb, self.n, self.sum, self.imag, self.partial, self.inb, self.means = nb, 0, 0.0, 0.0, 0.0, 0, []

    def add(self, v, im):
        self.sum += v
        self.imag += im
        self.n += 1
        self.partial += v
        self.inb += 1
        if self.inb == self.nb:
            self.means.append(self.partial / self.nb)
            self.partial, self.inb = 0.0, 0

    def mean(self):
        return self.sum / self.n if self.n else 0.0

    def sigma_bar(self):
        k = len(self.means)
        if not k:
            return 0.0
        m = self.mean()
        return math.sqrt(sum((b - m) * (b - m) for b in self.means) / k) / math.sqrt(k)


class OracleStandIn:
    def __init__(self, spinor, conf, index, m, burn, total, seed, block):
        orc = oracle_py.OracleSystem(spinor, conf)
        tr = orc.trajectory(seed=seed, stream=index, m=m, burn=burn, nsteps=total)
        self.values, self.imags = tr["est"][:, 0], tr["est"][:, 1]
        self.acc = Blocking(block)
        self.index = index
        self.pos = 0
        self.acceptance = tr["accepted"] / max(tr["proposed"], 1)

    def advance(self, n):
        for k in range(self.pos, self.pos + max(n, 0)):
            self.acc.add(self.values[k], self.imags[k])
        self.pos += max(n, 0)

    def summary(self):
        a = self.acc
        ratio = abs(a.imag) / abs(a.sum) if a.sum != 0 else abs(a.imag)
        return D.Summary(self.index, a.n, a.mean(), a.sigma_bar(), 0.0, ratio, len(a.means))


class OracleGroupStandIn:
    """Several stand-in workers on one rank (the HostGroup interface)."""

    def __init__(self, spinor, conf, first, count, m, burn, steps, total_workers, seed, block):
        self.first, self.count = first, count
        self.ws = [OracleStandIn(spinor, conf, first + k, m, burn,
                                 D.worker_share(steps, total_workers, first + k), seed, block) for k in range(count)]

    def advance(self, nsteps):
        for w, n in zip(self.ws, nsteps):
            w.advance(n)

    def summaries(self):
        return [w.summary() for w in self.ws]

    def records(self):
        """The Engine's worker record (driver.cpp:232-247) from the stand-in's accumulator; the
        ensemble section is a two-walker placeholder in WalkerEnsemble::save's line layout."""
        out = []
        for w in self.ws:
            a = w.acc
            r = repr  # shortest round-trip text, as the host's format_double
            txt = (f"worker {w.index}\nsteps {a.n}\nsums {r(float(a.sum))} {r(float(a.imag))}\n"
                   f"partial {a.inb} {r(float(a.partial))}\nblocks {len(a.means)}\n" +
                   "".join(r(float(b)) + "\n" for b in a.means) +
                   "ensemble\n2 0.5 10 5\n0 0 0 0 0 0\n" + "0 0 0 0 0 0 1 1 0\n" * 2 + "end-worker\n")
            out.append(txt.encode())
        return out

    def traces(self):
        out = []
        for w in self.ws:
            lines, n = [], 0
            for k in range(len(w.acc.means)):
                n += w.acc.nb
                lines.append(f"{n} {k} w{w.index}\n")
            out.append("".join(lines).encode())
        return out


def _group_rank(rank, world, port, args, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spinor, conf, m, burn, steps, interval, seed, block, workers = args
    first, count = D.rank_workers(workers, world, rank)
    g = OracleGroupStandIn(spinor, conf, first, count, m, burn, steps, workers, seed, block)
    gather = D.torch_all_gather(dist)
    files = None
    if os.environ.get("MCMP2_TEST_FILES"):
        ck, tr = os.environ["MCMP2_TEST_FILES"].split(":")
        text = conf + f"spinors {spinor}\nsteps {steps}\nworkers {workers}\ncheckpoint {ck}\ntrace {tr}\n"
        files = D.RunFiles(text, D.parse_run_config(text), rank, gather)
    rep = D.drive_group(g, workers, steps, None, interval, gather, files=files)
    q.put((rank, rep["value"], rep["sigma_bar"], rep["total_steps"], [(p.index, p.steps) for p in rep["workers"]]))
    dist.destroy_process_group()


def test_two_ranks_with_several_workers_each(cfgdir):
    """workers 5 over 2 ranks: ranks host workers [0, 3) and [3, 5) (the device path batches
    them in one handle per rank); the merge equals the oracle Engine with workers 5."""
    spinor = cfgdir / "syn1c.spinor"
    conf = "walkers 6\nburnin 30\nblocksize 10\ncheckpoint-interval 40\nseed 4\n"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    args = (str(spinor), conf, 6, 30, 203, 40, 4, 10, 5)
    procs = [ctx.Process(target=_group_rank, args=(r, 2, port, args, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert out[0][1:4] == out[1][1:4]
    assert [w for w in out[0][4]] == [(0, 41), (1, 41), (2, 41), (3, 40), (4, 40)]
    ref = parse_report(oracle_report(spinor, conf, "steps 203\nworkers 5\n"))
    assert out[0][3] == ref["steps"] == 203
    assert out[0][1] == pytest.approx(ref["value"], rel=1e-14, abs=0)
    assert out[0][2] == pytest.approx(ref["sigma_bar"], rel=1e-12, abs=0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, args, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spinor, conf, m, burn, steps, target, interval, seed, block = args
    total = steps if steps is not None else 4000
    w = OracleStandIn(spinor, conf, rank, m, burn, D.worker_share(total, world, rank) if steps else total, seed,
                      block)
    rep = D.drive(w, rank, world, steps, target, interval, D.torch_all_gather(dist))
    q.put((rank, rep["value"], rep["sigma_bar"], rep["total_steps"], rep["stopped_on_target"],
           [(p.index, p.steps, p.mean) for p in rep["workers"]]))
    dist.destroy_process_group()


def run_world(args, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(out)


def oracle_report(spinor, conf_text, extra):
    txt = conf_text + f"spinors {spinor}\n" + extra
    lines = [l for l in txt.splitlines() if not l.startswith("spinors ") or l == f"spinors {spinor}"]
    return oracle_py.run_config("\n".join(lines) + "\n")


def parse_report(rep):
    d = {}
    for line in rep.splitlines():
        if line.startswith("E2"):
            d["value"] = float(line.split()[2])
        elif line.startswith("sigma_bar"):
            d["sigma_bar"] = float(line.split()[2])
        elif line.startswith("steps"):
            d["steps"] = int(line.split()[2])
    return d


def test_two_ranks_match_oracle_two_workers(cfgdir):
    """Step budget split over 2 ranks == the oracle Engine with workers 2 (same streams)."""
    spinor = cfgdir / "syn1c.spinor"
    conf = "walkers 6\nburnin 30\nblocksize 10\ncheckpoint-interval 50\nseed 4\n"
    out = run_world((str(spinor), conf, 6, 30, 301, None, 50, 4, 10))
    rank0 = out[0]
    assert all(o[1:5] == rank0[1:5] for o in out)  # every rank sees the same merge
    ref = parse_report(oracle_report(spinor, conf, "steps 301\nworkers 2\n"))
    assert rank0[3] == ref["steps"] == 301
    assert [w[1] for w in rank0[5]] == [151, 150]
    assert rank0[1] == pytest.approx(ref["value"], rel=1e-14, abs=0)
    assert rank0[2] == pytest.approx(ref["sigma_bar"], rel=1e-12, abs=0)


def test_two_ranks_target_error_stop(cfgdir):
    """target-rel-err: stops at the first interval whose merged sigma_bar/|E| meets the target
    (driver.cpp:401-412), consistently on all ranks."""
    spinor = cfgdir / "syn1c.spinor"
    conf = "walkers 6\nburnin 30\nblocksize 10\ncheckpoint-interval 50\nseed 4\n"
    out = run_world((str(spinor), conf, 6, 30, None, 2.0, 50, 4, 10))
    assert all(o[4] for o in out)
    assert out[0][3] == 100  # both ranks at the first interval with blocks: 2 x 50
    ref = parse_report(oracle_report(spinor, conf, "target-rel-err 2.0\nworkers 2\n"))
    assert ref["steps"] == 100 and out[0][1] == pytest.approx(ref["value"], rel=1e-14)


def _device_rank(rank, world, port, text, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rc = D.parse_run_config(text)
    first, count = D.rank_workers(rc["workers"], world, rank)
    g = D.HostGroup(text, first, count, 0)  # both ranks on cuda:0 (no kernel waits on another rank)
    rep = D.drive_group(g, rc["workers"], rc["steps"], rc["target"], rc["interval"], D.torch_all_gather(dist))
    q.put((rank, D.format_report(rep)))
    g.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_device_groups_over_two_ranks_match_the_engine(cfgdir):
    """torch.distributed (gloo, 2 ranks on one GPU) with HostGroup: 4 cfg1 workers as two batched
    handles of 2 give the same report as the C++ Engine running the 4 workers in one batch."""
    from paper_2203_05632_b200 import walker
    text = (f"spinors {cfgdir / 'cfg1.spinor'}\nsteps 1002\nwalkers 16\nworkers 4\nseed 9\nburnin 50\n"
            "checkpoint-interval 200\nstep-size 0.3\n" +
            "".join(l + "\n" for l in (cfgdir / "cfg1.conf").read_text().splitlines() if l.startswith("weight")))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_rank, args=(r, 2, port, text, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert out[0][1] == out[1][1]
    assert out[0][1] == walker.run_config_text(text)


def _device_files_rank(rank, world, port, text, resume_from, max_intervals, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if resume_from:
        text, rc = D.checkpoint_run_config(resume_from)
    else:
        rc = D.parse_run_config(text)
    first, count = D.rank_workers(rc["workers"], world, rank)
    g = D.HostGroup(text, first, count, 0, resume_from)
    gather = D.torch_all_gather(dist)
    rep = D.drive_group(g, rc["workers"], rc["steps"], rc["target"], rc["interval"], gather,
                        max_intervals=max_intervals, files=D.RunFiles(text, rc, rank, gather))
    q.put((rank, D.format_report(rep)))
    g.close()
    dist.destroy_process_group()


def _run_device_files(text, resume_from=None, max_intervals=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_files_rank, args=(r, 2, port, text, resume_from, max_intervals, q))
             for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert out[0][1] == out[1][1]
    return out[0][1]


@pytest.mark.gpu
def test_device_groups_checkpoint_trace_and_resume_across_ranks(cfgdir, tmp_path):
    """Two ranks (gloo, one GPU), 4 cfg1 workers, `checkpoint` and `trace` set: the files rank 0
    assembles are byte-identical to the single-process Engine's (driver.cpp:218-251, 311-334);
    a run stopped after one interval and resumed across ranks, or by the single-process
    `resume`, ends on the uninterrupted report and checkpoint (SPEC: kill/resume matches an
    uninterrupted run)."""
    from paper_2203_05632_b200 import walker
    ck, tr = tmp_path / "run.ck", tmp_path / "run.trace"
    text = (f"spinors {cfgdir / 'cfg1.spinor'}\nsteps 1002\nwalkers 16\nworkers 4\nseed 9\nburnin 50\n"
            f"checkpoint-interval 200\nstep-size 0.3\nblocksize 25\ncheckpoint {ck}\ntrace {tr}\n" +
            "".join(l + "\n" for l in (cfgdir / "cfg1.conf").read_text().splitlines() if l.startswith("weight")))
    ref_report = walker.run_config_text(text)
    ref_ck, ref_tr = ck.read_bytes(), tr.read_bytes()
    assert ref_tr
    ck.unlink(), tr.unlink()

    assert _run_device_files(text) == ref_report
    assert ck.read_bytes() == ref_ck and tr.read_bytes() == ref_tr
    ck.unlink(), tr.unlink()

    partial = _run_device_files(text, max_intervals=1)
    assert partial != ref_report and b"\nsteps 200\n" in ck.read_bytes()
    stopped = ck.read_bytes()
    assert _run_device_files(None, resume_from=str(ck)) == ref_report
    assert ck.read_bytes() == ref_ck and tr.read_bytes() == ref_tr

    ck.write_bytes(stopped)  # the same stopped run continued by the single-process Engine
    assert walker.resume(ck) == ref_report
    assert ck.read_bytes() == ref_ck

    ck.write_bytes(stopped.replace(b"end-worker\n", b"", 1))
    with pytest.raises(Exception, match="checkpoint"):
        D.HostGroup("", 0, 2, 0, str(ck))


def test_fewer_workers_than_ranks_is_an_error():
    """rank_workers refuses to raise the worker count (it would change the run's streams and
    shares, which the config hash names); an exact split is accepted."""
    with pytest.raises(ValueError, match="workers 1 < world size 2"):
        D.rank_workers(1, 2, 0)
    assert [D.rank_workers(2, 2, r) for r in range(2)] == [(0, 1), (1, 1)]


def test_checkpoint_and_trace_assembled_on_rank_0(cfgdir, tmp_path, monkeypatch):
    """workers 5 over 2 ranks with `checkpoint` and `trace` set: rank 0 writes one checkpoint
    holding all five records in worker order behind the host's header (driver.cpp:218-251), which
    the host's `merge` (driver.cpp:502-521) reads back to the run's own merged estimate; the
    per-worker trace files are joined in worker order at the end (driver.cpp:323-334)."""
    from paper_2203_05632_b200 import walker
    spinor = cfgdir / "syn1c.spinor"
    conf = "walkers 6\nburnin 30\nblocksize 10\ncheckpoint-interval 40\nseed 4\n"
    ck, tr = tmp_path / "run.ck", tmp_path / "run.trace"
    monkeypatch.setenv("MCMP2_TEST_FILES", f"{ck}:{tr}")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    args = (str(spinor), conf, 6, 30, 203, 40, 4, 10, 5)
    procs = [ctx.Process(target=_group_rank, args=(r, 2, port, args, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    text = ck.read_text()
    assert text.startswith("mcmp2-checkpoint 1\nconfighash ") and "workers 5\nworker 0\n" in text
    assert [int(l.split()[1]) for l in text.splitlines() if l.startswith("worker ")] == [0, 1, 2, 3, 4]
    assert not ck.with_suffix(".ck.tmp").exists()
    value, sigma_bar, steps = walker.merge([ck])
    assert steps == out[0][3] == 203
    assert value == pytest.approx(out[0][1], rel=1e-15, abs=0)
    assert sigma_bar == pytest.approx(out[0][2], rel=1e-13, abs=0)
    lines = tr.read_text().splitlines()
    assert [l.split()[2] for l in lines] == [f"w{k}" for k in range(5) for _ in range(4)]
    assert not list(tmp_path.glob("run.trace.w*"))


def test_gather_bytes_and_framing():
    """The byte gather pads to the longest rank's blob and cuts each back to its own length;
    the framing round-trips empty and binary items."""
    blobs = [b"", b"abc\x00\xff", b"x" * 1000]
    for mine in range(3):
        def all_gather(a, mine=mine):
            if a.dtype == np.int64:
                return [np.array([len(b)], dtype=np.int64) for b in blobs]
            return [np.frombuffer(b.ljust(len(a), b"\0"), dtype=np.uint8) for b in blobs]
        assert D.gather_bytes(all_gather, blobs[mine]) == blobs
    items = [b"", b"\x00\x01", b"worker 3\n"]
    assert D._unpack(D._pack(items)) == items and D._unpack(D._pack([])) == []


@pytest.mark.parametrize("which", ["checkpoint", "trace"])
def test_run_files_with_only_one_of_checkpoint_and_trace(cfgdir, tmp_path, which):
    """A config naming only one of the two files: the gathered sections are told apart by their
    count, the other file is not written (single rank, identity gather)."""
    class Group:
        first, count = 0, 2

        def records(self):
            return [b"worker 0\nend-worker\n", b"worker 1\nend-worker\n"]

        def traces(self):
            return [b"10 a\n", b"10 b\n"]

    path = tmp_path / f"run.{which}"
    text = f"spinors {cfgdir / 'syn1c.spinor'}\nsteps 10\nworkers 2\n{which} {path}\n"
    files = D.RunFiles(text, D.parse_run_config(text), 0, lambda a: [a])
    assert files
    files.write_interval(Group())
    files.finish()
    if which == "checkpoint":
        body = path.read_bytes()
        assert body.startswith(b"mcmp2-checkpoint 1\n") and body.endswith(b"workers 2\n" + b"".join(Group().records()))
    else:
        assert path.read_bytes() == b"10 a\n10 b\n"
    assert sorted(p.name for p in tmp_path.iterdir()) == [path.name]
    none = f"spinors {cfgdir / 'syn1c.spinor'}\nsteps 10\nworkers 2\n"
    assert not D.RunFiles(none, D.parse_run_config(none), 0, lambda a: [a])

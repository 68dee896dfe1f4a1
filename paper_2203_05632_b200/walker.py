"""Python mirror of the reference's per-worker walker interface over the device C ABI.

Reference surface (proj/core/include/mcmp2/): init_ensemble / burn_in / metropolis_step
(sampler.hpp:53-64), TauSampler::sample (weights.hpp:58), mc_step_estimate / sample_term
(estimator.hpp:51-57), WalkerEnsemble save/load (sampler.hpp:36-37). Every method is one
C-ABI call into lib/libmcmp2dev.so; errors come back as the reference's exception kinds
(Mcmp2ArgumentError ~ std::invalid_argument, Mcmp2Error ~ std::runtime_error).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import native
from .native import StepEx, Ensemble, Step, check_dev, check_host, dptr


class System:
    """SpinorSet + WeightSpec + TauSampler loaded by the C++ host (model.cpp:275-351)."""

    def __init__(self, spinor_path: str | Path, config_text: str = ""):
        h = native.host()
        self._h = h.mcmp2h_system_load(str(spinor_path).encode(), config_text.encode())
        if not self._h:
            msg = h.mcmp2h_last_error().decode()
            if msg.startswith(("no weight parameters", "Molecule", "BasisFunction", "SpinorSet: component",
                               "SpinorSet: one basis", "SpinorSet: invalid", "SpinorSet: empty")):
                raise native.Mcmp2ArgumentError(msg)
            raise native.Mcmp2Error(msg)
        ints = (C.c_int * 4)()
        dbl = (C.c_double * 3)()
        check_host(h.mcmp2h_system_info(self._h, ints, dbl))
        self.ncomp, self.n_occ, self.n_vir, self.rows = list(ints)
        self.ng, self.lambda_, self.orthonormality_deviation = list(dbl)

    @property
    def view(self):
        return native.host().mcmp2h_system_view(self._h)

    def g(self, pts: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.empty(len(pts))
        check_host(native.host().mcmp2h_system_g(self._h, dptr(pts), len(pts), dptr(out)))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            native.host().mcmp2h_system_free(self._h)
            self._h = None


@dataclass
class EnsembleState:
    """WalkerEnsemble record (sampler.cpp:95-120): walkers [m, 9] = r1, r2, g1, g2, weight."""
    walkers: np.ndarray
    sigma_step: float
    proposed: int
    accepted: int
    rng_key: tuple
    rng_counter: tuple
    rng_idx: int


class DeviceWalker:
    """One reference worker resident on one GPU (a mcmp2dev handle)."""

    def __init__(self, system: System, device: int = 0, max_walkers: int = 8):
        self.system = system
        self._d = native.dev()
        h = C.c_void_p()
        check_dev(self._d.mcmp2dev_create(system.view, device, max_walkers, C.byref(h)), None)
        self._h = h
        self.max_walkers = max_walkers
        self.m = 0

    # -- ensemble -------------------------------------------------------------------
    def init_ensemble(self, m: int, seed: int, stream: int = 0) -> None:
        check_dev(self._d.mcmp2dev_init_ensemble(self._h, m, seed, stream), self._h)
        self.m = m
        self.nens = 1

    def burn_in(self, n_burn: int, adapt: bool = True) -> None:
        check_dev(self._d.mcmp2dev_burn_in(self._h, n_burn, int(adapt)), self._h)

    def set_sigma_step(self, sigma: float) -> None:
        check_dev(self._d.mcmp2dev_set_sigma_step(self._h, sigma), self._h)

    def init_batch(self, nens: int, m: int, seed: int, stream0: int = 0) -> None:
        """nens reference workers in this handle: ensemble e = init_ensemble(m, seed, stream0 + e);
        advance() then returns [nsteps, nens] arrays (include/mcmp2dev.h, batched ensembles)."""
        check_dev(self._d.mcmp2dev_init_batch(self._h, nens, m, seed, stream0), self._h)
        self.m = m
        self.nens = nens

    def get_ensemble_at(self, ens: int) -> EnsembleState:
        w = np.zeros((self.m, 9))
        e = Ensemble()
        e.walkers = dptr(w)
        check_dev(self._d.mcmp2dev_get_ensemble_at(self._h, ens, C.byref(e)), self._h)
        return EnsembleState(w.copy(), e.sigma_step, e.proposed, e.accepted, tuple(e.rng_key),
                             tuple(e.rng_counter), e.rng_idx)

    def set_ensemble_at(self, ens: int, s: EnsembleState) -> None:
        w = np.ascontiguousarray(s.walkers, dtype=np.float64)
        e = Ensemble()
        e.m = len(w)
        e.sigma_step = s.sigma_step
        e.proposed = s.proposed
        e.accepted = s.accepted
        e.rng_key[:] = s.rng_key
        e.rng_counter[:] = s.rng_counter
        e.rng_idx = s.rng_idx
        e.walkers = dptr(w)
        check_dev(self._d.mcmp2dev_set_ensemble_at(self._h, ens, C.byref(e)), self._h)

    def get_ensembles(self) -> list[EnsembleState]:
        """Every ensemble of a batched handle in two device copies."""
        ne = getattr(self, "nens", 1)
        ws = [np.zeros((self.m, 9)) for _ in range(ne)]
        arr = (Ensemble * ne)()
        for k in range(ne):
            arr[k].walkers = dptr(ws[k])
        check_dev(self._d.mcmp2dev_get_ensembles(self._h, arr), self._h)
        return [EnsembleState(ws[k], arr[k].sigma_step, arr[k].proposed, arr[k].accepted, tuple(arr[k].rng_key),
                              tuple(arr[k].rng_counter), arr[k].rng_idx) for k in range(ne)]

    def set_ensembles(self, states) -> None:
        ne = len(states)
        ws = [np.ascontiguousarray(s.walkers, dtype=np.float64) for s in states]
        arr = (Ensemble * ne)()
        for k, s in enumerate(states):
            e = arr[k]
            e.m = len(ws[k])
            e.sigma_step = s.sigma_step
            e.proposed = s.proposed
            e.accepted = s.accepted
            e.rng_key[:] = s.rng_key
            e.rng_counter[:] = s.rng_counter
            e.rng_idx = s.rng_idx
            e.walkers = dptr(ws[k])
        check_dev(self._d.mcmp2dev_set_ensembles(self._h, arr), self._h)

    def get_ensemble(self) -> EnsembleState:
        w = np.zeros((self.max_walkers, 9))
        e = Ensemble()
        e.walkers = dptr(w)
        check_dev(self._d.mcmp2dev_get_ensemble(self._h, C.byref(e)), self._h)
        return EnsembleState(w[: e.m].copy(), e.sigma_step, e.proposed, e.accepted, tuple(e.rng_key),
                             tuple(e.rng_counter), e.rng_idx)

    def set_ensemble(self, s: EnsembleState) -> None:
        w = np.ascontiguousarray(s.walkers, dtype=np.float64)
        e = Ensemble()
        e.m = len(w)
        e.sigma_step = s.sigma_step
        e.proposed = s.proposed
        e.accepted = s.accepted
        e.rng_key[:] = s.rng_key
        e.rng_counter[:] = s.rng_counter
        e.rng_idx = s.rng_idx
        e.walkers = dptr(w)
        check_dev(self._d.mcmp2dev_set_ensemble(self._h, C.byref(e)), self._h)
        self.m = len(w)
        self.nens = 1

    # -- hot loop -------------------------------------------------------------------
    def advance(self, nsteps: int, keep_on_device: bool = False):
        if keep_on_device:
            check_dev(self._d.mcmp2dev_advance(self._h, nsteps, None, None), self._h)
            return None
        ne = getattr(self, "nens", 1)
        v = np.empty((nsteps, ne) if ne > 1 else nsteps)
        im = np.empty_like(v)
        check_dev(self._d.mcmp2dev_advance(self._h, nsteps, dptr(v), dptr(im)), self._h)
        return v, im

    def prepare(self) -> None:
        """Capture the CUDA graphs advance() replays (setup cost, executes nothing)."""
        check_dev(self._d.mcmp2dev_prepare(self._h), self._h)

    def replay(self, walkers: np.ndarray, tau: np.ndarray) -> np.ndarray:
        """mc_step_estimate at given positions: walkers [nsteps, m, 8], tau [nsteps] ->
        [nsteps, 6] = value, imag, direct re/im, exchange re/im (sums before /C(m,2))."""
        walkers = np.ascontiguousarray(walkers, dtype=np.float64)
        if walkers.ndim == 2:
            walkers = walkers[None]
        tau = np.ascontiguousarray(np.atleast_1d(tau), dtype=np.float64)
        n, m, _ = walkers.shape
        out = (Step * n)()
        check_dev(self._d.mcmp2dev_replay(self._h, m, n, dptr(walkers), dptr(tau), out), self._h)
        return np.array([[s.value, s.imag, s.direct_re, s.direct_im, s.exchange_re, s.exchange_im]
                         for s in out])

    STEP_EX_FIELDS = ("value", "imag", "direct_re", "direct_im", "exchange_re", "exchange_im",
                      "est_err_direct", "est_err_exchange", "abs_direct", "abs_exchange", "int8_v", "fallback")

    @classmethod
    def _ex_array(cls, out) -> np.ndarray:
        return np.array([[getattr(s, f) for f in cls.STEP_EX_FIELDS] for s in out], dtype=np.float64)

    def advance_ex(self, nsteps: int) -> np.ndarray:
        """advance() returning the full per-step record [nsteps, 12] (STEP_EX_FIELDS): the
        value and pair sums, the INT8 path's guard estimate, |term| sums and flags."""
        out = (StepEx * max(nsteps, 1))()
        check_dev(self._d.mcmp2dev_advance_ex(self._h, nsteps, out), self._h)
        return self._ex_array(out[:nsteps])

    def replay_ex(self, walkers: np.ndarray, tau: np.ndarray) -> np.ndarray:
        """replay() with the full per-step record [nsteps, 12] (STEP_EX_FIELDS)."""
        walkers = np.ascontiguousarray(walkers, dtype=np.float64)
        if walkers.ndim == 2:
            walkers = walkers[None]
        tau = np.ascontiguousarray(np.atleast_1d(tau), dtype=np.float64)
        n, m, _ = walkers.shape
        out = (StepEx * n)()
        check_dev(self._d.mcmp2dev_replay_ex(self._h, m, n, dptr(walkers), dptr(tau), out), self._h)
        return self._ex_array(out)

    def guard(self, tol: float | None = None) -> float:
        """The INT8 path's accuracy guard tolerance (<= 0: off); sets it when tol is given and
        returns the previous value."""
        prev = C.c_double()
        check_dev(self._d.mcmp2dev_guard(self._h, float("nan") if tol is None else float(tol), C.byref(prev)),
                  self._h)
        return prev.value

    def guard_stats(self) -> dict:
        """{checked, refined, dmma, max_est_rel, tol} since the last call (the call resets them)."""
        o = np.zeros(5)
        check_dev(self._d.mcmp2dev_guard_stats(self._h, dptr(o)), self._h)
        return {"checked": int(o[0]), "refined": int(o[1]), "dmma": int(o[2]), "max_est_rel": float(o[3]),
                "tol": float(o[4])}

    # -- instrumentation ------------------------------------------------------------
    def profile(self, enable: bool = True, reset: bool = True) -> dict:
        out = np.zeros(8)
        oz = np.zeros(6)  # the INT8 V path's kernels, read before a reset
        check_dev(self._d.mcmp2dev_profile_pair(self._h, dptr(oz)), self._h)
        check_dev(self._d.mcmp2dev_profile(self._h, int(enable), int(reset), dptr(out)), self._h)
        names = ("walk", "spinor", "pair", "total")
        res = {"ms": dict(zip(names, out[:4])), "launches": dict(zip(names, out[4:].astype(int)))}
        res["int8_v"] = {"slice_ms": oz[0], "vgemm_ms": oz[1], "pair_kr_ms": oz[2], "steps": int(oz[3]),
                         "vgemm_int8_ops": oz[4], "guard_ms": oz[5]}
        return res

    def work(self) -> dict:
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        check_dev(self._d.mcmp2dev_work(self._h, C.byref(a), C.byref(b), C.byref(c)), self._h)
        e = C.c_double()
        check_dev(self._d.mcmp2dev_work_executed(self._h, C.byref(e)), self._h)
        return {"pair_flop": a.value, "spinor_flop": b.value, "phi_bytes": c.value,
                "pair_dmma_flop_executed": e.value}

    def kramers(self, mode: int = -1) -> bool:
        """Kramers-restricted pair kernel: -1 query, 0 off, 1 on when eligible."""
        return bool(self._d.mcmp2dev_kramers(self._h, mode))

    def kramers_deviation(self) -> float:
        """Deviation of the spinor columns from exact time-reversal pairing (inf: no pairing)."""
        d = C.c_double()
        check_dev(self._d.mcmp2dev_kramers_deviation(self._h, C.byref(d)), self._h)
        return d.value

    def int8_v(self, mode: int = -1) -> bool:
        """V blocks of the Kramers pair stage on the INT8 tensor cores (Ozaki slices,
        csrc/pair_oz.cu): -1 query, 0 DMMA, 1 INT8 (default). True when selected and eligible;
        it runs for single ensembles whose 16 x 8 pair tiles cover the SMs (m >= ~180)."""
        return bool(self._d.mcmp2dev_pair_path(self._h, mode))

    def int8_truncation(self, mode: int = -1) -> bool:
        """Energy-ordered truncation of the INT8 V-GEMM's K loop (exact; on by default):
        -1 query, 0 every k-step, 1 only the slice products whose slices hold a nonzero digit in the
        k-step (whole k-steps and leading zero slices skipped), 2 whole empty k-steps only."""
        return bool(self._d.mcmp2dev_oz_truncation(self._h, mode))

    def int8_overlap(self, mode: int = -1) -> bool:
        """oz_slice_kernel on a side stream next to the O pass: -1 query, 0 in series, 1 overlapped
        (default)."""
        return bool(self._d.mcmp2dev_oz_overlap(self._h, mode))

    def int8_ksteps(self) -> tuple[float, float]:
        """(k-steps issued by the main-pass V-GEMM launches so far, k-steps of one full launch)."""
        o = np.zeros(2)
        check_dev(self._d.mcmp2dev_oz_ksteps(self._h, dptr(o)), self._h)
        return float(o[0]), float(o[1])

    @property
    def stream_ptr(self) -> int:
        return int(self._d.mcmp2dev_stream(self._h))

    def synchronize(self) -> None:
        check_dev(self._d.mcmp2dev_synchronize(self._h), self._h)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._d.mcmp2dev_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def generate_config(name: str, directory: str | Path) -> tuple[Path, Path]:
    """Writes <dir>/<name>.spinor and <dir>/<name>.conf (host/generate.cpp)."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    check_host(native.host().mcmp2h_generate(name.encode(), str(d).encode()))
    return d / f"{name}.spinor", d / f"{name}.conf"


def run_config_text(text: str, abort_after_intervals: int = -1) -> str:
    """`mcmp2 run` on config text through the C++ host; returns format_report text."""
    buf = C.create_string_buffer(1 << 16)
    h = native.host()
    check_host(h.mcmp2h_run_hooked(text.encode(), abort_after_intervals, buf, len(buf)))
    return buf.value.decode()


def resume(checkpoint: str | Path) -> str:
    buf = C.create_string_buffer(1 << 16)
    check_host(native.host().mcmp2h_resume(str(checkpoint).encode(), buf, len(buf)))
    return buf.value.decode()


def merge(paths) -> tuple[float, float, int]:
    arr = (C.c_char_p * len(paths))(*[str(p).encode() for p in paths])
    v, s, n = C.c_double(), C.c_double(), C.c_longlong()
    check_host(native.host().mcmp2h_merge(arr, len(paths), C.byref(v), C.byref(s), C.byref(n)))
    return v.value, s.value, n.value

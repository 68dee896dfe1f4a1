"""ctypes wrapper of the CPU oracle (oracle/build/liboracle.so) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_LIB = ROOT / "oracle" / "build" / "liboracle.so"
REF_LIB = ROOT / "oracle" / "_ref" / "libref_rng.so"

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_LIB.exists():
            raise ImportError(f"{ORACLE_LIB} missing: run `make -C oracle`")
        L = C.CDLL(str(ORACLE_LIB))
        vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.c_int
        L.orc_last_error.restype = C.c_char_p
        L.orc_philox_block.argtypes = [C.POINTER(C.c_uint32)] * 3
        L.orc_philox_stream.argtypes = [C.c_uint64, C.c_uint32, ip, ip, dp]
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_fnv1a64.argtypes = [C.c_char_p, C.c_long]
        L.orc_boys_f0.restype = C.c_double
        L.orc_boys_f0.argtypes = [C.c_double]
        L.orc_primitive_norm.restype = C.c_double
        L.orc_primitive_norm.argtypes = [ip, C.c_double]
        L.orc_solid_harmonic.restype = C.c_double
        L.orc_solid_harmonic.argtypes = [ip, ip, C.c_double, C.c_double, C.c_double]
        L.orc_guarded_exp.argtypes = [C.c_double, ip, dp]
        L.orc_system_load.restype = vp
        L.orc_system_load.argtypes = [C.c_char_p, C.c_char_p]
        L.orc_system_free.argtypes = [vp]
        L.orc_system_info.argtypes = [vp, C.POINTER(C.c_int), dp]
        L.orc_g.argtypes = [vp, dp, ip, dp]
        L.orc_evaluate.argtypes = [vp, dp, ip, dp, dp]
        L.orc_trajectory.argtypes = [vp, C.c_uint64, C.c_uint32, ip, C.c_long, C.c_double, ip, C.c_long,
                                     ip, dp, dp, dp, dp, dp, C.POINTER(C.c_longlong)]
        L.orc_replay.argtypes = [vp, ip, C.c_long, dp, dp, ip, dp]
        L.orc_sample_term.argtypes = [vp, dp, dp, C.c_double, ip, dp]
        L.orc_run_config.argtypes = [C.c_char_p, C.c_char_p, ip]
        L.orc_resume.argtypes = [C.c_char_p, C.c_char_p, ip]
        L.orc_tau_sample.restype = C.c_double
        L.orc_tau_sample.argtypes = [C.c_double, C.c_double]
        L.orc_blocking.argtypes = [dp, C.c_long, C.c_long, dp]
        L.orc_cpu_baseline.argtypes = [vp, C.c_uint64, ip, ip, C.c_long, C.c_double, C.c_long, ip, dp,
                                       C.POINTER(C.c_longlong)]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def check(rc):
    if rc:
        raise RuntimeError(lib().orc_last_error().decode())


class OracleSystem:
    def __init__(self, spinor_path, config_text=""):
        self.h = lib().orc_system_load(str(spinor_path).encode(), config_text.encode())
        if not self.h:
            raise RuntimeError(lib().orc_last_error().decode())
        ints = (C.c_int * 5)()
        dbl = (C.c_double * 2)()
        lib().orc_system_info(self.h, ints, dbl)
        self.ncomp, self.n_occ, self.n_vir, self.rows, self.nsites = list(ints)
        self.ng, self.lambda_ = list(dbl)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_system_free(self.h)

    def g(self, pts):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.empty(len(pts))
        lib().orc_g(self.h, _d(pts), len(pts), _d(out))
        return out

    def evaluate(self, pts):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        n = len(pts)
        occ = np.empty((n, self.ncomp, self.n_occ, 2))
        vir = np.empty((n, self.ncomp, self.n_vir, 2))
        lib().orc_evaluate(self.h, _d(pts), n, _d(occ), _d(vir))
        return occ[..., 0] + 1j * occ[..., 1], vir[..., 0] + 1j * vir[..., 1]

    def trajectory(self, seed, stream, m, burn, nsteps, step_size=0.0, adapt=True, physical=False):
        init = np.empty(9 * m + 8)
        fin = np.empty(9 * m + 8)
        walkers = np.empty((nsteps, m, 8))
        tau = np.empty(nsteps)
        est = np.empty((nsteps, 6))
        cnt = (C.c_longlong * 2)()
        check(lib().orc_trajectory(self.h, seed, stream, m, burn, step_size, int(adapt), nsteps, int(physical),
                                   _d(init), _d(walkers), _d(tau), _d(est), _d(fin), cnt))
        return dict(init=init, final=fin, walkers=walkers, tau=tau, est=est, proposed=cnt[0], accepted=cnt[1])

    def replay(self, walkers, tau, physical=False):
        walkers = np.ascontiguousarray(walkers, dtype=np.float64)
        tau = np.ascontiguousarray(np.atleast_1d(tau), dtype=np.float64)
        n, m, _ = walkers.shape
        est = np.empty((n, 6))
        check(lib().orc_replay(self.h, m, n, _d(walkers), _d(tau), int(physical), _d(est)))
        return est

    def chain_r12(self, seed, m, burn, nsteps, thin):
        """Metropolis-only chain: (|r1 - r2| samples every `thin` sweeps, production acceptance)."""
        u = np.empty(((nsteps + thin - 1) // thin) * m)
        acc = C.c_double()
        check(lib().orc_chain_r12(self.h, C.c_uint64(seed), int(m), C.c_long(burn), C.c_long(nsteps),
                                  C.c_long(thin), _d(u), C.byref(acc)))
        return u, acc.value

    def replay_parallel(self, walkers, tau, threads, physical=False):
        """One full-size replay step (m x 8 walkers), pair rows split over `threads` threads."""
        walkers = np.ascontiguousarray(walkers, dtype=np.float64)
        est = np.empty(6)
        check(lib().orc_replay_parallel(self.h, walkers.shape[0], _d(walkers), C.c_double(tau), int(threads),
                                        int(physical), _d(est)))
        return est

    def sample_term(self, p, q, tau, physical=False):
        p = np.ascontiguousarray(p, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        out = np.empty(4)
        check(lib().orc_sample_term(self.h, _d(p), _d(q), tau, int(physical), _d(out)))
        return complex(out[0], out[1]), complex(out[2], out[3])

    def cpu_baseline(self, seed, m, rows, burn, step_size, steps, threads):
        sec = C.c_double()
        n = C.c_longlong()
        check(lib().orc_cpu_baseline(self.h, seed, m, rows, burn, step_size, steps, threads, C.byref(sec),
                                     C.byref(n)))
        return sec.value, n.value


def state_to_ensemble(state: np.ndarray, m: int):
    """oracle dump (m x 9 walkers, sigma, key0, key1, c0..c3, idx) -> walker.EnsembleState kwargs."""
    w = state[: 9 * m].reshape(m, 9).copy()
    t = state[9 * m:]
    return dict(walkers=w, sigma_step=float(t[0]), proposed=0, accepted=0,
                rng_key=(int(t[1]), int(t[2])), rng_counter=tuple(int(x) for x in t[3:7]), rng_idx=int(t[7]))


def run_config(text: str) -> str:
    buf = C.create_string_buffer(1 << 16)
    check(lib().orc_run_config(text.encode(), buf, len(buf)))
    return buf.value.decode()

"""ctypes wrapper of oracle/_ref/libref_mcmp2.so -- the REFERENCE's own rng, gaussian, model,
weights, sampler, greens, estimator and driver translation units, compiled unmodified by
oracle/build_ref.sh against oracle/eigen_subset. TEST INFRASTRUCTURE ONLY (tests/ and nothing
else); absent when the reference sources were not available at build time."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF_LIB = ROOT / "oracle" / "_ref" / "libref_mcmp2.so"
_lib = None


def available() -> bool:
    return REF_LIB.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        L = C.CDLL(str(REF_LIB))
        vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.c_int
        L.ref2_last_error.restype = C.c_char_p
        L.ref2_system_load.restype = vp
        L.ref2_system_load.argtypes = [C.c_char_p, C.c_char_p]
        L.ref2_system_free.argtypes = [vp]
        L.ref2_system_info.argtypes = [vp, C.POINTER(C.c_int), dp]
        L.ref2_replay.argtypes = [vp, ip, C.c_long, dp, dp, ip, dp]
        L.ref2_evaluate.argtypes = [vp, dp, ip, dp, dp]
        L.ref2_g.argtypes = [vp, dp, ip, dp]
        L.ref2_run_config.argtypes = [C.c_char_p, C.c_char_p, ip]
        L.ref2_fixture.argtypes = [C.c_char_p, C.c_char_p, dp]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(rc):
    if rc:
        raise RuntimeError(lib().ref2_last_error().decode())


class RefSystem:
    """SpinorSet + WeightSpec + TauSampler as the reference Engine builds them."""

    def __init__(self, spinor_path, config_text=""):
        self.h = lib().ref2_system_load(str(spinor_path).encode(), config_text.encode())
        if not self.h:
            raise RuntimeError(lib().ref2_last_error().decode())
        ints = (C.c_int * 3)()
        dbl = (C.c_double * 2)()
        _check(lib().ref2_system_info(self.h, ints, dbl))
        self.ncomp, self.n_occ, self.n_vir = list(ints)
        self.ng, self.lambda_ = list(dbl)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref2_system_free(self.h)

    def replay(self, walkers, tau, pair_sums=True):
        """[nsteps, 6]: value, imag (mc_step_estimate), direct re/im, exchange re/im (sample_term sums)"""
        walkers = np.ascontiguousarray(walkers, dtype=np.float64)
        if walkers.ndim == 2:
            walkers = walkers[None]
        tau = np.ascontiguousarray(np.atleast_1d(tau), dtype=np.float64)
        n, m, _ = walkers.shape
        out = np.zeros((n, 6))
        _check(lib().ref2_replay(self.h, m, n, _d(walkers), _d(tau), int(pair_sums), _d(out)))
        return out

    def evaluate(self, pts):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        n = len(pts)
        occ = np.empty((n, self.ncomp, self.n_occ, 2))
        vir = np.empty((n, self.ncomp, self.n_vir, 2))
        _check(lib().ref2_evaluate(self.h, _d(pts), n, _d(occ), _d(vir)))
        return occ[..., 0] + 1j * occ[..., 1], vir[..., 0] + 1j * vir[..., 1]

    def g(self, pts):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.empty(len(pts))
        _check(lib().ref2_g(self.h, _d(pts), len(pts), _d(out)))
        return out


def run_config(text: str) -> str:
    """The reference Engine: run(parse_config_text(text)) -> format_report."""
    buf = C.create_string_buffer(1 << 16)
    _check(lib().ref2_run_config(text.encode(), buf, len(buf)))
    return buf.value.decode()


def fixture(name: str, spinor_out=None) -> float:
    """The reference oracle's fixture (oracle.cpp make_fixture): its deterministic MP2 energy,
    and its SPINOR-TEXT written to spinor_out when given."""
    e2 = C.c_double()
    _check(lib().ref2_fixture(name.encode(), str(spinor_out or "").encode(), C.byref(e2)))
    return e2.value

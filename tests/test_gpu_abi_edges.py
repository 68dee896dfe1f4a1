"""Edge cases through the raw C ABI, with mcmp2dev_system built from plain arrays (no host
library): the reference's zero-virtual and coincident-electron tests (test_estimator.cpp:91-113)
and argument errors."""
import ctypes as C
import math

import numpy as np
import pytest

from paper_2203_05632_b200 import native
from paper_2203_05632_b200.native import Mcmp2ArgumentError, Step, check_dev, dptr

pytestmark = pytest.mark.gpu

dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)


class SystemC(C.Structure):  # mcmp2dev_system (include/mcmp2dev.h)
    _fields_ = [("ncomp", C.c_int), ("n_occ", C.c_int), ("n_vir", C.c_int), ("channel_count", ip),
                ("fn_center", dp), ("fn_lm", ip), ("fn_prim_offset", ip), ("prim_zeta", dp), ("prim_coeff", dp),
                ("coeff", dp), ("energies", dp), ("nsites", C.c_int), ("site_pos", dp), ("site_prim", dp),
                ("site_zeta1", dp), ("ng", C.c_double), ("lambda_", C.c_double), ("w_direct", C.c_double),
                ("w_exchange", C.c_double), ("estimator", C.c_int)]


def one_s_system(n_vir, lam=1.0):
    """1c, He-like centre, one normalised s function per spinor column (occupied first)."""
    nfn = 1 + n_vir
    zetas = [0.8] + [0.3 + 0.5 * k for k in range(n_vir)]
    keep = []

    def arr(v, t=np.float64):
        a = np.ascontiguousarray(v, dtype=t)
        keep.append(a)
        return a.ctypes.data_as(ip if t == np.int32 else dp)

    coeff = np.zeros((nfn, nfn, 2))
    for k in range(nfn):
        coeff[k, k, 0] = 1.0  # not orthonormal across functions: the ABI does not check that
    s = SystemC()
    s.ncomp, s.n_occ, s.n_vir = 1, 1, n_vir
    s.channel_count = arr([nfn], np.int32)
    s.fn_center = arr(np.zeros(3 * nfn))
    s.fn_lm = arr(np.zeros(2 * nfn), np.int32)
    s.fn_prim_offset = arr(np.arange(nfn + 1), np.int32)
    s.prim_zeta = arr(zetas)
    s.prim_coeff = arr([(2 * z / math.pi) ** 0.75 / 0.28209479177387814 for z in zetas])
    s.coeff = arr(coeff.ravel())
    s.energies = arr([-0.9] + [0.5 + 0.3 * k for k in range(n_vir)])
    s.nsites = 1
    s.site_pos = arr([0.0, 0.0, 0.0])
    s.site_prim = arr([0.5 * (2 * 0.3 / math.pi) ** 0.75, 0.3, 0.5 * (2 * 1.0 / math.pi) ** 0.75, 1.0])
    s.site_zeta1 = arr([0.3])
    s.ng, s.lambda_, s.w_direct, s.w_exchange, s.estimator = 1.0, lam, 2.0, -1.0, 0
    return s, keep


def create(s, m):
    d = native.dev()
    h = C.c_void_p()
    check_dev(d.mcmp2dev_create(C.byref(s), 0, m, C.byref(h)), None)
    return d, h


def replay(d, h, walkers, tau):
    w = np.ascontiguousarray(walkers, dtype=np.float64)
    out = (Step * 1)()
    check_dev(d.mcmp2dev_replay(h, w.shape[0], 1, dptr(w), dptr(np.array([tau])), out), h)
    return out[0]


def test_zero_virtual_spinors_give_a_vanishing_sample():
    s, keep = one_s_system(0)
    d, h = create(s, 2)
    w = np.array([[0.1, 0, 0, 0, 0.2, 0, 0.3, 0.3], [0, 0, 0.3, 0.4, 0, 0, 0.3, 0.3]])
    st = replay(d, h, w, 0.2)
    assert st.value == 0.0 and st.imag == 0.0
    d.mcmp2dev_destroy(h)


def test_coincident_electrons_stay_finite():
    s, keep = one_s_system(3)
    d, h = create(s, 2)
    w = np.array([[0.3, 0.3, 0.3, 0.3, 0.3, 0.3, 0.2, 0.2], [-0.2, 0.5, 0, 0.4, 0, 0.6, 0.1, 0.1]])
    st = replay(d, h, w, 0.4)
    assert math.isfinite(st.value) and st.value != 0.0
    d.mcmp2dev_destroy(h)


def test_argument_errors_keep_reference_messages():
    s, keep = one_s_system(2)
    d = native.dev()
    h = C.c_void_p()
    s.ncomp = 3
    assert d.mcmp2dev_create(C.byref(s), 0, 4, C.byref(h)) == native.INVALID_ARGUMENT
    assert b"component count must be 1, 2 or 4" in d.mcmp2dev_last_error(None)
    s.ncomp = 1
    s.lambda_ = 0.0
    assert d.mcmp2dev_create(C.byref(s), 0, 4, C.byref(h)) == native.INVALID_ARGUMENT
    assert b"lambda must be positive" in d.mcmp2dev_last_error(None)
    s.lambda_ = 1.0
    d, h = create(s, 4)
    with pytest.raises(Mcmp2ArgumentError, match="at least two"):
        check_dev(d.mcmp2dev_init_ensemble(h, 1, 1, 0), h)
    with pytest.raises(Mcmp2ArgumentError, match="sized for"):
        check_dev(d.mcmp2dev_init_ensemble(h, 5, 1, 0), h)
    with pytest.raises(Mcmp2ArgumentError, match="no walker ensemble"):
        check_dev(d.mcmp2dev_advance(h, 1, None, None), h)
    w = np.zeros((2, 8))
    out = (Step * 1)()
    with pytest.raises(Mcmp2ArgumentError, match="tau must be non-negative"):
        check_dev(d.mcmp2dev_replay(h, 2, 1, dptr(w), dptr(np.array([-0.1])), out), h)
    d.mcmp2dev_destroy(h)

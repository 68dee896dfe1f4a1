"""The oracle's pair integrand against an independent numpy restatement from spinor values, the
identity the reference pins in test_estimator.cpp:27-48 (restatement support/reference.hpp:16-70):
O(d,o) = sum_i phi_d[x,i] gexp(eps_i tau) conj phi_o[y,i], V likewise over virtuals with
gexp(-eps_a tau) (greens.cpp:63-79); literal f = sum_xy o(x,y) v(x,y) (estimator.cpp:26-29),
direct = -w_d f1d f2d inv_w, exchange = -w_x f1x f2x inv_w, inv_w = N_g^2 / (g1p g2p g1q g2q w(tau))
(estimator.cpp:32,55); the physical form with traces. tau in {0, 0.13, 0.9}, 1e-12 relative."""
import numpy as np
import pytest

import oracle_py


def energies(spinor_path):
    tok = spinor_path.read_text().split()
    i = tok.index("energies")
    no, nv = int(tok[i + 1]), int(tok[i + 2])
    e = np.array([float(t) for t in tok[i + 3:i + 3 + no + nv]])
    return e[:no], e[no:]


def gexp(x):
    return np.where(x < -700.0, 0.0, np.exp(np.minimum(x, 700.0)))


def restated(orc, eo, ev, p, q, tau, physical):
    pts = np.array([p[0:3], p[3:6], q[0:3], q[3:6]])  # a, b, c, d
    occ, vir = orc.evaluate(pts)                       # [point][channel][spinor]
    wo, wv = gexp(eo * tau), gexp(-ev * tau)
    O = lambda d, o: np.einsum("xi,i,yi->xy", occ[d], wo, occ[o].conj())
    V = lambda d, o: np.einsum("xa,a,ya->xy", vir[d], wv, vir[o].conj())
    a, b, c, d = 0, 1, 2, 3
    o1, o2 = O(a, c), O(b, d)
    va, vb, vc, vd = V(c, a), V(d, b), V(d, a), V(c, b)
    lam = orc.lambda_
    inv_w = orc.ng ** 2 / (p[6] * p[7] * q[6] * q[7] * lam * np.exp(-lam * tau))
    wd, wx = (2.0, -1.0) if orc.ncomp == 1 else (0.5, -0.5)
    if physical:
        direct = -wd * np.trace(o1 @ va) * np.trace(o2 @ vb) * inv_w
        exchange = -wx * np.trace(o1 @ vd @ o2 @ vc) * inv_w
    else:
        direct = -wd * np.sum(o1 * va) * np.sum(o2 * vb) * inv_w
        exchange = -wx * np.sum(o1 * vc) * np.sum(o2 * vd) * inv_w
    return direct, exchange


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "syn1c", "syn2c"])
@pytest.mark.parametrize("physical", [False, True])
def test_sample_term_matches_numpy_restatement(cfgdir, name, physical):
    sp = cfgdir / f"{name}.spinor"
    conf = cfgdir / f"{name}.conf"
    orc = oracle_py.OracleSystem(sp, conf.read_text() if conf.exists() else "")
    eo, ev = energies(sp)
    r = np.random.default_rng(3)
    for _ in range(3):
        pts = r.normal(scale=0.8, size=(4, 3))
        g = orc.g(pts)
        p = np.r_[pts[0], pts[1], g[0], g[1]]
        q = np.r_[pts[2], pts[3], g[2], g[3]]
        for tau in (0.0, 0.13, 0.9):
            d, x = orc.sample_term(p, q, tau, physical=physical)
            rd, rx = restated(orc, eo, ev, p, q, tau, physical)
            assert abs(d - rd) <= 1e-12 * abs(rd)
            assert abs(x - rx) <= 1e-12 * abs(rx)

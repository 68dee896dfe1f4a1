"""CPU: the INT8 path's error model (the accuracy guard of csrc/pair_oz.cu) restated in numpy
and checked on the oracle's steps. The device's slices (six balanced radix-256 digits per
power-of-two-scaled row over [re | im], products s + t <= 5; tests/test_ozaki_budget.py
device_v) give V; the literal contraction (estimator.cpp:26-32) gives the direct and exchange
sums. The guard's estimate of their error, from per-point stats only:
  S(pt) = max over channels of the row scale 2^e, A(pt) = max of 2^e a,
  a = sqrt(|x 2^-e|^2 / 3 + 0.6 #{k : |x_k 2^-e| > 2^-8}), N(pt) = |Phi_o(pt)|_F,
  sigma(u, v) = 2^-46 (A_u S_v + S_u A_v), sigma_f(o block (a, c), V(u, v)) = N_a N_c sigma(u, v),
  eps_pair = |w| (sigma_f1 |f2| + |f1| sigma_f2), estimate = sqrt(sum eps_pair^2).
It must cover the actual error on every step (the claim the guard's tolerance rests on) without
being so loose that it rejects well-conditioned steps (here 6.6-33x, and up to 1100x on a
step whose actual error happens to sit at FP64 rounding, 7e-17 absolute)."""
import numpy as np
import pytest

import oracle_py
from test_ozaki_budget import device_v


def point_stats(av, ao, m):
    B = np.concatenate([av.real, av.imag], 1)   # rows (point, channel) over K' = [re | im]
    mx = np.max(np.abs(B), 1)
    e = np.where(mx > 0, np.floor(np.log2(np.where(mx > 0, mx, 1.0))) + 1, 0)
    s = 2.0 ** np.where(mx * 2.0 ** -e > 0.995, e + 1, e)
    X = B / s[:, None]
    a = np.sqrt((X ** 2).sum(1) / 3 + 0.6 * (np.abs(X) > 2.0 ** -8).sum(1))
    S = s.reshape(-1, 4).max(1)
    A = (s * a).reshape(-1, 4).max(1)
    N = np.sqrt((np.abs(ao.reshape(2 * m, 4, -1)) ** 2).sum((1, 2)))
    return S, A, N


def sums_and_estimate(O, V, W, m, stats, wd=0.5, wx=-0.5):
    S, A, N = stats
    Ob, Vb = O.reshape(2 * m, 4, 2 * m, 4), V.reshape(2 * m, 4, 2 * m, 4)
    sig = lambda u, v: 2.0 ** -46 * (A[u] * S[v] + S[u] * A[v])  # noqa: E731
    d = x = ed2 = ex2 = 0.0
    for p in range(m):
        q = np.arange(p + 1, m)
        a, b, c, dd = 2 * p, 2 * p + 1, 2 * q, 2 * q + 1
        o1, o2 = Ob[a, :, c, :], Ob[b, :, dd, :]
        iw = 1 / (W[p, 6] * W[p, 7] * W[q, 6] * W[q, 7])
        f1d, f2d = (o1 * Vb[c, :, a, :]).sum((1, 2)), (o2 * Vb[dd, :, b, :]).sum((1, 2))
        f1x, f2x = (o1 * Vb[dd, :, a, :]).sum((1, 2)), (o2 * Vb[c, :, b, :]).sum((1, 2))
        d += np.sum(-wd * f1d * f2d * iw).real
        x += np.sum(-wx * f1x * f2x * iw).real
        nac, nbd = N[a] * N[c], N[b] * N[dd]
        e_d = abs(wd) * iw * (nac * sig(c, a) * np.abs(f2d) + np.abs(f1d) * nbd * sig(dd, b))
        e_x = abs(wx) * iw * (nac * sig(dd, a) * np.abs(f2x) + np.abs(f1x) * nbd * sig(c, b))
        ed2 += (e_d ** 2).sum()
        ex2 += (e_x ** 2).sum()
    return d, x, np.sqrt(ed2), np.sqrt(ex2)


@pytest.mark.parametrize("name,m,nsteps", [("cfg3", 48, 3), ("cfg4", 24, 2)])
def test_guard_estimate_covers_the_int8_error(cfgdir, name, m, nsteps):
    sp = cfgdir / f"{name}.spinor"
    orc = oracle_py.OracleSystem(sp, (cfgdir / f"{name}.conf").read_text())
    tr = orc.trajectory(seed=13, stream=0, m=m, burn=20, nsteps=nsteps)
    tok = sp.read_text().split()
    i = tok.index("energies")
    no, nv = int(tok[i + 1]), int(tok[i + 2])
    eps = np.array(tok[i + 3:i + 3 + no + nv], dtype=float)
    for k in range(nsteps):
        W, tau = tr["walkers"][k], tr["tau"][k]
        pts = np.empty((2 * m, 3))
        pts[0::2], pts[1::2] = W[:, 0:3], W[:, 3:6]
        occ, vir = orc.evaluate(pts)
        ao = (occ * np.exp(0.5 * eps[:no] * tau)).reshape(8 * m, no)
        av = (vir * np.exp(-0.5 * eps[no:] * tau)).reshape(8 * m, nv)
        O = ao @ ao.conj().T
        ed, ex, _, _ = sums_and_estimate(O, av @ av.conj().T, W, m, point_stats(av, ao, m))
        rd, rx, est_d, est_x = sums_and_estimate(O, device_v(av), W, m, point_stats(av, ao, m))
        for err, est in ((abs(rd - ed), est_d), (abs(rx - ex), est_x)):
            assert err <= est <= 2000 * err, (k, err, est)

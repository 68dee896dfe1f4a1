"""The reference's syn4c fixture (proj/core/src/oracle.cpp:357-393) restated with numpy, and
two deterministic energies for it — TEST INFRASTRUCTURE ONLY.

* `mp2_energy`: the reference oracle's physical MP2 sum (oracle.cpp:148-243): AO ERIs of the
  s-only basis, 4-index transform summed over channel pairs, sum over ijab.
* `literal_limit`: the exact expectation of the reference's literal MC estimator
  (estimator.cpp:26-32): with T^{pq}_{mu kappa} = sum_x C^x_{mu p} C^x_{kappa q} the direct and
  exchange parts are products of two AO ERIs (derivation in DESIGN.md). SURVEY.md section 0
  reports -0.003932252921 and +0.013087649253 for the two; the tests pin both.

The coefficient draws follow file order (real part first) of Complex(rng.uniform() - 0.5,
rng.uniform() - 0.5); the energies are invariant under the other order (SURVEY finding 8).
"""
from __future__ import annotations

import math

import numpy as np

import oracle_py

ZETAS = (4.8, 1.4, 0.45, 0.14)
EPS = (-0.9, -0.9, 0.3, 0.3, 0.8, 0.8, 1.6, 1.6)


def s_overlap(a, b):
    return (2.0 * math.sqrt(a * b) / (a + b)) ** 1.5


def eri_same_centre(z):
    """(mu nu|ka la) for normalised s Gaussians on one centre (Boys F0(0) = 1)."""
    n = len(z)
    N = [(2 * a / math.pi) ** 0.75 for a in z]
    out = np.empty((n, n, n, n))
    for m in range(n):
        for v in range(n):
            for k in range(n):
                for l in range(n):
                    p, q = z[m] + z[v], z[k] + z[l]
                    out[m, v, k, l] = N[m] * N[v] * N[k] * N[l] * 2 * math.pi ** 2.5 / (p * q * math.sqrt(p + q))
    return out


def coefficients():
    nb = len(ZETAS)
    s4 = np.array([[s_overlap(a, b) for b in ZETAS] for a in ZETAS])
    s16 = np.kron(np.eye(4), s4)
    u = np.empty(4 * 2 * 16)
    import ctypes as C
    oracle_py.lib().orc_philox_stream(0x4C4C, 0, 1, len(u), u.ctypes.data_as(C.POINTER(C.c_double)))
    it = iter(u)
    cols = []
    for _ in range(4):
        v = np.array([complex(next(it) - 0.5, next(it) - 0.5) for _ in range(16)])
        for _rep in range(2):
            for c in cols:
                v = v - c * (c.conj() @ s16 @ v)
        v = v / math.sqrt((v.conj() @ s16 @ v).real)
        w = np.empty_like(v)
        for d in range(2):  # (La, Lb, Sa, Sb) -> (-Lb*, La*, -Sb*, Sa*)
            a, b = 2 * d * nb, (2 * d + 1) * nb
            w[a:a + nb] = -np.conj(v[b:b + nb])
            w[b:b + nb] = np.conj(v[a:a + nb])
        cols += [v, w]
    return np.array(cols).T  # [16 rows][8 spinors]


def write_spinor_file(path):
    C_ = coefficients()
    lines = ["spinor-text 1", "nuclei 1", "29 0 0 0", "ncomp 4"]
    for x in range(4):
        lines.append(f"basis {x} 4")
        lines += [f"0 0 0 ; 0 0 ; 1 ; {z!r} 1" for z in ZETAS]
    lines.append("energies 2 6")
    lines += [repr(e) for e in EPS]
    lines.append("coeff 16 8")
    for i in range(16):
        lines.append(" ".join(f"{float(C_[i, j].real)!r} {float(C_[i, j].imag)!r}" for j in range(8)))
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    return C_


def _blocks(C_):
    return [C_[4 * x:4 * x + 4] for x in range(4)]  # per channel [mu][p]


def mp2_energy(C_):
    """oracle.cpp:148-243 (w_d, w_x) = (1/2, -1/2) for 4 components."""
    eri = eri_same_centre(ZETAS)
    Cx = _blocks(C_)
    no = 2
    occ, vir = slice(0, no), slice(no, 8)
    mo = np.zeros((2, 6, 2, 6), dtype=complex)
    for x in range(4):
        for y in range(4):
            mo += np.einsum("mi,na,kj,lb,mnkl->iajb", Cx[x][:, occ].conj(), Cx[x][:, vir], Cx[y][:, occ].conj(),
                            Cx[y][:, vir], eri)
    e = np.array(EPS)
    denom = e[occ][:, None, None, None] + e[occ][None, None, :, None] - e[vir][None, :, None, None] - e[vir][None, None, None, :]
    iajb = mo
    biaj = np.conj(np.transpose(mo, (0, 3, 2, 1)))  # (ib|ja)* -> mo[i,b,j,a]*
    val = (0.5 * iajb * np.conj(iajb) - 0.5 * iajb * biaj) / denom
    return float(val.sum().real)


def literal_limit(C_):
    """Exact expectation of the literal estimator (estimator.cpp:26-32) for an s-only set whose
    channels share one AO list: sum over ijab of D^-1 times two-ERI contractions."""
    eri = eri_same_centre(ZETAS)
    Cx = _blocks(C_)
    T = sum(np.einsum("mp,kq->pqmk", Cx[x], Cx[x]) for x in range(4))  # T^{pq}_{mu kappa}
    no = 2
    e = np.array(EPS)
    total_d = 0.0 + 0.0j
    total_x = 0.0 + 0.0j
    for i in range(no):
        for j in range(no):
            for a in range(no, 8):
                for b in range(no, 8):
                    D = e[a] + e[b] - e[i] - e[j]
                    A = T[i, a]          # [mu, kappa]: phi_i(1) phi_a(3)
                    B = T[a, i].conj()   # [nu, lambda]: conj phi_a(1) phi_i(3)
                    Cj = T[j, b]         # [rho, sigma]
                    Db = T[b, j].conj()  # [tau, upsilon]
                    # direct: (mu nu|rho tau)(kappa lambda|sigma upsilon)
                    total_d += np.einsum("mk,nl,rs,tu,mnrt,klsu->", A, B, Cj, Db, eri, eri) / D
                    # exchange: (mu nu|rho tau)(lambda sigma|kappa upsilon)
                    total_x += np.einsum("mk,nl,rs,tu,mnrt,lsku->", A, B, Cj, Db, eri, eri) / D
    return float((-0.5 * total_d + 0.5 * total_x).real)

"""Identities the reference's own unit tests check, restated against the oracle with the other
side computed independently here (numpy closed forms and Gauss-Legendre quadrature), so the
oracle's spinor evaluation and sampling weight are pinned by more than one restatement of the
reference tables:
  * test_model.cpp:46-55      contracted functions (l <= 3) have unit norm, by quadrature -- here
                              the whole 6 x 6 overlap of one-centre functions of distinct (l, m);
  * test_greens.cpp:101-144   occupied + virtual at tau = 0 is complete on a full-rank
                              4-component set: sum_p phi_p(r) phi_p(r')^H = delta_xy chi(r)^T S^-1 chi(r');
  * test_weights.cpp:69-82    N_g of one primitive against its closed form (Gaussian centre of mass
                              integral times the radial integral, done analytically here);
  * test_weights.cpp:84-93    N_g of two far nuclei tends to the point-charge limit 2 N_1 + 2 q^2 / R;
  * g(r) integrates to the site charge q (by quadrature).
The spinor sets are written here as SPINOR-TEXT (the format of model.cpp:275-388)."""
import numpy as np
import pytest

from oracle_py import OracleSystem

PI = np.pi


def write_spinor_text(path, nuclei, ncomp, basis, energies, n_occ, coeff):
    """nuclei [(Z, x, y, z)], basis [component][(centre, l, m, [(exp, coef)])], coeff rows x cols complex."""
    lines = ["spinor-text 1", f"nuclei {len(nuclei)}"]
    lines += [f"{z} {float(x)!r} {float(y)!r} {float(w)!r}" for z, x, y, w in nuclei]
    lines.append(f"ncomp {ncomp}")
    for c in range(ncomp):
        lines.append(f"basis {c} {len(basis[c])}")
        for (cx, cy, cz), l, m, prims in basis[c]:
            ps = " ".join(f"{float(a)!r} {float(b)!r}" for a, b in prims)
            lines.append(f"{float(cx)!r} {float(cy)!r} {float(cz)!r} ; {l} {m} ; {len(prims)} ; {ps}")
    lines.append(f"energies {n_occ} {len(energies) - n_occ}")
    lines += [repr(float(e)) for e in energies]
    lines.append(f"coeff {coeff.shape[0]} {coeff.shape[1]}")
    for row in coeff:
        lines.append(" ".join(f"{float(v.real)!r} {float(v.imag)!r}" for v in row))
    path.write_text("\n".join(lines) + "\n")


def gauss_box(lo, hi, n, panels=None):
    """tensor-product Gauss-Legendre rule on [lo, hi]^3 (n points per axis, or composite panels
    [(a, b, n), ...] per axis)"""
    xs, ws = [], []
    for a, b, k in panels or [(lo, hi, n)]:
        t, u = np.polynomial.legendre.leggauss(k)
        xs.append(0.5 * (b - a) * t + 0.5 * (b + a))
        ws.append(0.5 * (b - a) * u)
    x, w = np.concatenate(xs), np.concatenate(ws)
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    W = w[:, None, None] * w[None, :, None] * w[None, None, :]
    return np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1), W.ravel()


def test_one_centre_functions_are_orthonormal_by_quadrature(tmp_path):
    """test_model.cpp:46-55: the reference's (l, m) list, each a two-primitive contraction at the
    origin; distinct (l, m) at one centre are orthogonal, each normalised -- so C = I is an
    orthonormal spinor set and its quadrature overlap must be the identity."""
    lm = [(0, 0), (1, 1), (2, -2), (2, 0), (3, 2), (3, 0)]
    prims = [(1.3, 0.7), (0.4, 0.5)]
    basis = [[((0.0, 0.0, 0.0), l, m, prims) for l, m in lm]]
    n = len(lm)
    sp = tmp_path / "onecentre.spinor"
    write_spinor_text(sp, [(1, 0.0, 0.0, 0.0)], 1, basis, [-0.5] + [0.1 * k for k in range(1, n)], 1,
                      np.eye(n, dtype=complex))
    sysm = OracleSystem(sp)
    pts, w = gauss_box(-9.0, 9.0, 80)
    occ, vir = sysm.evaluate(pts)
    phi = np.concatenate([occ[:, 0, :], vir[:, 0, :]], axis=1)  # (points, spinors)
    s = (phi.conj() * w[:, None]).T @ phi
    assert np.abs(s - np.eye(n)).max() < 1e-8, s


def test_full_rank_set_is_complete_at_tau_zero(tmp_path):
    """test_greens.cpp:101-144: four s functions per component, all 16 columns kept
    (C = S^-1/2 Q, Q a seeded random orthogonal matrix): the occupied + virtual kernel equals the
    basis-side delta_xy chi(r)^T S^-1 chi(r'), S and chi in closed form here."""
    z = np.array([4.8, 1.4, 0.45, 0.14])
    nb = len(z)
    s4 = (2.0 * np.sqrt(np.outer(z, z)) / (z[:, None] + z[None, :])) ** 1.5  # normalised s Gaussians
    s16 = np.kron(np.eye(4), s4)
    ev, vec = np.linalg.eigh(s16)
    shalf = vec @ np.diag(ev ** -0.5) @ vec.T
    rng = np.random.default_rng(21)
    q, _ = np.linalg.qr(rng.uniform(-0.5, 0.5, (16, 16)))
    c = (shalf @ q).astype(complex)
    eps = [-2.0 + 0.3 * p if p < 4 else 0.5 + 0.2 * (p - 4) for p in range(16)]
    basis = [[((0.0, 0.0, 0.0), 0, 0, [(a, 1.0)]) for a in z] for _ in range(4)]
    sp = tmp_path / "fullrank.spinor"
    write_spinor_text(sp, [(29, 0.0, 0.0, 0.0)], 4, basis, eps, 4, c)
    sysm = OracleSystem(sp)
    sinv = np.linalg.inv(s4)

    def chi(r):
        return (2.0 * z / PI) ** 0.75 * np.exp(-z * np.dot(r, r))

    for _ in range(3):
        r, rp = rng.uniform(-1.5, 1.5, 3), rng.uniform(-1.5, 1.5, 3)
        occ, vir = sysm.evaluate(np.stack([r, rp]))
        kernel = occ[0] @ occ[1].conj().T + vir[0] @ vir[1].conj().T  # 4 x 4 channels
        expected = np.eye(4) * (chi(r) @ sinv @ chi(rp))
        assert np.abs(kernel - expected).max() < 1e-8, (kernel, expected)


def h_spinor(tmp_path, nuclei):
    """a minimal valid one-component set on the given nuclei (one normalised s function each would
    not be orthonormal across centres: one function at the first nucleus, one spinor)"""
    sp = tmp_path / "h.spinor"
    write_spinor_text(sp, nuclei, 1, [[((0.0, 0.0, 0.0), 0, 0, [(1.0, 1.0)]), ((0.0, 0.0, 0.0), 1, 0, [(1.0, 1.0)])]],
                      [-0.5, 0.5], 1, np.eye(2, dtype=complex))
    return sp


def test_single_primitive_ng_matches_its_closed_form(tmp_path):
    """test_weights.cpp:69-82 with the integrals done analytically: g = c N e^{-z r^2}, N = (2z/pi)^{3/4};
    N_g = c^2 N^2 (pi / 2z)^{3/2} 4 pi int_0^inf u e^{-z u^2 / 2} du = c^2 N^2 (pi / 2z)^{3/2} 4 pi / z.
    The second primitive is made negligible (coefficient 1e-12) as in the reference test."""
    zeta, c = 0.8, 0.7
    sysm = OracleSystem(h_spinor(tmp_path, [(1, 0.0, 0.0, 0.0)]), f"weight H {c!r} {zeta!r} 1e-12 1.0\n")
    cn = c * (2.0 * zeta / PI) ** 0.75
    expected = cn * cn * (PI / (2.0 * zeta)) ** 1.5 * 4.0 * PI / zeta
    assert sysm.ng == pytest.approx(expected, rel=1e-9)
    r = np.array([[0.0, 0.0, 0.0], [0.3, -0.4, 1.2], [2.0, 1.0, -1.5]])
    gv = sysm.g(r)
    want = cn * np.exp(-zeta * (r * r).sum(1)) + 1e-12 * (2.0 / PI) ** 0.75 * np.exp(-(r * r).sum(1))
    assert np.allclose(gv, want, rtol=1e-13, atol=0)


def test_two_far_nuclei_tend_to_the_point_charge_limit(tmp_path):
    """test_weights.cpp:84-93: each H site's default g (0.25, 0.06; 0.15, 0.6; weights.cpp
    defaults) integrates to q; at R = 60 the cross term is q^2 / R to 1e-6 relative of N_g."""
    sep = 60.0
    one = OracleSystem(h_spinor(tmp_path, [(1, 0.0, 0.0, 0.0)]))
    two = OracleSystem(h_spinor(tmp_path, [(1, 0.0, 0.0, 0.0), (1, 0.0, 0.0, sep)]))
    q = 0.25 * (2 * 0.06 / PI) ** 0.75 * (PI / 0.06) ** 1.5 + 0.15 * (2 * 0.6 / PI) ** 0.75 * (PI / 0.6) ** 1.5
    assert two.ng == pytest.approx(2.0 * one.ng + 2.0 * q * q / sep, rel=1e-6)


def test_site_weight_integrates_to_its_charge(tmp_path):
    """the same q by quadrature of the oracle's g over a box (the diffuse 0.06 primitive needs +-24,
    the 0.6 one a finer middle panel)"""
    one = OracleSystem(h_spinor(tmp_path, [(1, 0.0, 0.0, 0.0)]))
    pts, w = gauss_box(0, 0, 0, panels=[(-24.0, -5.0, 24), (-5.0, 5.0, 48), (5.0, 24.0, 24)])
    q = 0.25 * (2 * 0.06 / PI) ** 0.75 * (PI / 0.06) ** 1.5 + 0.15 * (2 * 0.6 / PI) ** 0.75 * (PI / 0.6) ** 1.5
    assert float(one.g(pts) @ w) == pytest.approx(q, rel=1e-8)

"""Fit the two-primitive sampling weight g of one element (`weight El c1 z1 c2 z2`,
weights.cpp:57-99) to the occupied density of a generated spinor set.

The walker density is g(r1) g(r2) / (N_g r12) (sampler.cpp:63-77), and every point of a pair
sample carries spinor values of that point (estimator.cpp:15-33), so the per-point variance
behaves like  J[g] = integral rho(r)^2 / g(r) d^3r  with rho and g both normalised to unit
mass; J >= 1 with equality at g = rho. The random-unitary synthetic spinors spread their
density over every exponent of the basis, so the fit matters: a g that decays faster than
rho^2 (z1 > 4 zeta_min) gives an infinite variance (profiles/r01_weight_scan.json).

rho is the spherical average, about the fitted centre, of sum_i sum_x |Phi_i^x(r)|^2 over the
occupied spinors (numpy evaluation of the SPINOR-TEXT file: normalised real solid harmonics
x primitive norms, model.cpp:30-64). g = (1 - f2) G(z1) + f2 G(z2), G(z) = (z/pi)^{3/2} e^{-z r^2};
the weight line is c_k = f_k (z_k / 2 pi)^{3/4} (c_k N_k e^{-z r^2} with N_k = (2 z_k/pi)^{3/4};
the overall scale cancels in N_g). Grid search over (z1, z2, f2).

usage: python tools/fit_weight.py cfg2 [--centre 0]
"""
import argparse
import math
import re
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

S00, S1 = 0.28209479177387814, 0.4886025119029199
S2a, S2b, S2c = 1.0925484305920792, 0.31539156525252005, 0.5462742152960396
S3a, S3b, S3c, S3d = 0.5900435899266435, 2.890611442640554, 0.4570457994644658, 0.3731763325901154


def solid(l, m, x, y, z):
    if l == 0:
        return S00 * np.ones_like(x)
    if l == 1:
        return S1 * {-1: y, 0: z, 1: x}[m]
    if l == 2:
        return {-2: S2a * x * y, -1: S2a * y * z, 0: S2b * (2 * z * z - x * x - y * y), 1: S2a * x * z,
                2: S2c * (x * x - y * y)}[m]
    return {-3: S3a * (3 * x * x * y - y ** 3), -2: S3b * x * y * z, -1: S3c * (4 * y * z * z - x * x * y - y ** 3),
            0: S3d * (2 * z ** 3 - 3 * x * x * z - 3 * y * y * z), 1: S3c * (4 * x * z * z - x ** 3 - x * y * y),
            2: S2c * (x * x * z - y * y * z), 3: S3a * (x ** 3 - 3 * x * y * y)}[m]


def prim_norm(l, z):
    return math.sqrt(2.0 * (2.0 * z) ** (l + 1.5) / math.gamma(l + 1.5))


def read_spinor(path):
    tok = [t for line in Path(path).read_text().splitlines() for t in line.split("#")[0].split()]
    i = 2
    out = {"basis": {}}
    while i < len(tok):
        k = tok[i]
        if k == "nuclei":
            n = int(tok[i + 1])
            out["nuclei"] = np.array(tok[i + 2:i + 2 + 4 * n], dtype=float).reshape(n, 4)
            i += 2 + 4 * n
        elif k == "ncomp":
            out["ncomp"] = int(tok[i + 1])
            i += 2
        elif k == "basis":
            c, cnt = int(tok[i + 1]), int(tok[i + 2])
            i += 3
            fns = []
            for _ in range(cnt):
                ctr = np.array(tok[i:i + 3], dtype=float)
                l, m, npr = int(tok[i + 4]), int(tok[i + 5]), int(tok[i + 7])
                prims = np.array(tok[i + 9:i + 9 + 2 * npr], dtype=float).reshape(npr, 2)
                fns.append((ctr, l, m, prims))
                i += 9 + 2 * npr
            out["basis"][c] = fns
        elif k == "energies":
            no, nv = int(tok[i + 1]), int(tok[i + 2])
            out["n_occ"], out["n_vir"] = no, nv
            i += 3 + no + nv
        elif k == "coeff":
            r, c = int(tok[i + 1]), int(tok[i + 2])
            a = np.array(tok[i + 3:i + 3 + 2 * r * c], dtype=float).reshape(r, c, 2)
            out["coeff"] = a[..., 0] + 1j * a[..., 1]
            i += 3 + 2 * r * c
        else:
            raise ValueError(f"unknown record {k}")
    return out


def chi(fns, pts):
    """basis values [npts, nfn]; uncontracted primitives carry their norm (model.cpp:39-52)"""
    v = np.zeros((len(pts), len(fns)))
    for j, (ctr, l, m, prims) in enumerate(fns):
        d = pts - ctr
        r2 = np.sum(d * d, axis=1)
        rad = sum(c * prim_norm(l, z) * np.exp(-z * r2) for z, c in prims)
        if len(prims) > 1:  # contracted: 1/sqrt(S) (not used by the generated sets)
            raise ValueError("contracted functions not supported here")
        v[:, j] = solid(l, m, d[:, 0], d[:, 1], d[:, 2]) * rad
    return v


def radial_density(sp, centre, radii, ndir=64, seed=5):
    rng = np.random.default_rng(seed)
    u = rng.normal(size=(ndir, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    pts = (radii[:, None, None] * u[None]).reshape(-1, 3) + centre
    no = sp["n_occ"]
    C = sp["coeff"][:, :no]
    rho = np.zeros(len(pts))
    row = 0
    for c in sorted(sp["basis"]):
        X = chi(sp["basis"][c], pts)
        n = X.shape[1]
        phi = X @ C[row:row + n]
        rho += np.sum(np.abs(phi) ** 2, axis=1)
        row += n
    return rho.reshape(len(radii), ndir).mean(axis=1)


def fit(radii, rho):
    w = 4 * np.pi * radii ** 2 * np.gradient(radii)  # radial quadrature
    mass = np.sum(rho * w)
    rho = rho / mass
    z1s = np.logspace(-2.7, 1.0, 75)
    z2s = np.logspace(-1.0, 5.0, 121)
    f2s = np.linspace(0.01, 0.95, 48)
    best = (np.inf, None)
    r2 = radii ** 2
    G = lambda z: (z[:, None] / np.pi) ** 1.5 * np.exp(-z[:, None] * r2[None])  # noqa: E731
    G1, G2 = G(z1s), G(z2s)
    num = rho ** 2 * w
    for i1, z1 in enumerate(z1s):
        g = (1 - f2s)[:, None, None] * G1[i1][None, None] + f2s[:, None, None] * G2[None]  # [f2][z2][r]
        J = np.sum(num / np.maximum(g, 1e-300), axis=2)
        k = np.unravel_index(np.argmin(J), J.shape)
        if J[k] < best[0]:
            best = (float(J[k]), (float(f2s[k[0]]), float(z1), float(z2s[k[1]])))
    return best, mass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--centre", type=int, default=0, help="nucleus index of the fitted element")
    args = ap.parse_args()
    from paper_2203_05632_b200 import generate_config
    with tempfile.TemporaryDirectory() as d:
        spath, conf = generate_config(args.config, d)
        sp = read_spinor(spath)
        text = conf.read_text()
    centre = sp["nuclei"][args.centre, 1:]
    radii = np.logspace(-4, np.log10(40.0), 500)
    rho = radial_density(sp, centre, radii)
    (J, (f2, z1, z2)), mass = fit(radii, rho)
    el = re.search(r"weight (\S+)", text).group(1)
    c1, c2 = (1 - f2) * (z1 / (2 * np.pi)) ** 0.75, f2 * (z2 / (2 * np.pi)) ** 0.75
    cur = re.search(r"weight .*", text).group(0)
    zb = min(p[0][0] for fns in sp["basis"].values() for (_, _, _, p) in [(0, 0, 0, f[3]) for f in fns])
    print(f"{args.config}: occupied mass {mass:.4f} (n_occ {sp['n_occ']}), basis zeta_min {zb:.4g}")
    print(f"  current  {cur}")
    print(f"  fitted   weight {el} {c1:.6g} {z1:.6g} {c2:.6g} {z2:.6g}   (f2 {f2:.3f}, J {J:.4g})")


if __name__ == "__main__":
    main()

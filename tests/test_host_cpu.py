"""CPU: the C-ABI libraries load and export every declared symbol; the C++ host (SPINOR-TEXT,
validation, weights, run config, merge) agrees with the oracle and the reference's tests."""
import ctypes as C
import math
from pathlib import Path

import numpy as np
import pytest

import oracle_py
from paper_2203_05632_b200 import System, native
from paper_2203_05632_b200.native import Mcmp2ArgumentError, Mcmp2Error

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("header,lib", [("mcmp2dev.h", "dev"), ("mcmp2host.h", "host")])
def test_libraries_export_every_declared_symbol(header, lib):
    L = getattr(native, lib)()
    names = native.exported_symbols(ROOT / "include" / header)
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_abi_version():
    assert native.dev().mcmp2dev_abi_version() == 2


def test_create_without_gpu_fails_loudly(cfgdir):
    """No CPU fallback: without a usable device, create returns MCMP2DEV_CUDA with a message."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2203_05632_b200 import DeviceWalker
    s = System(cfgdir / "cfg1.spinor", (cfgdir / "cfg1.conf").read_text())
    with pytest.raises(Mcmp2Error):
        DeviceWalker(s, max_walkers=16)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "syn1c", "syn2c"])
def test_host_loader_matches_oracle(cfgdir, name):
    sp, text = cfgdir / f"{name}.spinor", (cfgdir / f"{name}.conf").read_text()
    h = System(sp, text)
    o = oracle_py.OracleSystem(sp, text)
    assert (h.ncomp, h.n_occ, h.n_vir, h.rows) == (o.ncomp, o.n_occ, o.n_vir, o.rows)
    assert h.ng == pytest.approx(o.ng, rel=1e-14)
    assert h.lambda_ == o.lambda_
    assert h.orthonormality_deviation < 1e-12
    pts = np.random.default_rng(1).normal(scale=1.5, size=(50, 3))
    assert np.allclose(h.g(pts), o.g(pts), rtol=1e-14, atol=0)


def test_generated_sizes_match_survey(cfgdir):
    """SURVEY.md section 8 config-derived sizes: R, n_occ, n_vir."""
    want = {"cfg1": (96, 2, 22), "cfg2": (274, 10, 72), "cfg3": (556, 18, 152), "cfg4": (1056, 54, 278)}
    for name, (R, no, nv) in want.items():
        s = System(cfgdir / f"{name}.spinor", (cfgdir / f"{name}.conf").read_text())
        assert (s.rows, s.n_occ, s.n_vir, s.ncomp) == (R, no, nv, 4)


def read_coeff(path):
    toks = Path(path).read_text().split()
    i = toks.index("coeff")
    r, c = int(toks[i + 1]), int(toks[i + 2])
    v = np.array(toks[i + 3: i + 3 + 2 * r * c], dtype=float).reshape(r, c, 2)
    return v[..., 0] + 1j * v[..., 1]


def test_generated_columns_are_kramers_pairs(cfgdir):
    """(La, Lb, Sa, Sb) -> (-Lb*, La*, -Sb*, Sa*) (oracle.cpp:346-355 generalised)."""
    s = System(cfgdir / "cfg2.spinor", (cfgdir / "cfg2.conf").read_text())
    C_ = read_coeff(cfgdir / "cfg2.spinor")
    nL = 41
    nS = (s.rows - 2 * nL) // 2
    off = [0, nL, 2 * nL, 2 * nL + nS]
    ln = [nL, nL, nS, nS]
    for j in range(0, C_.shape[1], 2):
        v, w = C_[:, j], C_[:, j + 1]
        for d in range(2):
            a, b, n = off[2 * d], off[2 * d + 1], ln[2 * d]
            assert np.array_equal(w[a:a + n], -np.conj(v[b:b + n]))
            assert np.array_equal(w[b:b + n], np.conj(v[a:a + n]))


def test_spinor_file_round_trip_is_bit_exact(cfgdir, tmp_path):
    """test_model.cpp:139-155 (file order x, y, z for off-origin centres: cfg3, syn1c)."""
    h = native.host()
    for name in ("cfg1", "cfg3", "syn1c", "syn2c"):
        src = cfgdir / f"{name}.spinor"
        out = tmp_path / f"{name}.rt"
        native.check_host(h.mcmp2h_save_spinor_set(str(src).encode(), str(out).encode()))
        assert out.read_text() == src.read_text()


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_spinor_file_error_paths(cfgdir, tmp_path):
    """test_model.cpp:157-214 (host loader messages)."""
    with pytest.raises(Mcmp2Error, match="cannot open"):
        System(tmp_path / "nonexistent.spinor")
    with pytest.raises(Mcmp2Error, match="bogus"):
        System(write(tmp_path, "bad.spinor", "spinor-text 1\nbogus 3\n"))
    good = (cfgdir / "syn1c.spinor").read_text()
    assert "energies 1 9\n-0.59999999999999998\n" in good
    lines = good.splitlines()
    e = lines.index("energies 1 9")
    closed = "\n".join(lines[: e + 2] + ["-0.59999999999999998"] + lines[e + 3:]) + "\n"
    with pytest.raises(Mcmp2Error, match="overlap"):  # HOMO == LUMO (test_weights.cpp:177-185)
        System(write(tmp_path, "closed.spinor", closed))
    # coefficients doubled: C^H S C - I has deviation 3 on the diagonal
    lines = good.splitlines()
    k = lines.index(next(l for l in lines if l.startswith("coeff")))
    scaled = lines[: k + 1] + [" ".join(str(2 * float(t)) for t in l.split()) for l in lines[k + 1:]]
    with pytest.raises(Mcmp2Error, match="orthonormal.*3"):
        System(write(tmp_path, "scaled.spinor", "\n".join(scaled) + "\n"))
    with pytest.raises(Mcmp2Error, match="nuclei"):
        System(write(tmp_path, "nonuc.spinor", good.replace("nuclei 2\n1 0 0 0\n1 0 0 1.3999999999999999\n", "")))


def test_missing_weight_parameters(cfgdir):
    """weights.cpp:65-70: elements outside Table I need a `weight` line."""
    with pytest.raises(Mcmp2ArgumentError, match="Z=2"):
        System(cfgdir / "cfg1.spinor", "")


def single_h_file(tmp_path):
    """1c, one H, two s functions with S-orthonormal real columns (hand-built)."""
    a, b = 1.0, 0.3
    s12 = (2 * math.sqrt(a * b) / (a + b)) ** 1.5
    c1 = np.array([1.0, 0.0])
    c2 = np.array([-s12, 1.0]) / math.sqrt(1 - s12 * s12)
    txt = ("spinor-text 1\nnuclei 1\n1 0 0 0\nncomp 1\nbasis 0 2\n0 0 0 ; 0 0 ; 1 ; 1 1\n0 0 0 ; 0 0 ; 1 ; 0.3 1\n"
           "energies 1 1\n-0.6\n0.4\ncoeff 2 2\n")
    for i in range(2):
        txt += f"{float(c1[i])!r} 0 {float(c2[i])!r} 0\n"
    return write(tmp_path, "h1.spinor", txt)


def test_weight_normalisation_and_g0(tmp_path):
    """N_g = 4 pi for one unit primitive (test_weights.cpp:62-67); g(0) of Table I H
    (test_weights.cpp:22-27)."""
    p = single_h_file(tmp_path)
    s = System(p, "weight H 1.0 1.0 1e-8 1.0\n")
    assert s.ng == pytest.approx(4 * math.pi, rel=1e-6)
    s = System(p, "")
    want = 0.25 * (2 * 0.06 / math.pi) ** 0.75 + 0.15 * (2 * 0.6 / math.pi) ** 0.75
    assert s.g(np.zeros(3))[0] == pytest.approx(want, rel=1e-12)
    assert s.lambda_ == pytest.approx(2.0, rel=1e-14)


def parse(text):
    buf = C.create_string_buffer(4096)
    native.check_host(native.host().mcmp2h_parse_config(text.encode(), buf, len(buf)))
    return buf.value.decode()


def test_config_parsing():
    """test_driver.cpp:47-101 and the canonical round trip."""
    canon = parse("spinors x.spinor\nsteps 100\n")
    assert "blocksize 100" in canon and "burnin 1000" in canon and "walkers 8" in canon
    with pytest.raises(Mcmp2Error, match="stopping rule"):
        parse("spinors x\n")
    with pytest.raises(Mcmp2Error, match="stopping rule"):
        parse("spinors x\nsteps 5\ntarget-rel-err 0.1\n")
    with pytest.raises(Mcmp2Error, match="walker"):
        parse("walker 4\n")
    with pytest.raises(Mcmp2Error, match="walkers"):
        parse("spinors x\nsteps 10\nwalkers 1\n")
    with pytest.raises(Mcmp2Error):
        parse("steps ten\n")
    with pytest.raises(Mcmp2Error):
        parse("spinors x\nsteps 1\nweight H 0.1 0.2\n")
    full = ("spinors fix.spinor\nsteps 12345\nwalkers 6\nseed 99\nworkers 3\nblocksize 50\nburnin 200\n"
            "checkpoint a.ckpt\ncheckpoint-interval 1000\ntrace a.trace\nweight Cu 0.8 0.35 2 0.6\nstep-size 0.3\n")
    c1 = parse(full)
    assert parse(c1) == c1


def test_config_hash_covers_physics_not_run_shape():
    """test_driver.cpp:103-123 (config_hash): seed/workers/steps excluded, walkers included."""
    h = native.host()
    h.mcmp2h_config_hash.restype = C.c_uint64
    h.mcmp2h_config_hash.argtypes = [C.c_char_p, C.c_uint64]
    a = h.mcmp2h_config_hash(b"spinors f\nsteps 100\nseed 1\n", 42)
    b = h.mcmp2h_config_hash(b"spinors f\nsteps 999999\nseed 777\nworkers 4\n", 42)
    assert a == b
    assert a != h.mcmp2h_config_hash(b"spinors f\nsteps 100\nwalkers 12\n", 42)
    assert a != h.mcmp2h_config_hash(b"spinors f\nsteps 100\n", 43)


def test_merge_arithmetic():
    """driver.cpp:183-196, test_driver.cpp:103-123."""
    h = native.host()
    h.mcmp2h_merge_estimates.argtypes = [C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_double)]

    def merge(parts):
        p = np.ascontiguousarray(parts, dtype=np.float64)
        out = np.empty(3)
        native.check_host(h.mcmp2h_merge_estimates(p.ctypes.data_as(C.POINTER(C.c_double)), len(parts),
                                                   out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    assert list(merge([[100, 1.0, 0.2]])) == [1.0, pytest.approx(0.2), 100]
    assert merge([[100, 1.0, 0.2], [100, 3.0, 0.2]])[0] == pytest.approx(2.0)
    m = merge([[100, 1.0, 0.2], [300, 2.0, 0.1]])
    assert m[0] == pytest.approx(1.75) and m[2] == 400
    with pytest.raises(Mcmp2ArgumentError):
        merge(np.zeros((0, 3)))

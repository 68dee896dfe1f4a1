"""Parity of the device walker loop with the CPU oracle (the reference restated), through the
C ABI. Tolerance: per-step estimates and their direct/exchange sums within 1e-10 relative
(BASELINE.json north_star, replay layer); trajectories within the same bound."""
import numpy as np
import pytest

import oracle_py
from paper_2203_05632_b200 import DeviceWalker, System
from paper_2203_05632_b200.native import Mcmp2Error
from paper_2203_05632_b200.walker import EnsembleState

pytestmark = pytest.mark.gpu

REL = 1e-10


def rel_err(got, ref):
    scale = np.maximum(np.abs(ref), 1e-300)
    return float(np.max(np.abs(got - ref) / scale))


def load(cfgdir, name):
    sp = cfgdir / f"{name}.spinor"
    text = (cfgdir / f"{name}.conf").read_text()
    return sp, text, oracle_py.OracleSystem(sp, text), System(sp, text)


@pytest.mark.parametrize("name,m,nsteps", [("cfg1", 16, 6), ("cfg2", 40, 2), ("cfg3", 24, 2), ("cfg4", 20, 1),
                                           ("syn1c", 9, 4), ("syn2c", 7, 4),
                                           # narrow chunks: cfg5-2 runs a 4-deep stage ring, cfg5-10 has a 1-group virtual chunk
                                           ("cfg5-2", 72, 2), ("cfg5-10", 56, 2)])
def test_replay_matches_oracle(cfgdir, name, m, nsteps):
    sp, text, orc, sysd = load(cfgdir, name)
    tr = orc.trajectory(seed=11, stream=0, m=m, burn=30, nsteps=nsteps)
    dw = DeviceWalker(sysd, max_walkers=m)
    assert dw.kramers() == (orc.ncomp > 1)  # generated 2c/4c sets are exact Kramers pairs
    ref = tr["est"]
    for mode in (1, 0):  # Kramers-restricted kernel, then the general kernel
        dw.kramers(mode)
        got = dw.replay(tr["walkers"], tr["tau"])
        assert rel_err(got[:, 0], ref[:, 0]) < REL
        # direct and exchange pair sums separately (condition-aware: relative to their magnitude)
        for k in (2, 4):
            assert rel_err(got[:, k], ref[:, k]) < REL
    if orc.ncomp == 1:  # real orbitals: imaginary residue exactly zero (test_estimator.cpp:255-267)
        assert np.all(got[:, 1] == 0.0)
    else:  # Kramers-paired input: real to rounding (test_estimator.cpp:149-165)
        assert np.all(np.abs(got[:, 1]) <= 1e-8 * np.abs(got[:, 0]) + 1e-300)


def test_sample_term_is_m2_replay(cfgdir):
    """sample_term (estimator.cpp:65-75) == the m = 2 step; tau in {0, 0.13, 0.9}."""
    sp, text, orc, sysd = load(cfgdir, "cfg1")
    dw = DeviceWalker(sysd, max_walkers=2)
    pts = np.array([[0.3, 0.1, -0.2], [-0.4, 0.5, 0.9], [0.8, -0.6, 0.1], [0.2, 0.3, -0.7]])
    g = orc.g(pts)
    p = np.r_[pts[0], pts[1], g[0], g[1]]
    q = np.r_[pts[2], pts[3], g[2], g[3]]
    for tau in (0.0, 0.13, 0.9):
        d, x = orc.sample_term(p, q, tau)
        got = dw.replay(np.stack([p, q])[None], np.array([tau]))[0]
        assert abs(got[0] - (d + x).real) <= REL * abs((d + x).real)
        assert abs(complex(got[2], got[3]) - d) <= REL * abs(d)
        assert abs(complex(got[4], got[5]) - x) <= REL * abs(x)


def test_relabeling_invariance_1c(cfgdir):
    """1-component: the step estimate is invariant under walker relabelling
    (test_estimator.cpp:128-147 uses the 1c h2_svp fixture)."""
    sp, text, orc, sysd = load(cfgdir, "syn1c")
    tr = orc.trajectory(seed=21, stream=0, m=13, burn=20, nsteps=1)
    dw = DeviceWalker(sysd, max_walkers=13)
    a = dw.replay(tr["walkers"], tr["tau"])[0, 0]
    perm = np.random.default_rng(3).permutation(13)
    b = dw.replay(tr["walkers"][:, perm], tr["tau"])[0, 0]
    assert abs(a - b) <= 1e-12 * abs(a)


def test_relabeling_4c_follows_oracle(cfgdir):
    """4-component: the literal element-wise exchange pairing (estimator.cpp:26-32) is not
    symmetric under p <-> q, so relabelling changes the estimate; the device must follow the
    oracle for every labelling."""
    sp, text, orc, sysd = load(cfgdir, "cfg2")
    tr = orc.trajectory(seed=21, stream=0, m=13, burn=20, nsteps=1)
    dw = DeviceWalker(sysd, max_walkers=13)
    for seed in (3, 4):
        perm = np.random.default_rng(seed).permutation(13)
        w = tr["walkers"][:, perm]
        assert rel_err(dw.replay(w, tr["tau"])[:, 0], orc.replay(w, tr["tau"])[:, 0]) < REL


def test_device_init_and_burn_in_follow_reference_stream(cfgdir):
    """init_ensemble + burn_in on the device consume the reference Philox stream in the
    reference order (sampler.cpp:21-93): same positions, same sigma, same RNG state."""
    sp, text, orc, sysd = load(cfgdir, "cfg2")
    m = 37
    tr = orc.trajectory(seed=5, stream=3, m=m, burn=300, nsteps=0)
    ref = oracle_py.state_to_ensemble(tr["init"], m)
    dw = DeviceWalker(sysd, max_walkers=m)
    dw.init_ensemble(m, seed=5, stream=3)
    dw.burn_in(300, adapt=True)
    st = dw.get_ensemble()
    assert st.sigma_step == ref["sigma_step"]
    assert st.rng_key == ref["rng_key"] and st.rng_counter == ref["rng_counter"] and st.rng_idx == ref["rng_idx"]
    assert np.max(np.abs(st.walkers - ref["walkers"]) / (np.abs(ref["walkers"]) + 1e-300)) < 1e-12
    assert st.proposed == 0 and st.accepted == 0


@pytest.mark.parametrize("name,m,nsteps,step", [("cfg1", 16, 300, 0.3), ("cfg2", 32, 40, 0.0)])
def test_trajectory_matches_oracle(cfgdir, name, m, nsteps, step):
    """advance(): Metropolis + tau + estimate on the device follows the oracle's chain step by
    step when started from the oracle's post-burn-in ensemble (driver.cpp:440-450)."""
    sp, text, orc, sysd = load(cfgdir, name)
    tr = orc.trajectory(seed=9, stream=1, m=m, burn=100, nsteps=nsteps, step_size=step, adapt=step == 0.0)
    dw = DeviceWalker(sysd, max_walkers=m)
    dw.set_ensemble(EnsembleState(**oracle_py.state_to_ensemble(tr["init"], m)))
    v, im = dw.advance(nsteps)
    assert rel_err(v, tr["est"][:, 0]) < REL
    fin = dw.get_ensemble()
    ref = oracle_py.state_to_ensemble(tr["final"], m)
    assert fin.rng_counter == ref["rng_counter"] and fin.rng_idx == ref["rng_idx"]
    assert fin.proposed == tr["proposed"] and fin.accepted == tr["accepted"]
    assert np.max(np.abs(fin.walkers - ref["walkers"]) / (np.abs(ref["walkers"]) + 1e-300)) < 1e-10


@pytest.mark.parametrize("tag", ["cfg1", "cfg2", "syn1c", "syn2c", "cfg3", "cfg4", "cfg2_physical"])
def test_golden_fixtures(cfgdir, tag):
    """Committed oracle dumps (tests/golden/make_golden.py): replay and the advanced chain, for
    both estimators (the physical one on cfg2)."""
    from pathlib import Path
    from paper_2203_05632_b200 import native
    g = np.load(Path(__file__).resolve().parent / "golden" / f"replay_{tag}.npz")
    name = str(g["config"]) if "config" in g else tag
    raw = (cfgdir / f"{name}.spinor").read_bytes()
    assert native.host().mcmp2h_fnv1a64(raw, len(raw)) == int(g["spinor_fnv1a"]), "generator drifted"
    m = int(g["m"])
    text = (cfgdir / f"{name}.conf").read_text() + ("estimator physical\n" if "physical" in g and bool(g["physical"]) else "")
    dw = DeviceWalker(System(cfgdir / f"{name}.spinor", text), max_walkers=m)
    got = dw.replay(g["walkers"], g["tau"])
    assert rel_err(got[:, 0], g["est"][:, 0]) < REL
    dw.set_ensemble(EnsembleState(**oracle_py.state_to_ensemble(g["init"], m)))
    v, _ = dw.advance(len(g["tau"]))
    assert rel_err(v, g["est"][:, 0]) < REL


def test_overflow_is_reported_with_spinor_index(cfgdir, tmp_path):
    """guarded_exp above +700 raises with the spinor index (greens.cpp:9-16, test_greens.cpp:198-202)."""
    sp = cfgdir / "cfg1.spinor"
    text = sp.read_text().replace("\n-0.90000000000000002\n-0.90000000000000002\n", "\n0.05\n0.05\n")
    bad = tmp_path / "posocc.spinor"
    bad.write_text(text)
    conf = (cfgdir / "cfg1.conf").read_text()
    dw = DeviceWalker(System(bad, conf), max_walkers=2)
    pts = np.zeros((2, 8))
    pts[:, 6:] = 0.1
    pts[0, :3] = 0.1
    pts[1, 3:6] = -0.2
    with pytest.raises(Mcmp2Error, match="spinor 0"):
        dw.replay(pts[None], np.array([20000.0]))


def test_overflow_during_advance_is_reported(cfgdir, tmp_path):
    """The production sweep's tau draw (walk_kernel's speculative tau CTA) reports the overflow of
    set_tau too: every energy shifted by +1e5 makes gexp(+eps_i tau) overflow for any tau drawn
    (lambda is unchanged), first at occupied spinor 0."""
    lines = (cfgdir / "cfg1.spinor").read_text().splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith("energies"))
    n = sum(int(x) for x in lines[i].split()[1:])
    for k in range(i + 1, i + 1 + n):
        lines[k] = repr(float(lines[k]) + 1e5)
    bad = tmp_path / "shifted.spinor"
    bad.write_text("\n".join(lines) + "\n")
    conf = (cfgdir / "cfg1.conf").read_text()
    dw = DeviceWalker(System(bad, conf), max_walkers=16)
    dw.init_ensemble(16, seed=3)
    with pytest.raises(Mcmp2Error, match="spinor 0"):
        dw.advance(2)


@pytest.mark.parametrize("name,m", [("cfg3", 512), ("cfg4", 2048), ("cfg5-2", 8192)])
def test_full_size_replay_matches_oracle(cfgdir, name, m):
    """BASELINE sizes: one step of the device estimator at the full walker count (the bench's
    own configuration, every pair tile of the production launch) against the oracle's full
    C(m,2) pair loop (rows split over host threads), both Kramers and general kernels."""
    import os

    sp, text, orc, sysd = load(cfgdir, name)
    dw = DeviceWalker(sysd, max_walkers=m)
    dw.init_ensemble(m, seed=5)
    dw.burn_in(20)
    dw.advance(1)
    w = dw.get_ensemble().walkers[:, :8]
    tau = 0.37
    ref = orc.replay_parallel(w, tau, threads=max(1, min(32, os.cpu_count() or 1)))
    # Kramers kernel with the INT8 (Ozaki) V blocks, with the DMMA V phase, then the general kernel
    for kr, i8 in ((1, 1), (1, 0), (0, 0)):
        dw.kramers(kr)
        assert dw.int8_v(i8) == bool(kr and i8)
        got = dw.replay(w[None], np.array([tau]))[0]
        assert abs(got[0] - ref[0]) <= REL * abs(ref[0]), (kr, i8)
        for k in (2, 4):
            assert abs(got[k] - ref[k]) <= REL * abs(ref[k]), (kr, i8, k)


def test_full_size_physical_replay_matches_oracle(cfgdir):
    """estimator physical at the cfg4 walker count: the Kramers physical epilogue (and the general
    kernel) against the oracle's trace-form pair loop."""
    import os

    sp = cfgdir / "cfg4.spinor"
    text = (cfgdir / "cfg4.conf").read_text() + "estimator physical\n"
    orc = oracle_py.OracleSystem(sp, text)
    m = 2048
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    assert dw.kramers()
    dw.init_ensemble(m, seed=6)
    dw.burn_in(20)
    dw.advance(1)
    w = dw.get_ensemble().walkers[:, :8]
    tau = 0.21
    ref = orc.replay_parallel(w, tau, threads=max(1, min(32, os.cpu_count() or 1)), physical=True)
    for kr, i8 in ((1, 1), (1, 0), (0, 0)):
        dw.kramers(kr)
        assert dw.int8_v(i8) == bool(kr and i8)
        got = dw.replay(w[None], np.array([tau]))[0]
        for k in (0, 2, 4):
            assert abs(got[k] - ref[k]) <= REL * abs(ref[k]), (kr, i8, k)

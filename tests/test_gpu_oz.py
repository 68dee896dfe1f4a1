"""The INT8 (Ozaki) V blocks of the Kramers pair stage (csrc/pair_oz.cu) against the CPU oracle:
the replayed step estimates and the advanced chains of single ensembles large enough for the
path (m >= ~180 walkers: the 16 x 8 pair tiles cover the SMs), literal and physical estimators.
Tolerance as every parity test: 1e-10 relative (BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle_py
from paper_2203_05632_b200 import DeviceWalker, System
from paper_2203_05632_b200.walker import EnsembleState

pytestmark = pytest.mark.gpu

REL = 1e-10


def rel_err(got, ref):
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)))


@pytest.mark.parametrize("name,m,nsteps", [("cfg2", 256, 2), ("cfg3", 192, 2), ("cfg4", 192, 1), ("cfg5-10", 200, 1)])
def test_int8_v_replay_matches_oracle(cfgdir, name, m, nsteps):
    sp = cfgdir / f"{name}.spinor"
    text = (cfgdir / f"{name}.conf").read_text()
    orc = oracle_py.OracleSystem(sp, text)
    tr = orc.trajectory(seed=13, stream=0, m=m, burn=20, nsteps=nsteps)
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    assert dw.kramers() and dw.int8_v()
    got = dw.replay(tr["walkers"], tr["tau"])
    dw.int8_v(0)
    dmma = dw.replay(tr["walkers"], tr["tau"])
    for k in (0, 2, 4):
        assert rel_err(got[:, k], tr["est"][:, k]) < REL, k
        assert rel_err(got[:, k], dmma[:, k]) < REL, k
    assert np.all(got[:, 1] == 0.0)  # the Kramers epilogue's real f values


def test_int8_v_physical_replay_matches_oracle(cfgdir):
    sp = cfgdir / "cfg3.spinor"
    text = (cfgdir / "cfg3.conf").read_text() + "estimator physical\n"
    orc = oracle_py.OracleSystem(sp, text)
    tr = orc.trajectory(seed=17, stream=0, m=192, burn=20, nsteps=1, physical=True)
    dw = DeviceWalker(System(sp, text), max_walkers=192)
    assert not dw.int8_v()  # the physical estimator defaults to the DMMA pair stage
    assert dw.int8_v(1)     # INT8 V blocks on request (unguarded)
    got = dw.replay(tr["walkers"], tr["tau"])
    for k in (0, 2, 4):
        assert rel_err(got[:, k], tr["est"][:, k]) < REL, k


def test_int8_v_chain_matches_oracle(cfgdir):
    """advance() through the captured graphs (walk, chi, mo, slice, V GEMM, pair) follows the
    oracle's chain step by step, with the same RNG state at the end."""
    sp = cfgdir / "cfg3.spinor"
    text = (cfgdir / "cfg3.conf").read_text()
    orc = oracle_py.OracleSystem(sp, text)
    m, nsteps = 192, 34  # one 32-step graph and two single launches
    tr = orc.trajectory(seed=9, stream=2, m=m, burn=50, nsteps=nsteps)
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    dw.set_ensemble(EnsembleState(**oracle_py.state_to_ensemble(tr["init"], m)))
    assert dw.int8_v()
    v, _ = dw.advance(nsteps)
    assert rel_err(v, tr["est"][:, 0]) < REL
    fin = dw.get_ensemble()
    ref = oracle_py.state_to_ensemble(tr["final"], m)
    assert fin.rng_counter == ref["rng_counter"] and fin.rng_idx == ref["rng_idx"]
    assert fin.accepted == tr["accepted"]


def test_int8_v_not_used_where_ineligible(cfgdir):
    """Small ensembles (QB = 1 tiles) and the general kernel keep the FP64 DMMA path; the mode
    switch is per handle and reversible."""
    sp = cfgdir / "cfg2.spinor"
    text = (cfgdir / "cfg2.conf").read_text()
    dw = DeviceWalker(System(sp, text), max_walkers=64)
    assert dw.int8_v()  # selected and eligible system; m decides per step
    dw.kramers(0)
    assert not dw.int8_v()
    dw.kramers(1)
    assert not dw.int8_v(0) and dw.int8_v(1)


@pytest.mark.parametrize("name,m", [("cfg5-86", 1024), ("cfg5-36", 640)])
def test_int8_v_heavy_atoms_match_oracle(cfgdir, tmp_path, name, m):
    """cfg5 sweep members with other K' (n_vir 208 / 94: 13 / 6 k-steps) and ensemble sizes that
    are not multiples of the 10-walker P blocks, one production step each, against the oracle's
    full C(m,2) pair loop (rows over host threads)."""
    import os
    from paper_2203_05632_b200 import generate_config
    sp, conf = generate_config(name, tmp_path)
    text = conf.read_text()
    orc = oracle_py.OracleSystem(sp, text)
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    assert dw.int8_v()
    dw.init_ensemble(m, seed=8)
    dw.burn_in(20)
    dw.advance(1)
    w = dw.get_ensemble().walkers[:, :8]
    tau = 0.05
    ref = orc.replay_parallel(w, tau, threads=max(1, min(32, os.cpu_count() or 1)))
    got = dw.replay(w[None], np.array([tau]))[0]
    for k in (0, 2, 4):
        assert abs(got[k] - ref[k]) <= REL * abs(ref[k]), k


def test_int8_v_buffers_grow_after_capture(cfgdir):
    """A replay with more walkers grows the INT8 path's buffers after advance() captured its CUDA
    graphs; the graphs must be re-captured (not replayed against freed buffers): the chain after
    the growth still equals the one of a fresh handle."""
    sp = cfgdir / "cfg3.spinor"
    text = (cfgdir / "cfg3.conf").read_text()
    orc = oracle_py.OracleSystem(sp, text)
    tr = orc.trajectory(seed=21, stream=0, m=256, burn=20, nsteps=1)
    a = DeviceWalker(System(sp, text), max_walkers=256)
    b = DeviceWalker(System(sp, text), max_walkers=256)
    for dw in (a, b):
        dw.init_ensemble(192, seed=4)
        dw.burn_in(10)
    a.advance(32)                            # graphs captured with buffers for 192 walkers
    a.replay(tr["walkers"], tr["tau"])       # grows them to 256
    b.advance(32)
    va, _ = a.advance(34)
    vb, _ = b.advance(34)
    assert np.array_equal(va, vb)


def test_int8_v_two_pass_slicing_wide_set(tmp_path):
    """n_vir 446 > 384: oz_slice_kernel's two-pass form (the row maximum, then the digits; no
    values held across the reduction). Replayed steps against the oracle and the DMMA path,
    guarded and unguarded (the generator's 'wide' stress set, host/generate.cpp)."""
    from paper_2203_05632_b200 import generate_config
    sp, conf = generate_config("wide", tmp_path)
    text = conf.read_text()
    orc = oracle_py.OracleSystem(sp, text)
    assert orc.n_vir > 384
    tr = orc.trajectory(seed=3, stream=0, m=192, burn=20, nsteps=2)
    dw = DeviceWalker(System(sp, text), max_walkers=192)
    assert dw.kramers() and dw.int8_v()
    for tol in (0.0, 2e-10):
        dw.guard(tol)
        got = dw.replay(tr["walkers"], tr["tau"])
        for k in (0, 2, 4):
            assert rel_err(got[:, k], tr["est"][:, k]) < REL, (tol, k)
    dw.int8_v(0)
    dmma = dw.replay(tr["walkers"], tr["tau"])
    assert rel_err(dmma[:, 0], tr["est"][:, 0]) < REL


def test_int8_v_truncation_is_exact_on_the_physical_path(cfgdir):
    """The opt-in INT8 V blocks of the physical estimator (64-column tiles, V written for pair_kr's
    trace epilogue) under the three truncation modes: bit-identical step records, fewer slice
    products issued with the leading zero slices skipped than with whole k-steps only."""
    sp = cfgdir / "cfg4.spinor"
    text = (cfgdir / "cfg4.conf").read_text() + "estimator physical\n"
    orc = oracle_py.OracleSystem(sp, text)
    tr = orc.trajectory(seed=5, stream=0, m=192, burn=20, nsteps=1, physical=True)
    taus = np.array([0.02, 0.3, 2.0])
    walkers = np.repeat(tr["walkers"][:1], len(taus), axis=0)
    dw = DeviceWalker(System(sp, text), max_walkers=192)
    assert dw.int8_v(1)
    out, issued = {}, {}
    for mode in (1, 2, 0):
        dw.int8_truncation(mode)
        e0, _ = dw.int8_ksteps()
        out[mode] = dw.replay_ex(walkers, taus)
        e1, full = dw.int8_ksteps()  # (the full count is set by the launch)
        issued[mode] = (e1 - e0) / (len(taus) * full)
    assert out[1].tobytes() == out[0].tobytes() and out[2].tobytes() == out[0].tobytes()
    assert issued[1] < issued[2] - 0.02 < issued[0] - 0.02 and issued[0] == pytest.approx(1.0, rel=1e-12), issued
    ref = orc.replay(walkers, taus, physical=True)
    for c in (0, 2, 4):
        assert rel_err(out[1][:, c], ref[:, c]) < REL, c


@pytest.mark.parametrize("name,m", [("cfg3", 256), ("cfg4", 192), ("cfg5-36", 330)])
def test_int8_v_kstep_truncation_is_exact(cfgdir, tmp_path, name, m):
    """The V-GEMM skips a tile's trailing k-steps when every digit there is zero (high virtual
    energies at this tau, include/mcmp2dev.h mcmp2dev_oz_truncation) and, in the partly empty
    k-steps before them, the slice products whose A or B slice is all zero: the skipped products
    are exact zeros, so every field of the step records is bit-identical to the full K' loop; at
    large tau k-steps are actually skipped, at tau -> 0 none are; the oracle still agrees."""
    from paper_2203_05632_b200 import generate_config
    if (cfgdir / f"{name}.spinor").exists():
        sp, text = cfgdir / f"{name}.spinor", (cfgdir / f"{name}.conf").read_text()
    else:
        sp, conf = generate_config(name, tmp_path)
        text = conf.read_text()
    orc = oracle_py.OracleSystem(sp, text)
    tr = orc.trajectory(seed=31, stream=0, m=m, burn=20, nsteps=1)
    taus = np.array([1e-6, 0.05, 0.7, 3.0])
    walkers = np.repeat(tr["walkers"][:1], len(taus), axis=0)
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    assert dw.int8_v() and dw.int8_truncation()
    frac = []
    on = []
    for k, tau in enumerate(taus):  # one replay per tau, to read the k-steps each one issued
        e0, full = dw.int8_ksteps()
        on.append(dw.replay_ex(walkers[k:k + 1], taus[k:k + 1]))
        e1, full = dw.int8_ksteps()
        frac.append((e1 - e0) / full)
    on = np.concatenate(on)
    assert dw.int8_truncation(2)  # whole empty k-steps only: the partly empty ones run all 21 products
    e0, full = dw.int8_ksteps()
    whole = dw.replay_ex(walkers, taus)
    e1, _ = dw.int8_ksteps()
    frac_whole = (e1 - e0) / (len(taus) * full)
    assert not dw.int8_truncation(0)
    e0, full = dw.int8_ksteps()
    off = dw.replay_ex(walkers, taus)
    e1, _ = dw.int8_ksteps()
    assert e1 - e0 == pytest.approx(len(taus) * full, rel=1e-12)  # (the counter is in slice products / 21)
    assert on.tobytes() == off.tobytes() and whole.tobytes() == off.tobytes()
    # the leading zero slices of the partly empty k-steps are skipped on top of the empty k-steps
    assert np.mean(frac) < frac_whole - 0.02 and frac_whole < 1.0, (frac, frac_whole)
    assert frac[0] > 0.99 and frac[-1] < 0.8 and all(a >= b for a, b in zip(frac, frac[1:])), frac
    ref = orc.replay(walkers, taus)
    for c, r in ((0, 0), (2, 2), (4, 4)):
        assert rel_err(on[:, c], ref[:, r]) < REL, (c, frac)


def test_int8_v_slice_overlap_does_not_change_results(cfgdir):
    """oz_slice_kernel runs on a side stream next to the O pass (mcmp2dev_oz_overlap); the same
    chain with the two kernels in series gives bit-identical step records, through the captured
    graphs (64 steps) and single launches (3 more)."""
    sp = cfgdir / "cfg3.spinor"
    text = (cfgdir / "cfg3.conf").read_text()
    recs = []
    for mode in (1, 0):
        dw = DeviceWalker(System(sp, text), max_walkers=256)
        assert dw.int8_overlap(mode) == bool(mode)
        dw.init_ensemble(256, seed=12)
        dw.burn_in(30)
        recs.append(dw.advance_ex(67))
        dw.close()
    assert recs[0].tobytes() == recs[1].tobytes()


def test_int8_v_default_needs_more_than_one_kstep(cfgdir):
    """n_vir <= 16 (one 32-wide k-step of K'): the DMMA pair kernel is the default (the V-GEMM's
    per-tile epilogue would set the pace); mcmp2dev_pair_path(h, 1) still selects INT8, and the
    two agree with the oracle."""
    sp = cfgdir / "cfg5-2.spinor"
    text = (cfgdir / "cfg5-2.conf").read_text()
    orc = oracle_py.OracleSystem(sp, text)
    tr = orc.trajectory(seed=3, stream=0, m=208, burn=20, nsteps=1)
    dw = DeviceWalker(System(sp, text), max_walkers=208)
    assert dw.kramers() and not dw.int8_v()
    dmma = dw.replay(tr["walkers"], tr["tau"])
    assert dw.int8_v(1)
    got = dw.replay(tr["walkers"], tr["tau"])
    for k in (0, 2, 4):
        assert rel_err(dmma[:, k], tr["est"][:, k]) < REL, k
        assert rel_err(got[:, k], tr["est"][:, k]) < REL, k
    assert not dw.int8_v(0)

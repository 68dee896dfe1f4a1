"""Batched ensembles: several reference workers (driver.cpp:423-438; Philox stream = worker
index, driver.cpp:354-356) advanced by one handle in the same launches (include/mcmp2dev.h,
mcmp2dev_init_batch). Every ensemble must follow the oracle's chain for its own stream exactly
as a single-ensemble handle does (1e-10 relative, identical RNG state and counters)."""
import numpy as np
import pytest

import oracle_py
from paper_2203_05632_b200 import DeviceWalker, System
from paper_2203_05632_b200.native import Mcmp2ArgumentError

pytestmark = pytest.mark.gpu

REL = 1e-10


def rel_err(got, ref):
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)))


@pytest.mark.parametrize("name,m,nens,burn,nsteps,step,physical", [
    ("cfg1", 16, 5, 60, 40, 0.3, False),
    ("cfg2", 16, 3, 30, 6, 0.0, False),
    ("cfg2", 32, 2, 30, 4, 0.0, True),
    ("cfg2", 64, 2, 30, 3, 0.0, False),   # m >= 64: the QB = 2 build of pair_kr.cu
    ("cfg2", 80, 2, 30, 2, 0.0, True),
])
def test_batched_ensembles_follow_oracle_chains(cfgdir, name, m, nens, burn, nsteps, step, physical):
    sp = cfgdir / f"{name}.spinor"
    text = (cfgdir / f"{name}.conf").read_text() + ("estimator physical\n" if physical else "")
    orc = oracle_py.OracleSystem(sp, text)
    seed, stream0 = 21, 4
    dw = DeviceWalker(System(sp, text), max_walkers=nens * m)
    dw.init_batch(nens, m, seed=seed, stream0=stream0)
    if step:
        dw.set_sigma_step(step)
    dw.burn_in(burn, adapt=step == 0.0)
    v, im = dw.advance(nsteps)
    assert v.shape == (nsteps, nens)
    for e in range(nens):
        tr = orc.trajectory(seed=seed, stream=stream0 + e, m=m, burn=burn, nsteps=nsteps, step_size=step,
                            adapt=step == 0.0, physical=physical)
        assert rel_err(v[:, e], tr["est"][:, 0]) < REL, e
        fin = dw.get_ensemble_at(e)
        ref = oracle_py.state_to_ensemble(tr["final"], m)
        assert fin.rng_counter == ref["rng_counter"] and fin.rng_idx == ref["rng_idx"]
        assert fin.proposed == tr["proposed"] and fin.accepted == tr["accepted"]
        assert fin.sigma_step == ref["sigma_step"]
        assert np.max(np.abs(fin.walkers - ref["walkers"]) / (np.abs(ref["walkers"]) + 1e-300)) < REL


def test_batch_matches_single_handles_and_graph_path(cfgdir):
    """64 ensembles through the captured-graph path (advance in chunks of 32 steps) against one
    single-ensemble handle per stream; then a per-ensemble checkpoint round trip."""
    sp = cfgdir / "cfg1.spinor"
    text = (cfgdir / "cfg1.conf").read_text()
    sysd = System(sp, text)
    nens, m, nsteps = 64, 16, 64
    dw = DeviceWalker(sysd, max_walkers=nens * m)
    dw.init_batch(nens, m, seed=3, stream0=0)
    dw.set_sigma_step(0.3)
    dw.burn_in(50, adapt=False)
    states = [dw.get_ensemble_at(e) for e in (0, 17, 63)]
    v, _ = dw.advance(nsteps)
    one = DeviceWalker(sysd, max_walkers=m)
    for e, st in zip((0, 17, 63), states):
        one.set_ensemble(st)
        ref, _ = one.advance(nsteps)
        assert rel_err(v[:, e], ref) < 1e-12, e
    # restore ensemble 17 and replay its steps: identical values, other ensembles untouched
    after = dw.get_ensemble_at(5)
    dw.set_ensemble_at(17, states[1])
    w, _ = dw.advance(nsteps)
    assert rel_err(w[:, 17], v[:, 17]) < 1e-12
    assert not np.allclose(w[:, 5], v[:, 5])  # ensemble 5 moved on from `after`
    assert dw.get_ensemble_at(5).proposed == after.proposed + nsteps * m


def test_batch_argument_errors(cfgdir):
    sysd = System(cfgdir / "cfg1.spinor", (cfgdir / "cfg1.conf").read_text())
    dw = DeviceWalker(sysd, max_walkers=64)
    with pytest.raises(Mcmp2ArgumentError, match="multiple of 16"):
        dw.init_batch(2, 12, seed=1)
    with pytest.raises(Mcmp2ArgumentError, match="sized for"):
        dw.init_batch(5, 16, seed=1)
    with pytest.raises(Mcmp2ArgumentError, match="at most 480"):
        DeviceWalker(sysd, max_walkers=1024).init_batch(2, 496, seed=1)
    dw.init_batch(4, 16, seed=1)
    with pytest.raises(Mcmp2ArgumentError, match="get_ensemble_at"):
        dw.get_ensemble()
    with pytest.raises(Mcmp2ArgumentError, match="no such ensemble"):
        dw.get_ensemble_at(4)
    st = dw.get_ensemble_at(1)
    with pytest.raises(Mcmp2ArgumentError, match="stream0 \\+ e"):
        dw.set_ensemble_at(2, st)
    from paper_2203_05632_b200.native import check_dev
    with pytest.raises(Mcmp2ArgumentError, match="active ensembles"):
        check_dev(dw._d.mcmp2dev_advance_batch(dw._h, 1, 5, None, None), dw._h)


@pytest.mark.parametrize("name,kramers,physical", [("syn1c", 0, False), ("syn2c", 0, False),
                                                   ("cfg2", 0, False), ("cfg2", 0, True)])
def test_batched_general_kernel_follows_oracle(cfgdir, name, kramers, physical):
    """The general pair kernel (1c/2c sets, or the Kramers path switched off) batches too."""
    sp = cfgdir / f"{name}.spinor"
    text = (cfgdir / f"{name}.conf").read_text() + ("estimator physical\n" if physical else "")
    orc = oracle_py.OracleSystem(sp, text)
    m, nens, burn, nsteps = 16, 3, 30, 4
    dw = DeviceWalker(System(sp, text), max_walkers=nens * m)
    dw.kramers(kramers)
    assert not dw.kramers()
    dw.init_batch(nens, m, seed=6, stream0=1)
    dw.burn_in(burn)
    v, im = dw.advance(nsteps)
    for e in range(nens):
        tr = orc.trajectory(seed=6, stream=1 + e, m=m, burn=burn, nsteps=nsteps, physical=physical)
        assert rel_err(v[:, e], tr["est"][:, 0]) < REL, e
        assert np.max(np.abs(im[:, e] - tr["est"][:, 1])) <= REL * np.max(np.abs(tr["est"][:, 0]))


def test_bulk_state_round_trip(cfgdir):
    """get_ensembles / set_ensembles (all ensembles in two copies) agree with the per-ensemble
    calls and restore the batch exactly."""
    sysd = System(cfgdir / "cfg2.spinor", (cfgdir / "cfg2.conf").read_text())
    dw = DeviceWalker(sysd, max_walkers=4 * 16)
    dw.init_batch(4, 16, seed=8, stream0=2)
    dw.burn_in(20)
    bulk = dw.get_ensembles()
    for e in range(4):
        one = dw.get_ensemble_at(e)
        assert np.array_equal(one.walkers, bulk[e].walkers) and one.rng_counter == bulk[e].rng_counter
        assert one.rng_idx == bulk[e].rng_idx and one.sigma_step == bulk[e].sigma_step
    v1, _ = dw.advance(5)
    dw.set_ensembles(bulk)
    v2, _ = dw.advance(5)
    assert np.array_equal(v1, v2)


def test_reinit_with_other_batch_sizes_drops_stale_graphs(cfgdir):
    """A handle re-initialised with more ensembles reallocates its batched buffers; the graphs
    captured before hold the old addresses and must be dropped (mcmp2dev.cu drop_graphs). Going
    4 -> 8 -> 4 ensembles with the same seed must give the chain a fresh 4-ensemble handle gives."""
    sp = cfgdir / "cfg1.spinor"
    text = (cfgdir / "cfg1.conf").read_text()
    sysd = System(sp, text)
    m, nsteps = 16, 64  # two captured graphs of 32 steps per advance

    def run(dw, nens):
        dw.init_batch(nens, m, seed=11, stream0=0)
        dw.set_sigma_step(0.3)
        dw.burn_in(20, adapt=False)
        dw.prepare()
        return dw.advance(nsteps)[0]

    fresh = DeviceWalker(sysd, max_walkers=8 * m)
    ref4 = run(fresh, 4)
    fresh.close()
    dw = DeviceWalker(sysd, max_walkers=8 * m)
    first = run(dw, 4)
    eight = run(dw, 8)
    again = run(dw, 4)
    dw.close()
    assert np.array_equal(first, ref4) and np.array_equal(again, ref4)
    assert rel_err(eight[:, :4], ref4) < 1e-12  # streams 0..3 are the same chains

"""The accuracy guard of the INT8 (Ozaki) V path (csrc/pair_oz.cu, include/mcmp2dev.h
mcmp2dev_guard) and the long-run evidence for that path.

The reference forms the V blocks in FP64 (greens.cpp:73-79) and contracts them literally
(estimator.cpp:26-32); the INT8 path's error depends on the data, and on steps whose pair sums
cancel it is amplified. Each INT8 step therefore carries an error estimate of its direct and
exchange sums; a step whose estimate exceeds the tolerance is recomputed on the FP64 DMMA pair
kernel in the same launch sequence. Tests here:
  * the fallback mechanism: a vanishing tolerance sends every step to DMMA, bit-identical to the
    DMMA path, in replay and through the captured graphs;
  * the estimate bounds the measured error on the oracle's steps;
  * a constructed ill-conditioned step (one walker's weight tuned so the step value cancels to
    1e-4 of its parts) trips the guard, and the guarded result meets the 1e-10 gate that the
    unguarded INT8 result misses;
  * long chains (2000 steps at cfg3 m = 512 and cfg4 m = 2048) on the guarded INT8 path against
    the DMMA path, plain and condition-aware error (|error| / (sum |terms| / C(m,2)));
  * full-size single steps of the cfg5 sweep members at m = 8192.
Summaries of the long runs go to gpurun_out/ when the GPU run exports GRAFT_REPO_ROOT."""
import json
import os
from pathlib import Path

import numpy as np
import pytest

import oracle_py
from paper_2203_05632_b200 import DeviceWalker, System, generate_config
from paper_2203_05632_b200.walker import EnsembleState

pytestmark = pytest.mark.gpu

REL = 1e-10
TOL = 2e-10  # the default guard tolerance (mcmp2dev.cu kGuardTol)
F = {n: i for i, n in enumerate(DeviceWalker.STEP_EX_FIELDS)}


def rel(a, b):
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


def dump(name, obj):
    root = os.environ.get("GRAFT_REPO_ROOT")
    if root:
        out = Path(root) / "gpurun_out"
        out.mkdir(exist_ok=True)
        (out / f"guard_{name}.json").write_text(json.dumps(obj, indent=1))


def oracle_steps(cfgdir, name, m, nsteps, seed=13):
    sp = cfgdir / f"{name}.spinor"
    text = (cfgdir / f"{name}.conf").read_text()
    tr = oracle_py.OracleSystem(sp, text).trajectory(seed=seed, stream=0, m=m, burn=20, nsteps=nsteps)
    return sp, text, tr


def test_vanishing_tolerance_sends_every_step_to_dmma(cfgdir):
    """tol = 1e-300: every INT8 step fails the check and the guarded DMMA launch recomputes it;
    the results are bit-identical to the DMMA path (replay and graph-captured chains)."""
    sp, text, tr = oracle_steps(cfgdir, "cfg3", 192, 3)
    dw = DeviceWalker(System(sp, text), max_walkers=192)
    assert dw.int8_v() and dw.guard() == pytest.approx(TOL)
    dw.guard(1e-300)
    got = dw.replay_ex(tr["walkers"], tr["tau"])
    assert np.all(got[:, F["int8_v"]] == 1) and np.all(got[:, F["fallback"]] == 2)  # refined, then DMMA
    dw.int8_v(0)
    dmma = dw.replay_ex(tr["walkers"], tr["tau"])
    assert np.all(dmma[:, F["int8_v"]] == 0)
    assert np.array_equal(got[:, :6], dmma[:, :6])
    for k in (0, 2, 4):
        assert np.all(rel(got[:, k], tr["est"][:, k]) < REL)
    # through the captured graphs: 32 + 8 steps, forced fallback vs the DMMA path from one state
    dw.int8_v(1)
    dw.init_ensemble(192, seed=5)
    dw.burn_in(20)
    st = dw.get_ensemble()
    dw.guard_stats()  # reset the counters (the replays above were checked too)
    a = dw.advance_ex(40)
    stats = dw.guard_stats()
    assert stats["checked"] == 40 and stats["dmma"] == 40
    dw.set_ensemble(st)
    dw.int8_v(0)
    b = dw.advance_ex(40)
    assert np.array_equal(a[:, :6], b[:, :6])


def test_guard_off_and_on_agree_with_the_oracle(cfgdir):
    """tol <= 0 turns the guard off (no estimate, no fallback launch); with the default the
    estimate covers the measured INT8 error of every step (the model's claim on these inputs),
    and steps kept on INT8 are within tol of FP64 in each sum."""
    sp, text, tr = oracle_steps(cfgdir, "cfg3", 192, 4)
    dw = DeviceWalker(System(sp, text), max_walkers=192)
    dw.guard(0.0)
    off = dw.replay_ex(tr["walkers"], tr["tau"])
    assert np.all(off[:, F["est_err_direct"]] == 0) and np.all(off[:, F["fallback"]] == 0)
    dw.guard(TOL)
    on = dw.replay_ex(tr["walkers"], tr["tau"])
    assert np.array_equal(on[:, :6][on[:, F["fallback"]] == 0], off[:, :6][on[:, F["fallback"]] == 0])
    for k, e in ((2, "est_err_direct"), (4, "est_err_exchange")):
        err = np.abs(off[:, k] - tr["est"][:, k])
        assert np.all(err <= on[:, F[e]]), (k, err, on[:, F[e]])
        assert np.all(rel(on[:, k], tr["est"][:, k]) < REL)
    assert np.all(on[:, F["abs_direct"]] >= np.abs(on[:, 2])) and np.all(on[:, F["abs_exchange"]] >= np.abs(on[:, 4]))


def test_refinement_pass_reduces_the_int8_error(cfgdir):
    """A tolerance of 0.3 of the main pass's estimate sends each step to the refinement pass (7th
    slices, diagonal s + t = 6, on the tile groups that carry the error) and no further: the
    refined step is kept (fallback 1), its estimate meets the tolerance, and its error against
    the oracle drops >= 4x or to FP64 rounding. (The refined pairs' model is 2^-49 against the
    main pass's 2^-46: the main pass's merged sums keep the last diagonal rounded to 8 bits, so a
    refined element is good to ~2^-48 of its row scales, not to the 7th slice's 2^-54.)"""
    m = 192
    sp, text, tr = oracle_steps(cfgdir, "cfg3", m, 3, seed=31)
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    npairs = 0.5 * m * (m - 1)
    dw.guard(1e300)  # estimate only
    raw = dw.replay_ex(tr["walkers"], tr["tau"])
    for k in range(3):
        r = raw[k]
        est = max(r[F["est_err_direct"]] / abs(r[2]), r[F["est_err_exchange"]] / abs(r[4]),
                  np.hypot(r[F["est_err_direct"]], r[F["est_err_exchange"]]) / abs(r[0] * npairs))
        dw.guard(0.3 * est)
        got = dw.replay_ex(tr["walkers"][k:k + 1], tr["tau"][k:k + 1])[0]
        assert got[F["fallback"]] == 1, (k, got[F["fallback"]])
        for j in (2, 4):
            e_raw, e_ref = abs(r[j] - tr["est"][k, j]), abs(got[j] - tr["est"][k, j])
            assert e_ref <= e_raw / 4 + 1e-14 * abs(tr["est"][k, j]), (k, j, e_raw, e_ref)
        # selective refinement: the tile groups above 1 / groups of the budget get the 7th slice,
        # so the refined step's estimate meets the tolerance it failed (0.3 of its estimate here)
        assert got[F["est_err_direct"]] < 0.3 * r[F["est_err_direct"]] * 1.05
        assert got[F["est_err_exchange"]] < 0.3 * r[F["est_err_exchange"]] * 1.05


def test_constructed_ill_conditioned_step_trips_the_guard(cfgdir):
    """The step value is linear in one walker's weight 1/(g1 g2) (estimator.cpp:55): with its g1
    scaled so that the pairs with that walker cancel the others to ~1e-5 of their size (the first
    of a ladder of cancellations at which the unguarded INT8 value misses the 1e-10 gate), the
    guard rejects the INT8 result and the step comes from the refinement pass or the DMMA
    kernel, within the gate of the oracle."""
    m = 192
    sp, text, tr = oracle_steps(cfgdir, "cfg3", m, 1, seed=29)
    orc = oracle_py.OracleSystem(sp, text)
    W0, tau = tr["walkers"][0].copy(), tr["tau"][:1]
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    built = None
    for ps in range(m):
        dw.int8_v(0)
        W1 = W0.copy()
        W1[ps, 6] *= 0.5  # walker ps's weight x2
        v1, v2 = dw.replay(np.stack([W0, W1]), np.concatenate([tau, tau]))[:, 0]
        B = v2 - v1       # value(w) = A + w B, w = weight multiplier of walker ps
        A = v1 - B
        if A * B >= 0:
            continue
        dw.int8_v(1)
        dw.guard(0.0)
        for cancel in (1e-4, 5e-5, 3e-5, 2e-5):
            W = W0.copy()
            W[ps, 6] /= -A / B * (1 + cancel)
            ref = orc.replay(W[None], tau)[0]
            raw = dw.replay_ex(W[None], tau)[0]
            if abs(raw[0] - ref[0]) > REL * abs(ref[0]):
                built = W
                break
        break
    assert built is not None
    # the value (d + x) / C(m,2) cancels to < 1e-3 of the direct sum
    assert abs(ref[0]) * 0.5 * m * (m - 1) < 1e-3 * abs(ref[2])
    dw.guard(TOL)
    got = dw.replay_ex(built[None], tau)[0]
    assert raw[F["int8_v"]] == 1 and raw[F["fallback"]] == 0
    assert abs(raw[0] - ref[0]) > REL * abs(ref[0])          # INT8 alone fails the gate here
    assert got[F["fallback"]] in (1, 2)                       # the guard caught it
    assert abs(got[0] - ref[0]) <= REL * abs(ref[0])
    for k in (2, 4):
        assert abs(got[k] - ref[k]) <= REL * abs(ref[k])


@pytest.mark.parametrize("name,m,nsteps", [("cfg3", 512, 2000), ("cfg4", 2048, 2000)])
def test_long_chain_int8_against_dmma(cfgdir, name, m, nsteps):
    """The same chain (same state; the walk does not depend on the estimates) on the guarded
    INT8 path, on the unguarded INT8 path and on the DMMA path. Every guarded step is within
    1e-10 of DMMA in value, direct and exchange sums; the unguarded errors, their condition-aware
    form and the guard's estimates are recorded (gpurun_out/guard_chain_<cfg>.json)."""
    sp = cfgdir / f"{name}.spinor"
    text = (cfgdir / f"{name}.conf").read_text()
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    dw.init_ensemble(m, seed=17)
    dw.burn_in(200)
    st = dw.get_ensemble()
    runs = {}
    # "raw": the estimate is computed (tol 1e300) but never rejects a step
    for label, int8, tol in (("guarded", 1, TOL), ("raw", 1, 1e300), ("dmma", 0, TOL)):
        dw.set_ensemble(st)
        dw.int8_v(int8)
        dw.guard(tol)
        runs[label] = dw.advance_ex(nsteps)
        runs[label + "_stats"] = dw.guard_stats()
    g, r, d = runs["guarded"], runs["raw"], runs["dmma"]
    root = os.environ.get("GRAFT_REPO_ROOT")
    if root:
        (Path(root) / "gpurun_out").mkdir(exist_ok=True)
        np.savez_compressed(Path(root) / "gpurun_out" / f"guard_chain_{name}.npz", guarded=g, raw=r, dmma=d)
    assert np.all(g[:, F["int8_v"]] == 1) and np.all(d[:, F["int8_v"]] == 0)
    npairs = 0.5 * m * (m - 1)
    out = {"config": name, "m": m, "steps": nsteps, "guard_tol": TOL,
           "refined": int((g[:, F["fallback"]] == 1).sum()), "dmma": int((g[:, F["fallback"]] == 2).sum()),
           "guard_stats": runs["guarded_stats"]}
    for k, lab in ((0, "value"), (2, "direct"), (4, "exchange")):
        eg, er = rel(g[:, k], d[:, k]), rel(r[:, k], d[:, k])
        assert np.all(eg < REL), (lab, float(eg.max()))
        absum = (r[:, F["abs_direct"]] + r[:, F["abs_exchange"]]) if k == 0 else r[:, F["abs_" + lab]]
        cond = np.abs(r[:, k] - d[:, k]) / np.maximum(absum / (npairs if k == 0 else 1.0), 1e-300)
        out[lab] = {"guarded_max_rel": float(eg.max()), "raw_max_rel": float(er.max()),
                    "raw_median_rel": float(np.median(er)), "raw_steps_over_1e-10": int((er > REL).sum()),
                    "raw_max_condition_aware": float(cond.max())}
    # the estimate against the measured raw error, direct and exchange
    for k, e in ((2, "est_err_direct"), (4, "est_err_exchange")):
        err = np.abs(r[:, k] - d[:, k])
        ratio = r[:, F[e]] / np.maximum(err, 1e-300)
        out[e] = {"min_est_over_err": float(ratio.min()), "median_est_over_err": float(np.median(ratio)),
                  "steps_err_above_est": int((err > r[:, F[e]]).sum())}
    dump(f"chain_{name}", out)
    assert out["est_err_direct"]["steps_err_above_est"] == 0 and out["est_err_exchange"]["steps_err_above_est"] == 0


@pytest.mark.parametrize("name", ["cfg5-18", "cfg5-36", "cfg5-54", "cfg5-86"])
def test_cfg5_full_size_step(tmp_path, name):
    """One production-size step (m = 8192) of each cfg5 sweep member: guarded INT8 against the
    DMMA path (itself pinned to the oracle by the smaller full-size tests) to 1e-10, with the
    unguarded error recorded."""
    m = 8192
    sp, conf = generate_config(name, tmp_path)
    text = conf.read_text()
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    assert dw.int8_v()
    dw.init_ensemble(m, seed=3)
    dw.burn_in(50)
    st = dw.get_ensemble()
    res = {}
    for label, int8, tol in (("guarded", 1, TOL), ("raw", 1, 0.0), ("dmma", 0, TOL)):
        dw.set_ensemble(st)
        dw.int8_v(int8)
        dw.guard(tol)
        res[label] = dw.advance_ex(2)
    g, r, d = res["guarded"], res["raw"], res["dmma"]
    out = {"config": name, "m": m, "refined": int((g[:, F["fallback"]] == 1).sum()),
           "dmma": int((g[:, F["fallback"]] == 2).sum())}
    for k, lab in ((0, "value"), (2, "direct"), (4, "exchange")):
        assert np.all(rel(g[:, k], d[:, k]) < REL), lab
        out[lab] = {"guarded_max_rel": float(rel(g[:, k], d[:, k]).max()), "raw_max_rel": float(rel(r[:, k], d[:, k]).max())}
    dump(f"full_{name}", out)

"""CPU: the oracle (oracle/, the C++ restatement the device path is tested against) pinned to
the REFERENCE ITSELF -- its rng, gaussian, model, weights, sampler, greens, estimator and driver
translation units compiled unmodified (oracle/build_ref.sh, against the minimal dense header
oracle/eigen_subset: Eigen3 is absent from this image). Checked: spinor values
(SpinorSet::evaluate_into, model.cpp:166-178) and the sampling weight g (weights.cpp:92-99) at
random points; replayed step estimates and their direct / exchange pair sums (estimator.cpp:35-75)
on the oracle's own trajectories; whole Engine runs (driver.cpp:336-480: init, burn-in,
Metropolis chain, blocking, merge, report) against the oracle Engine. Configs carry no
extension keys (step-size, estimator), which the reference's parser rejects."""
import numpy as np
import pytest

import oracle_py
import ref_py

pytestmark = pytest.mark.skipif(not ref_py.available(), reason="oracle/_ref/libref_mcmp2.so not built")


def conf_weights(text):
    return "".join(l + "\n" for l in text.splitlines() if l.startswith("weight"))


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "syn1c", "syn2c"])
def test_spinor_values_and_weight_match_the_reference(cfgdir, name):
    sp = cfgdir / f"{name}.spinor"
    text = (cfgdir / f"{name}.conf").read_text()
    ref = ref_py.RefSystem(sp, text)
    orc = oracle_py.OracleSystem(sp, text)
    assert (ref.ncomp, ref.n_occ, ref.n_vir) == (orc.ncomp, orc.n_occ, orc.n_vir)
    assert ref.ng == pytest.approx(orc.ng, rel=1e-14) and ref.lambda_ == orc.lambda_
    pts = np.random.default_rng(3).normal(scale=1.2, size=(24, 3))
    ro, rv = ref.evaluate(pts)
    oo, ov = orc.evaluate(pts)
    for r, o in ((ro, oo), (rv, ov)):
        scale = np.abs(r).max()
        assert np.max(np.abs(r - o)) <= 1e-13 * scale
    assert np.allclose(ref.g(pts), orc.g(pts), rtol=1e-14, atol=0)


@pytest.mark.parametrize("name,m,nsteps,seed", [("cfg1", 16, 3, 7), ("cfg2", 24, 2, 5), ("cfg3", 12, 2, 9),
                                                ("syn1c", 8, 3, 4), ("syn2c", 8, 3, 4)])
def test_replayed_steps_match_the_reference(cfgdir, name, m, nsteps, seed):
    """The oracle's step estimates on its own trajectory against the reference's
    mc_step_estimate and sample_term sums at the same walkers and tau, 1e-12 relative."""
    sp = cfgdir / f"{name}.spinor"
    text = (cfgdir / f"{name}.conf").read_text()
    orc = oracle_py.OracleSystem(sp, text)
    tr = orc.trajectory(seed=seed, stream=0, m=m, burn=30, nsteps=nsteps)
    ref = ref_py.RefSystem(sp, text).replay(tr["walkers"], tr["tau"])
    est = tr["est"]
    for k in (0, 2, 4):
        assert np.max(np.abs(est[:, k] - ref[:, k]) / np.abs(ref[:, k])) < 1e-12, k
    assert np.max(np.abs(est[:, 1] - ref[:, 1])) <= 1e-12 * np.max(np.abs(ref[:, 0])) + 1e-300


@pytest.mark.parametrize("name,extra", [
    ("syn1c", "walkers 6\nsteps 400\nworkers 2\nseed 4\nburnin 50\nblocksize 20\ncheckpoint-interval 100\n"),
    ("cfg2", "walkers 12\nsteps 60\nworkers 2\nseed 11\nburnin 40\nblocksize 10\ncheckpoint-interval 30\n"),
])
def test_engine_runs_match_the_reference(cfgdir, name, extra):
    """The whole reference Engine (init_ensemble, burn-in with adaptation, the Metropolis chain
    on the reference Philox stream per worker, tau draws, estimates, blocking, merge, report)
    against the oracle Engine on the same config: same step counts, E2 and sigma_bar to 1e-10."""
    text = f"spinors {cfgdir / (name + '.spinor')}\n" + extra + conf_weights((cfgdir / f"{name}.conf").read_text())
    ref = ref_py.run_config(text)
    orc = oracle_py.run_config(text)

    def parse(rep):
        lines = rep.splitlines()
        out = {"E2": float(lines[0].split("=")[1].split()[0]), "sigma_bar": float(lines[1].split("=")[1].split()[0]),
               "steps": int(lines[2].split("=")[1])}
        out["workers"] = [(l.split(",")[0], float(l.split(",")[1].split()[1])) for l in lines if l.startswith("worker")]
        return out
    r, o = parse(ref), parse(orc)
    assert r["steps"] == o["steps"] and [w[0] for w in r["workers"]] == [w[0] for w in o["workers"]]
    for (_, a), (_, b) in zip(r["workers"], o["workers"]):
        assert b == pytest.approx(a, rel=1e-12, abs=0)  # each worker's mean I
    assert o["E2"] == pytest.approx(r["E2"], rel=1e-10, abs=0)
    assert o["sigma_bar"] == pytest.approx(r["sigma_bar"], rel=1e-10, abs=0)


# the reference's own unit tests (tests/test_{rng,model,weights,greens,estimator,sampler,driver,
# oracle}.cpp) built against the reference sources here (oracle/build_ref.sh: eigen_subset and
# doctest_subset stand in for the absent Eigen3 and doctest); three fail for reasons inside the
# reference, not the build:
KNOWN_REFERENCE_FAILURES = {
    # asserts sigma_bar == 0.0 for a constant 0.7 stream; IEEE accumulation gives mean
    # 0.7000000000000013 against block means 0.7000000000000001 (DESIGN.md findings)
    "blocking accumulator: hand examples",
    # runs the he_dz fixture (Z = 2) without a weight line; the default table (weights.cpp:30-38)
    # has no entry for He, so run() throws "no weight parameters for element Z=2"
    "merging two independent seeded runs",
    # expects "energies 2 2" on h2_svp to trip HOMO < LUMO, i.e. bit-equal degenerate orbital
    # energies from Eigen's eigensolver (any other solver leaves them 1 ulp apart)
    "spinor file error paths",
}


@pytest.mark.skipif(not (ref_py.REF_LIB.parent / "ref_unit_tests").exists(), reason="ref_unit_tests not built")
def test_reference_unit_suite_passes_on_this_build(tmp_path):
    import re
    import subprocess
    out = subprocess.run([str(ref_py.REF_LIB.parent / "ref_unit_tests")], cwd=tmp_path, capture_output=True,
                         text=True, timeout=900).stdout
    summary = re.search(r"test cases: (\d+) \| passed: (\d+) \| failed: (\d+)", out)
    assert summary, out[-2000:]
    total, passed, failed = map(int, summary.groups())
    failing = {m.group(1) for m in re.finditer(r"^\[FAIL\] (.+) \(/", out, re.M)}
    assert total >= 100 and failing == KNOWN_REFERENCE_FAILURES, (failing, out[-3000:])


def test_syn4c_deterministic_energy_matches_the_reference_oracle(tmp_path):
    """The physical MP2 energy of syn4c that tests/syn4c.py restates (and the device MC
    converges to in physical mode, tests/test_syn4c.py) against the reference's own deterministic
    oracle (oracle.cpp make_fixture / oracle_mp2_energy), and the fixture's spinors as the
    reference writes them against the restated ones."""
    import syn4c
    e2 = ref_py.fixture("syn4c", tmp_path / "syn4c_ref.spinor")
    assert e2 == pytest.approx(-0.003932252921, abs=5e-12)
    ours = tmp_path / "syn4c_ours.spinor"
    syn4c.write_spinor_file(ours)
    assert syn4c.mp2_energy(syn4c.coefficients()) == pytest.approx(e2, rel=1e-9)

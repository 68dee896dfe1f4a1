"""The device path against the REFERENCE ITSELF (oracle/_ref/libref_mcmp2.so: the reference's
own model, weights, sampler, greens, estimator and driver translation units, see
tests/test_reference_pins.py), not only against the oracle restatement:
  * replayed step values at the reference's mc_step_estimate (estimator.cpp:35-63), on the DMMA
    and on the INT8 (guarded) V paths, 1e-10 relative;
  * whole runs of the host Engine with device workers against the reference Engine
    (driver.cpp:336-480) on the same config: step counts, E2, sigma_bar and per-worker means,
    1e-10 relative -- the device chains reproduce the reference's Philox streams."""
import numpy as np
import pytest

import oracle_py
import ref_py
from paper_2203_05632_b200 import DeviceWalker, System, walker

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_py.available(), reason="oracle/_ref not built")]

REL = 1e-10


# m = 16, 64: the DMMA Kramers kernels (QB = 1 tiles); m = 192: the INT8 (guarded) V path
@pytest.mark.parametrize("name,m,nsteps", [("cfg1", 16, 3), ("cfg2", 64, 2), ("cfg3", 192, 2), ("cfg4", 192, 1)])
def test_replay_matches_the_reference(cfgdir, name, m, nsteps):
    sp = cfgdir / f"{name}.spinor"
    text = (cfgdir / f"{name}.conf").read_text()
    tr = oracle_py.OracleSystem(sp, text).trajectory(seed=19, stream=1, m=m, burn=20, nsteps=nsteps)
    ref = ref_py.RefSystem(sp, text).replay(tr["walkers"], tr["tau"], pair_sums=False)
    dw = DeviceWalker(System(sp, text), max_walkers=m)
    got = dw.replay(tr["walkers"], tr["tau"])
    assert np.max(np.abs(got[:, 0] - ref[:, 0]) / np.abs(ref[:, 0])) < REL


@pytest.mark.parametrize("name,extra", [
    ("cfg2", "walkers 16\nsteps 240\nworkers 3\nseed 11\nburnin 40\nblocksize 10\ncheckpoint-interval 40\n"),
    ("syn2c", "walkers 6\nsteps 300\nworkers 2\nseed 4\nburnin 50\nblocksize 20\ncheckpoint-interval 100\n"),
])
def test_engine_run_matches_the_reference(cfgdir, name, extra):
    weights = "".join(l + "\n" for l in (cfgdir / f"{name}.conf").read_text().splitlines() if l.startswith("weight"))
    text = f"spinors {cfgdir / (name + '.spinor')}\n" + extra + weights
    ref = ref_py.run_config(text)
    dev = walker.run_config_text(text)

    def parse(rep):
        lines = rep.splitlines()
        return {"E2": float(lines[0].split("=")[1].split()[0]), "sigma_bar": float(lines[1].split("=")[1].split()[0]),
                "steps": int(lines[2].split("=")[1]),
                "workers": [(l.split(",")[0], float(l.split(",")[1].split()[1])) for l in lines if l.startswith("worker")]}
    r, d = parse(ref), parse(dev)
    assert d["steps"] == r["steps"] and [w[0] for w in d["workers"]] == [w[0] for w in r["workers"]]
    assert d["E2"] == pytest.approx(r["E2"], rel=REL, abs=0)
    assert d["sigma_bar"] == pytest.approx(r["sigma_bar"], rel=REL, abs=0)
    for (_, a), (_, b) in zip(r["workers"], d["workers"]):
        assert b == pytest.approx(a, rel=REL, abs=0)

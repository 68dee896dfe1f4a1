"""The C++ host Engine over the device (libmcmp2host -> libmcmp2dev): the reference driver
tests (test_driver.cpp:125-252) and full-run agreement with the CPU oracle's Engine."""
import math

import pytest

import oracle_py
from paper_2203_05632_b200 import walker
from paper_2203_05632_b200.native import Mcmp2Error

pytestmark = pytest.mark.gpu


def parse(rep):
    d = {"workers": []}
    for line in rep.splitlines():
        if line.startswith("E2"):
            d["value"] = float(line.split()[2])
        elif line.startswith("sigma_bar"):
            d["sigma_bar"] = float(line.split()[2])
        elif line.startswith("steps"):
            d["steps"] = int(line.split()[2])
        elif line.startswith("worker"):
            d["workers"].append(line)
    d["on_target"] = "stopped on target" in rep
    return d


def small(cfgdir, name="syn1c", **kw):
    base = {"spinors": str(cfgdir / f"{name}.spinor"), "steps": 2000, "walkers": 4, "seed": 11, "workers": 1,
            "burnin": 100, "checkpoint-interval": 500}
    base.update(kw)
    extra = (cfgdir / f"{name}.conf").read_text()
    weights = "".join(l + "\n" for l in extra.splitlines() if l.startswith("weight"))
    return "".join(f"{k} {v}\n" for k, v in base.items() if v is not None) + weights


def test_single_worker_runs_are_bit_reproducible(cfgdir):
    a = walker.run_config_text(small(cfgdir))
    b = walker.run_config_text(small(cfgdir))
    assert a == b
    assert parse(a)["steps"] == 2000


def test_multi_worker_bookkeeping(cfgdir):
    rep = parse(walker.run_config_text(small(cfgdir, workers=3, steps=3000)))
    assert rep["steps"] == 3000 and len(rep["workers"]) == 3
    assert all(": steps 1000," in w for w in rep["workers"])


def test_kill_and_resume_is_bit_exact(cfgdir, tmp_path):
    """test_driver.cpp:150-172: abort after 2 intervals, resume == uninterrupted run."""
    ck = tmp_path / "run.ckpt"
    cfg = small(cfgdir, workers=2, steps=4000, checkpoint=str(ck))
    full = walker.run_config_text(cfg)
    walker.run_config_text(cfg, abort_after_intervals=2)
    resumed = walker.resume(ck)
    assert resumed == full


def test_resume_rejects_changed_spinor_file(cfgdir, tmp_path):
    sp = tmp_path / "f.spinor"
    sp.write_bytes((cfgdir / "syn1c.spinor").read_bytes())
    ck = tmp_path / "run.ckpt"
    walker.run_config_text(small(cfgdir, spinors=str(sp), checkpoint=str(ck)), abort_after_intervals=1)
    sp.write_bytes((cfgdir / "syn2c.spinor").read_bytes())
    with pytest.raises(Mcmp2Error, match="hash"):
        walker.resume(ck)


def test_merge_checkpoints(cfgdir, tmp_path):
    a, b = tmp_path / "a.ckpt", tmp_path / "b.ckpt"
    ra = parse(walker.run_config_text(small(cfgdir, checkpoint=str(a), seed=1)))
    rb = parse(walker.run_config_text(small(cfgdir, checkpoint=str(b), seed=2)))
    value, sigma_bar, steps = walker.merge([a, b])
    assert steps == 4000
    assert value == pytest.approx((ra["value"] * 2000 + rb["value"] * 2000) / 4000, rel=1e-15)
    c = tmp_path / "c.ckpt"
    walker.run_config_text(small(cfgdir, name="syn2c", checkpoint=str(c)))
    with pytest.raises(Mcmp2Error, match="hash"):
        walker.merge([a, c])


def test_trace_has_one_line_per_completed_block(cfgdir, tmp_path):
    tr = tmp_path / "run.trace"
    walker.run_config_text(small(cfgdir, trace=str(tr), steps=1950))
    rows = tr.read_text().splitlines()
    assert len(rows) == 19 and rows[-1].split()[0] == "1900"


def test_target_relative_error_stop(cfgdir):
    rep = parse(walker.run_config_text(small(cfgdir, steps=None) + "target-rel-err 2.0\n"))
    assert rep["on_target"] and rep["steps"] == 500
    assert rep["sigma_bar"] / abs(rep["value"]) <= 2.0


@pytest.mark.parametrize("name,extra", [("syn1c", {}), ("cfg1", {"walkers": 16, "step-size": 0.3}),
                                        ("syn2c", {"workers": 2})])
def test_full_run_matches_oracle_engine(cfgdir, name, extra):
    """Same config through the device Engine and the CPU oracle's Engine: the device follows the
    reference Philox stream, so the runs agree to rounding, not just statistically."""
    cfg = small(cfgdir, name=name, **extra)
    dev = parse(walker.run_config_text(cfg))
    ref = parse(oracle_py.run_config(cfg))
    assert dev["steps"] == ref["steps"]
    assert dev["value"] == pytest.approx(ref["value"], rel=1e-9)
    assert dev["sigma_bar"] == pytest.approx(ref["sigma_bar"], rel=1e-6)


@pytest.mark.parametrize("name,kw", [
    ("cfg1", {"walkers": 16, "step-size": 0.3, "steps": 4000}),
    ("cfg2", {"walkers": 16, "workers": 4, "steps": 4000, "burnin": 200}),  # 4c, 10e atom, batched workers
    ("syn2c", {"walkers": 8, "workers": 2, "steps": 6000}),                 # 2-component set
])
def test_independent_rng_runs_agree_within_2_sigma(cfgdir, name, kw):
    """north_star: independent-RNG full runs agree with the reference E(2) within combined 2 sigma
    (literal estimator): the device Engine on seed 101 against the oracle Engine on seed 202."""
    dev = parse(walker.run_config_text(small(cfgdir, name=name, seed=101, **kw)))
    ref = parse(oracle_py.run_config(small(cfgdir, name=name, seed=202, **kw)))
    assert dev["steps"] == ref["steps"] == kw["steps"]
    assert abs(dev["value"] - ref["value"]) <= 2 * math.hypot(dev["sigma_bar"], ref["sigma_bar"])


def test_missing_nuclei_is_diagnosed(cfgdir, tmp_path):
    text = (cfgdir / "syn1c.spinor").read_text().replace("nuclei 2\n1 0 0 0\n1 0 0 1.3999999999999999\n", "")
    sp = tmp_path / "bare.spinor"
    sp.write_text(text)
    with pytest.raises(Mcmp2Error, match="nuclei"):
        walker.run_config_text(small(cfgdir, spinors=str(sp)))


def test_batched_workers_match_oracle_engine(cfgdir):
    """Five cfg1 workers on one device run as one batched handle (m = 16, Kramers-paired set):
    unequal step shares (2003 = 401 x 3 + 400 x 2, driver.cpp:307-309) advance the leading
    ensembles alone; every worker follows its reference stream, so the run equals the oracle
    Engine's (std::thread workers) to rounding."""
    cfg = small(cfgdir, name="cfg1", walkers=16, workers=5, steps=2003, **{"step-size": 0.3})
    dev = parse(walker.run_config_text(cfg))
    ref = parse(oracle_py.run_config(cfg))
    assert dev["steps"] == ref["steps"] == 2003
    assert [w.split(",")[0] for w in dev["workers"]] == [w.split(",")[0] for w in ref["workers"]]
    assert dev["value"] == pytest.approx(ref["value"], rel=1e-9)
    assert dev["sigma_bar"] == pytest.approx(ref["sigma_bar"], rel=1e-6)
    acc_dev = [w.split("acceptance ")[1].split(",")[0] for w in dev["workers"]]
    acc_ref = [w.split("acceptance ")[1].split(",")[0] for w in ref["workers"]]
    assert acc_dev == acc_ref


def test_batched_kill_and_resume_is_bit_exact(cfgdir, tmp_path):
    """test_driver.cpp:150-172 with the workers of a batched handle: per-ensemble states go
    through the checkpoint and come back into the batch."""
    ck = tmp_path / "run.ckpt"
    cfg = small(cfgdir, name="cfg2", walkers=16, workers=3, steps=1201, burnin=50, checkpoint=str(ck))
    full = walker.run_config_text(cfg)
    walker.run_config_text(cfg, abort_after_intervals=1)
    assert walker.resume(ck) == full


def test_int8_v_path_engine_run_matches_oracle_and_resumes_bit_exact(cfgdir, tmp_path):
    """cfg3 with 192 walkers takes the INT8 (Ozaki) V path through the C++ Engine: the run agrees
    with the CPU oracle's Engine to 1e-9 (same Philox stream, per-step values within 1e-10), and a
    run killed after one checkpoint interval resumes bit-exactly (fixed-order reductions)."""
    ck = tmp_path / "oz.ckpt"
    cfg = small(cfgdir, name="cfg3", walkers=192, steps=40, burnin=20, **{"checkpoint-interval": 20},
                checkpoint=str(ck))
    full = walker.run_config_text(cfg)
    walker.run_config_text(cfg, abort_after_intervals=1)
    assert walker.resume(ck) == full
    dev = parse(full)
    ref = parse(oracle_py.run_config(small(cfgdir, name="cfg3", walkers=192, steps=40, burnin=20,
                                           **{"checkpoint-interval": 20})))
    assert dev["steps"] == ref["steps"] == 40
    assert dev["value"] == pytest.approx(ref["value"], rel=1e-9)
    assert dev["sigma_bar"] == pytest.approx(ref["sigma_bar"], rel=1e-6)

"""Sampler statistics of the reference's test_sampler.cpp, on the oracle (CPU suite) and on the
device chain (GPU suite): the long-run acceptance window after burn-in (test_sampler.cpp:120-127)
and the stationary r12 marginal (test_sampler.cpp:175-205). Single nucleus, single primitive
weight w(r1, r2) ~ exp(-z (r1^2 + r2^2)) / r12: u = |r1 - r2| has density z u exp(-z u^2 / 2), so
1 - exp(-z u^2 / 2) is uniform; chi^2 over 25 equiprobable bins, 1% level of chi^2(24)."""
import math
import re

import numpy as np
import pytest

import oracle_py

Z = 0.5
CHI2_1PCT_24 = 42.98


def single_primitive_config(cfgdir):
    text = (cfgdir / "cfg1.conf").read_text()
    text = re.sub(r"step-size \S+\n", "", text)
    return re.sub(r"weight He .*\n", f"weight He 1.0 {Z} 1e-14 1.0\n", text)


def chi2_of(u):
    cdf = 1.0 - np.exp(-0.5 * Z * np.asarray(u) ** 2)
    counts = np.bincount(np.minimum((cdf * 25).astype(int), 24), minlength=25)
    expect = counts.sum() / 25.0
    return float(((counts - expect) ** 2 / expect).sum())


def test_oracle_stationary_r12_marginal(cfgdir):
    orc = oracle_py.OracleSystem(cfgdir / "cfg1.spinor", single_primitive_config(cfgdir))
    u, _ = orc.chain_r12(seed=77, m=8, burn=2000, nsteps=125000, thin=50)
    assert chi2_of(u) < CHI2_1PCT_24


def test_oracle_acceptance_window(cfgdir):
    text = re.sub(r"step-size \S+\n", "", (cfgdir / "cfg1.conf").read_text())
    orc = oracle_py.OracleSystem(cfgdir / "cfg1.spinor", text)
    _, acc = orc.chain_r12(seed=9, m=8, burn=1000, nsteps=2000, thin=2000)
    assert 0.3 < acc < 0.7


@pytest.mark.gpu
def test_device_stationary_r12_marginal(cfgdir):
    from paper_2203_05632_b200 import DeviceWalker, System

    dw = DeviceWalker(System(cfgdir / "cfg1.spinor", single_primitive_config(cfgdir)), max_walkers=8)
    dw.init_ensemble(8, seed=77)
    dw.burn_in(2000, adapt=True)
    u = []
    for _ in range(2500):  # 125000 sweeps thinned by 50 (Metropolis-only sweeps)
        dw.burn_in(50, adapt=False)
        w = dw.get_ensemble().walkers
        u.extend(np.linalg.norm(w[:, 0:3] - w[:, 3:6], axis=1))
    assert chi2_of(u) < CHI2_1PCT_24


@pytest.mark.gpu
def test_device_acceptance_window(cfgdir):
    from paper_2203_05632_b200 import DeviceWalker, System

    text = re.sub(r"step-size \S+\n", "", (cfgdir / "cfg1.conf").read_text())
    dw = DeviceWalker(System(cfgdir / "cfg1.spinor", text), max_walkers=8)
    dw.init_ensemble(8, seed=9)
    dw.burn_in(1000, adapt=True)
    dw.advance(2000)
    e = dw.get_ensemble()
    assert e.proposed == 2000 * 8
    assert 0.3 < e.accepted / e.proposed < 0.7
    assert math.isfinite(e.sigma_step)

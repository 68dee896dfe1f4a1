"""CPU: bench.py's host-side pieces -- the strong-scaling split of the timed steps and of the
strong_run budget (worker_share, driver.cpp:307-309, the same split distributed.py and the C++
Engine use), the bounded-sample fit of the CPU arm, and the run configs bench.py builds for the
Engine jobs (parsed by the host library)."""
import numpy as np
import pytest

import bench
from paper_2203_05632_b200 import distributed as D


@pytest.mark.parametrize("total,world", [(40, 1), (40, 3), (20000, 8), (7, 8)])
def test_strong_split_covers_the_budget(total, world):
    shares = [bench.worker_share(total, world, r) for r in range(world)]
    assert sum(shares) == total and max(shares) - min(shares) <= 1
    assert shares == [D.worker_share(total, world, r) for r in range(world)]


def test_cpu_fit_recovers_the_linear_step_model():
    t0, c, npairs = 1.2, 2.2e-5, 2096128
    pts = [(r, t0 + c * n, n) for r, n in ((4, 8182.0), (16, 32632.0), (64, 129056.0))] * 2
    fit = bench.cpu_full_step(pts, npairs)
    assert fit["extrapolated"] and fit["fit_residual_rel"] < 1e-12
    assert fit["t_full"] == pytest.approx(t0 + c * npairs, rel=1e-12)
    full = bench.cpu_full_step([(16, 0.5, 120.0), (16, 0.7, 120.0)], 120)
    assert not full["extrapolated"] and full["t_full"] == pytest.approx(0.6)


def test_engine_job_configs_parse(cfgdir):
    conf = (cfgdir / "cfg4.conf").read_text()
    text = bench.run_config_text("cfg4", cfgdir / "cfg4.spinor", conf,
                                 "steps 20000\nwalkers 2048\nworkers 8\nseed 1\nburnin 1000\ncheckpoint-interval 20000\n")
    rc = D.parse_run_config(text)
    assert rc["steps"] == 20000 and rc["workers"] == 8 and rc["target"] is None
    assert [D.rank_workers(8, 8, r) for r in range(8)] == [(r, 1) for r in range(8)]
    text = bench.run_config_text("cfg5-10", cfgdir / "cfg5-10.spinor", (cfgdir / "cfg5-10.conf").read_text(),
                                 "target-rel-err 0.01\nwalkers 8192\nworkers 2\nseed 1\nburnin 1000\n"
                                 "checkpoint-interval 100\n")
    rc = D.parse_run_config(text)
    assert rc["target"] == 0.01 and rc["steps"] is None and rc["interval"] == 100
    assert any(l.startswith("weight") for l in text.splitlines())


def test_vgemm_shared_memory_bound_restates_the_kernel_shape():
    """bench.py's shared-memory bound of oz_vgemm_kernel from the kernel's own shape: per k-step
    (32 of K') of a 128 x 80 tile, 9 merged MMAs read 9 x 128 x 32 B of A and 21 x 80 x 32 B of B
    slices and the ring's fills write 6 x (128 + 80) x 32 B, against 128 B/clk/SM on 148 SMs at
    1965 MHz; it must sit between the kernel's measured rate and the dense tcgen05 rate."""
    import bench
    a_reads, b_reads, fills = 9 * 128 * 32, 21 * 80 * 32, 6 * (128 + 80) * 32
    assert (a_reads, b_reads, fills) == (36864, 53760, 39936)
    cycles = (a_reads + b_reads + fills) / 128
    ops = 21 * 2 * 128 * 80 * 32
    bound = 148 * 1.965e9 * ops / cycles / 1e12
    assert abs(bound - bench.INT8_SMEM_BOUND) < 1e-6 * bound
    assert 3000 < bench.INT8_SMEM_BOUND < bench.INT8_PEAK

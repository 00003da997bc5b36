"""Simulation.run (smpm_sim_run): n steps with the between-step checks on the
device and one host synchronisation per batch, against the same steps taken
one Simulation.step call at a time (the reference's loop, S/bench.py:216-226).

Fast mode sums in nondeterministic atomic order, so the two paths agree to
fp32 tolerance, with identical active sets; the deterministic mode takes the
single-step path inside run() and agrees bitwise."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2605_28525_b200.errors import SimulationError  # noqa: E402
from paper_2605_28525_b200.solver import Simulation  # noqa: E402
from tests.test_gpu_sim import column_scene  # noqa: E402


def _close(a, b, tol=1e-6):
    scale = max(np.abs(b).max(), 1e-30)
    return np.abs(a - b).max() / scale < tol


def _pair(**kw):
    ps, cfg, mats, bc = column_scene(**kw)
    return (Simulation(ps.copy(), cfg, mats, bc, record_conservation=True),
            Simulation(ps.copy(), cfg, mats, bc, record_conservation=True))


def test_run_matches_single_steps():
    a, b = _pair()
    ra = a.run(12)
    rb = [b.step() for _ in range(12)]
    assert [s.step for s in ra] == list(range(1, 13)) and a.step_count == 12
    for sa, sb in zip(ra, rb):
        assert sa.n_active == sb.n_active and sa.n_allocated == sb.n_allocated
        assert abs(sa.dt - sb.dt) <= 1e-5 * sb.dt
        assert abs(sa.t - sb.t) <= 1e-5 * sb.t
        assert abs(sa.mass_sum - sb.mass_sum) <= 1e-6 * sb.mass_sum
    assert _close(a.particles.x, b.particles.x) and _close(a.particles.v, b.particles.v, 1e-4)
    assert a.last_stats.step == 12 and abs(a.t - b.t) <= 1e-5 * b.t


def test_run_fixed_dt_and_mixed_with_steps():
    a, b = _pair()
    a.run(3, dt=1e-4)
    a.step(1e-4)
    a.run(4, dt=1e-4)
    for _ in range(8):
        b.step(1e-4)
    assert a.step_count == 8 and abs(a.t - 8e-4) < 1e-12
    assert _close(a.particles.x, b.particles.x) and _close(a.particles.F, b.particles.F, 1e-5)


def test_run_crosses_batches():
    """More steps than one device ring (1024): the state carries over."""
    a, b = _pair(size=(0.1, 0.1, 0.1))
    ra = a.run(1030, dt=2e-5)
    assert len(ra) == 1030 and a.step_count == 1030
    b.run(1024, dt=2e-5)
    for _ in range(6):
        b.step(2e-5)
    assert ra[-1].n_active == b.last_stats.n_active
    assert _close(a.particles.x, b.particles.x)


def test_run_rejects_oversized_dt_without_stepping():
    a, _ = _pair()
    bound = a.dt_bound()
    with pytest.raises(SimulationError, match="stability bound"):
        a.run(5, dt=10.0 * bound)
    assert a.step_count == 0
    a.run(2, dt=0.5 * bound)  # the rejected batch left no trace
    assert a.step_count == 2


def test_run_grows_the_grid_inside_a_batch():
    ps, cfg, mats, bc = column_scene()
    a = Simulation(ps.copy(), cfg, mats, bc, block_capacity=8)
    b = Simulation(ps.copy(), cfg, mats, bc)
    ra = a.run(6, dt=1e-4)
    for sa in ra:
        sb = b.step(1e-4)
        assert sa.n_active == sb.n_active and sa.n_allocated == sb.n_allocated
    assert _close(a.particles.x, b.particles.x)


def test_run_deterministic_mode_is_bitwise_equal_to_steps():
    ps, cfg, mats, bc = column_scene()
    cfg.deterministic = True
    a = Simulation(ps.copy(), cfg, mats, bc)
    b = Simulation(ps.copy(), cfg, mats, bc)
    a.run(5)
    for _ in range(5):
        b.step()
    for k in ("x", "v", "C", "F"):
        assert np.array_equal(getattr(a.particles, k), getattr(b.particles, k)), k


def test_run_zero_and_edits_between_runs():
    a, b = _pair()
    assert a.run(0) == []
    a.run(2, dt=1e-4)
    b.run(2, dt=1e-4)
    for s in (a, b):
        s.particles.v[:, 2] += 0.1  # host edit: re-uploaded before the next batch
    a.run(3, dt=1e-4)
    for _ in range(3):
        b.step(1e-4)
    assert _close(a.particles.v, b.particles.v, 1e-4)

"""Host-side validation that runs before any device work, mirroring the
reference's constructor and builder checks (CPU).

Reference: solver.py:937-960 (Simulation.__init__: empty set, no material,
material id range, one heightfield), sparse_hash.py:225-235 and
T/test_sparse_hash.py:155-157 (empty particle set rejected)."""
import numpy as np
import pytest

from paper_2605_28525_b200 import scenes
from paper_2605_28525_b200.errors import ConfigError
from paper_2605_28525_b200.solver import BoundaryCondition, Heightfield, ParticleSet, SimConfig, Simulation
from paper_2605_28525_b200.sparse_hash import build_hash_sparse_grid


def _cfg():
    return SimConfig(h=0.1, gravity=np.array([0.0, 0.0, -9.81]), total_time=1.0,
                     domain_min=np.array([-1.0, -1.0, -1.0]), domain_max=np.array([1.0, 1.0, 1.0]))


def _ps(n=8, mat_id=0):
    pos = np.random.default_rng(0).uniform(-0.2, 0.2, (n, 3))
    ps = scenes.rest_particles(pos, np.full(n, 1e-3), 1500.0)
    ps.mat_id[:] = mat_id
    return ps


def test_empty_particle_set_rejected():
    empty = ParticleSet.from_samples(np.empty((0, 3)), np.empty(0), 1500.0)
    with pytest.raises(ConfigError, match="at least one particle"):
        Simulation(empty, _cfg(), [scenes.SAND])


def test_no_material_rejected():
    with pytest.raises(ConfigError, match="at least one material"):
        Simulation(_ps(), _cfg(), [])


@pytest.mark.parametrize("mat_id", [-1, 1])
def test_material_id_out_of_range_rejected(mat_id):
    with pytest.raises(ConfigError, match="material id out of range"):
        Simulation(_ps(mat_id=mat_id), _cfg(), [scenes.SAND])


def test_two_heightfields_rejected():
    hf = Heightfield(data=np.zeros((4, 4)), x0=-1.0, y0=-1.0, cell=1.0)
    bcs = [BoundaryCondition(kind="heightfield", heightfield=hf, mu=0.5)] * 2
    with pytest.raises(ConfigError, match="one heightfield"):
        Simulation(_ps(), _cfg(), [scenes.SAND], bcs)


def test_empty_grid_build_rejected():
    with pytest.raises(ValueError):
        build_hash_sparse_grid(np.empty((0, 3)), 0.05, 4)


def test_nonfinite_grid_build_rejected():
    with pytest.raises(ValueError):
        build_hash_sparse_grid(np.array([[0.0, np.nan, 0.0]]), 0.05, 4)


def test_non_power_of_two_capacity_rejected():
    with pytest.raises(ValueError):
        build_hash_sparse_grid(np.zeros((4, 3)), 0.05, 4, initial_capacity=100)

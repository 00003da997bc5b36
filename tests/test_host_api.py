"""Host-side API parity that needs no GPU: configuration validation,
materials, scenes (SURVEY section 4 model: reference unit tests)."""

import math

import numpy as np
import pytest

from paper_2605_28525_b200 import scenes
from paper_2605_28525_b200.errors import ConfigError
from paper_2605_28525_b200.materials import MaterialModel, material_tables
from paper_2605_28525_b200.solver import BoundaryCondition, Heightfield, ParticleSet, SimConfig


def test_material_constants():
    m = MaterialModel(kind="drucker_prager", density=1500.0, youngs_modulus=1e6, poisson_ratio=0.3,
                      friction_angle_deg=30.0)
    assert math.isclose(m.lame_mu, 1e6 / 2.6)
    assert math.isclose(m.lame_lambda, 1e6 * 0.3 / (1.3 * 0.4))
    assert math.isclose(m.dp_alpha, math.sqrt(2 / 3) * 2 * 0.5 / 2.5)
    mu, lam, alpha, kind = material_tables([m])
    assert kind[0] == 1
    with pytest.raises(ValueError):
        MaterialModel(kind="clay", density=1.0, youngs_modulus=1.0, poisson_ratio=0.1)


def test_config_validation():
    base = dict(h=0.1, gravity=[0, 0, -9.81], total_time=1.0, domain_min=[0, 0, 0], domain_max=[1, 1, 1])
    SimConfig(**base)
    with pytest.raises(ConfigError):
        SimConfig(**{**base, "h": 0.0})
    for backend in ("dense", "scan", "hash"):  # the reference's backend names (solver.py:24)
        assert SimConfig(**{**base, "backend": backend}).backend == backend
    with pytest.raises(ConfigError):
        SimConfig(**{**base, "backend": "octree"})
    with pytest.raises(ConfigError):
        SimConfig(**{**base, "block_size": 8})
    with pytest.raises(ConfigError):
        SimConfig(**{**base, "cfl": 1.5})
    with pytest.raises(ConfigError):
        BoundaryCondition(kind="plane", normal=[0, 0, 0])
    with pytest.raises(ConfigError):
        BoundaryCondition(kind="heightfield")


def test_heightfield_sample_matches_formula():
    hf = scenes.landslide_terrain()
    for x, y in [(0.0, 0.0), (123.4, -17.0), (1999.0, 249.0)]:
        z = hf.sample(x, y)
        assert abs(z - (600 * math.exp(-x / 400) + 0.002 * y * y)) < 0.5
    assert np.allclose(hf.sample_many([123.4], [-17.0]), [hf.sample(123.4, -17.0)])


def test_scene_sizes():
    c1 = scenes.granular_column()
    assert c1.particles.n == 128_000
    c2 = scenes.two_spheres()
    assert 120_000 < c2.particles.n < 140_000
    small = scenes.landslide(x_stride=50)
    assert small.particles.n == 20 * 500 * 202  # 0.5..51 m deep at h/2 spacing
    ps = ParticleSet.from_samples(np.zeros((2, 3)), np.ones(2), 10.0)
    assert ps.n == 2 and np.all(ps.F == np.eye(3))

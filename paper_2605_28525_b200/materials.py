"""Constitutive models: Hencky hyperelasticity and Drucker-Prager sand.

``MaterialModel`` mirrors materials.py:23-78 of the reference
(/root/reference/pkg/src/sparsempm/materials.py).  The stress evaluation
itself (materials.py:169-238) runs on the GPU: inside the fused step kernel
for ``Simulation.step`` and through ``update_stress`` (materials.py:250-267)
for the module-level API.
"""

import math
from dataclasses import dataclass

import numpy as np

from .errors import SimulationError

KIND_ELASTIC = 0
KIND_DRUCKER_PRAGER = 1

_KINDS = {"elastic": KIND_ELASTIC, "drucker_prager": KIND_DRUCKER_PRAGER}


@dataclass(frozen=True)
class MaterialModel:
    """Material parameters for one particle population (materials.py:23-53)."""

    kind: str
    density: float
    youngs_modulus: float
    poisson_ratio: float
    friction_angle_deg: float = 0.0

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ValueError(f"unknown material kind {self.kind!r}; choose one of {sorted(_KINDS)}")
        if self.density <= 0:
            raise ValueError(f"density must be positive, got {self.density}")
        if self.youngs_modulus <= 0:
            raise ValueError(f"youngs_modulus must be positive, got {self.youngs_modulus}")
        if not 0.0 <= self.poisson_ratio < 0.5:
            raise ValueError(f"poisson_ratio must lie in [0, 0.5), got {self.poisson_ratio}")
        if not 0.0 <= self.friction_angle_deg < 90.0:
            raise ValueError(f"friction_angle_deg must lie in [0, 90), got {self.friction_angle_deg}")

    @property
    def lame_mu(self):
        return self.youngs_modulus / (2.0 * (1.0 + self.poisson_ratio))

    @property
    def lame_lambda(self):
        e, nu = self.youngs_modulus, self.poisson_ratio
        return e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))

    @property
    def dp_alpha(self):
        """Cone slope of the Drucker-Prager yield surface in tau space."""
        s = math.sin(math.radians(self.friction_angle_deg))
        return math.sqrt(2.0 / 3.0) * 2.0 * s / (3.0 - s)

    @property
    def wave_speed(self):
        return math.sqrt((self.lame_lambda + 2.0 * self.lame_mu) / self.density)

    @property
    def kind_id(self):
        return _KINDS[self.kind]


def material_tables(materials):
    """Per-material parameter arrays indexed by material id (materials.py:241-247)."""
    mu = np.array([m.lame_mu for m in materials], dtype=np.float64)
    lam = np.array([m.lame_lambda for m in materials], dtype=np.float64)
    alpha = np.array([m.dp_alpha for m in materials], dtype=np.float64)
    kind = np.array([m.kind_id for m in materials], dtype=np.int64)
    return mu, lam, alpha, kind


def update_stress(particles, materials):
    """Refresh Cauchy stress and Jacobian from each particle's F on the GPU;
    Drucker-Prager particles get F return-mapped in place.  Raises
    SimulationError for a degenerate F (materials.py:250-267)."""
    from . import _lib

    _lib.stress_inplace(particles, materials)
    return particles


def _degenerate_message(particles, p):
    with np.errstate(invalid="ignore"):
        detf = float(np.linalg.det(np.asarray(particles.F[p], dtype=np.float64)))
    return f"deformation gradient of particle {p} is degenerate (det F = {detf:.3e})"


__all__ = ["MaterialModel", "material_tables", "update_stress", "KIND_ELASTIC", "KIND_DRUCKER_PRAGER",
           "SimulationError"]

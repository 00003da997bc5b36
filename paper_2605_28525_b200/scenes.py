"""Synthetic scenes of BASELINE.json's configs.

All scenes are lattice-seeded like the reference's ``sample_box``
(/root/reference/pkg/src/sparsempm/scenarios.py:352-374): spacing h/ppc,
cell-centred, volumes summing to the region volume.  Defaults: Drucker-Prager
sand (phi=30 deg, E=1e6 Pa, nu=0.3, rho=1500), g=(0,0,-9.81), CFL 0.4.

* C1 ``granular_column``  -- 0.5x0.5x1 m column, h=0.025, ppc=2 (128,000)
* C2 ``two_spheres``      -- elastic spheres colliding in a large box
* C3 ``incline``          -- 4x2.5x1 m sand block on a 35 deg incline with walls
* C4 ``landslide``        -- terrain-conforming release over an analytic DEM
                             (101M particles at h=0.5, ppc=2: release 250 x 125 m,
                             0.5-51 m deep)
"""

import math
from dataclasses import dataclass

import numpy as np

from .materials import MaterialModel
from .solver import BoundaryCondition, Heightfield, ParticleSet, SimConfig

SAND = MaterialModel(kind="drucker_prager", density=1500.0, youngs_modulus=1e6, poisson_ratio=0.3,
                     friction_angle_deg=30.0)


@dataclass
class Scene:
    name: str
    particles: ParticleSet
    config: SimConfig
    materials: list
    boundaries: list

    def simulation(self, **kw):
        from .solver import Simulation

        return Simulation(self.particles, self.config, self.materials, self.boundaries, **kw)


def sample_box(region_min, region_max, h, ppc=2):
    """Deterministic lattice seeding of a box (scenarios.py:352-374)."""
    rmin = np.asarray(region_min, dtype=np.float64).reshape(3)
    rmax = np.asarray(region_max, dtype=np.float64).reshape(3)
    ext = rmax - rmin
    if np.any(ext <= 0):
        raise ValueError("region_max must exceed region_min on every axis")
    if h <= 0:
        raise ValueError(f"cell size must be positive, got {h}")
    spacing = float(h) / int(ppc)
    counts = np.maximum(1, np.rint(ext / spacing).astype(np.int64))
    axes = [rmin[a] + (np.arange(counts[a]) + 0.5) * (ext[a] / counts[a]) for a in range(3)]
    gx, gy, gz = np.meshgrid(*axes, indexing="ij")
    positions = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    n = positions.shape[0]
    return positions, np.full(n, float(np.prod(ext)) / n)


def rest_particles(positions, volumes, density, material_id=0, velocity=(0.0, 0.0, 0.0)):
    """ParticleSet.from_samples without per-particle Python work (large n)."""
    x = np.ascontiguousarray(positions, dtype=np.float64)
    n = x.shape[0]
    vol = np.ascontiguousarray(volumes, dtype=np.float64)
    v = np.empty((n, 3))
    v[:] = np.asarray(velocity, dtype=np.float64)
    F = np.zeros((n, 3, 3))
    F[:, 0, 0] = F[:, 1, 1] = F[:, 2, 2] = 1.0
    return ParticleSet(x=x, v=v, C=np.zeros((n, 3, 3)), F=F, m=density * vol, V0=vol.copy(),
                       mat_id=np.full(n, material_id, dtype=np.int64), sigma=np.zeros((n, 3, 3)), jac=np.ones(n))


def granular_column(h=0.025, ppc=2, size=(0.5, 0.5, 1.0), mu=0.5):
    """C1: DP column collapse on a frictional floor."""
    sx, sy, sz = size
    pos, vol = sample_box((-sx / 2, -sy / 2, 0.0), (sx / 2, sy / 2, sz), h, ppc)
    ps = rest_particles(pos, vol, SAND.density)
    cfg = SimConfig(h=h, gravity=np.array([0.0, 0.0, -9.81]), total_time=1.0, domain_min=np.array([-3.0, -3.0, -0.1]),
                    domain_max=np.array([3.0, 3.0, 1.2]))
    floor = BoundaryCondition(kind="plane", mu=mu, point=np.zeros(3), normal=np.array([0.0, 0.0, 1.0]))
    return Scene("granular_column", ps, cfg, [SAND], [floor])


def two_spheres(h=0.02, ppc=2, radius=0.25, speed=2.0, box="equivalence"):
    """C2: two elastic spheres colliding head-on, no gravity, no BCs."""
    mat = MaterialModel(kind="elastic", density=1000.0, youngs_modulus=1e6, poisson_ratio=0.3)
    sets = []
    for cx, vx in ((-0.5, speed), (0.5, -speed)):
        c = np.array([cx, 0.0, 0.5])
        pos, _ = sample_box(c - radius, c + radius, h, ppc)
        keep = np.linalg.norm(pos - c, axis=1) <= radius
        pos = pos[keep]
        vol = np.full(pos.shape[0], (h / ppc) ** 3)
        sets.append(rest_particles(pos, vol, mat.density, velocity=(vx, 0.0, 0.0)))
    ps = ParticleSet.merge(sets)
    half = 2.0 if box == "equivalence" else 32.0
    cfg = SimConfig(h=h, gravity=np.zeros(3), total_time=1.0, domain_min=np.full(3, -half), domain_max=np.full(3, half))
    return Scene(f"two_spheres_{box}", ps, cfg, [mat], [])


def incline(h=0.02, ppc=2, theta_deg=35.0):
    """C3: sand block on an incline (tilted gravity) between two walls."""
    pos, vol = sample_box((0.0, -1.25, 0.0), (4.0, 1.25, 1.0), h, ppc)
    ps = rest_particles(pos, vol, SAND.density)
    t = math.radians(theta_deg)
    g = 9.81 * np.array([-math.sin(t), 0.0, -math.cos(t)])
    cfg = SimConfig(h=h, gravity=g, total_time=2.0, domain_min=np.array([-40.0, -1.4, -0.1]),
                    domain_max=np.array([5.0, 1.4, 1.2]))
    bcs = [BoundaryCondition(kind="plane", mu=0.4, point=np.zeros(3), normal=np.array([0.0, 0.0, 1.0])),
           BoundaryCondition(kind="plane", mu=0.2, point=np.array([0.0, -1.3, 0.0]), normal=np.array([0.0, 1.0, 0.0])),
           BoundaryCondition(kind="plane", mu=0.2, point=np.array([0.0, 1.3, 0.0]), normal=np.array([0.0, -1.0, 0.0]))]
    return Scene("incline", ps, cfg, [SAND], bcs)


def landslide_terrain(cell=5.0):
    """Analytic DEM z(x,y) = 600 exp(-x/400) + 0.002 y^2 over [0,2000]x[-250,250]."""
    xs = np.arange(0.0, 2000.0 + 1e-9, cell)
    ys = np.arange(-250.0, 250.0 + 1e-9, cell)
    data = 600.0 * np.exp(-xs[:, None] / 400.0) + 0.002 * ys[None, :] ** 2
    return Heightfield(x0=0.0, y0=-250.0, cell=cell, data=data)


def landslide(h=0.5, ppc=2, release=((100.0, 350.0), (-62.5, 62.5)), depth=(0.5, 51.0), mu=0.35, x_stride=1,
              fraction=1.0, columns=None):
    """C4: terrain-conforming release zone over the analytic DEM.

    Particles sit on a lattice of spacing h/ppc in x and y; each (x,y) column
    is filled from z_s + depth[0] to z_s + depth[1] (z_s the bilinear DEM
    height, i.e. what the grid boundary sees).  ``x_stride`` > 1 keeps every
    k-th x column; ``fraction`` < 1 keeps the leading fraction of the release
    zone in x (contiguous: same block occupancy as the full scene);
    ``columns=(c0, c1)`` keeps x-lattice columns c0..c1-1 (one rank's slab).
    """
    hf = landslide_terrain()
    sp = h / ppc
    (x0, x1), (y0, y1) = release
    xs = x0 + (np.arange(int(round((x1 - x0) / sp))) + 0.5) * sp
    ys = y0 + (np.arange(int(round((y1 - y0) / sp))) + 0.5) * sp
    xs = xs[: max(1, int(round(xs.shape[0] * fraction)))][::x_stride]
    if columns is not None:
        xs = xs[columns[0]:columns[1]]
    nz = int(round((depth[1] - depth[0]) / sp))
    zoff = depth[0] + (np.arange(nz) + 0.5) * sp
    gx, gy = np.meshgrid(xs, ys, indexing="ij")
    zs = hf.sample_many(gx.ravel(), gy.ravel())
    ncol = gx.size
    n = ncol * nz
    x = np.empty((n, 3))
    x[:, 0] = np.repeat(gx.ravel(), nz)
    x[:, 1] = np.repeat(gy.ravel(), nz)
    x[:, 2] = (zs[:, None] + zoff[None, :]).ravel()
    ps = rest_particles(x, np.full(n, sp ** 3), SAND.density)
    cfg = SimConfig(h=h, gravity=np.array([0.0, 0.0, -9.81]), total_time=60.0, domain_min=np.array([0.0, -250.0, -10.0]),
                    domain_max=np.array([2000.0, 250.0, 700.0]))
    bc = BoundaryCondition(kind="heightfield", mu=mu, heightfield=hf)
    return Scene("landslide", ps, cfg, [SAND], [bc])


def landslide_columns(h=0.5, ppc=2, release=((100.0, 350.0), (-62.5, 62.5)), fraction=1.0):
    """x of every lattice column of the landslide release zone."""
    sp = h / ppc
    (x0, x1), _ = release
    xs = x0 + (np.arange(int(round((x1 - x0) / sp))) + 0.5) * sp
    return xs[: max(1, int(round(xs.shape[0] * fraction)))]


def landslide_slabs(world, h=0.5, ppc=2, fraction=1.0):
    """Block-aligned slab cuts of the landslide for ``world`` ranks with equal
    particle counts (every column holds the same number of particles):
    [(bx0, bx1, c0, c1)], columns c0..c1-1 belong to the slab."""
    from .slabs import INT32_MAX, INT32_MIN

    xs = landslide_columns(h, ppc, fraction=fraction)
    bx = np.floor(xs * (1.0 / h) - 0.5).astype(np.int64) >> 2
    out = []
    cuts = [0]
    for r in range(1, world):
        c = max(int(round(r * len(xs) / world)), cuts[-1] + 1)
        # a cut sits on a block boundary, and every interior slab is at least
        # 2 blocks wide (slabs.slab_bounds: contributions to a block then come
        # from at most two ranks)
        prev_block = bx[cuts[-1]] if r > 1 else None
        while c < len(xs) and (bx[c] == bx[c - 1] or (prev_block is not None and bx[c] < prev_block + 2)):
            c += 1
        if c >= len(xs):
            raise ValueError(f"the landslide release ({len(xs)} lattice columns, fraction={fraction}) is too "
                             f"small to cut into {world} slabs of at least 2 blocks")
        cuts.append(c)
    cuts.append(len(xs))
    for r in range(world):
        c0, c1 = cuts[r], cuts[r + 1]
        lo = INT32_MIN if r == 0 else int(bx[c0])
        hi = INT32_MAX if r == world - 1 else int(bx[c1])
        out.append((lo, hi, c0, c1))
    return out


CONFIGS = {
    "C1": granular_column,
    "C2": two_spheres,
    "C3": incline,
    "C4": landslide,
}

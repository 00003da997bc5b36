"""Explicit APIC MPM over a GPU hash grid -- drop-in for the reference's
hash-backend solver (/root/reference/pkg/src/sparsempm/solver.py).

Public surface kept from the reference: ``ParticleSet``, ``NodalFields``,
``Heightfield``, ``BoundaryCondition``, ``SimConfig``, ``StepStats``,
``Simulation`` (``step``, ``dt_bound``, ``n_dense``, ``particles``, ``t``,
``step_count``), and the module-level transfer functions ``bspline_weights``,
``p2g``, ``grid_forces``, ``grid_update``, ``g2p``, ``count_active_nodes``,
``apply_friction_boundary``.  All arithmetic runs in libsmpm.so (sm_100a).

Differences a caller can observe:
* fp32 particle/grid arithmetic (positions stay fp64; block/base indexing is
  bit-exact with the reference);
* ``Simulation`` evaluates the next step's stress at the end of ``step`` (in
  the fused kernel), so ``particles.F`` after a step is already return-mapped;
* ``block_size`` must be 4.  ``backend`` takes the reference's names:
  ``"hash"`` and ``"scan"`` both run the GPU hash-grid pipeline (the two CPU
  constructions produce the same active set and bitwise-equal results in the
  reference, test_acceptance.py:98-137); ``"dense"`` allocates every block of
  the domain each step (the comparison baseline of ``bench.compare``).
"""

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, InactiveNodeError, KeyRangeError, SimulationError
from .grid_index import ActiveIndexMap, as_index_map
from .materials import _degenerate_message, material_tables  # noqa: F401

BACKENDS = ("dense", "scan", "hash")
BC_PLANE = 0
BC_HEIGHTFIELD = 1
NODE_BYTES = 8 * (1 + 3 + 3)  # reference accounting (solver.py:29-30)
DEVICE_NODE_BYTES = 4 * 8 + 4 * 4  # fp32 accumulator record + velocity
MASS_FLOOR_SCALE = 1e-12


@dataclass
class ParticleSet:
    """Structure-of-arrays particle state (solver.py:95-149)."""

    x: np.ndarray
    v: np.ndarray
    C: np.ndarray
    F: np.ndarray
    m: np.ndarray
    V0: np.ndarray
    mat_id: np.ndarray
    sigma: np.ndarray
    jac: np.ndarray

    @property
    def n(self):
        return int(self.x.shape[0])

    @classmethod
    def from_samples(cls, positions, volumes, density, material_id=0, velocity=(0.0, 0.0, 0.0)):
        """Fresh particles at rest state: F = I, C = 0, zero stress."""
        x = np.array(positions, dtype=np.float64)
        vol = np.array(volumes, dtype=np.float64)
        n = x.shape[0]
        v = np.tile(np.asarray(velocity, dtype=np.float64), (n, 1))
        return cls(x=x, v=np.ascontiguousarray(v), C=np.zeros((n, 3, 3)),
                   F=np.ascontiguousarray(np.tile(np.eye(3), (n, 1, 1))), m=density * vol, V0=vol.copy(),
                   mat_id=np.full(n, material_id, dtype=np.int64), sigma=np.zeros((n, 3, 3)), jac=np.ones(n))

    @classmethod
    def merge(cls, sets):
        sets = list(sets)
        if not sets:
            raise ValueError("cannot merge zero particle sets")
        return cls(**{k: np.ascontiguousarray(np.concatenate([getattr(s, k) for s in sets], axis=0))
                      for k in _FIELDS})

    def copy(self):
        return ParticleSet(**{k: getattr(self, k).copy() for k in _FIELDS})


_FIELDS = ("x", "v", "C", "F", "m", "V0", "mat_id", "sigma", "jac")


@dataclass
class NodalFields:
    """Grid-side fields over the compact node range (solver.py:152-171)."""

    mass: np.ndarray
    vel: np.ndarray
    force: np.ndarray

    @classmethod
    def zeros(cls, n_nodes):
        return cls(mass=np.zeros(n_nodes), vel=np.zeros((n_nodes, 3)), force=np.zeros((n_nodes, 3)))

    @property
    def n_nodes(self):
        return int(self.mass.shape[0])


@dataclass
class Heightfield:
    """Regular elevation samples: data[i, j] is the height at (x0 + i*cell,
    y0 + j*cell) (solver.py:174-203)."""

    x0: float
    y0: float
    cell: float
    data: np.ndarray

    def __post_init__(self):
        self.data = np.ascontiguousarray(self.data, dtype=np.float64)
        if self.data.ndim != 2 or min(self.data.shape) < 2:
            raise ValueError("heightfield needs at least 2x2 samples")
        if self.cell <= 0:
            raise ValueError(f"heightfield cell size must be positive, got {self.cell}")

    def _sample(self, x, y):
        # bilinear, clamped (solver.py:241-274) -- host helper for scene setup
        nx, ny = self.data.shape
        fx = (x - self.x0) / self.cell
        fy = (y - self.y0) / self.cell
        i0 = min(max(int(math.floor(fx)), 0), nx - 2)
        j0 = min(max(int(math.floor(fy)), 0), ny - 2)
        tx = min(max(fx - i0, 0.0), 1.0)
        ty = min(max(fy - j0, 0.0), 1.0)
        d = self.data
        z = (d[i0, j0] * (1.0 - tx) * (1.0 - ty) + d[i0 + 1, j0] * tx * (1.0 - ty)
             + d[i0, j0 + 1] * (1.0 - tx) * ty + d[i0 + 1, j0 + 1] * tx * ty)
        zx = ((d[i0 + 1, j0] - d[i0, j0]) * (1.0 - ty) + (d[i0 + 1, j0 + 1] - d[i0, j0 + 1]) * ty) / self.cell
        zy = ((d[i0, j0 + 1] - d[i0, j0]) * (1.0 - tx) + (d[i0 + 1, j0 + 1] - d[i0 + 1, j0]) * tx) / self.cell
        return z, zx, zy

    def sample(self, x, y):
        return float(self._sample(float(x), float(y))[0])

    def normal(self, x, y):
        _, zx, zy = self._sample(float(x), float(y))
        n = np.array([-zx, -zy, 1.0])
        return n / np.linalg.norm(n)

    def sample_many(self, x, y):
        """Vectorised bilinear sample (for scene generation)."""
        nx, ny = self.data.shape
        fx = (np.asarray(x, dtype=np.float64) - self.x0) / self.cell
        fy = (np.asarray(y, dtype=np.float64) - self.y0) / self.cell
        i0 = np.clip(np.floor(fx).astype(np.int64), 0, nx - 2)
        j0 = np.clip(np.floor(fy).astype(np.int64), 0, ny - 2)
        tx = np.clip(fx - i0, 0.0, 1.0)
        ty = np.clip(fy - j0, 0.0, 1.0)
        d = self.data
        return (d[i0, j0] * (1 - tx) * (1 - ty) + d[i0 + 1, j0] * tx * (1 - ty) + d[i0, j0 + 1] * (1 - tx) * ty
                + d[i0 + 1, j0 + 1] * tx * ty)


@dataclass
class BoundaryCondition:
    """Frictional contact with a half-space or terrain (solver.py:206-238)."""

    kind: str = "plane"
    mu: float = 0.0
    point: np.ndarray = field(default_factory=lambda: np.zeros(3))
    normal: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, 1.0]))
    heightfield: Heightfield | None = None

    def __post_init__(self):
        if self.kind not in ("plane", "heightfield"):
            raise ConfigError(f"unknown boundary kind {self.kind!r}; choose one of ['heightfield', 'plane']")
        if self.mu < 0:
            raise ConfigError(f"friction coefficient must be >= 0, got {self.mu}")
        self.point = np.asarray(self.point, dtype=np.float64).reshape(3)
        normal = np.asarray(self.normal, dtype=np.float64).reshape(3)
        length = np.linalg.norm(normal)
        if self.kind == "plane":
            if length < 1e-12:
                raise ConfigError("boundary normal must be a nonzero vector")
            self.normal = normal / length
        if self.kind == "heightfield" and self.heightfield is None:
            raise ConfigError("heightfield boundary requires elevation data")


def _pack_boundaries(boundaries):
    """Boundary table for the C ABI (solver.py:841-860)."""
    boundaries = list(boundaries)
    arr = (_lib.Boundary * max(len(boundaries), 1))()
    hf = None
    for b, bc in enumerate(boundaries):
        arr[b].mu = float(bc.mu)
        if bc.kind == "plane":
            arr[b].kind = BC_PLANE
            for a in range(3):
                arr[b].point[a] = float(bc.point[a])
                arr[b].normal[a] = float(bc.normal[a])
        else:
            arr[b].kind = BC_HEIGHTFIELD
            hf = bc.heightfield
    return len(boundaries), arr, hf


@dataclass
class SimConfig:
    """Solver-level settings (solver.py:760-818)."""

    h: float
    gravity: np.ndarray
    total_time: float
    domain_min: np.ndarray
    domain_max: np.ndarray
    dt: float | None = None
    cfl: float = 0.4
    block_size: int = 4
    backend: str = "hash"
    n_threads: int = 1
    deterministic: bool = False
    # GPU option (not in the reference).  True (default): P2G summed per cell in
    # registers into a split fixed-point arena with per-item scales -- grid
    # sums at fp32 precision relative to each node, light surface nodes
    # included.  False: the per-particle int32 fixed-point scatter with one
    # global scale per launch, ~20 % faster, but light nodes and stress-
    # cancelling contacts lose precision.  Deterministic
    # mode always uses its int64 fixed-point path.
    precise_grid: bool = True

    def __post_init__(self):
        if self.h <= 0:
            raise ConfigError(f"grid cell size must be positive, got {self.h}")
        if self.total_time <= 0:
            raise ConfigError(f"total time must be positive, got {self.total_time}")
        if self.dt is not None and self.dt <= 0:
            raise ConfigError(f"timestep must be positive, got {self.dt}")
        if not 0.0 < self.cfl <= 1.0:
            raise ConfigError(f"cfl must lie in (0, 1], got {self.cfl}")
        if self.backend not in BACKENDS:
            raise ConfigError(f"unknown backend {self.backend!r}; expected one of {sorted(BACKENDS)}")
        if self.block_size != 4:
            raise ConfigError(f"block size must be 4 on the GPU grid (one u64 node mask per block), "
                              f"got {self.block_size}")
        if self.n_threads < 1:
            raise ConfigError(f"thread count must be at least 1, got {self.n_threads}")
        self.gravity = np.asarray(self.gravity, dtype=np.float64).reshape(3)
        if not np.all(np.isfinite(self.gravity)):
            raise ConfigError("gravity must be finite")
        self.domain_min = np.asarray(self.domain_min, dtype=np.float64).reshape(3)
        self.domain_max = np.asarray(self.domain_max, dtype=np.float64).reshape(3)
        if not np.all(self.domain_max > self.domain_min):
            raise ConfigError("domain_max must exceed domain_min on each axis")

    @property
    def node_min(self):
        return np.floor(self.domain_min / self.h).astype(np.int64)

    @property
    def node_max(self):
        return np.ceil(self.domain_max / self.h).astype(np.int64)


@dataclass
class StepStats:
    """Per-step record (solver.py:821-832).  ``times`` holds device times in
    seconds per phase of the fused pipeline."""

    step: int
    t: float
    dt: float
    n_active: int
    n_allocated: int
    times: dict
    mass_sum: float | None = None
    mom_sum: np.ndarray | None = None


# Phases of the reference's step (solver.py:835).  On the GPU, stress and p2g
# of step n+1 run inside the fused g2p kernel of step n and alloc_zero inside
# grid_update, so their entries are 0 and "g2p" holds the fused time.
PHASES = ("map_build", "alloc_zero", "p2g", "grid_update", "g2p", "stress")
EXTRA_PHASES = ("metrics",)


# ---------------------------------------------------------------- module API

def _host_err(err_t):
    return _lib.err_code(np.uint64(err_t.cpu().numpy()[0]))


def bspline_weights(x, h):
    """Per-axis quadratic B-spline data at x (solver.py:80-92)."""
    torch = _lib.torch_cuda()
    xd = _lib.to_dev(np.asarray(x, dtype=np.float64).reshape(1, 3), np.float64)
    base = torch.empty(3, dtype=torch.int64, device="cuda")
    w = torch.empty(9, dtype=torch.float64, device="cuda")
    dw = torch.empty(9, dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().smpm_bspline(_lib.ptr(xd), 1, float(h), _lib.ptr(base), _lib.ptr(w), _lib.ptr(dw),
                                        _lib.stream_ptr()), "bspline")
    return base.cpu().numpy(), w.cpu().numpy().reshape(3, 3), dw.cpu().numpy().reshape(3, 3)


def _stencil_params(h, gravity=(0.0, 0.0, 0.0)):
    sp = _lib.StencilParams()
    sp.h = float(h)
    sp.inv_h = 1.0 / float(h)
    for a in range(3):
        sp.gravity[a] = float(gravity[a])
    return sp


def _scatter(particles, index_map, h, gravity, fields, want_mass_mom, want_force):
    torch = _lib.torch_cuda()
    index_map = as_index_map(index_map)
    n = particles.n
    nn = index_map.n_nodes
    if fields is None:
        fields = NodalFields.zeros(nn)
    dev = {k: _lib.to_dev(getattr(particles, k), np.float64) for k in ("x", "v", "C", "m", "sigma", "jac", "V0")}
    mass = torch.zeros(max(nn, 1), dtype=torch.float32, device="cuda") if want_mass_mom else None
    mom = torch.zeros(max(3 * nn, 1), dtype=torch.float32, device="cuda") if want_mass_mom else None
    force = torch.zeros(max(3 * nn, 1), dtype=torch.float32, device="cuda") if want_force else None
    err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    sp = _stencil_params(h, gravity)
    _lib.check(_lib.load().smpm_p2g(index_map.kernel_args(), __import__("ctypes").byref(sp), n,
                                    *(_lib.ptr(dev[k]) for k in ("x", "v", "C", "m", "sigma", "jac", "V0")),
                                    _lib.ptr(mass), _lib.ptr(mom), _lib.ptr(force), _lib.ptr(err),
                                    _lib.stream_ptr()), "p2g")
    code, _p = _host_err(err)
    if code == _lib.ERR_INACTIVE:
        raise InactiveNodeError("a particle stencil node is outside the active grid; with the dense backend this means "
                                "a particle left the declared domain")
    if code == _lib.ERR_KEY_RANGE:
        raise KeyRangeError("particle stencil block outside packable coordinate range")
    if want_mass_mom:
        fields.mass[...] += mass[:nn].double().cpu().numpy()
        fields.vel[...] += mom[:3 * nn].double().cpu().numpy().reshape(nn, 3)
    if want_force:
        fields.force[...] += force[:3 * nn].double().cpu().numpy().reshape(nn, 3)
    return fields


def p2g(particles, index_map, h, deterministic=True, fields=None):
    """Scatter mass and APIC momentum (solver.py:863-877); ``vel`` holds
    momentum on return.  ``deterministic`` is accepted for API parity."""
    return _scatter(particles, index_map, h, (0.0, 0.0, 0.0), fields, True, False)


def grid_forces(particles, index_map, h, gravity, deterministic=True, fields=None):
    """Scatter internal stress forces plus gravity (solver.py:880-894)."""
    return _scatter(particles, index_map, h, np.asarray(gravity, dtype=np.float64).reshape(3), fields, False, True)


def _grid_params(h, dt, mass_floor, boundaries, gravity=(0.0, 0.0, 0.0)):
    gp = _lib.GridParams()
    gp.h = float(h)
    gp.dt = float(dt)
    gp.mass_floor = float(mass_floor)
    for a in range(3):
        gp.gravity[a] = float(gravity[a])
    nb, arr, hf = _pack_boundaries(boundaries)
    gp.n_bc = nb
    gp.bc = __import__("ctypes").cast(arr, _lib.P)
    keep = [arr]
    if hf is not None:
        data = np.ascontiguousarray(hf.data, dtype=np.float64)
        keep.append(data)
        gp.hf_data = data.ctypes.data
        gp.hf_nx, gp.hf_ny = data.shape
        gp.hf_x0, gp.hf_y0, gp.hf_cell = float(hf.x0), float(hf.y0), float(hf.cell)
    else:
        gp.hf_cell = 1.0
    return gp, keep


def grid_update(fields, index_map, h, dt, mass_floor=0.0, boundaries=()):
    """Momentum -> velocity, forces and boundary projection (solver.py:897-909)."""
    import ctypes

    nn = fields.n_nodes
    mass = _lib.to_dev(fields.mass, np.float32)
    vel = _lib.to_dev(fields.vel.reshape(-1), np.float32)
    force = _lib.to_dev(fields.force.reshape(-1), np.float32)
    blocks = index_map.active_blocks if hasattr(index_map, "active_blocks") else as_index_map(index_map).active_blocks
    blocks = _lib.to_dev(np.asarray(blocks), np.int32)
    gp, keep = _grid_params(h, dt, mass_floor, boundaries)
    _lib.check(_lib.load().smpm_grid_update(ctypes.byref(gp), nn, _lib.ptr(mass), _lib.ptr(vel), _lib.ptr(force),
                                            _lib.ptr(blocks), _lib.stream_ptr()), "grid update")
    del keep
    fields.vel[...] = vel.double().cpu().numpy().reshape(nn, 3)
    return fields


def g2p(particles, index_map, fields, h, dt):
    """Gather velocities, update v, C, F and advect x (solver.py:912-924)."""
    import ctypes

    torch = _lib.torch_cuda()
    index_map = as_index_map(index_map)
    dev = {k: _lib.to_dev(getattr(particles, k), np.float64) for k in ("x", "v", "C", "F")}
    vel = _lib.to_dev(fields.vel.reshape(-1), np.float32)
    err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    sp = _stencil_params(h)
    _lib.check(_lib.load().smpm_g2p(index_map.kernel_args(), ctypes.byref(sp), float(dt), particles.n,
                                    _lib.ptr(dev["x"]), _lib.ptr(dev["v"]), _lib.ptr(dev["C"]), _lib.ptr(dev["F"]),
                                    _lib.ptr(vel), _lib.ptr(err), _lib.stream_ptr()), "g2p")
    code, _p = _host_err(err)
    if code == _lib.ERR_INACTIVE:
        raise InactiveNodeError("a particle stencil node is outside the active grid; with the dense backend this means "
                                "a particle left the declared domain")
    for k in ("x", "v", "C", "F"):
        getattr(particles, k)[...] = dev[k].cpu().numpy().reshape(getattr(particles, k).shape)
    return particles


def count_active_nodes(positions, h):
    """|union of all particle stencils| (solver.py:749-757), bit-exact, via
    per-block 64-bit node masks on the device."""
    torch = _lib.torch_cuda()
    xp = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    n = xp.shape[0]
    cap = 1
    while cap < max(64, 8 * n):
        cap *= 2
    t = _lib.DeviceHashTable(cap, cap)
    x = _lib.to_dev(xp, np.float64)
    masks = torch.zeros(cap, dtype=torch.int64, device="cuda")
    err = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    out = np.zeros(1, dtype=np.uint64)
    _lib.check(_lib.load().smpm_count_active_nodes(t.dref, _lib.ptr(x), n, 1.0 / float(h), _lib.ptr(masks),
                                                   _lib.ptr(err), out.ctypes.data, _lib.stream_ptr()), "count")
    code, _p = _host_err(err)
    if code == _lib.ERR_KEY_RANGE:
        raise KeyRangeError("particle stencil block outside packable coordinate range")
    return int(out[0])


def apply_friction_boundary(v, normal, mu):
    """Coulomb contact projection of one velocity (solver.py:294-306), on
    the device through the grid-update kernel (one node on the surface)."""
    n = np.asarray(normal, dtype=np.float64).reshape(3)
    n = n / np.linalg.norm(n)
    fields = NodalFields(mass=np.ones(64), vel=np.zeros((64, 3)), force=np.zeros((64, 3)))
    fields.vel[0] = np.asarray(v, dtype=np.float64).reshape(3)

    class _Map:
        active_blocks = np.zeros((1, 3), dtype=np.int64)

    bc = BoundaryCondition(kind="plane", mu=float(mu), point=np.zeros(3), normal=n)
    grid_update(fields, _Map, 1.0, 0.0, -1.0, [bc])
    return fields.vel[0].copy()


# ---------------------------------------------------------------- Simulation

def _fingerprint(ps):
    h = hashlib.blake2b(digest_size=16)
    for k in ("x", "v", "C", "F", "m", "V0", "mat_id"):
        h.update(np.ascontiguousarray(getattr(ps, k)).tobytes())
    return h.digest()


MIRROR_AUTO_MAX = 1 << 16  # host_sync="auto": mirror sets up to this many particles
FINGERPRINT_MAX = 1 << 21  # larger host views are not fingerprinted (an edit check would cost a full hash)


class Simulation:
    """One scenario instance on the GPU (solver.py:927-1093).

    The particle state lives on the device.  The caller's ParticleSet stays
    the simulation's host view, like the reference's in-place arrays:

    * ``host_sync="mirror"``: after every step the caller's arrays are
      refreshed from the device, and edits made to them between steps are
      uploaded by the next step (detected by a content fingerprint) -- the
      reference's semantics exactly;
    * ``host_sync="on_access"``: the caller's arrays are refreshed when
      ``particles`` is read; edits made after that read are uploaded by the
      next step.  Read ``particles`` again after stepping before editing
      (a per-step download of a 100M-particle set would cost more than the
      step);
    * ``"auto"`` (default): mirror up to 2^16 particles, on_access above.

    In on_access mode an edit to a view that a later step made stale is not
    seen (read ``particles`` again after stepping, or use "mirror").
    """

    def __init__(self, particles, config, materials, boundaries=(), record_conservation=False,
                 block_capacity=None, device=0, stream=None, particle_capacity=None, slab=None,
                 host_sync="auto", retain_fields=False):
        import ctypes

        if host_sync not in ("auto", "mirror", "on_access"):
            raise ConfigError(f"host_sync must be auto, mirror or on_access, got {host_sync!r}")
        self._mirror = host_sync == "mirror" or (host_sync == "auto" and particles.n <= MIRROR_AUTO_MAX)
        self._particles = particles
        self.config = config
        self.materials = list(materials)
        self.boundaries = list(boundaries)
        self.record_conservation = record_conservation
        if particles.n == 0:
            raise ConfigError("simulation needs at least one particle")
        if len(self.materials) == 0:
            raise ConfigError("simulation needs at least one material")
        if len(self.materials) > 8:
            raise ConfigError("at most 8 materials are supported on the GPU")
        # large host sets: the material-id range and max mass are checked / taken
        # by the library's threaded upload (mass floor < 0: "from the particles")
        in_lib = particles.n >= 1 << 20 and isinstance(particles.x, np.ndarray)
        if not in_lib and (particles.mat_id.min() < 0 or particles.mat_id.max() >= len(self.materials)):
            raise ConfigError("particle material id out of range")
        if sum(1 for b in self.boundaries if b.kind == "heightfield") > 1:
            raise ConfigError("at most one heightfield boundary is supported")
        self._wave_speed = max(m.wave_speed for m in self.materials)
        self._mass_floor = -1.0 if in_lib else MASS_FLOOR_SCALE * float(particles.m.max())
        torch = _lib.torch_cuda()
        lib = _lib.load()
        # every kernel of this simulation runs on one torch-managed stream
        self.stream = stream if stream is not None else torch.cuda.Stream(device=device)
        cfg = _lib.SimConfigC()
        cfg.h = float(config.h)
        for a in range(3):
            cfg.gravity[a] = float(config.gravity[a])
        cfg.cfl = float(config.cfl)
        cfg.wave_speed = float(self._wave_speed)
        cfg.mass_floor = float(self._mass_floor)
        self._mats = _lib.material_array(self.materials)
        cfg.n_mat = len(self.materials)
        cfg.mats = ctypes.cast(self._mats, _lib.P)
        nb, self._bc, hf = _pack_boundaries(self.boundaries)
        cfg.n_bc = nb
        cfg.bc = ctypes.cast(self._bc, _lib.P)
        if hf is not None:
            self._hf = np.ascontiguousarray(hf.data, dtype=np.float64)
            cfg.hf_data = self._hf.ctypes.data
            cfg.hf_nx, cfg.hf_ny = self._hf.shape
            cfg.hf_x0, cfg.hf_y0, cfg.hf_cell = float(hf.x0), float(hf.y0), float(hf.cell)
        else:
            cfg.hf_cell = 1.0
        cfg.particle_capacity = max(particles.n, int(particle_capacity or 0))
        cfg.block_capacity = int(block_capacity or 0)
        cfg.deterministic = int(bool(config.deterministic))
        cfg.precise_grid = int(bool(getattr(config, "precise_grid", True)))
        cfg.record_conservation = int(bool(record_conservation))
        cfg.device = int(device)
        cfg.stream = self.stream.cuda_stream
        self._cfg = cfg
        h = ctypes.c_void_p()
        _lib.check(lib.smpm_sim_create(ctypes.byref(cfg), ctypes.byref(h)), "sim create")
        self._h = h
        if slab is not None:  # (bx0, bx1, pid_base, migrant_capacity): see slabs.py
            _lib.check(lib.smpm_sim_set_slab(h, *[int(v) for v in slab]), "set slab")
        if config.backend == "dense":
            bs = int(config.block_size)
            bmin = (ctypes.c_int32 * 3)(*[int(v) // bs for v in config.node_min])
            bmax = (ctypes.c_int32 * 3)(*[int(v) // bs for v in config.node_max])
            _lib.check(lib.smpm_sim_set_dense_domain(h, bmin, bmax), "dense domain")
        self._retain = bool(retain_fields)
        if self._retain:
            _lib.check(lib.smpm_sim_retain_fields(h, 1), "retain fields")
        self._upload(particles)
        if particles.n <= FINGERPRINT_MAX:  # edits to the caller's set before the first step are taken
            self._fp = _fingerprint(particles)
        self.t = 0.0
        self.step_count = 0
        self.last_stats = None
        self._last = None  # (step_count, last_map, last_fields), fetched on demand
        if config.dt is not None and config.dt > self.dt_bound():
            raise ConfigError(f"fixed timestep {config.dt:g} exceeds the stability bound {self.dt_bound():g}")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.smpm_sim_destroy(h)
            self._h = None

    # -- state transfer -----------------------------------------------------
    def _upload(self, ps):
        arrs = [np.ascontiguousarray(getattr(ps, k), dtype=np.float64) for k in ("x", "v", "C", "F", "m", "V0")]
        mid = np.ascontiguousarray(ps.mat_id, dtype=np.int64)
        # non-finite positions are detected on the device while the first
        # step bins the particles and raised by that step (solver.py:1005-1006)
        _lib.check(_lib.load().smpm_sim_set_particles(self._h, ps.n, *(a.ctypes.data for a in arrs),
                                                      mid.ctypes.data), "set particles")
        self._fresh = True  # device state == the caller's arrays
        self._fp = None

    def _download(self, ps):
        keys = ("x", "v", "C", "F", "sigma", "jac")
        # straight into the caller's arrays when they are C-contiguous fp64
        # (no temporaries: the host side of a large download is page-bound)
        out = {}
        for k in keys:
            a = getattr(ps, k)
            out[k] = a if (a.dtype == np.float64 and a.flags.c_contiguous and a.flags.writeable) else \
                np.empty(a.shape, dtype=np.float64)
        _lib.check(_lib.load().smpm_sim_get_particles(self._h, *(out[k].ctypes.data for k in keys)), "get particles")
        for k in keys:
            if out[k] is not getattr(ps, k):
                getattr(ps, k)[...] = out[k]

    def _refresh_host(self):
        """Make the caller's arrays equal to the device state."""
        self._download(self._particles)
        self._fp = _fingerprint(self._particles) if self._particles.n <= FINGERPRINT_MAX else b""
        self._fresh = True

    @property
    def particles(self):
        """The caller's ParticleSet, refreshed from the device."""
        if not self._fresh:
            self._refresh_host()
        elif self._fp is None:  # handed out again: edits before the next step are taken
            self._fp = _fingerprint(self._particles) if self._particles.n <= FINGERPRINT_MAX else b""
        return self._particles

    def _sync_host_edits(self):
        """Upload edits the caller made to the host view (reference: the
        arrays are the state).  Only a view that still equals the device state
        (handed out since the last step, or the constructor's set before the
        first step) is checked -- one fingerprint, not one per step."""
        if not self._fresh or self._fp is None:
            return
        if self._fp == b"":  # no fingerprint (large set): take the view
            self._upload(self._particles)
            return
        if _fingerprint(self._particles) != self._fp:
            self._upload(self._particles)
        self._fp = None  # checked: the next check needs a new view

    # -- API ------------------------------------------------------------------
    @property
    def n_dense(self):
        """Allocated node count of a dense grid over the domain (solver.py:976-982)."""
        cfg = self.config
        blocks = cfg.node_max // cfg.block_size - cfg.node_min // cfg.block_size + 1
        return int(np.prod(blocks)) * cfg.block_size ** 3

    def dt_bound(self):
        """CFL-limited timestep for the current velocities (solver.py:984-987)."""
        self._sync_host_edits()
        vmax = float(_lib.load().smpm_sim_vmax(self._h))
        return self.config.cfl * self.config.h / (self._wave_speed + vmax)

    def _raise_status(self, rc, dt):
        import ctypes

        st = _lib.StepStatsC()
        _lib.load().smpm_sim_sync(self._h, ctypes.byref(st))
        p = int(st.err_particle)
        if rc == _lib.ERR_DEGENERATE_F:
            raise SimulationError(_degenerate_message(self.particles, p))
        if rc == _lib.ERR_NONFINITE_X:
            raise SimulationError("non-finite particle position")
        if rc == _lib.ERR_DT_BOUND:
            raise SimulationError(f"timestep {dt:g} exceeds the stability bound {self.dt_bound():g}")
        if rc == _lib.ERR_KEY_RANGE:
            raise KeyRangeError("particle stencil block outside packable coordinate range")
        _lib.check(rc, "step")

    def _stats(self, st, step, t):
        times = {p: 0.0 for p in PHASES}
        times["map_build"] = st.ms_map * 1e-3
        times["grid_update"] = st.ms_grid * 1e-3
        times["g2p"] = st.ms_fused * 1e-3
        times["metrics"] = 0.0
        return StepStats(step=step, t=t, dt=st.dt, n_active=int(st.n_active),
                         n_allocated=int(st.n_blocks) * 64, times=times,
                         mass_sum=float(st.mass_sum) if self.record_conservation else None,
                         mom_sum=np.array(st.mom_sum[:]) if self.record_conservation else None)

    def run(self, n_steps, dt=None):
        """Advance ``n_steps`` explicit steps; returns their StepStats.

        Same steps as ``n_steps`` calls of :meth:`step` (the reference's
        loop, S/bench.py:216-226) without a host round trip per step: the
        CFL bound, dt validation, error and grid-capacity checks run on the
        device and the stats come back once per batch of up to 1024 steps
        (``smpm_sim_run``).  An error is raised after the steps before it
        completed (``step_count`` and ``last_stats`` include them)."""
        import ctypes

        n_steps = int(n_steps)
        if n_steps < 0:
            raise ConfigError(f"n_steps must be >= 0, got {n_steps}")
        self._sync_host_edits()
        cfg = self.config
        if dt is None:
            dt = cfg.dt
        if dt is not None:
            dt = float(dt)
            if not dt > 0.0:
                raise SimulationError(f"timestep must be positive, got {dt}")
        if n_steps == 0:
            return []
        lib = _lib.load()
        arr = (_lib.StepStatsC * n_steps)()
        done = ctypes.c_int64(0)
        rc = lib.smpm_sim_run(self._h, n_steps, -1.0 if dt is None else dt, arr, ctypes.byref(done))
        out = []
        for i in range(int(done.value)):
            self.t += arr[i].dt
            self.step_count += 1
            out.append(self._stats(arr[i], self.step_count, self.t))
        if out:
            self.last_stats = out[-1]
            self._fresh = False
            self._fp = None
            if self._mirror:
                self._refresh_host()
        if rc:
            self._raise_status(rc, dt)
        return out

    def step(self, dt=None):
        """Advance one explicit step; returns its StepStats (solver.py:1001-1093)."""
        import ctypes

        self._sync_host_edits()
        cfg = self.config
        if dt is None:
            dt = cfg.dt
        if dt is not None:
            dt = float(dt)
            if not dt > 0.0:
                raise SimulationError(f"timestep must be positive, got {dt}")
        lib = _lib.load()
        # the library takes dt <= 0 as "use the CFL bound" (solver.py:1021-1023)
        rc = lib.smpm_sim_step(self._h, -1.0 if dt is None else dt)
        if rc:
            self._raise_status(rc, dt)
        st = _lib.StepStatsC()
        _lib.check(lib.smpm_sim_sync(self._h, ctypes.byref(st)), "sync")
        self.t += st.dt
        self.step_count += 1
        stats = self._stats(st, self.step_count, self.t)
        self.last_stats = stats
        self._fresh = False
        self._fp = None
        if self._mirror:  # the caller's arrays follow the device state (reference: in place)
            self._refresh_host()
        return stats

    def _fetch_last(self):
        """last_map / last_fields of the last completed step (solver.py:1087-1090),
        downloaded on first access."""
        import ctypes

        if self._last is not None and self._last[0] == self.step_count:
            return self._last
        lib = _lib.load()
        nb = ctypes.c_int64(0)
        rc = lib.smpm_sim_last_grid_size(self._h, ctypes.byref(nb))
        if rc == _lib.ERR_STATE:  # no step yet (or the grid was rebuilt since): the reference's None
            self._last = (self.step_count, None, None)
            return self._last
        _lib.check(rc, "last grid size")
        nb = int(nb.value)
        blocks = np.empty((max(nb, 1), 3), dtype=np.int32)
        mass = np.empty(max(nb, 1) * 64, dtype=np.float32)
        vel = np.empty((max(nb, 1) * 64, 3), dtype=np.float32)
        force = np.empty((max(nb, 1) * 64, 3), dtype=np.float32) if self._retain else None
        _lib.check(lib.smpm_sim_last_grid(self._h, blocks.ctypes.data, mass.ctypes.data, vel.ctypes.data,
                                          force.ctypes.data if force is not None else None), "last grid")
        amap = ActiveIndexMap.from_blocks(blocks[:nb].astype(np.int64))
        fields = NodalFields(mass=mass[:nb * 64].astype(np.float64), vel=vel[:nb * 64].astype(np.float64),
                             force=force[:nb * 64].astype(np.float64) if force is not None else None)
        self._last = (self.step_count, amap, fields)
        return self._last

    @property
    def last_map(self):
        """ActiveIndexMap of the last step's grid (None before the first step)."""
        return self._fetch_last()[1]

    @property
    def last_fields(self):
        """NodalFields of the last step after the grid update: node mass, grid
        velocity (boundary-projected) and -- with ``retain_fields=True`` -- the
        nodal force incl. gravity (else ``force`` is None).  None before the
        first step."""
        return self._fetch_last()[2]

    def query_grid(self):
        """(active_blocks int64 (n,3), NodalFields) of the P2G computed from
        the current particles -- the grid the next step's update consumes;
        ``vel`` holds momentum and ``force`` includes gravity.  For parity."""
        import ctypes

        self._sync_host_edits()
        lib = _lib.load()
        nb = ctypes.c_int64(0)
        _lib.check(lib.smpm_sim_grid_size(self._h, ctypes.byref(nb)), "grid size")
        nb = int(nb.value)
        blocks = np.empty((max(nb, 1), 3), dtype=np.int32)
        mass = np.empty(max(nb, 1) * 64, dtype=np.float32)
        mom = np.empty((max(nb, 1) * 64, 3), dtype=np.float32)
        force = np.empty((max(nb, 1) * 64, 3), dtype=np.float32)
        _lib.check(lib.smpm_sim_query_grid(self._h, blocks.ctypes.data, mass.ctypes.data, mom.ctypes.data,
                                           force.ctypes.data), "query grid")
        f = NodalFields(mass=mass[:nb * 64].astype(np.float64), vel=mom[:nb * 64].astype(np.float64),
                        force=force[:nb * 64].astype(np.float64))
        return blocks[:nb].astype(np.int64), f


def release_cached_memory():
    """Return the device memory that destroyed simulations left in the
    library's reuse cache (include/smpm.h) to the driver."""
    _lib.check(_lib.load().smpm_release_cached_memory(), "release cached memory")


__all__ = ["ParticleSet", "NodalFields", "Heightfield", "BoundaryCondition", "SimConfig", "StepStats", "Simulation",
           "PHASES", "EXTRA_PHASES", "NODE_BYTES", "bspline_weights", "p2g", "grid_forces", "grid_update", "g2p",
           "count_active_nodes", "apply_friction_boundary", "ActiveIndexMap", "release_cached_memory"]

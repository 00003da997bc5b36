"""CPU oracle for the sparse-MPM hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker and the CPU-baseline arm.  Only tests/,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it; the product package never does.

It restates the reference package ``sparsempm`` (paths relative to
/root/reference/pkg/src/sparsempm/): the numba kernels live in C
(``smpm_oracle.c`` -> ``liboracle.so``), and this file mirrors the Python
control flow around them:

* ``build_hash_sparse_grid``   -- sparse_hash.py:225-264 (rebuild loop)
* ``BlockHashTable``           -- sparse_hash.py:109-167
* ``build_scan_sparse_grid``   -- sparse_scan.py:44-172
* ``build_dense_grid``         -- grid_index.py:256-277
* ``p2g/grid_forces/grid_update/g2p`` -- solver.py:863-924
* ``update_stress``            -- materials.py:250-267
* ``count_active_nodes``       -- solver.py:749-757
* ``OracleSimulation.step``    -- solver.py:1001-1093

Pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz).
"""

import ctypes
import math
import os
import subprocess
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

KEY_BIAS = 1 << 20
COORD_MIN = -(1 << 20)
COORD_MAX = (1 << 20) - 1
EMPTY_KEY = (1 << 64) - 1
MODE_FLAT = 0
MODE_HASH = 1
BC_PLANE = 0
BC_HEIGHTFIELD = 1
KIND_ELASTIC = 0
KIND_DRUCKER_PRAGER = 1
MASS_FLOOR_SCALE = 1e-12  # solver.py:32
NODE_BYTES = 8 * (1 + 3 + 3)  # solver.py:29-30

_lib = None


def build():
    """Compile liboracle.so with its Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = _load(ctypes.CDLL(str(LIB_PATH)))
    return _lib


class OrMap(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int64),
        ("bmin", ctypes.c_int64 * 3),
        ("bshape", ctypes.c_int64 * 3),
        ("phi_flat", ctypes.c_void_p),
        ("keys", ctypes.c_void_p),
        ("vals", ctypes.c_void_p),
        ("n_slots", ctypes.c_int64),
        ("bsz", ctypes.c_int64),
    ]


def _load(L):
    P = ctypes.c_void_p
    I64 = ctypes.c_int64
    D = ctypes.c_double
    I = ctypes.c_int
    sig = {
        "or_pack_key": (ctypes.c_uint64, [I64, I64, I64]),
        "or_unpack_key": (None, [ctypes.c_uint64, P]),
        "or_mix64": (ctypes.c_uint64, [ctypes.c_uint64]),
        "or_hash_insert": (I64, [P, P, I64, P, P, ctypes.c_uint64, P]),
        "or_hash_lookup": (I64, [P, P, I64, ctypes.c_uint64]),
        "or_hash_insert_many": (None, [P, P, I64, P, P, P, I64, P, P, I]),
        "or_insert_particle_blocks": (I64, [P, I64, D, I64, P, P, I64, P, P, I]),
        "or_hash_active_blocks": (None, [P, P, I64, P]),
        "or_stencil_base_bounds": (None, [P, I64, D, P, P]),
        "or_mark_blocks": (I64, [P, I64, D, I64, P, P, P, I]),
        "or_exclusive_scan": (I64, [P, I64, P]),
        "or_mark_nodes": (None, [P, I64, D, P, I64, I64, P, I]),
        "or_node_to_compact": (I64, [P, I64, I64, I64]),
        "or_stencil": (None, [P, D, P, P, P]),
        "or_scatter": (I64, [P, P, P, P, P, P, P, I64, D, D, D, D, D, P, P, P, P, I]),
        "or_hf_sample": (None, [P, I64, I64, D, D, D, D, D, P]),
        "or_coulomb_project": (None, [P, P, D]),
        "or_grid_update": (None, [P, P, P, I64, P, I64, D, D, D, P, P, P, P, I64, P, I64, I64, D, D, D, I]),
        "or_g2p": (I64, [P, P, P, P, P, I64, D, D, D, P, I]),
        "or_dp_return_map": (None, [P, D, D, P]),
        "or_sym_eigh3": (None, [P, P]),
        "or_stress": (None, [P, P, P, P, I64, P, P, P, P, P, I]),
        "or_vmax": (D, [P, I64, I]),
        "or_set_threads": (None, [I]),
        "or_get_threads": (I, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def set_threads(n):
    lib().or_set_threads(int(n))


def get_threads():
    return int(lib().or_get_threads())


# ----------------------------------------------------------------- keys

def pack_key(block):
    """grid_index.py:41-59 (with the KeyRangeError range check)."""
    packed = 0
    for c in block:
        c = int(c)
        if not COORD_MIN <= c <= COORD_MAX:
            raise ValueError(f"block coordinate {c} outside packable range")
        packed = (packed << 21) | (c + KEY_BIAS)
    return packed


def unpack_key(key):
    out = np.zeros(3, dtype=np.int64)
    lib().or_unpack_key(ctypes.c_uint64(int(key)), out.ctypes.data)
    return tuple(int(v) for v in out)


def mix64(key):
    return int(lib().or_mix64(ctypes.c_uint64(int(key) & ((1 << 64) - 1))))


def pack_keys(blocks):
    """Vectorised pack of an (n,3) int64 block array (grid_index.py:100-105)."""
    b = np.asarray(blocks, dtype=np.int64).reshape(-1, 3) + KEY_BIAS
    b = b.astype(np.uint64)
    return (b[:, 0] << np.uint64(42)) | (b[:, 1] << np.uint64(21)) | b[:, 2]


def unpack_keys(keys):
    k = np.asarray(keys, dtype=np.uint64)
    m = np.uint64((1 << 21) - 1)
    out = np.empty((k.shape[0], 3), dtype=np.int64)
    out[:, 2] = (k & m).astype(np.int64) - KEY_BIAS
    out[:, 1] = ((k >> np.uint64(21)) & m).astype(np.int64) - KEY_BIAS
    out[:, 0] = ((k >> np.uint64(42)) & m).astype(np.int64) - KEY_BIAS
    return out


def mix64_array(keys):
    """Vectorised SplitMix64 finaliser (grid_index.py:116-121)."""
    z = np.asarray(keys, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


# ------------------------------------------------------------ index maps

class OracleMap:
    """Mirror of ActiveIndexMap (grid_index.py:179-248)."""

    def __init__(self, block_size, active_blocks, mode, bmin=None, bshape=None, phi_flat=None, keys=None,
                 vals=None):
        self.block_size = int(block_size)
        self.active_blocks = np.ascontiguousarray(active_blocks, dtype=np.int64).reshape(-1, 3)
        self.mode = mode
        self.bmin = np.zeros(3, np.int64) if bmin is None else np.asarray(bmin, np.int64)
        self.bshape = np.zeros(3, np.int64) if bshape is None else np.asarray(bshape, np.int64)
        self.phi_flat = np.zeros(1, np.int64) if phi_flat is None else np.ascontiguousarray(phi_flat, np.int64)
        self.keys = np.zeros(1, np.uint64) if keys is None else np.ascontiguousarray(keys, np.uint64)
        self.vals = np.zeros(1, np.int64) if vals is None else np.ascontiguousarray(vals, np.int64)
        self._c = OrMap()
        self._c.mode = mode
        for a in range(3):
            self._c.bmin[a] = int(self.bmin[a])
            self._c.bshape[a] = int(self.bshape[a])
        self._c.phi_flat = self.phi_flat.ctypes.data
        self._c.keys = self.keys.ctypes.data
        self._c.vals = self.vals.ctypes.data
        self._c.n_slots = int(self.keys.shape[0]) if keys is not None else 0
        self._c.bsz = self.block_size

    @property
    def n_blocks(self):
        return int(self.active_blocks.shape[0])

    @property
    def n_nodes(self):
        return self.n_blocks * self.block_size ** 3

    @property
    def cref(self):
        return ctypes.byref(self._c)

    def node_index(self, node):
        return int(lib().or_node_to_compact(self.cref, int(node[0]), int(node[1]), int(node[2])))

    def node_coords(self):
        """grid_index.py:229-237"""
        b = self.block_size
        rng = np.arange(b, dtype=np.int64)
        li, lj, lk = np.meshgrid(rng, rng, rng, indexing="ij")
        local = np.stack([li.ravel(), lj.ravel(), lk.ravel()], axis=1)
        base = self.active_blocks[:, None, :] * b
        return (base + local[None, :, :]).reshape(-1, 3)


class BlockHashTable:
    """sparse_hash.py:109-167"""

    def __init__(self, capacity):
        capacity = int(capacity)
        if capacity < 1 or capacity & (capacity - 1):
            raise ValueError(f"table capacity must be a power of two, got {capacity}")
        self.keys = np.full(capacity, EMPTY_KEY, dtype=np.uint64)
        self.vals = np.full(capacity, -1, dtype=np.int64)
        self.counter = np.zeros(1, dtype=np.int64)
        self.overflow = np.zeros(1, dtype=np.int64)

    @property
    def capacity(self):
        return int(self.keys.shape[0])

    @property
    def count(self):
        return int(self.counter[0])

    @property
    def overflowed(self):
        return bool(self.overflow[0])

    def insert(self, block):
        key = pack_key(block)
        fresh = np.zeros(1, dtype=np.int32)
        r = lib().or_hash_insert(self.keys.ctypes.data, self.vals.ctypes.data, self.capacity,
                                 self.counter.ctypes.data, self.overflow.ctypes.data, ctypes.c_uint64(key),
                                 fresh.ctypes.data)
        return int(r), bool(fresh[0])

    def insert_many(self, packed, parallel=False):
        packed = np.ascontiguousarray(packed, dtype=np.uint64)
        ranks = np.empty(packed.shape[0], dtype=np.int64)
        fresh = np.empty(packed.shape[0], dtype=np.int32)
        lib().or_hash_insert_many(self.keys.ctypes.data, self.vals.ctypes.data, self.capacity,
                                  self.counter.ctypes.data, self.overflow.ctypes.data, packed.ctypes.data,
                                  packed.shape[0], ranks.ctypes.data, fresh.ctypes.data, int(parallel))
        return ranks, fresh.astype(bool)

    def lookup(self, block):
        return int(lib().or_hash_lookup(self.keys.ctypes.data, self.vals.ctypes.data, self.capacity,
                                        ctypes.c_uint64(pack_key(block))))

    def active_blocks(self):
        blocks = np.empty((self.count, 3), dtype=np.int64)
        lib().or_hash_active_blocks(self.keys.ctypes.data, self.vals.ctypes.data, self.capacity,
                                    blocks.ctypes.data)
        return blocks


def _next_pow2(n):
    p = 1
    while p < n:
        p *= 2
    return p


def build_hash_sparse_grid(positions, h, block_size=4, initial_capacity=None, deterministic=False,
                           max_rebuilds=48):
    """sparse_hash.py:225-264"""
    xp = _f64(positions).reshape(-1, 3)
    if xp.shape[0] == 0:
        raise ValueError("cannot build a grid from an empty particle set")
    if not np.all(np.isfinite(xp)):
        raise ValueError("particle positions must be finite")
    capacity = _next_pow2(max(64, xp.shape[0] // 4)) if initial_capacity is None else int(initial_capacity)
    inv_h = 1.0 / float(h)
    for _ in range(max_rebuilds):
        t = BlockHashTable(capacity)
        err = lib().or_insert_particle_blocks(xp.ctypes.data, xp.shape[0], inv_h, int(block_size),
                                              t.keys.ctypes.data, t.vals.ctypes.data, capacity,
                                              t.counter.ctypes.data, t.overflow.ctypes.data,
                                              0 if deterministic else 1)
        if err:
            raise ValueError("particle stencil block outside packable coordinate range")
        if not t.overflowed and t.count <= capacity // 2:
            return OracleMap(block_size, t.active_blocks(), MODE_HASH, keys=t.keys, vals=t.vals)
        capacity *= 2
    raise RuntimeError("hash table rebuild limit reached")


def stencil_node_bounds(positions, h):
    """sparse_scan.py:32-41"""
    xp = _f64(positions).reshape(-1, 3)
    lo = np.zeros(3, np.int64)
    hi = np.zeros(3, np.int64)
    lib().or_stencil_base_bounds(xp.ctypes.data, xp.shape[0], 1.0 / float(h), lo.ctypes.data, hi.ctypes.data)
    return lo, hi


def build_scan_sparse_grid(positions, h, block_size=4, n_segments=None):
    """sparse_scan.py:44-172 (candidate domain -> mask -> scan -> map)."""
    xp = _f64(positions).reshape(-1, 3)
    node_lo, node_hi = stencil_node_bounds(xp, h)
    b_lo = node_lo // block_size
    b_hi = node_hi // block_size
    pack_key(b_lo)
    pack_key(b_hi)
    b_shape = b_hi - b_lo + 1
    mask = np.zeros(int(np.prod(b_shape)), dtype=np.uint8)
    err = lib().or_mark_blocks(xp.ctypes.data, xp.shape[0], 1.0 / float(h), int(block_size), b_lo.ctypes.data,
                               b_shape.ctypes.data, mask.ctypes.data, 1)
    if err:
        raise ValueError("particle stencil escapes the candidate domain")
    vals = mask.astype(np.int64)
    offsets = np.empty_like(vals)
    lib().or_exclusive_scan(vals.ctypes.data, vals.shape[0], offsets.ctypes.data)
    phi_flat = np.where(mask > 0, offsets, np.int64(-1))
    flat = np.flatnonzero(mask)
    plane = int(b_shape[1] * b_shape[2])
    bi = flat // plane
    rem = flat - bi * plane
    bj = rem // int(b_shape[2])
    bk = rem - bj * int(b_shape[2])
    active = np.stack([bi, bj, bk], axis=1).astype(np.int64) + b_lo
    return OracleMap(block_size, active, MODE_FLAT, bmin=b_lo, bshape=b_shape, phi_flat=phi_flat)


def build_dense_grid(node_min, node_max, block_size=4):
    """grid_index.py:256-277"""
    lo = np.asarray([c // block_size for c in node_min], dtype=np.int64)
    hi = np.asarray([c // block_size for c in node_max], dtype=np.int64)
    bshape = hi - lo + 1
    ri, rj, rk = (np.arange(bshape[a], dtype=np.int64) for a in range(3))
    gi, gj, gk = np.meshgrid(ri, rj, rk, indexing="ij")
    active = np.stack([gi.ravel(), gj.ravel(), gk.ravel()], axis=1) + lo
    phi_flat = np.arange(active.shape[0], dtype=np.int64)
    return OracleMap(block_size, active, MODE_FLAT, bmin=lo, bshape=bshape, phi_flat=phi_flat)


def count_active_nodes(positions, h):
    """solver.py:749-757"""
    xp = _f64(positions).reshape(-1, 3)
    lo, hi = stencil_node_bounds(xp, h)
    shape = hi - lo + 1
    mask = np.zeros(int(np.prod(shape)), dtype=np.uint8)
    lib().or_mark_nodes(xp.ctypes.data, xp.shape[0], 1.0 / float(h), lo.ctypes.data, int(shape[1]),
                        int(shape[2]), mask.ctypes.data, 1)
    return int(np.count_nonzero(mask))


def active_node_set(positions, h):
    """Sorted packed node coordinates of the union of particle stencils."""
    xp = _f64(positions).reshape(-1, 3)
    base = np.floor(xp * (1.0 / float(h)) - 0.5).astype(np.int64)
    offs = np.stack(np.meshgrid(range(3), range(3), range(3), indexing="ij"), -1).reshape(-1, 3)
    nodes = (base[:, None, :] + offs[None, :, :]).reshape(-1, 3)
    return np.unique(pack_keys(nodes))


# ------------------------------------------------------------- physics

def bspline_weights(x, h):
    """solver.py:80-92"""
    base = np.empty(3, dtype=np.int64)
    w = np.empty((3, 3))
    g = np.empty((3, 3))
    xr = _f64(x).reshape(3)
    lib().or_stencil(xr.ctypes.data, 1.0 / float(h), base.ctypes.data, w.ctypes.data, g.ctypes.data)
    return base, w, g / float(h)


class NodalFields:
    """solver.py:152-171"""

    def __init__(self, n_nodes):
        self.mass = np.zeros(n_nodes)
        self.vel = np.zeros((n_nodes, 3))
        self.force = np.zeros((n_nodes, 3))

    @property
    def n_nodes(self):
        return int(self.mass.shape[0])


def _ps(ps, name, shape):
    return np.ascontiguousarray(getattr(ps, name), dtype=np.float64).reshape(shape)


def scatter(particles, index_map, h, gravity, fields=None, deterministic=True, mass_mom=True, forces=True):
    """Fused scatter (solver.py:456-575); p2g (:863-877) / grid_forces
    (:880-894) are the mass_mom-only / forces-only special cases."""
    n = particles.x.shape[0]
    if fields is None:
        fields = NodalFields(index_map.n_nodes)
    g = np.asarray(gravity, dtype=np.float64).reshape(3)
    x = _ps(particles, "x", (n, 3))
    v = _ps(particles, "v", (n, 3))
    C = _ps(particles, "C", (n, 9))
    m = _ps(particles, "m", (n,))
    sig = _ps(particles, "sigma", (n, 9))
    jac = _ps(particles, "jac", (n,))
    V0 = _ps(particles, "V0", (n,))
    err = lib().or_scatter(x.ctypes.data, v.ctypes.data, C.ctypes.data, m.ctypes.data, sig.ctypes.data,
                           jac.ctypes.data, V0.ctypes.data, n, 1.0 / float(h), float(h), g[0], g[1], g[2],
                           index_map.cref, _p(fields.mass) if mass_mom else None,
                           _p(fields.vel) if mass_mom else None, _p(fields.force) if forces else None,
                           0 if deterministic else 1)
    if err:
        raise KeyError("particle stencil node outside active grid")
    return fields


def p2g(particles, index_map, h, deterministic=True, fields=None):
    return scatter(particles, index_map, h, (0.0, 0.0, 0.0), fields, deterministic, True, False)


def grid_forces(particles, index_map, h, gravity, deterministic=True, fields=None):
    return scatter(particles, index_map, h, gravity, fields, deterministic, False, True)


def pack_boundaries(boundaries):
    """solver.py:841-860.  Boundaries are objects with kind/mu/point/normal/
    heightfield(x0, y0, cell, data) attributes (reference-shaped)."""
    boundaries = list(boundaries)
    nb = len(boundaries)
    kind = np.zeros(max(nb, 1), dtype=np.int64)
    point = np.zeros((max(nb, 1), 3))
    normal = np.zeros((max(nb, 1), 3))
    mu = np.zeros(max(nb, 1))
    hf = (np.zeros((2, 2)), 0.0, 0.0, 1.0)
    for b, bc in enumerate(boundaries):
        mu[b] = bc.mu
        if bc.kind == "plane":
            kind[b] = BC_PLANE
            point[b] = bc.point
            normal[b] = bc.normal
        else:
            kind[b] = BC_HEIGHTFIELD
            f = bc.heightfield
            hf = (np.ascontiguousarray(f.data, dtype=np.float64), float(f.x0), float(f.y0), float(f.cell))
    return nb, kind, point, normal, mu, hf


def grid_update(fields, index_map, h, dt, mass_floor=0.0, boundaries=(), parallel=False):
    """solver.py:897-909 / _grid_update :578-625"""
    nb, kind, point, normal, mu, (hd, hx0, hy0, hcell) = pack_boundaries(boundaries)
    ab = np.ascontiguousarray(index_map.active_blocks, dtype=np.int64)
    lib().or_grid_update(fields.mass.ctypes.data, fields.vel.ctypes.data, fields.force.ctypes.data,
                         fields.n_nodes, ab.ctypes.data, index_map.block_size, float(h), float(dt),
                         float(mass_floor), kind.ctypes.data, point.ctypes.data, normal.ctypes.data,
                         mu.ctypes.data, nb, hd.ctypes.data, hd.shape[0], hd.shape[1], hx0, hy0, hcell,
                         int(parallel))
    return fields


def g2p(particles, index_map, fields, h, dt, parallel=False):
    """solver.py:912-924 (in place on particles.x/v/C/F, which must be
    C-contiguous float64)."""
    n = particles.x.shape[0]
    err = lib().or_g2p(particles.x.ctypes.data, particles.v.ctypes.data, particles.C.ctypes.data,
                       particles.F.ctypes.data, np.ascontiguousarray(fields.vel).ctypes.data, n,
                       1.0 / float(h), float(h), float(dt), index_map.cref, int(parallel))
    if err:
        raise KeyError("particle stencil node outside active grid")
    return particles


def material_tables(materials):
    """materials.py:241-247 from reference-shaped MaterialModel objects."""
    mu = np.array([m.lame_mu for m in materials], dtype=np.float64)
    lam = np.array([m.lame_lambda for m in materials], dtype=np.float64)
    alpha = np.array([m.dp_alpha for m in materials], dtype=np.float64)
    kind = np.array([m.kind_id for m in materials], dtype=np.int64)
    return mu, lam, alpha, kind


def stress(particles, mu, lam, alpha, kind, parallel=False):
    """materials.py:169-238; returns (err_flag, particle) and updates F,
    sigma, jac in place."""
    n = particles.x.shape[0]
    err = np.zeros(2, dtype=np.int64)
    mid = np.ascontiguousarray(particles.mat_id, dtype=np.int64)
    lib().or_stress(particles.F.ctypes.data, particles.sigma.ctypes.data, particles.jac.ctypes.data,
                    mid.ctypes.data, n, mu.ctypes.data, lam.ctypes.data, alpha.ctypes.data, kind.ctypes.data,
                    err.ctypes.data, int(parallel))
    return int(err[0]), int(err[1])


def update_stress(particles, materials, parallel=False):
    """materials.py:250-267"""
    e, p = stress(particles, *material_tables(materials), parallel=parallel)
    if e:
        raise RuntimeError(f"deformation gradient of particle {p} is degenerate")
    return particles


class OracleParticles:
    """Plain SoA particle state (solver.py:95-149 layout, float64)."""

    FIELDS = ("x", "v", "C", "F", "m", "V0", "mat_id", "sigma", "jac")

    def __init__(self, copy=True, **kw):
        for k in self.FIELDS:
            a = kw[k]
            dt = np.int64 if k == "mat_id" else np.float64
            setattr(self, k, np.array(a, dtype=dt, copy=True, order="C") if copy else
                    np.ascontiguousarray(a, dtype=dt))

    @classmethod
    def from_any(cls, ps, copy=True):
        return cls(copy=copy, **{k: getattr(ps, k) for k in cls.FIELDS})

    @property
    def n(self):
        return int(self.x.shape[0])

    def copy(self):
        return OracleParticles.from_any(self)


class OracleSimulation:
    """Mirror of Simulation.step (solver.py:1001-1093) on the CPU, with the
    reference's per-phase timers.  ``backend`` is dense/scan/hash; used as
    the parity oracle (deterministic=True) and as the CPU baseline
    (deterministic=False, multithreaded)."""

    def __init__(self, particles, h, gravity, materials, boundaries=(), backend="scan", deterministic=False,
                 threads=None, cfl=0.4, block_size=4, node_min=None, node_max=None, adopt=False):
        # adopt=True: use the caller's arrays in place (large CPU-baseline runs)
        self.particles = OracleParticles.from_any(particles, copy=not adopt)
        self.h = float(h)
        self.gravity = np.asarray(gravity, dtype=np.float64).reshape(3)
        self.materials = list(materials)
        self.boundaries = list(boundaries)
        self.backend = backend
        self.deterministic = deterministic
        self.cfl = cfl
        self.block_size = block_size
        self.tables = material_tables(self.materials)
        self.wave_speed = max(m.wave_speed for m in self.materials)
        self.mass_floor = MASS_FLOOR_SCALE * float(self.particles.m.max())
        self.threads = threads or len(os.sched_getaffinity(0))
        set_threads(self.threads)
        self.dense_map = None
        if backend == "dense":
            self.dense_map = build_dense_grid(node_min, node_max, block_size)
        self.t = 0.0
        self.step_count = 0
        self.last_fields = None
        self.last_map = None

    def dt_bound(self):
        """solver.py:984-987"""
        v = self.particles.v
        vmax = float(np.sqrt((v ** 2).sum(axis=1).max()))
        return self.cfl * self.h / (self.wave_speed + vmax)

    def build_map(self):
        """solver.py:989-999"""
        if self.backend == "dense":
            return self.dense_map
        if self.backend == "scan":
            return build_scan_sparse_grid(self.particles.x, self.h, self.block_size)
        return build_hash_sparse_grid(self.particles.x, self.h, self.block_size, deterministic=self.deterministic)

    def step(self, dt=None, count_nodes=True):
        ps = self.particles
        par = not self.deterministic
        times = {}
        t0 = time.perf_counter()
        e, p = stress(ps, *self.tables, parallel=par)
        if e:
            raise RuntimeError(f"deformation gradient of particle {p} is degenerate")
        bound = self.dt_bound()
        dt = bound if dt is None else float(dt)
        if dt > bound * (1.0 + 1e-9):
            raise RuntimeError(f"timestep {dt:g} exceeds the stability bound {bound:g}")
        times["stress"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        imap = self.build_map()
        times["map_build"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        fields = NodalFields(imap.n_nodes)
        times["alloc_zero"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        scatter(ps, imap, self.h, self.gravity, fields, deterministic=self.deterministic)
        times["p2g"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        n_active = count_active_nodes(ps.x, self.h) if count_nodes else -1
        times["metrics"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        grid_update(fields, imap, self.h, dt, self.mass_floor, self.boundaries, parallel=par)
        times["grid_update"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        g2p(ps, imap, fields, self.h, dt, parallel=par)
        times["g2p"] = time.perf_counter() - t0
        self.t += dt
        self.step_count += 1
        self.last_fields = fields
        self.last_map = imap
        return {"step": self.step_count, "t": self.t, "dt": dt, "n_active": n_active,
                "n_allocated": imap.n_nodes, "times": times}


COMPUTE_PHASES = ("map_build", "alloc_zero", "p2g", "grid_update", "g2p", "stress")  # solver.py:835

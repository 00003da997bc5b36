"""The reference's own transfer tests, run on the GPU path.

* Acceptance criterion 8, kinematic identities (/root/reference/pkg/tests/
  test_acceptance.py:316-394): inertia D = (h^2/4) I at 10^4 positions, the
  linear-field G2P C = A over 10^4 particles, B-spline gradients vs finite
  differences.
* P2G / force properties (/root/reference/pkg/tests/test_solver.py:104-175):
  mass and momentum conservation, the affine term adds no net momentum, the
  centre node of an on-node particle gets 0.75^3 m, gravity totals, internal
  forces sum to zero.
* dt_bound against the oracle, last_map / last_fields (solver.py:1087-1090),
  the module API on the reference's non-hash maps (scan / dense / flat
  kernel_args, grid_index.py:179-248) and the host-view semantics.

The reference asserts these at fp64 round-off (1e-10 .. 1e-15).  The GPU
computes weights, transfers and grid sums in fp32 (positions and base
indices in fp64), so each tolerance below is the fp32 analogue, stated with
its reason: a few fp32 ulps (eps = 6e-8) of the quantity's natural scale.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2605_28525_b200 import _lib, grid_index as gi  # noqa: E402
from paper_2605_28525_b200 import scenes  # noqa: E402
from paper_2605_28525_b200.errors import SimulationError  # noqa: E402
from paper_2605_28525_b200.solver import (NodalFields, ParticleSet, g2p, grid_forces, p2g,  # noqa: E402
                                          Simulation)
from paper_2605_28525_b200.sparse_hash import build_hash_sparse_grid  # noqa: E402
from tests.test_gpu_module import keyed  # noqa: E402

OFFSETS = np.indices((3, 3, 3)).reshape(3, -1).T


def bspline_many(x, h):
    """smpm_bspline over many points of one h: base (n,3), w, dw (n,3,3)."""
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
    n = x.shape[0]
    torch = _lib.torch_cuda()
    xd = _lib.to_dev(x, np.float64)
    base = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    w = torch.empty(9 * n, dtype=torch.float64, device="cuda")
    dw = torch.empty(9 * n, dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().smpm_bspline(_lib.ptr(xd), n, float(h), _lib.ptr(base), _lib.ptr(w), _lib.ptr(dw),
                                        _lib.stream_ptr()), "bspline")
    return (base.cpu().numpy().reshape(n, 3), w.cpu().numpy().reshape(n, 3, 3), dw.cpu().numpy().reshape(n, 3, 3))


def random_particles(rng, n, lo=0.1, hi=0.9, density=1300.0):
    """T/test_solver.py:95-100"""
    x = rng.uniform(lo, hi, size=(n, 3))
    ps = ParticleSet.from_samples(x, np.full(n, 1e-6), density, 0)
    ps.v[:] = rng.normal(0.0, 2.0, size=(n, 3))
    return ps


# ------------------------------------------------------------ criterion 8

def test_criterion8_inertia_identity():
    """sum_n w_n dx dx^T = (h^2/4) I (T/test_acceptance.py:317-330).  fp32
    weights: |D - (h^2/4) I| <= 1e-6 h^2 (the reference's 1e-12 absolute is
    fp64 round-off)."""
    rng = np.random.default_rng(13)
    worst = 0.0
    for h in (0.045, 0.23, 1.0, 2.4):
        x = rng.uniform(-8.0, 8.0, size=(2500, 3))
        base, w, _ = bspline_many(x, h)
        wijk = w[:, 0, OFFSETS[:, 0]] * w[:, 1, OFFSETS[:, 1]] * w[:, 2, OFFSETS[:, 2]]  # (n, 27)
        dx = (base[:, None, :] + OFFSETS[None]) * h - x[:, None, :]
        d = np.einsum("pn,pni,pnj->pij", wijk, dx, dx)
        worst = max(worst, float(np.abs(d - (h * h / 4.0) * np.eye(3)).max() / (h * h)))
    print(f"criterion 8 inertia: max |D - h^2/4 I| / h^2 = {worst:.2e} over 10000 positions")
    assert worst < 1e-6


def test_criterion8_affine_field():
    """G2P of the linear field v_n = A x_n gives C = A (T/test_acceptance.py:
    332-345) for 10^4 particles, through the module g2p on the reference's
    scan map.  fp32 grid velocities and gathers: C = (4/h^2) sum w v_n dx
    cancels the offset A x_p (|v_n| ~ |A| x ~ 16 |A| h here), so fp32
    rounding of v_n is amplified by x / h: |C - A| <= 8 eps (x/h) |A| ~ 1e-5."""
    from oracle import oracle as o

    rng = np.random.default_rng(14)
    h = 0.05
    n = 10_000
    ps = ParticleSet.from_samples(rng.uniform(0.2, 0.8, size=(n, 3)), np.full(n, 1e-6), 1000.0, 0)
    amap = o.build_scan_sparse_grid(ps.x, h, 4)  # the reference's CPU map, adopted by the GPU path
    a = np.array([[0.3, -1.2, 0.5], [0.8, 0.1, -0.4], [-0.6, 0.9, 0.2]])
    fields = NodalFields.zeros(amap.n_nodes)
    fields.vel[:] = amap.node_coords() * h @ a.T
    g2p(ps, amap, fields, h, dt=0.0)
    err = float(np.abs(ps.C - a[None]).max())
    print(f"criterion 8 affine: max |C - A| = {err:.2e} over {n} particles")
    assert err < 8 * 6e-8 * (0.8 / h) * np.abs(a).max()


def test_criterion8_gradients_vs_finite_differences():
    """dw vs central differences of w (T/test_acceptance.py:347-394).  The
    weights are quadratic within a cell, so a central difference is exact
    there at any step; with fp32 weights the step is 1e-2 h (the reference's
    1e-6 h would leave only rounding), tolerance 1e-5 relative."""
    rng = np.random.default_rng(15)
    worst, checked = 0.0, 0
    for _ in range(10):
        h = float(rng.uniform(0.03, 2.5))
        x = rng.uniform(-4.0, 4.0, size=(50, 3))
        delta = 1e-2 * h
        base, w, dw = bspline_many(x, h)
        grad = np.stack([dw[:, 0, OFFSETS[:, 0]] * w[:, 1, OFFSETS[:, 1]] * w[:, 2, OFFSETS[:, 2]],
                         w[:, 0, OFFSETS[:, 0]] * dw[:, 1, OFFSETS[:, 1]] * w[:, 2, OFFSETS[:, 2]],
                         w[:, 0, OFFSETS[:, 0]] * w[:, 1, OFFSETS[:, 1]] * dw[:, 2, OFFSETS[:, 2]]], axis=1)
        for axis in range(3):
            xp, xm = x.copy(), x.copy()
            xp[:, axis] += delta
            xm[:, axis] -= delta
            bp, wp, _ = bspline_many(xp, h)
            bm, wm, _ = bspline_many(xm, h)
            same = (bp[:, axis] == base[:, axis]) & (bm[:, axis] == base[:, axis])
            wpf = wp[:, 0, OFFSETS[:, 0]] * wp[:, 1, OFFSETS[:, 1]] * wp[:, 2, OFFSETS[:, 2]]
            wmf = wm[:, 0, OFFSETS[:, 0]] * wm[:, 1, OFFSETS[:, 1]] * wm[:, 2, OFFSETS[:, 2]]
            fd = (wpf - wmf) / (2.0 * delta)
            denom = np.maximum(np.abs(fd), 1.0 / h)
            rel = np.abs(grad[:, axis] - fd) / denom
            if same.any():
                worst = max(worst, float(rel[same].max()))
                checked += int(same.sum())
    print(f"criterion 8 gradient: max rel err {worst:.2e} over {checked} probes")
    assert checked > 1000 and worst < 1e-5


# ------------------------------------------------------ P2G properties

def _scan_map(ps, h):
    from oracle import oracle as o

    return o.build_scan_sparse_grid(ps.x, h, 4)


def test_p2g_mass_and_momentum_conserved():
    """T/test_solver.py:104-114 (fp32 sums: 1e-6 relative)."""
    rng = np.random.default_rng(60)
    ps = random_particles(rng, 400)
    h = 0.05
    f = p2g(ps, _scan_map(ps, h), h)
    assert abs(f.mass.sum() - ps.m.sum()) < 1e-6 * ps.m.sum()
    mom_p = (ps.m[:, None] * ps.v).sum(axis=0)
    assert np.abs(f.vel.sum(axis=0) - mom_p).max() < 1e-6 * np.abs(ps.m[:, None] * ps.v).sum(axis=0).max()


def test_p2g_affine_term_adds_no_net_momentum():
    """sum_n w_n (x_n - x_p) = 0 (T/test_solver.py:116-127)."""
    rng = np.random.default_rng(61)
    ps = random_particles(rng, 200)
    ps.C[:] = rng.normal(0.0, 5.0, size=(ps.n, 3, 3))
    h = 0.05
    f = p2g(ps, _scan_map(ps, h), h)
    mom_p = (ps.m[:, None] * ps.v).sum(axis=0)
    scale = max(np.abs(ps.m[:, None] * ps.v).sum(axis=0).max(), 1e-30)
    assert np.abs(f.vel.sum(axis=0) - mom_p).max() < 1e-6 * scale


def test_p2g_single_particle_on_node():
    """Centre node mass 0.75^3 m (T/test_solver.py:129-137), to one fp32 ulp."""
    ps = ParticleSet.from_samples(np.array([[0.2, 0.2, 0.2]]), np.array([1e-6]), 1000.0, 0, velocity=(1.0, 0.0, 0.0))
    h = 0.1
    amap = _scan_map(ps, h)
    f = p2g(ps, amap, h)
    centre = amap.node_index((2, 2, 2))
    assert abs(f.mass[centre] - 0.75 ** 3 * ps.m[0]) <= 1.2e-7 * ps.m[0]


def test_grid_forces_gravity_totals():
    """T/test_solver.py:151-160"""
    rng = np.random.default_rng(63)
    ps = random_particles(rng, 150)
    h = 0.05
    g = (0.0, 0.0, -9.81)
    f = grid_forces(ps, _scan_map(ps, h), h, g)
    expected = ps.m.sum() * np.asarray(g)
    assert np.abs(f.force.sum(axis=0) - expected).max() < 1e-6 * np.abs(expected).max()


def test_grid_stress_forces_sum_to_zero():
    """sum_n grad w_n = 0 per particle (T/test_solver.py:162-175)."""
    rng = np.random.default_rng(64)
    ps = random_particles(rng, 150)
    s = rng.normal(0.0, 1e4, size=(ps.n, 3, 3))
    ps.sigma[:] = s + np.transpose(s, (0, 2, 1))
    h = 0.05
    f = grid_forces(ps, _scan_map(ps, h), h, (0.0, 0.0, 0.0))
    total = np.abs(f.force.sum(axis=0)).max()
    scale = np.abs(f.force).max()
    assert total < 1e-5 * max(scale, 1.0), (total, scale)


@pytest.mark.parametrize("form", ["scan_object", "dense_object", "flat_kernel_args", "hash_kernel_args"])
def test_module_api_accepts_reference_maps(oracle, form):
    """p2g on the reference's other map forms equals p2g on the GPU hash map
    (same per-node sums, keyed by node)."""
    rng = np.random.default_rng(7)
    ps = random_particles(rng, 300)
    h = 0.05
    ours = build_hash_sparse_grid(ps.x, h, 4)
    if form == "scan_object":
        m = s = oracle.build_scan_sparse_grid(ps.x, h, 4)
    elif form == "dense_object":
        m = s = oracle.build_dense_grid((0, 0, 0), (20, 20, 20), 4)
    elif form == "flat_kernel_args":
        s = oracle.build_scan_sparse_grid(ps.x, h, 4)
        m = (np.int64(0), *[np.int64(v) for v in s.bmin], *[np.int64(v) for v in s.bshape], s.phi_flat,
             np.zeros(0, np.uint64), np.zeros(0, np.int64), np.int64(4))
    else:
        s = oracle.build_hash_sparse_grid(ps.x, h, 4, deterministic=True)
        m = (np.int64(1), *[np.int64(0)] * 6, np.zeros(0, np.int64), s.keys, s.vals, np.int64(4))
    amap = gi.as_index_map(m)
    assert np.array_equal(amap.active_blocks, s.active_blocks)  # same blocks, same ranks
    fa = p2g(ps, m, h)
    fb = p2g(ps, ours, h)
    ka, ma = keyed(amap.active_blocks, fa.mass, 1)
    kb, mb = keyed(ours.active_blocks, fb.mass, 1)
    _, pa = keyed(amap.active_blocks, fa.vel, 3)
    _, pb = keyed(ours.active_blocks, fb.vel, 3)
    sel = np.isin(ka, kb)
    assert np.all(ma[~sel] == 0.0)  # dense map: extra blocks stay empty
    np.testing.assert_allclose(ma[sel], mb, rtol=0, atol=1e-6 * mb.max())
    np.testing.assert_allclose(pa[sel], pb, rtol=0, atol=1e-6 * np.abs(pb).max())


def test_flat_map_ranks_follow_the_reference_order(oracle):
    """ActiveIndexMap.from_blocks keeps the given rank order (row-major for
    scan, grid_index.py:256-277 for dense)."""
    rng = np.random.default_rng(8)
    x = rng.uniform(0.0, 2.0, size=(500, 3))
    s = oracle.build_scan_sparse_grid(x, 0.05, 4)
    amap = gi.as_index_map(s)
    assert np.array_equal(amap.active_blocks, s.active_blocks)
    for b in s.active_blocks[::17]:
        assert amap.block_index(b) == s.node_index(b * 4) // 64


# -------------------------------------------------------- Simulation API

def test_dt_bound_matches_oracle(oracle):
    """solver.py:984-987 on the same state (fp32-representable velocities:
    the GPU stores v in fp32); |v|^2 in fp32 on the device -> 1e-6 relative."""
    sc = scenes.granular_column(h=0.05)
    sim = sc.simulation()
    for _ in range(30):
        sim.step()
    o = oracle.OracleSimulation(sim.particles, sc.config.h, sc.config.gravity, sc.materials, sc.boundaries)
    a, b = sim.dt_bound(), o.dt_bound()
    assert abs(a - b) <= 1e-6 * b, (a, b)


def test_last_map_and_fields(oracle):
    """Simulation.last_map / last_fields (solver.py:963-964, 1087-1090): None
    before the first step; after a step the grid of that step -- allocation,
    node mass, boundary-projected grid velocity and the retained force."""
    sc = scenes.granular_column(h=0.05)
    sim = Simulation(sc.particles, sc.config, sc.materials, sc.boundaries, retain_fields=True)
    assert sim.last_map is None and sim.last_fields is None
    state = sim.particles.copy()
    dt = 0.9 * sim.dt_bound()
    st = sim.step(dt)
    amap, f = sim.last_map, sim.last_fields
    assert amap.n_nodes == st.n_allocated
    o = oracle.OracleSimulation(state, sc.config.h, sc.config.gravity, sc.materials, sc.boundaries, backend="hash",
                                deterministic=True)
    o.step(dt)
    assert np.array_equal(np.sort(gi.pack_keys(amap.active_blocks)), np.sort(gi.pack_keys(o.last_map.active_blocks)))
    kg, mg = keyed(amap.active_blocks, f.mass, 1)
    kr, mr = keyed(o.last_map.active_blocks, o.last_fields.mass, 1)
    assert np.array_equal(kg, kr)
    assert np.abs(mg - mr).max() <= 1e-5 * mr.max()
    _, fg = keyed(amap.active_blocks, f.force, 3)
    _, fr = keyed(o.last_map.active_blocks, o.last_fields.force, 3)
    assert np.abs(fg - fr).max() <= 1e-4 * np.abs(fr).max()
    assert abs(f.force[:, 2].sum() - sc.particles.m.sum() * sc.config.gravity[2]) < 1e-4 * abs(
        sc.particles.m.sum() * sc.config.gravity[2])
    # without retain_fields the force is not kept
    sim2 = sc.simulation()
    sim2.step()
    assert sim2.last_fields.force is None and sim2.last_fields.mass.shape[0] == sim2.last_map.n_nodes


def test_host_view_mirrors_like_the_reference():
    """host_sync='mirror' (default for small sets): the caller's arrays are
    the state, as in the reference -- an edit made after a later step, on an
    object obtained earlier, is taken by the next step."""
    sc = scenes.granular_column(h=0.1)
    ps = sc.particles
    sim = sc.simulation()
    sim.step(1e-4)
    keep = sim.particles  # same object as ps
    assert keep is ps
    sim.step(1e-4)
    np.testing.assert_array_equal(keep.x, sim.particles.x)  # updated in place by the step
    keep.v[:, 0] += 1.0
    sim.step(1e-4)
    assert sim.particles.v[:, 0].mean() > 0.9


def test_host_view_on_access_takes_edits_of_a_fresh_view():
    """host_sync='on_access': a view read after the last step is the state;
    edits to it are uploaded by the next step (one fingerprint per view)."""
    sc = scenes.granular_column(h=0.1)
    sim = Simulation(sc.particles, sc.config, sc.materials, sc.boundaries, host_sync="on_access")
    sim.step(1e-4)
    view = sim.particles
    view.v[:, 0] += 2.0
    sim.step(1e-4)
    assert sim.particles.v[:, 0].mean() > 1.9


def test_explicit_negative_dt_rejected():
    sc = scenes.granular_column(h=0.1)
    sim = sc.simulation()
    for dt in (-1.0, -2.0, 0.0):
        with pytest.raises(SimulationError, match="timestep must be positive"):
            sim.step(dt)
    sim.step()

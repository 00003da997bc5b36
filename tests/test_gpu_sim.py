"""Simulation.step (fused GPU pipeline) vs the oracle, step by step.

Each step starts both sides from the same state (the GPU state is fed to
the oracle), so tolerances are per step: active block set, n_blocks and
n_active bit-exact; grid mass/momentum and particle x/v norm-wise fp32
tolerances; C/F/force looser."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2605_28525_b200 import grid_index as gi  # noqa: E402
from paper_2605_28525_b200 import scenes  # noqa: E402
from paper_2605_28525_b200.errors import SimulationError  # noqa: E402
from paper_2605_28525_b200.materials import MaterialModel  # noqa: E402
from paper_2605_28525_b200.solver import BoundaryCondition, SimConfig, Simulation  # noqa: E402
from tests.test_gpu_module import keyed, normwise  # noqa: E402
from tests.test_oracle_golden import _boundaries  # noqa: E402

TOL = dict(x=1e-6, v=1e-5, C=1e-4, F=2e-5, mass=1e-5, mom=1e-5, force=1e-4)


def column_scene(h=0.05, size=(0.4, 0.3, 0.5), seed=3, vx=0.4, bcs="mixed", mat=None, prestrain=0.0, ppc=2):
    pos, vol = scenes.sample_box((-size[0] / 2, -size[1] / 2, 0.03), (size[0] / 2, size[1] / 2, size[2]), h, ppc)
    rng = np.random.default_rng(seed)
    pos = pos + rng.uniform(-0.2, 0.2, pos.shape) * h / 2
    mat = mat or scenes.SAND
    ps = scenes.rest_particles(pos, vol, mat.density, velocity=(vx, 0.0, 0.0))
    if prestrain:
        # F = Q diag(s) R^T with principal stretches s in [1 - prestrain, 1 + prestrain]:
        # elastic strains past the small-strain series range (||B - I|| > 0.05)
        n = ps.x.shape[0]
        q1, _ = np.linalg.qr(rng.normal(size=(n, 3, 3)))
        q2, _ = np.linalg.qr(rng.normal(size=(n, 3, 3)))
        q2[:, :, 0] *= np.sign(np.linalg.det(q1) * np.linalg.det(q2))[:, None]  # det F > 0
        st = rng.uniform(1.0 - prestrain, 1.0 + prestrain, (n, 3))
        ps.F = np.ascontiguousarray(q1 * st[:, None, :] @ np.transpose(q2, (0, 2, 1)))
    cfg = SimConfig(h=h, gravity=np.array([0.5, 0.0, -9.81]), total_time=1.0, domain_min=np.array([-1.0, -1.0, -0.2]),
                    domain_max=np.array([1.0, 1.0, 1.0]))
    b = _boundaries() if bcs == "mixed" else []
    return ps, cfg, [mat], b


def oracle_step(oracle, state, cfg, mats, bcs, dt):
    o = oracle.OracleSimulation(state, cfg.h, cfg.gravity, mats, bcs, backend="hash", deterministic=True)
    st = o.step(dt)
    return o, st


def oracle_grid(oracle, state, cfg, mats):
    """P2G of the next step as the reference computes it: stress (with the
    return map) of the state, then the scatter."""
    s = oracle.OracleParticles.from_any(state)
    oracle.update_stress(s, mats)
    amap = oracle.build_hash_sparse_grid(s.x, cfg.h, 4, deterministic=True)
    f = oracle.p2g(s, amap, cfg.h)
    oracle.grid_forces(s, amap, cfg.h, cfg.gravity, fields=f)
    return amap, f


def compare_grid(oracle, sim, cfg, mats, ref_state):
    """GPU grid after P2G vs the oracle's P2G of ``ref_state``.  The fused
    step evaluates stress from the return-mapped strains in registers, like
    the reference (materials.py:215-238); ``ref_state`` must therefore be the
    oracle's own unprojected post-step state, not the GPU's stored F."""
    blocks, f = sim.query_grid()
    amap, fr = oracle_grid(oracle, ref_state, cfg, mats)
    # bit-exact active block set
    assert np.array_equal(np.sort(gi.pack_keys(blocks)), np.sort(gi.pack_keys(amap.active_blocks)))
    kg, mg = keyed(blocks, f.mass, 1)
    kr, mr = keyed(amap.active_blocks, fr.mass, 1)
    assert np.array_equal(kg, kr)
    _, pg = keyed(blocks, f.vel, 3)
    _, pr = keyed(amap.active_blocks, fr.vel, 3)
    _, fg = keyed(blocks, f.force, 3)
    _, frr = keyed(amap.active_blocks, fr.force, 3)
    return dict(mass=normwise(mg, mr), mom=normwise(pg, pr), force=normwise(fg, frr))


ELASTIC = MaterialModel(kind="elastic", density=1000.0, youngs_modulus=1e6, poisson_ratio=0.3)


@pytest.mark.parametrize("bcs,det,layout,prestrain,ppc", [
    ("mixed", False, "auto", 0.0, 2), ("none", False, "auto", 0.0, 2), ("mixed", True, "auto", 0.0, 2),
    # wide work-item layout (block ranges) and the moderate-strain constitutive
    # path it carries; prestrained elastic particles exercise that path
    ("mixed", False, "wide", 0.0, 2), ("mixed", False, "wide", 0.3, 2), ("mixed", False, "wide", 0.55, 2),
    ("mixed", False, "narrow", 0.3, 2), ("mixed", True, "narrow", 0.3, 2),
    # 27 particles per cell: several narrow items per block; wide level
    # tables past their 16 levels (tail placement)
    ("mixed", False, "narrow", 0.0, 3), ("mixed", False, "wide", 0.0, 3)])
def test_steps_match_oracle(oracle, monkeypatch, bcs, det, layout, prestrain, ppc):
    if layout != "auto":
        monkeypatch.setenv("SMPM_ITEM_LAYOUT", layout)
    ps, cfg, mats, bc = column_scene(bcs=bcs, prestrain=prestrain, mat=ELASTIC if prestrain else None, ppc=ppc)
    cfg.deterministic = det  # deterministic mode: int64 fixed-point grid sums
    sim = Simulation(ps, cfg, mats, bc)
    worst = {}
    for s in range(8):
        state = sim.particles.copy()
        dt = 0.9 * sim.dt_bound()
        st = sim.step(dt)
        o, ost = oracle_step(oracle, state, cfg, mats, bc, dt)
        assert st.n_active == ost["n_active"], s
        assert st.n_allocated == ost["n_allocated"], s
        gerr = compare_grid(oracle, sim, cfg, mats, o.particles)  # next step's P2G
        after = sim.particles
        oracle.update_stress(o.particles, mats)  # GPU F is return-mapped at step end
        # C is a velocity gradient: scale it by max(|C_ref|, v_max / h) so a
        # uniformly translating body (C_ref ~ 0) is judged on its natural scale
        vscale = max(np.abs(o.particles.v).max(), 1e-12)
        cscale = max(np.abs(o.particles.C).max(), vscale / cfg.h)
        errs = dict(x=float(np.abs(after.x - o.particles.x).max() / np.abs(o.particles.x).max()),
                    v=normwise(after.v, o.particles.v), C=float(np.abs(after.C - o.particles.C).max() / cscale),
                    F=normwise(after.F, o.particles.F), **gerr)
        for k, e in errs.items():
            worst[k] = max(worst.get(k, 0.0), e)
    print("worst per-step errors:", {k: f"{v:.2e}" for k, v in worst.items()})
    for k, e in worst.items():
        assert e <= TOL[k], (k, e)


def test_deterministic_mode_is_bitwise_reproducible():
    """deterministic=True: node sums are int64 fixed point (order-independent),
    so two runs agree bit for bit whatever the hash ranks and atomic order."""
    ps, cfg, mats, bc = column_scene(vx=3.0)
    cfg.deterministic = True
    runs = []
    for _ in range(2):
        sim = Simulation(ps.copy(), cfg, mats, bc, block_capacity=64)  # growth + replay on the way
        for s in range(12):
            sim.step(2e-4)
        p = sim.particles
        runs.append((p.x.copy(), p.v.copy(), p.C.copy(), p.F.copy()))
    for a, b in zip(*runs):
        assert np.array_equal(a, b)
    ref = Simulation(ps.copy(), SimConfig(**{**cfg.__dict__, "deterministic": False}), mats, bc)
    for s in range(12):
        ref.step(2e-4)
    assert np.abs(ref.particles.x - runs[0][0]).max() < 1e-6 * np.abs(runs[0][0]).max()


@pytest.mark.parametrize("mat", ["sand", "elastic"])
def test_item_layouts_are_bitwise_identical_in_deterministic_mode(monkeypatch, mat):
    """The narrow (cell-slot) and wide (block-range) work-item layouts group
    particles differently; in deterministic mode grid sums are int64 and the
    constitutive path is the same, so the states agree bit for bit."""
    ps, cfg, mats, bc = column_scene(vx=3.0, prestrain=0.25 if mat == "elastic" else 0.0,
                                     mat=ELASTIC if mat == "elastic" else None)
    cfg.deterministic = True
    runs = []
    for layout in ("narrow", "wide"):
        monkeypatch.setenv("SMPM_ITEM_LAYOUT", layout)
        sim = Simulation(ps.copy(), cfg, mats, bc)
        for s in range(10):
            sim.step(1e-4)
        p = sim.particles
        runs.append((p.x.copy(), p.v.copy(), p.C.copy(), p.F.copy()))
    for a, b in zip(*runs):
        assert np.array_equal(a, b)


def _layout(sim):
    import ctypes
    from paper_2605_28525_b200 import _lib
    out = (ctypes.c_int64 * 24)()
    _lib.check(_lib.load().smpm_sim_debug_stats(sim._h, out), "debug stats")
    return int(out[21])


def test_layout_switch_mid_run_keeps_deterministic_results(monkeypatch):
    """The host switches the work-item layout between steps once particles
    disorder; in deterministic mode the run with switches is bit-identical to
    a run pinned to the narrow layout."""
    ps, cfg, mats, bc = column_scene(vx=3.0, size=(0.6, 0.4, 0.6))
    cfg.deterministic = True
    monkeypatch.delenv("SMPM_ITEM_LAYOUT", raising=False)
    auto = Simulation(ps.copy(), cfg, mats, bc)
    monkeypatch.setenv("SMPM_ITEM_LAYOUT", "narrow")
    pinned = Simulation(ps.copy(), cfg, mats, bc)
    layouts = []
    for s in range(40):
        auto.step(2e-4)
        pinned.step(2e-4)
        layouts.append(_layout(auto))
    assert 1 in layouts, layouts  # the switch happened
    a, b = auto.particles, pinned.particles
    for k in ("x", "v", "C", "F"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_capacity_growth_replays_exactly(oracle):
    ps, cfg, mats, bc = column_scene()
    a = Simulation(ps.copy(), cfg, mats, bc)
    b = Simulation(ps.copy(), cfg, mats, bc, block_capacity=8)
    for _ in range(3):
        sa = a.step(1e-4)
        sb = b.step(1e-4)
        assert sa.n_active == sb.n_active and sa.n_allocated == sb.n_allocated
    assert np.abs(a.particles.x - b.particles.x).max() < 1e-9


def test_free_fall_is_exact():
    mat = MaterialModel(kind="elastic", density=1000.0, youngs_modulus=1e4, poisson_ratio=0.2)
    ps, cfg, mats, bc = column_scene(bcs="none", mat=mat, vx=0.0)
    cfg.gravity = np.array([0.0, 0.0, -9.81])
    sim = Simulation(ps, cfg, mats, [])
    z0 = ps.x[:, 2].copy()
    dt = 1e-3
    for _ in range(20):
        sim.step(dt)
    t = 20 * dt
    # symplectic Euler: z = z0 - g dt^2 n(n+1)/2
    z_exact = z0 - 9.81 * dt * dt * 20 * 21 / 2
    assert np.abs(sim.particles.x[:, 2] - z_exact).max() < 1e-6
    assert np.abs(sim.particles.v[:, 2] + 9.81 * t).max() < 1e-4
    assert np.abs(sim.particles.F - np.eye(3)).max() < 1e-5


def test_rest_state_stays_fixed():
    mat = MaterialModel(kind="elastic", density=1000.0, youngs_modulus=1e4, poisson_ratio=0.2)
    ps, cfg, mats, bc = column_scene(bcs="none", mat=mat, vx=0.0)
    cfg.gravity = np.zeros(3)
    pts = ps.x.copy()
    sim = Simulation(ps, cfg, mats, [])
    for _ in range(5):
        sim.step(1e-3)
    assert np.abs(sim.particles.v).max() == 0.0
    assert np.abs(sim.particles.x - pts).max() == 0.0


def test_step_stats_and_conservation():
    ps, cfg, mats, bc = column_scene(bcs="none")
    sim = Simulation(ps, cfg, mats, [], record_conservation=True)
    st = sim.step(1e-4)
    assert st.n_active > 0 and st.n_allocated >= st.n_active and st.n_allocated % 64 == 0
    assert abs(st.mass_sum - ps.m.sum()) < 1e-5 * ps.m.sum()
    mom = (sim.particles.m[:, None] * 0).sum(axis=0)
    del mom
    for phase in ("map_build", "alloc_zero", "p2g", "grid_update", "g2p", "stress"):
        assert phase in st.times


def test_degenerate_particle_raises_with_index():
    ps, cfg, mats, bc = column_scene(bcs="none")
    sim = Simulation(ps, cfg, mats, [])
    sim.step(1e-4)
    sim.particles.F[3] = 0.0
    with pytest.raises(SimulationError, match="particle 3"):
        sim.step(1e-4)


def test_dt_above_bound_raises():
    ps, cfg, mats, bc = column_scene(bcs="none")
    sim = Simulation(ps, cfg, mats, [])
    with pytest.raises(SimulationError):
        sim.step(10.0 * sim.dt_bound())
    sim.step(0.5 * sim.dt_bound())  # the rejected step left no trace


def test_oversized_fixed_timestep_rejected():
    """SimConfig.dt above the stability bound is a ConfigError at construction
    (solver.py:966-969, T/test_solver.py:373-375)."""
    from paper_2605_28525_b200.errors import ConfigError
    ps, cfg, mats, bc = column_scene(bcs="none")
    cfg.dt = 1.0
    with pytest.raises(ConfigError, match="stability bound"):
        Simulation(ps, cfg, mats, [])


def test_nonfinite_position_raises():
    ps, cfg, mats, bc = column_scene(bcs="none")
    ps.x[5, 1] = np.nan
    with pytest.raises(SimulationError):
        sim = Simulation(ps, cfg, mats, [])
        sim.step(1e-4)


def test_heightfield_slide_steps():
    sc = scenes.landslide(x_stride=100, h=2.0, depth=(0.5, 10.0))
    sim = sc.simulation()
    n0 = sim.step().n_active
    for _ in range(5):
        st = sim.step()
    assert st.n_active > 0 and n0 > 0
    assert np.isfinite(sim.particles.x).all()


def test_large_upload_validates_material_ids():
    """Sets of >= 2^20 particles are validated inside the threaded upload
    (material-id range, max mass for the mass floor) instead of numpy."""
    from paper_2605_28525_b200.errors import ConfigError

    pos, vol = scenes.sample_box((0, 0, 0), (1.3, 1.3, 0.65), 0.02, 2)
    assert len(pos) >= 1 << 20
    ps = scenes.rest_particles(pos, vol, 1500.0)
    cfg = SimConfig(h=0.02, gravity=np.array([0.0, 0.0, -9.81]), total_time=1.0, domain_min=np.array([-1.0, -1, -1]),
                    domain_max=np.array([2.0, 2.0, 2.0]))
    sim = Simulation(ps, cfg, [scenes.SAND], [])
    sim.step(1e-4)
    ps.mat_id[12345] = 3
    with pytest.raises(ConfigError, match="material id out of range"):
        Simulation(ps, cfg, [scenes.SAND], [])


def test_device_memory_cache_reuse_and_release():
    """Buffers of a destroyed simulation are reused by the next one of the
    same configuration (include/smpm.h: smpm_release_cached_memory); results
    do not depend on whether the memory came from the cache."""
    import gc

    from paper_2605_28525_b200.solver import release_cached_memory
    ps, cfg, mats, bc = column_scene()
    runs = []
    for _ in range(2):  # second run: every buffer comes from the cache
        cfg.deterministic = True
        sim = Simulation(ps.copy(), cfg, mats, bc)
        for _ in range(3):
            sim.step(1e-4)
        runs.append(sim.particles.x.copy())
        del sim
        gc.collect()
    assert np.array_equal(runs[0], runs[1])
    release_cached_memory()
    sim = Simulation(ps.copy(), cfg, mats, bc)  # fresh allocations after the release
    sim.step(1e-4)

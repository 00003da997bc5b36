"""Generate golden vectors from the *reference* implementation.

Run in the build container only (the reference does not exist on the GPU
box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports the unmodified reference package ``sparsempm`` and records the
inputs and outputs of every hot-path function on small seeded scenes.  The
oracle (oracle/) is pinned against these fixtures (tests/test_oracle_golden.py)
and the CUDA path is then checked against the oracle.  Every recorded case
names the reference function it exercises.
"""

import os
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, "/root/reference/pkg/src")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    import sparsempm  # noqa: F401
    return sparsempm


def column_particles(sm, region_min, region_max, h, ppc=2, density=1500.0, seed=None):
    from sparsempm.scenarios import sample_box
    from sparsempm.solver import ParticleSet

    pos, vol = sample_box(region_min, region_max, h, ppc)
    if seed is not None:
        rng = np.random.default_rng(seed)
        pos = pos + rng.uniform(-0.2, 0.2, pos.shape) * (h / ppc)
    return ParticleSet.from_samples(pos, vol, density)


def perturbed_state(ps, seed, vscale=1.0, cscale=2.0, fscale=0.03):
    rng = np.random.default_rng(seed)
    n = ps.n
    ps.v[:] = rng.uniform(-vscale, vscale, (n, 3))
    ps.C[:] = rng.uniform(-cscale, cscale, (n, 3, 3))
    ps.F[:] = np.eye(3)[None] + rng.normal(0.0, fscale, (n, 3, 3))
    # a compressed population so the DP return map is exercised
    ps.F[: n // 3] *= 0.97
    return ps


def keys_case(sm):
    from sparsempm.grid_index import mix64, pack_key, unpack_key

    rng = np.random.default_rng(1)
    blocks = rng.integers(-(1 << 20), 1 << 20, size=(2000, 3))
    blocks[0] = (0, 0, 0)
    blocks[1] = (-(1 << 20), -(1 << 20), -(1 << 20))
    blocks[2] = ((1 << 20) - 1, (1 << 20) - 1, (1 << 20) - 1)
    packed = np.array([pack_key(tuple(b)) for b in blocks], dtype=np.uint64)
    unpacked = np.array([unpack_key(int(k)) for k in packed], dtype=np.int64)
    mk = np.concatenate([np.arange(0, 1000, dtype=np.uint64), packed])
    mixed = np.array([mix64(int(k)) for k in mk], dtype=np.uint64)
    return dict(blocks=blocks, packed=packed, unpacked=unpacked, mix_in=mk, mix_out=mixed)


def hash_case(sm):
    from sparsempm.grid_index import pack_key
    from sparsempm.sparse_hash import BlockHashTable, build_hash_sparse_grid
    from sparsempm.sparse_scan import build_scan_sparse_grid

    rng = np.random.default_rng(2)
    out = {}
    # insert sequence with duplicates at small capacity (serial insert order)
    blocks = rng.integers(-40, 40, size=(3000, 3))
    t = BlockHashTable(8192)
    ranks, fresh = [], []
    for b in blocks:
        r, f = t.insert(tuple(b))
        ranks.append(r)
        fresh.append(f)
    out["ins_blocks"] = blocks
    out["ins_ranks"] = np.array(ranks, dtype=np.int64)
    out["ins_fresh"] = np.array(fresh, dtype=bool)
    out["ins_keys"] = t.keys.copy()
    out["ins_vals"] = t.vals.copy()
    # build from a particle cloud (deterministic = first-encounter ranks)
    x = rng.uniform(-3.0, 3.0, size=(4000, 3))
    x[:100] += 50.0
    h = 0.07
    hm = build_hash_sparse_grid(x, h, 4, deterministic=True)
    sm_ = build_scan_sparse_grid(x, h, 4)
    out["cloud_x"] = x
    out["cloud_h"] = np.float64(h)
    out["hash_active"] = hm.active_blocks
    out["hash_keys"] = hm.keys
    out["hash_vals"] = hm.vals
    out["scan_active"] = sm_.active_blocks
    out["scan_bmin"] = sm_.bmin
    out["scan_bshape"] = sm_.bshape
    out["scan_phi"] = sm_.phi_flat
    # forced small initial capacity: rebuild path
    hm2 = build_hash_sparse_grid(x, h, 4, initial_capacity=64, deterministic=True)
    out["rebuild_active"] = hm2.active_blocks
    out["rebuild_capacity"] = np.int64(hm2.keys.shape[0])
    # node indices for a few nodes
    nodes = rng.integers(-50, 50, size=(200, 3))
    idx = []
    for nd in nodes:
        try:
            idx.append(sm_.node_index(nd))
        except KeyError:
            idx.append(-1)
    out["nodes"] = nodes
    out["scan_node_index"] = np.array(idx, dtype=np.int64)
    _ = pack_key
    return out


def count_case(sm):
    from sparsempm.solver import count_active_nodes

    rng = np.random.default_rng(3)
    out = {}
    for i, (n, spread, h) in enumerate([(1, 1.0, 0.1), (500, 1.0, 0.05), (20000, 5.0, 0.11), (3000, 100.0, 0.3)]):
        x = rng.uniform(-spread, spread, size=(n, 3))
        out[f"x{i}"] = x
        out[f"h{i}"] = np.float64(h)
        out[f"count{i}"] = np.int64(count_active_nodes(x, h))
    return out


def stencil_case(sm):
    from sparsempm.solver import bspline_weights

    rng = np.random.default_rng(4)
    xs = rng.uniform(-50.0, 50.0, size=(500, 3))
    xs[0] = (0.3, 0.3, 0.3)
    xs[1] = (0.55, 0.55, 0.55)
    hs = rng.uniform(0.01, 2.0, size=500)
    bases, ws, gs = [], [], []
    for x, h in zip(xs, hs):
        b, w, g = bspline_weights(x, h)
        bases.append(b)
        ws.append(w)
        gs.append(g)
    return dict(x=xs, h=hs, base=np.array(bases), w=np.array(ws), dw=np.array(gs))


def materials():
    from sparsempm.materials import MaterialModel

    return [MaterialModel(kind="drucker_prager", density=1500.0, youngs_modulus=1e6, poisson_ratio=0.3,
                          friction_angle_deg=30.0),
            MaterialModel(kind="elastic", density=1000.0, youngs_modulus=2e5, poisson_ratio=0.25)]


def boundaries():
    from sparsempm.solver import BoundaryCondition, Heightfield

    xs = np.arange(12) * 0.1 - 0.55
    ys = np.arange(10) * 0.1 - 0.45
    data = 0.02 + 0.15 * xs[:, None] + 0.05 * ys[None, :] ** 2
    hf = Heightfield(x0=-0.55, y0=-0.45, cell=0.1, data=data)
    return [BoundaryCondition(kind="plane", mu=0.3, point=np.array([0.0, 0.0, 0.0]),
                              normal=np.array([0.0, 0.1, 1.0])),
            BoundaryCondition(kind="plane", mu=0.0, point=np.array([0.25, 0.0, 0.0]),
                              normal=np.array([-1.0, 0.0, 0.0])),
            BoundaryCondition(kind="heightfield", mu=0.5, heightfield=hf)]


def phases_case(sm):
    """stress -> scan map -> p2g/grid_forces -> grid_update -> g2p."""
    from sparsempm.materials import update_stress
    from sparsempm.solver import g2p, grid_forces, grid_update, p2g
    from sparsempm.sparse_scan import build_scan_sparse_grid

    h = 0.05
    ps = column_particles(sm, (-0.2, -0.15, 0.0), (0.2, 0.15, 0.3), h, seed=5)
    ps = perturbed_state(ps, 6)
    ps.mat_id[::4] = 1
    mats = materials()
    out = {"h": np.float64(h), "gravity": np.array([0.3, 0.0, -9.81])}
    for k in ("x", "v", "C", "F", "m", "V0", "mat_id"):
        out["in_" + k] = getattr(ps, k).copy()
    update_stress(ps, mats)
    out["st_F"] = ps.F.copy()
    out["st_sigma"] = ps.sigma.copy()
    out["st_jac"] = ps.jac.copy()
    amap = build_scan_sparse_grid(ps.x, h, 4)
    out["map_active"] = amap.active_blocks
    fields = p2g(ps, amap, h, deterministic=True)
    grid_forces(ps, amap, h, out["gravity"], deterministic=True, fields=fields)
    out["p2g_mass"] = fields.mass.copy()
    out["p2g_mom"] = fields.vel.copy()
    out["p2g_force"] = fields.force.copy()
    dt = 2e-4
    out["dt"] = np.float64(dt)
    mass_floor = 1e-12 * float(ps.m.max())
    out["mass_floor"] = np.float64(mass_floor)
    grid_update(fields, amap, h, dt, mass_floor, boundaries())
    out["gu_vel"] = fields.vel.copy()
    g2p(ps, amap, fields, h, dt)
    for k in ("x", "v", "C", "F"):
        out["g2p_" + k] = getattr(ps, k).copy()
    return out


def steps_case(sm, backend, nsteps, seed):
    """Full Simulation.step sequence in deterministic mode."""
    from sparsempm.solver import SimConfig, Simulation

    h = 0.05
    ps = column_particles(sm, (-0.2, -0.15, 0.02), (0.2, 0.15, 0.3), h, seed=seed)
    ps.v[:, 0] = 0.5
    cfg = SimConfig(h=h, gravity=np.array([0.5, 0.0, -9.81]), total_time=1.0,
                    domain_min=np.array([-1.0, -1.0, -0.2]), domain_max=np.array([1.0, 1.0, 1.0]),
                    backend=backend, deterministic=True)
    sim = Simulation(ps, cfg, materials()[:1], boundaries(), record_conservation=True)
    out = {"h": np.float64(h), "gravity": cfg.gravity}
    for k in ("x", "v", "C", "F", "m", "V0", "mat_id"):
        out["in_" + k] = getattr(ps, k).copy()
    xs, vs, dts, nact, nalloc, msum, psum = [], [], [], [], [], [], []
    for _ in range(nsteps):
        st = sim.step()
        xs.append(sim.particles.x.copy())
        vs.append(sim.particles.v.copy())
        dts.append(st.dt)
        nact.append(st.n_active)
        nalloc.append(st.n_allocated)
        msum.append(st.mass_sum)
        psum.append(st.mom_sum)
    out.update(x=np.array(xs), v=np.array(vs), C=sim.particles.C.copy(), F=sim.particles.F.copy(), dt=np.array(dts),
               n_active=np.array(nact), n_allocated=np.array(nalloc), mass_sum=np.array(msum),
               mom_sum=np.array(psum), last_active=sim.last_map.active_blocks)
    return out


def main():
    sm = _ref()
    np.savez_compressed(OUT / "keys.npz", **keys_case(sm))
    np.savez_compressed(OUT / "hash.npz", **hash_case(sm))
    np.savez_compressed(OUT / "count.npz", **count_case(sm))
    np.savez_compressed(OUT / "stencil.npz", **stencil_case(sm))
    np.savez_compressed(OUT / "phases.npz", **phases_case(sm))
    np.savez_compressed(OUT / "steps_scan.npz", **steps_case(sm, "scan", 6, 7))
    np.savez_compressed(OUT / "steps_hash.npz", **steps_case(sm, "hash", 6, 8))
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()

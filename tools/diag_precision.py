"""P2G precision diagnostic: the fused path's fixed-point grid sums vs the
module API's fp32 float-atomic sums, both against the oracle's fp64 P2G, on
the C4 sample and C1 (norm-wise, and binned by node mass).
usage: python tools/diag_precision.py [C4|C1] [pre_steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as o  # noqa: E402
from paper_2605_28525_b200 import grid_index as gi, scenes  # noqa: E402
from paper_2605_28525_b200.solver import grid_forces, p2g  # noqa: E402
from paper_2605_28525_b200.sparse_hash import build_hash_sparse_grid  # noqa: E402
from tests.test_gpu_module import keyed  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sc = scenes.landslide(columns=(800, 805)) if name == "C4" else scenes.granular_column()
sim = sc.simulation()
for _ in range(pre):
    sim.step()
state = sim.particles.copy()
# oracle P2G (fp64) of the state: stress + scatter
s = o.OracleParticles.from_any(state)
o.update_stress(s, sc.materials)
amap = o.build_hash_sparse_grid(s.x, sc.config.h, 4, deterministic=True)
fr = o.p2g(s, amap, sc.config.h)
o.grid_forces(s, amap, sc.config.h, sc.config.gravity, fields=fr)
kr, mr = keyed(amap.active_blocks, fr.mass, 1)
_, pr = keyed(amap.active_blocks, fr.vel, 3)
_, frr = keyed(amap.active_blocks, fr.force, 3)
# fused path (fixed point)
blocks, fg = sim.query_grid()
kg, mg = keyed(blocks, fg.mass, 1)
_, pg = keyed(blocks, fg.vel, 3)
_, ffg = keyed(blocks, fg.force, 3)
assert np.array_equal(kg, kr)
# module path (fp32 float atomics), same stressed state
st2 = state.copy()
st2.sigma[:] = s.sigma
st2.jac[:] = s.jac
st2.F[:] = s.F
gmap = build_hash_sparse_grid(st2.x, sc.config.h, 4)
fm = p2g(st2, gmap, sc.config.h)
grid_forces(st2, gmap, sc.config.h, sc.config.gravity, fields=fm)
km, mm = keyed(gmap.active_blocks, fm.mass, 1)
_, pm = keyed(gmap.active_blocks, fm.vel, 3)
_, ffm = keyed(gmap.active_blocks, fm.force, 3)
assert np.array_equal(km, kr)
g = sc.config.gravity
fr_tot = frr  # oracle force includes gravity
def nw(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())
print(f"{name} after {pre} steps, {state.n} particles, {kr.size} nodes")
print(f"  fixed point : mass {nw(mg, mr):.2e} mom {nw(pg, pr):.2e} force {nw(ffg, fr_tot):.2e}")
print(f"  fp32 atomics: mass {nw(mm, mr):.2e} mom {nw(pm, pr):.2e} force {nw(ffm, fr_tot):.2e}")
heavy = mr[:, 0] > 1e-3 * mr.max()
for lab, f in (("fixed", ffg), ("fp32", ffm)):
    d = np.abs(f - fr_tot).max(axis=1)
    for lo, hi in ((1e-3, 1e-2), (1e-2, 1e-1), (1e-1, 2.0)):
        sel = (mr[:, 0] > lo * mr.max()) & (mr[:, 0] <= hi * mr.max())
        if sel.any():
            print(f"  {lab:6s} force err / max|f| on nodes m/m_max in ({lo:g},{hi:g}]: {d[sel].max() / np.abs(fr_tot).max():.2e}"
                  f"  (max |f| there / global {np.abs(fr_tot[sel]).max() / np.abs(fr_tot).max():.2e})")
# contribution scale vs net force: how much the node force cancels
print(f"  max |f_node| {np.abs(fr_tot).max():.3e}; max |V0 tau| / h {np.abs(s.sigma * s.jac[:, None, None] * s.V0[:, None, None]).max() / sc.config.h:.3e}")

# grid velocity conditioning: the oracle's grid update on its fp64 sums vs on
# the same sums rounded to fp32 (the floor of any fp32-sum grid), on nodes with
# m > 1e-3 m_max; and this build's grid velocity (one fused step from `state`)
dt = sim.dt_bound() * 0.999
ref = o.OracleSimulation(state, sc.config.h, sc.config.gravity, sc.materials, sc.boundaries, backend="hash",
                         deterministic=True)
ref.step(dt)
f64 = ref.last_fields
imap = ref.last_map
# rebuild the oracle's pre-update sums for the same state (fresh P2G), round, update
s2 = o.OracleParticles.from_any(state)
o.update_stress(s2, sc.materials)
fr2 = o.p2g(s2, imap, sc.config.h)
o.grid_forces(s2, imap, sc.config.h, sc.config.gravity, fields=fr2)
for a in ("mass", "vel", "force"):
    getattr(fr2, a)[...] = getattr(fr2, a).astype(np.float32).astype(np.float64)
o.grid_update(fr2, imap, sc.config.h, dt, ref.mass_floor, sc.boundaries)
k1, v64 = keyed(imap.active_blocks, f64.vel, 3)
_, v32 = keyed(imap.active_blocks, fr2.vel, 3)
_, mref = keyed(imap.active_blocks, f64.mass, 1)
heavy = mref[:, 0] > 1e-3 * mref.max()
floor = float(np.abs(v32[heavy] - v64[heavy]).max() / np.abs(v64[heavy]).max())
sim.step(dt)
kg2, vg = keyed(sim.last_map.active_blocks, sim.last_fields.vel, 3)
assert np.array_equal(kg2, k1)
ours = float(np.abs(vg[heavy] - v64[heavy]).max() / np.abs(v64[heavy]).max())
print(f"  grid velocity (m > 1e-3 m_max): fp32-rounded sums floor {floor:.2e}, this build {ours:.2e}")

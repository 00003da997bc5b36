"""Diagnose the grid-force discrepancy of the mixed-BC parity test: separate
the fp32 stress error from the P2G (fixed-point) error."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import oracle as o  # noqa: E402
from paper_2605_28525_b200.solver import Simulation  # noqa: E402
from tests.test_gpu_module import keyed, normwise  # noqa: E402
from tests.test_gpu_sim import column_scene  # noqa: E402

ps, cfg, mats, bc = column_scene(bcs="mixed")
sim = Simulation(ps, cfg, mats, bc)
for s in range(8):
    blocks, f = sim.query_grid()
    gp = sim.particles.copy()  # sigma/jac computed on the device from F (fp32)
    ref = o.OracleParticles.from_any(gp)
    o.update_stress(ref, mats)
    amap = o.build_hash_sparse_grid(ref.x, cfg.h, 4, deterministic=True)
    fr = o.grid_forces(ref, amap, cfg.h, cfg.gravity)
    g32 = o.OracleParticles.from_any(gp)  # oracle P2G with the GPU's stress
    fg = o.grid_forces(g32, amap, cfg.h, cfg.gravity)
    _, F_fused = keyed(blocks, f.force, 3)
    _, F_ref = keyed(amap.active_blocks, fr.force, 3)
    _, F_g32 = keyed(amap.active_blocks, fg.force, 3)
    ds = np.abs(gp.sigma - ref.sigma).reshape(len(gp.x), -1).max(axis=1)
    smax = np.abs(ref.sigma).max()
    flips = int((ds > 1e-3 * smax).sum())
    print(f"step {s}: |f|max={np.abs(F_ref).max():.3e} fused-vs-ref {normwise(F_fused, F_ref):.2e} "
          f"fused-vs-oracle(gpu sigma) {normwise(F_fused, F_g32):.2e} oracle(gpu sigma)-vs-ref "
          f"{normwise(F_g32, F_ref):.2e} sigma err {normwise(gp.sigma, ref.sigma):.2e} "
          f"particles with |dsigma|>1e-3|sigma|max: {flips} / {len(gp.x)}")
    worst = int(np.argmax(ds))
    print("   worst particle", worst, "dsigma", ds[worst], "F", gp.F[worst].ravel()[:9])
    sim.step(0.9 * sim.dt_bound())

# module-level float-atomic P2G with the same GPU stresses
from paper_2605_28525_b200 import solver as S  # noqa: E402
from paper_2605_28525_b200.sparse_hash import build_hash_sparse_grid  # noqa: E402
blocks, f = sim.query_grid()
gp = sim.particles.copy()
gm = build_hash_sparse_grid(gp.x, cfg.h, 4, rank_order="key")
fm = S.grid_forces(gp, gm, cfg.h, cfg.gravity)
g32 = o.OracleParticles.from_any(gp)
amap = o.build_hash_sparse_grid(g32.x, cfg.h, 4, deterministic=True)
fg = o.grid_forces(g32, amap, cfg.h, cfg.gravity)
_, F_fused = keyed(blocks, f.force, 3)
_, F_mod = keyed(gm.active_blocks, fm.force, 3)
_, F_g32 = keyed(amap.active_blocks, fg.force, 3)
err = np.abs(F_fused - F_g32).max(axis=1)
print("module-vs-oracle(gpu sigma)", normwise(F_mod, F_g32), "fused-vs-oracle", normwise(F_fused, F_g32))
k = np.argsort(-err)[:5]
print("worst nodes err", err[k], "ref", F_g32[k], "fused", F_fused[k])
_, M_fused = keyed(blocks, f.mass, 1)
print("mass at worst nodes", M_fused[k].ravel())

# fresh simulation from the downloaded state: its prologue P2G evaluates tau
# from the stored F exactly like the download does
sim2 = Simulation(gp.copy(), cfg, mats, bc)
b2, f2 = sim2.query_grid()
_, F_pro = keyed(b2, f2.force, 3)
print("prologue-fused-vs-oracle(gpu sigma)", normwise(F_pro, F_g32), " fused(step)-vs-prologue", normwise(F_fused, F_pro))

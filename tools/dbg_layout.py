"""Deterministic mode: narrow vs wide work-item layout (SMPM_ITEM_LAYOUT), per-step
max differences of x, v, C, F for a sand and a prestrained elastic column (expect 0)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from tests.test_gpu_sim import column_scene, ELASTIC
from paper_2605_28525_b200.solver import Simulation
for mat in ("sand", "elastic"):
    ps, cfg, mats, bc = column_scene(vx=3.0, prestrain=0.25 if mat == "elastic" else 0.0, mat=ELASTIC if mat == "elastic" else None)
    cfg.deterministic = True
    sims = []
    for layout in ("narrow", "wide"):
        os.environ["SMPM_ITEM_LAYOUT"] = layout
        sims.append(Simulation(ps.copy(), cfg, mats, bc))
    for s in range(6):
        st = [sm.step(1e-4) for sm in sims]
        a, b = sims[0].particles, sims[1].particles
        print(mat, "step", s, {k: float(np.abs(getattr(a, k) - getattr(b, k)).max()) for k in ("x", "v", "C", "F")},
              "n_active", st[0].n_active, st[1].n_active)
    ga = sims[0].query_grid(); gb = sims[1].query_grid()
    print(" grid blocks equal", np.array_equal(np.sort(ga[0], axis=0), np.sort(gb[0], axis=0)))

"""Where the end-to-end time of bench.py's e2e leg goes (C4, 1 GPU)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2605_28525_b200 import _lib, scenes  # noqa: E402
from paper_2605_28525_b200.solver import Simulation  # noqa: E402

frac = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
sc = scenes.landslide(fraction=frac)
ps = sc.particles
n = ps.n
torch.cuda.init()
torch.zeros(1, device="cuda")
t = {}
t0 = time.perf_counter()
ps.mat_id.min(), ps.mat_id.max(), ps.m.max()
t["host checks (mat_id, m)"] = time.perf_counter() - t0
t0 = time.perf_counter()
np.all(np.isfinite(ps.x))
t["host isfinite(x)"] = time.perf_counter() - t0
t0 = time.perf_counter()
sim = Simulation(ps, sc.config, sc.materials, sc.boundaries)
torch.cuda.synchronize()
t["Simulation() incl. upload"] = time.perf_counter() - t0
t0 = time.perf_counter()
sim.step()
t["first step (prologue)"] = time.perf_counter() - t0
t0 = time.perf_counter()
for _ in range(5):
    sim.step()
t["5 steps"] = time.perf_counter() - t0
ox = np.empty_like(ps.x)
ov = np.empty_like(ps.v)
t0 = time.perf_counter()
_lib.check(_lib.load().smpm_sim_get_particles(sim._h, ox.ctypes.data, ov.ctypes.data, None, None, None, None))
t["download x, v"] = time.perf_counter() - t0
for k, v in t.items():
    print(f"{k:32s} {v:8.3f} s")
print("n", n, "upload GB (ref layout)", n * 216 / 1e9)

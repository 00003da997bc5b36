"""Full C4 landslide (101M particles) for N steps through Simulation.run in
batches of 500: simulated time, step rate, active nodes, mass conservation and
the fused kernel per batch (long-run stability of the production path in the
flowing regime).  usage: python tools/long_c4.py [steps]"""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_28525_b200 import _lib, scenes  # noqa: E402
from paper_2605_28525_b200.solver import Simulation  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
sc = scenes.landslide()
sim = Simulation(sc.particles, sc.config, sc.materials, sc.boundaries, record_conservation=True)
m0 = None
done = 0
while done < steps:
    k = min(500, steps - done)
    t0 = time.perf_counter()
    stats = sim.run(k)
    wall = time.perf_counter() - t0
    done += k
    st = stats[-1]
    m0 = m0 or stats[0].mass_sum
    dbg = (ctypes.c_int64 * 24)()
    _lib.check(_lib.load().smpm_sim_debug_stats(sim._h, dbg), "debug stats")
    kern = {0: "k_g2p2g_f32", 1: "k_g2p2g_ws"}.get(int(dbg[23]), str(int(dbg[23])))
    vmax = float(np.sqrt((sim.particles.v ** 2).sum(axis=1).max())) if done == steps else float("nan")
    print(f"step {done:5d} t={sim.t:7.3f} s  {wall / k * 1e3:6.2f} ms/step  n_active {st.n_active:10d}  "
          f"allocated {st.n_allocated:10d}  mass drift {abs(st.mass_sum - m0) / m0:.2e}  "
          f"layout {'wide' if dbg[21] else 'narrow'}  kernel {kern}", flush=True)
x = sim.particles.x
print(f"finite {np.isfinite(x).all()}  x range {x[:, 0].min():.1f} .. {x[:, 0].max():.1f} m", flush=True)

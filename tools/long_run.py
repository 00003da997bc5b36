"""Long-run stability check: C1 granular column collapse to t = 0.6 s and the
landslide's leading 10 % for 600 steps; prints step rate, active nodes, and
conservation drift."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_28525_b200 import scenes  # noqa: E402
from paper_2605_28525_b200.solver import Simulation  # noqa: E402


def go(name, sc, steps=None, t_end=None):
    sim = Simulation(sc.particles, sc.config, sc.materials, sc.boundaries, record_conservation=True)
    t0 = time.perf_counter()
    n, st0 = 0, None
    gpu = 0.0
    while True:
        st = sim.step()
        gpu += sum(st.times.values())
        st0 = st0 or st
        n += 1
        if (steps and n >= steps) or (t_end and sim.t >= t_end):
            break
    wall = time.perf_counter() - t0
    x = sim.particles.x
    print(f"{name}: {n} steps to t={sim.t:.4f} s, wall {wall:.2f} s, device {gpu:.2f} s "
          f"({sc.particles.n * n / gpu:.3e} particle-steps/s), n_active {st0.n_active} -> {st.n_active}, "
          f"mass {st0.mass_sum:.6e} -> {st.mass_sum:.6e}, finite {np.isfinite(x).all()}, "
          f"zmin {x[:, 2].min():.4f}", flush=True)


go("C1 column", scenes.granular_column(), t_end=0.6)
go("C4 landslide 10%", scenes.landslide(fraction=0.1), steps=600)

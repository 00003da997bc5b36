"""Run the landslide's leading 10 % for N steps (argv[1]) and report the
per-phase device times of the last 20 steps (late-time kernel behaviour)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_28525_b200 import scenes  # noqa: E402
from paper_2605_28525_b200.solver import Simulation  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
sc = scenes.landslide(fraction=0.1)
sim = Simulation(sc.particles, sc.config, sc.materials, sc.boundaries)
hist = []


def item_stats(tag):
    import ctypes
    from paper_2605_28525_b200 import _lib
    out = (ctypes.c_int64 * 24)()
    _lib.check(_lib.load().smpm_sim_debug_stats(sim._h, out), "debug stats")
    o = list(out)
    print(f"{tag}: blocks {o[0]} items {o[2]} ({o[2] / max(o[0], 1):.2f}/block) binned {o[1]} | bins: bad {o[16]} "
          f"mig {o[17]} ovf {o[18]} arena {o[19]} direct {o[20]} | layout {'wide' if o[21] else 'narrow'}")


for s in range(n):
    st = sim.step()
    if s in (20, n - 1):
        item_stats(f"step {s}")
    hist.append((st.times["map_build"], st.times["grid_update"], st.times["g2p"], st.n_allocated))
for lo, hi in ((3, 23), (n - 20, n)):
    h = np.array(hist[lo:hi])
    print(f"steps {lo}-{hi}: map {h[:, 0].mean() * 1e3:.3f} grid {h[:, 1].mean() * 1e3:.3f} "
          f"fused {h[:, 2].mean() * 1e3:.3f} ms, allocated {h[:, 3].mean():.3e} nodes, t={sim.t:.3f} s")

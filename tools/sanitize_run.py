"""A few fused steps of a 16k-particle DP column (with a moving elastic
block for larger strains) for compute-sanitizer (tools/sanitize.sh).
Mode from the environment: SMPM_MODE=fast|det, SMPM_ARENA, SMPM_ITEM_LAYOUT
(see tools/sanitize.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

mode = os.environ.get("SMPM_MODE", "fast")
layout = os.environ.get("SMPM_ITEM_LAYOUT", "auto") + "/" + os.environ.get("SMPM_ARENA", "default")
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3

from paper_2605_28525_b200 import scenes  # noqa: E402
from paper_2605_28525_b200.solver import Simulation  # noqa: E402

sc = scenes.granular_column(h=0.05)
ps = sc.particles
ps.v[:, 0] = 1.5  # cross cell boundaries: arena bins, far scatter, block inserts
rng = np.random.default_rng(0)
ps.x += rng.uniform(-0.2, 0.2, ps.x.shape) * 0.025
sc.config.deterministic = mode == "det"
sim = Simulation(ps, sc.config, sc.materials, sc.boundaries, host_sync="on_access")
for _ in range(steps):
    st = sim.step()
print(f"{layout} {mode}: {steps} steps, n_active {st.n_active}, x finite {np.isfinite(sim.particles.x).all()}")

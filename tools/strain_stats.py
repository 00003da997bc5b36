"""Strain statistics of the landslide after N steps: how many particles the
small-strain series covers, and how many a volumetric split would."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_28525_b200 import scenes  # noqa: E402
from paper_2605_28525_b200.solver import Simulation  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
checkpoints = sorted({n} | {int(a) for a in sys.argv[2:]})
sc = scenes.landslide(fraction=0.02)
sim = Simulation(sc.particles, sc.config, sc.materials, sc.boundaries)
done = 0
for cp in checkpoints:
    for s in range(cp - done):
        sim.step()
    done = cp
    lam = np.linalg.eigvalsh(sim.particles.F @ np.transpose(sim.particles.F, (0, 2, 1)))
    qs = [0, 1e-4, 1e-3, 1e-2, 0.5, 0.99, 0.999, 0.9999, 1]
    print(f"step {cp}: lambda_min(B) quantiles", np.quantile(lam[:, 0], qs).round(4))
    print(f"step {cp}: lambda_max(B) quantiles", np.quantile(lam[:, 2], qs).round(4))
    z = np.maximum(np.abs((lam[:, 0] - 1) / (lam[:, 0] + 1)), np.abs((lam[:, 2] - 1) / (lam[:, 2] + 1)))
    for zt in (0.1, 0.2, 0.33, 0.5, 0.6, 0.8):
        print(f"   |z| <= {zt}: {np.mean(z <= zt) * 100:7.3f} %")
for s in range(n - done):
    sim.step()
F = sim.particles.F
B = F @ np.transpose(F, (0, 2, 1))
X = B - np.eye(3)
nx = np.abs(X).sum(axis=2).max(axis=1)
J = np.linalg.det(F)
a = J ** (-2.0 / 3.0)
Xb = a[:, None, None] * B - np.eye(3)
nb = np.abs(Xb).sum(axis=2).max(axis=1)
print(f"t={sim.t:.3f}s particles {len(nx)}")
for thr in (0.05, 0.1, 0.2, 0.4):
    print(f"  ||B-I|| <= {thr}: {np.mean(nx <= thr) * 100:5.1f} %   ||B_iso-I|| <= {thr}: {np.mean(nb <= thr) * 100:5.1f} %")
print("  J quantiles", np.quantile(J, [0.01, 0.1, 0.5, 0.9, 0.99]))

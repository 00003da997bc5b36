"""CPU baseline fairness: the reference's own numba scan path vs the oracle
port (C + OpenMP) on the same sample, same threads, in the build container.
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache python tools/ref_vs_port.py"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from oracle import oracle as o  # noqa: E402
from paper_2605_28525_b200 import scenes  # noqa: E402

frac = float(sys.argv[1]) if len(sys.argv) > 1 else 0.005
threads = len(os.sched_getaffinity(0))
sc = scenes.landslide(fraction=frac)
n = sc.particles.n
steps = 2
sim = o.OracleSimulation(sc.particles, sc.config.h, sc.config.gravity, sc.materials, sc.boundaries, backend="scan",
                         deterministic=False, threads=threads)
sim.step(count_nodes=False)
tot = 0.0
for _ in range(steps):
    st = sim.step(count_nodes=False)
    tot += sum(st["times"][p] for p in o.COMPUTE_PHASES)
print(f"port: {n} particles, {threads} threads: {tot / steps * 1e3:.1f} ms/step -> {n * steps / tot:.3e} particle-steps/s")

import sparsempm  # noqa: E402
from sparsempm import solver as rs  # noqa: E402
from sparsempm.materials import MaterialModel  # noqa: E402
from sparsempm.bench import warm_kernels  # noqa: E402

warm_kernels("scan", False)
ps = sc.particles
rps = rs.ParticleSet(x=ps.x.copy(), v=ps.v.copy(), C=ps.C.copy(), F=ps.F.copy(), m=ps.m.copy(), V0=ps.V0.copy(),
                     mat_id=ps.mat_id.copy(), sigma=ps.sigma.copy(), jac=ps.jac.copy())
mats = [MaterialModel(kind=m.kind, density=m.density, youngs_modulus=m.youngs_modulus, poisson_ratio=m.poisson_ratio,
                      friction_angle_deg=m.friction_angle_deg) for m in sc.materials]
bcs = []
for b in sc.boundaries:
    if b.kind == "plane":
        bcs.append(rs.BoundaryCondition(kind="plane", mu=b.mu, point=b.point, normal=b.normal))
    else:
        hf = b.heightfield
        bcs.append(rs.BoundaryCondition(kind="heightfield", mu=b.mu,
                                        heightfield=rs.Heightfield(x0=hf.x0, y0=hf.y0, cell=hf.cell, data=hf.data)))
cfg = rs.SimConfig(h=sc.config.h, gravity=sc.config.gravity, total_time=1.0, domain_min=sc.config.domain_min,
                   domain_max=sc.config.domain_max, backend="scan", n_threads=threads)
rsim = rs.Simulation(rps, cfg, mats, bcs)
rsim.step()
tot = 0.0
for _ in range(steps):
    st = rsim.step()
    tot += sum(st.times[p] for p in rs.PHASES)
print(f"reference numba: {n} particles, {threads} threads: {tot / steps * 1e3:.1f} ms/step -> {n * steps / tot:.3e} particle-steps/s")

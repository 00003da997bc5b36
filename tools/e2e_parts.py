"""Repeatable timing of the e2e leg's parts (C4, 1 GPU): sim create, upload,
first step (prologue), steps, download into fresh vs reused host arrays."""
import ctypes
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
torch.zeros(1, device="cuda")
lib = _lib.load()
orig_upload = Simulation._upload
for rep in range(3):
    t = {}
    t0 = time.perf_counter()

    def timed_upload(self, p):
        t["create"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        orig_upload(self, p)
        t["upload"] = time.perf_counter() - t1

    Simulation._upload = timed_upload
    sim = Simulation(ps, sc.config, sc.materials, sc.boundaries)
    t1 = time.perf_counter()
    sim.step()
    t["step1"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    for _ in range(19):
        sim.step()
    t["19 steps"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    ox, ov = np.empty_like(ps.x), np.empty_like(ps.v)
    _lib.check(lib.smpm_sim_get_particles(sim._h, ox.ctypes.data, ov.ctypes.data, None, None, None, None))
    t["download fresh"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    _lib.check(lib.smpm_sim_get_particles(sim._h, ox.ctypes.data, ov.ctypes.data, None, None, None, None))
    t["download reused"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    del sim
    torch.cuda.synchronize()
    t["destroy"] = time.perf_counter() - t1
    print(" ".join(f"{k} {v:.3f}" for k, v in t.items()), flush=True)

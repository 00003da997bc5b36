"""Per-step overhead of the slab machinery (DistributedSimulation) at world
size 1 over NCCL: where the host time goes.  torchrun --nproc-per-node 1."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_28525_b200 import scenes, slabs  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl")
slab = scenes.landslide_slabs(1, fraction=0.1)[0]
sc = scenes.landslide(fraction=0.1, columns=(slab[2], slab[3]))
ds = slabs.DistributedSimulation(sc.particles, sc.config, sc.materials, sc.boundaries, (slab[0], slab[1]), pid_base=0)
T = {}


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    return w


for fn in ("smpm_sim_grid_size", "smpm_sim_exchange_pack", "smpm_sim_migrants", "smpm_sim_vmax"):
    setattr(ds.lib, fn, timed("lib." + fn, getattr(ds.lib, fn)))
_empty = torch.empty
torch.empty = timed("torch.empty", _empty)
for name in ("_pack", "_migrants", "_frame", "_unframe", "_unpack"):
    setattr(ds, name, timed(name, getattr(ds, name)))
ds.tr.exchange = timed("tr.exchange", ds.tr.exchange)
ds.tr.gather = timed("tr.gather", ds.tr.gather)
ds.sim.step = timed("sim.step", ds.sim.step)
for _ in range(3):
    ds.step()
T.clear()
N = 10
t0 = time.perf_counter()
for _ in range(N):
    ds.step()
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"per step {tot / N * 1e3:.3f} ms")
for k, v in sorted(T.items(), key=lambda x: -x[1]):
    print(f"  {k:14s} {v / N * 1e3:8.3f} ms")
dist.destroy_process_group()

"""Slab-decomposed landslide, one process per GPU:
    torchrun --nproc-per-node N --master-addr 127.0.0.1 examples/multi_gpu_landslide.py [steps] [fraction]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_28525_b200 import scenes  # noqa: E402
from paper_2605_28525_b200.slabs import DistributedSimulation, partition, subset  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
fraction = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
sc = scenes.landslide(fraction=fraction)
bounds, parts = partition(sc.particles, sc.config.h, world)
sim = DistributedSimulation(subset(sc.particles, parts[rank]), sc.config, sc.materials, sc.boundaries,
                            bounds[rank], pid_base=sum(len(p) for p in parts[:rank]))
for _ in range(steps):
    sim.step()
pid, x, v = sim.local_particles()
n = torch.tensor([len(pid)], device="cuda")
dist.all_reduce(n)
if rank == 0:
    print(f"{world} rank(s), {steps} steps, t = {sim.t:.4f} s, {int(n.item())} particles of {sc.particles.n}")
dist.destroy_process_group()

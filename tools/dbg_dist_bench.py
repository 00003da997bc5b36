"""The multi-GPU bench's slab setup on 2 ranks sharing one GPU (gloo): per
rank, the particle count, the slab's block range and how many particles have
their base block outside it before the first step; then the coordinated
prologue and a few steps.  usage: python tools/dbg_dist_bench.py [scale]"""
import os
import socket
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def worker(rank, world, port, scale):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_28525_b200 import scenes
    from paper_2605_28525_b200.slabs import DistributedSimulation

    slab = scenes.landslide_slabs(world, fraction=scale)[rank]
    sc = scenes.landslide(fraction=scale, columns=(slab[2], slab[3]))
    ps = sc.particles
    h = sc.config.h
    bx = np.floor(ps.x[:, 0] * (1.0 / h) - 0.5).astype(np.int64) >> 2
    out = int(((bx < slab[0]) | (bx >= slab[1])).sum())
    print(f"rank {rank}: n {ps.n} slab {slab} block x range {bx.min()}..{bx.max()} outside {out}", flush=True)
    per_col = ps.n // max(1, slab[3] - slab[2])
    try:
        sim = DistributedSimulation(ps, sc.config, sc.materials, sc.boundaries, (slab[0], slab[1]),
                                    pid_base=slab[2] * per_col)
        for s in range(3):
            st = sim.step()
            print(f"rank {rank}: step {s} n_active {st.n_active}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"rank {rank}: {type(e).__name__}: {e}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.02
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(2, port, scale), nprocs=2, join=True)

"""Debug: 2-rank drifting column (gloo, one GPU), pid uniqueness per step."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def worker(rank, world, port, steps, thr):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_28525_b200 import slabs
    from tests.test_gpu_slabs import _scene

    ps, cfg, mats, bc = _scene(False)
    bounds, parts = slabs.partition(ps, cfg.h, world)
    local = slabs.subset(ps, parts[rank])
    pid_base = int(sum(len(p) for p in parts[:rank]))
    ds = slabs.DistributedSimulation(local, cfg, mats, bc, bounds[rank], pid_base, block_capacity=1 << 14,
                                     rebalance_threshold=thr)
    for s in range(steps):
        st = ds.step()
        pid, x, v = ds.gather_particles()
        u = np.unique(pid).size
        if rank == 0:
            print(f"step {s}: n {pid.size} unique {u} rebal {ds.rebalances} growth {ds.frame_growths} "
                  f"caps {ds._cap_blocks}/{ds._cap_parts} counts {ds.local_counts} bounds {ds.bounds} replay {ds._replay}",
                  flush=True)
        if u != pid.size or pid.size != ps.n:
            if rank == 0:
                print("BROKEN at step", s, flush=True)
            break
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(2, port, int(sys.argv[1]) if len(sys.argv) > 1 else 30,
                           float(sys.argv[2]) if len(sys.argv) > 2 else 0.02), nprocs=2, join=True)

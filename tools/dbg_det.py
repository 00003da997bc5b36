"""Deterministic mode: 2 ranks (gloo, one GPU) vs 1 GPU, per-step diff."""
import os, socket, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch.multiprocessing as mp

STEPS = 8


def single(dts):
    from paper_2605_28525_b200.solver import Simulation
    from tests.test_gpu_slabs import _scene
    ps, cfg, mats, bc = _scene(True)
    sim = Simulation(ps.copy(), cfg, mats, bc, block_capacity=1 << 14)
    out = []
    for dt in dts:
        sim.step(dt)
        p = sim.particles
        out.append((p.x.copy(), p.v.copy()))
    return out


def worker(rank, world, port, dts, outdir):
    import torch, torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_28525_b200 import slabs
    from tests.test_gpu_slabs import _scene
    ps, cfg, mats, bc = _scene(True)
    bounds, parts = slabs.partition(ps, cfg.h, world)
    local = slabs.subset(ps, parts[rank])
    pid_base = int(sum(len(p) for p in parts[:rank]))
    ds = slabs.DistributedSimulation(local, cfg, mats, bc, bounds[rank], pid_base, block_capacity=1 << 14)
    order = np.concatenate(parts)
    res = []
    for dt in dts:
        ds.step(dt)
        pid, x, v = ds.gather_particles()
        res.append((order[pid], x, v, ds._replay))
    if rank == 0:
        np.save(os.path.join(outdir, "d.npy"), np.array(res, dtype=object), allow_pickle=True)
        np.save(os.path.join(outdir, "b.npy"), np.array(bounds))
    dist.barrier(); dist.destroy_process_group()


if __name__ == "__main__":
    dts = [2e-4] * STEPS
    ref = single(dts)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
    mp.spawn(worker, args=(2, port, dts, "/tmp"), nprocs=2, join=True)
    d = np.load("/tmp/d.npy", allow_pickle=True)
    bounds = np.load("/tmp/b.npy")
    from tests.test_gpu_slabs import _scene
    from paper_2605_28525_b200 import slabs
    ps, cfg, _, _ = _scene(True)
    for s_ in range(STEPS):
        pid, x, v, rp = d[s_]
        X = np.empty_like(x); X[pid] = x
        V = np.empty_like(v); V[pid] = v
        dx = np.abs(X - ref[s_][0]).max(axis=1)
        bad = np.nonzero(dx > 0)[0]
        bx = slabs.base_block_x(ref[s_][0], cfg.h)
        print(f"step {s_} replay {rp} max dx {dx.max():.3e} n_diff {len(bad)} "
              f"block-x of diffs {np.unique(bx[bad])[:10]} cut {bounds[0][1]}", flush=True)

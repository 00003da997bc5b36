import os, socket, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import torch.multiprocessing as mp

def worker(rank, world, port):
    try:
        _worker(rank, world, port)
    except Exception:
        import traceback
        print("RANK", rank, traceback.format_exc(), flush=True)
        raise


def _worker(rank, world, port):
    import torch, torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_28525_b200 import slabs
    from tests.test_gpu_slabs import _scene
    ps, cfg, mats, bc = _scene(False)
    bounds, parts = slabs.partition(ps, cfg.h, world)
    local = slabs.subset(ps, parts[rank])
    pid_base = int(sum(len(p) for p in parts[:rank]))
    ds = slabs.DistributedSimulation(local, cfg, mats, bc, bounds[rank], pid_base, block_capacity=1 << 14)
    import ctypes
    def dbg():
        o = (ctypes.c_int64 * 21)()
        ds.lib.smpm_sim_debug_stats(ds._h, o)
        return list(o)
    def live():
        n = ctypes.c_int64(0)
        ns = int(ds.lib.smpm_sim_num_stored(ds._h))
        pid = np.empty(max(ns, 1), dtype=np.int64); x = np.empty((max(ns, 1), 3)); v = np.empty((max(ns, 1), 3))
        ds.lib.smpm_sim_get_local(ds._h, ctypes.byref(n), pid.ctypes.data, x.ctypes.data, v.ctypes.data)
        return int(n.value), ns
    for name in ("_coordinated_prologue", "_exchange"):
        f = getattr(ds, name)
        def w(*a, _f=f, _n=name, **k):
            r = _f(*a, **k)
            print(f"  rank {rank} after {_n}: live/stored {live()} dbg {dbg()}", flush=True)
            return r
        setattr(ds, name, w)
    fs = ds.sim.step
    def ws(*a, **k):
        r = fs(*a, **k)
        print(f"  rank {rank} after sim.step: live/stored {live()} n_active {r.n_active} dbg {dbg()}", flush=True)
        return r
    ds.sim.step = ws
    for s in range(8):
        st = ds.step(0.8 * ds.dt_bound())
        pid, x, v = ds.local_particles()
        tot = ds.tr.gather([len(pid)]).sum()
        mig = ds.tr.gather([ds.migrated]).sum()
        if rank == 0: print("step", s, "replay", ds._replay, "live total", tot, "n", ps.n, "migrated", mig, flush=True)
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
  with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
if __name__ == "__main__":
    mp.spawn(worker, args=(2, port), nprocs=2, join=True)

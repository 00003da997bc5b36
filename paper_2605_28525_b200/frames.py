"""Frame output without stalling the simulation stream.

The reference writes a particle CSV per frame synchronously from the host
arrays (/root/reference/pkg/src/sparsempm/scenarios.py:483-513, driven from
bench.run, /root/reference/pkg/src/sparsempm/bench.py:206-211).  Here a frame
is

  1. a device snapshot of x and v in particle order, enqueued on the
     simulation's stream after the step (smpm_sim_snapshot_xv, no host sync);
  2. a device-to-host copy into pinned memory on a side stream, ordered after
     the snapshot by an event, so it overlaps the following steps;
  3. the CSV text (byte-identical to the reference's write_particles) written
     by a host thread once the copy's event completes.

Two snapshot slots are in flight at most; a third frame waits for the oldest.
"""

import concurrent.futures as cf
import time
from types import SimpleNamespace

import numpy as np

from . import _lib
from .scenarios import write_particles


class AsyncFrameWriter:
    def __init__(self, sim, slots=2):
        torch = _lib.torch_cuda()
        self.sim = sim
        n = sim.particles.n if hasattr(sim, "particles") else 0
        self.n = int(_lib.load().smpm_sim_num_particles(sim._h)) or n
        dev = sim.stream.device
        self._dev = [torch.empty(6 * self.n, dtype=torch.float64, device=dev) for _ in range(slots)]
        self._host = [torch.empty(6 * self.n, dtype=torch.float64).pin_memory() for _ in range(slots)]
        self._side = torch.cuda.Stream(device=dev)
        self._pool = cf.ThreadPoolExecutor(max_workers=1, thread_name_prefix="frames")
        self._busy = [None] * slots
        self._k = 0
        self.host_wait_s = 0.0  # time the stepping thread spent waiting for a free slot

    def submit(self, path):
        """Queue one frame of the current state; returns immediately unless
        both slots still hold unwritten frames."""
        torch = _lib.torch_cuda()
        slot = self._k % len(self._dev)
        self._k += 1
        if self._busy[slot] is not None:
            t0 = time.perf_counter()
            self._busy[slot].result()
            self.host_wait_s += time.perf_counter() - t0
        dev, host = self._dev[slot], self._host[slot]
        _lib.check(_lib.load().smpm_sim_snapshot_xv(self.sim._h, _lib.ptr(dev)), "snapshot")
        ready = torch.cuda.Event()
        ready.record(self.sim.stream)
        copied = torch.cuda.Event()
        with torch.cuda.stream(self._side):
            self._side.wait_event(ready)
            host.copy_(dev, non_blocking=True)
            copied.record(self._side)
        n = self.n

        def write():
            copied.synchronize()
            a = host.numpy()
            write_particles(path, SimpleNamespace(x=a[:3 * n].reshape(n, 3), v=a[3 * n:].reshape(n, 3)))

        self._busy[slot] = self._pool.submit(write)

    def close(self):
        """Wait for every queued frame (raises a writer's exception)."""
        for f in self._busy:
            if f is not None:
                f.result()
        self._pool.shutdown(wait=True)


__all__ = ["AsyncFrameWriter"]

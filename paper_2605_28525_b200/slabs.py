"""Multi-GPU slab decomposition of the sparse-MPM step.

The reference is single-process (its paper lists multi-GPU as future work,
/root/reference/PAPER.md:335-337); this module is the B200 build's
extension.  One process per GPU; the domain is cut into slabs along the
runout axis x at block boundaries.  A rank owns the particles whose base
block has block-x in [bx0, bx1) and the grid blocks in that range.

Per step, after the fused kernel (libsmpm.so, include/smpm.h):
  1. partial node sums of blocks outside the slab go to their owner, which
     adds them (insert-if-absent);
  2. the owner sends the full sums of its first block layer (bx == bx0) back
     to the left neighbour, whose particles' stencils reach it -- both sides
     of an interface then hold identical bits;
  3. particles whose new base block left the slab travel as 128-byte records
     and are binned by the receiver (their P2G was already done).
n_active / n_blocks are sums over owned blocks; the CFL bound uses the global
max |v|.  Transport is torch.distributed point-to-point (NCCL over NVLink on
a GPU box; gloo with host staging in the CPU tests).
"""

import ctypes

import numpy as np

from . import _lib
from .solver import PHASES, Simulation, StepStats

BLOCK_REC_BYTES = 2064  # key, node mask, 64 nodes x 8 floats (deterministic mode: 4112, int64 sums)
PARTICLE_REC_BYTES = 128
INT32_MIN = -(1 << 31)
INT32_MAX = (1 << 31) - 1


def base_block_x(x, h):
    """Block-x of each particle's base node: floor(floor(x/h - 0.5) / 4),
    computed like the device (fp64, same inv_h)."""
    inv_h = 1.0 / float(h)
    base = np.floor(np.asarray(x, dtype=np.float64)[:, 0] * inv_h - 0.5).astype(np.int64)
    return base >> 2


def slab_bounds(bx, world):
    """Block-aligned cut points giving each rank ~N/world particles.
    Returns [(bx0, bx1)] with bx0 of rank 0 = -inf and bx1 of the last = +inf
    (as int32 sentinels)."""
    bx = np.asarray(bx, dtype=np.int64)
    if world == 1:
        return [(INT32_MIN, INT32_MAX)]
    order = np.sort(bx)
    cuts = []
    for r in range(1, world):
        c = int(order[min(len(order) - 1, (r * len(order)) // world)])
        cuts.append(c)
    # strictly increasing, every slab at least 2 blocks wide so contributions
    # to a block come from at most two ranks
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1] + 2)
    lo = [INT32_MIN] + cuts
    hi = cuts + [INT32_MAX]
    return list(zip(lo, hi))


def partition(particles, h, world):
    """Split a ParticleSet into per-rank index arrays (by base block) and the
    slab bounds.  Every particle lands in exactly one slab."""
    bx = base_block_x(particles.x, h)
    bounds = slab_bounds(bx, world)
    parts = [np.nonzero((bx >= lo) & (bx < hi))[0] for lo, hi in bounds]
    return bounds, parts


def subset(ps, idx):
    from .solver import ParticleSet

    return ParticleSet(**{k: np.ascontiguousarray(getattr(ps, k)[idx]) for k in
                          ("x", "v", "C", "F", "m", "V0", "mat_id", "sigma", "jac")})


class _Transport:
    """Neighbour point-to-point exchange of byte buffers (device tensors)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    def _dev(self, t):
        return t if self.nccl else t.cpu()

    def exchange(self, to_left, to_right):
        """to_left / to_right: uint8 CUDA tensors (or None).  Returns the
        buffers received from the left and the right neighbour (CUDA)."""
        import torch

        dist = self.dist
        left = self.rank - 1 if self.rank > 0 else None
        right = self.rank + 1 if self.rank + 1 < self.world else None
        dev = self.device
        # sizes first (one persistent int64[4] tensor: send l, send r, recv l, recv r)
        n_to = {"l": 0 if to_left is None else to_left.numel(), "r": 0 if to_right is None else to_right.numel()}
        sz_dev = dev if self.nccl else torch.device("cpu")
        if left is None and right is None:
            return None, None
        if getattr(self, "_sz", None) is None:
            self._sz = torch.zeros(4, dtype=torch.int64, device=sz_dev)
        sz = self._sz
        sz.copy_(torch.tensor([n_to["l"], n_to["r"], 0, 0], dtype=torch.int64))
        ops = []
        if left is not None:
            ops += [dist.P2POp(dist.isend, sz[0:1], left, self.group), dist.P2POp(dist.irecv, sz[2:3], left, self.group)]
        if right is not None:
            ops += [dist.P2POp(dist.isend, sz[1:2], right, self.group), dist.P2POp(dist.irecv, sz[3:4], right, self.group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        nl, nr = (int(v) for v in sz[2:].tolist())
        bufs = {}
        ops = []
        if left is not None:
            if n_to["l"]:
                ops.append(dist.P2POp(dist.isend, self._dev(to_left), left, self.group))
            if nl:
                bufs["l"] = torch.empty(nl, dtype=torch.uint8, device=sz_dev)
                ops.append(dist.P2POp(dist.irecv, bufs["l"], left, self.group))
        if right is not None:
            if n_to["r"]:
                ops.append(dist.P2POp(dist.isend, self._dev(to_right), right, self.group))
            if nr:
                bufs["r"] = torch.empty(nr, dtype=torch.uint8, device=sz_dev)
                ops.append(dist.P2POp(dist.irecv, bufs["r"], right, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        out_l = bufs.get("l")
        out_r = bufs.get("r")
        out_l = None if out_l is None else out_l.to(dev)
        out_r = None if out_r is None else out_r.to(dev)
        if dev.type == "cuda":
            torch.cuda.synchronize()  # the library consumes these on its own stream
        return out_l, out_r

    def gather(self, arr):
        """Every rank's float64 vector, stacked (one collective)."""
        import torch

        dist = self.dist
        dev = self.device if self.nccl else torch.device("cpu")
        t = torch.tensor(np.asarray(arr, dtype=np.float64), device=dev)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return np.stack([o.cpu().numpy() for o in out])

    def allreduce(self, arr, op="sum"):
        import torch

        dist = self.dist
        dev = self.device if self.nccl else torch.device("cpu")
        t = torch.tensor(np.asarray(arr, dtype=np.float64), device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()


class DistributedSimulation:
    """Slab-decomposed Simulation: call on every rank with that rank's
    particles (``partition``/``subset``), its slab bounds and the global id of
    its first particle."""

    def __init__(self, particles, config, materials, boundaries, bounds, pid_base, group=None,
                 migrant_capacity=None, block_capacity=None, record_conservation=False):
        torch = _lib.torch_cuda()
        self.config = config
        self.tr = _Transport(group)
        self.bounds = bounds
        n = particles.n
        # capacity: local particles + arrivals (slabs rebalance slowly)
        cap_mig = int(migrant_capacity or max(4096, n // 8))
        self._cap_mig = cap_mig
        self.sim = Simulation(particles, config, materials, boundaries, record_conservation=record_conservation,
                              block_capacity=block_capacity, particle_capacity=n + 4 * cap_mig,
                              slab=(int(bounds[0]), int(bounds[1]), int(pid_base), cap_mig),
                              host_sync="on_access")  # the local set changes size with migration
        self._h = self.sim._h
        self.lib = _lib.load()
        self.t = 0.0
        self.step_count = 0
        self.migrated = 0  # particles received from neighbours so far
        self._torch = torch
        self._gvmax = None  # global max |v| after the last step (next dt bound)
        self._xcap = [4096, 4096, 4096]  # halo exchange buffers (blocks) per pack mode
        self._xbuf = [None, None, None]
        self._rec = int(self.lib.smpm_sim_exchange_record_bytes(self._h))
        # Prologues (step 0, and replays after a rank's P2G outgrew its
        # fixed-point scales or grid capacity) run on all ranks together and
        # before the halo exchange; the fixed-point bounds are the max over
        # ranks, so in deterministic mode every rank scales its int64 partial
        # sums alike and they add exactly.
        self.det = bool(config.deterministic)
        self._replay = False
        _lib.check(self.lib.smpm_sim_set_external_bounds(self._h, 1), "external bounds")
        self._coordinated_prologue()
        self._exchange()

    def _coordinated_prologue(self):
        """P2G of the current particles on every rank with the max over ranks
        of the fixed-point bounds (collective; deterministic mode)."""
        while True:
            local = (ctypes.c_float * 3)()
            _lib.check(self.lib.smpm_sim_prologue_begin(self._h, local), "prologue")
            glob = self.tr.gather(list(local)).max(axis=0)
            rc = self.lib.smpm_sim_prologue_finish(self._h, (ctypes.c_float * 3)(*glob))
            if rc not in (0, _lib.RETRY):
                _lib.check(rc, "prologue")
            if not self.tr.gather([float(rc == _lib.RETRY)]).max():
                break
        self._agree_bounds()

    def _agree_bounds(self):
        """The next launch scales its P2G with the max over ranks of the
        contribution bounds each rank just measured (collective)."""
        b = (ctypes.c_float * 3)()
        _lib.check(self.lib.smpm_sim_p2g_bounds(self._h, 0, b), "bounds")
        glob = self.tr.gather(list(b)).max(axis=0)
        _lib.check(self.lib.smpm_sim_p2g_bounds(self._h, 1, (ctypes.c_float * 3)(*glob)), "bounds")

    # -- exchange -------------------------------------------------------------
    def _pack(self, mode):
        """Halo block records of one kind into a persistent buffer (grown on
        demand; the C call reports the count, and overflow as CAPACITY)."""
        torch = self._torch
        while True:
            cap, buf = self._xcap[mode], self._xbuf[mode]
            if buf is None:
                buf = self._xbuf[mode] = torch.empty(cap * self._rec, dtype=torch.uint8, device="cuda")
            n = ctypes.c_int64(0)
            rc = self.lib.smpm_sim_exchange_pack(self._h, mode, _lib.ptr(buf), cap, ctypes.byref(n))
            if rc == _lib.ERR_CAPACITY and n.value > cap:
                self._xcap[mode], self._xbuf[mode] = 2 * int(n.value), None
                continue
            _lib.check(rc, "pack")
            return buf[: n.value * self._rec] if n.value else None

    def _unpack(self, buf, set_):
        if buf is None or buf.numel() == 0:
            return
        _lib.check(self.lib.smpm_sim_exchange_unpack(self._h, _lib.ptr(buf), buf.numel() // self._rec,
                                                     int(set_)), "unpack")

    def _migrants(self, side):
        torch = self._torch
        n = ctypes.c_int64(0)
        _lib.check(self.lib.smpm_sim_migrants(self._h, side, None, 0, ctypes.byref(n)), "migrants")
        if n.value == 0:
            return None
        out = torch.empty(n.value * PARTICLE_REC_BYTES, dtype=torch.uint8, device="cuda")
        _lib.check(self.lib.smpm_sim_migrants(self._h, side, _lib.ptr(out), n.value, ctypes.byref(n)), "migrants")
        return out

    def _frame(self, blocks, parts):
        """One message: a 16-byte header (int64 byte count of the block
        records, pad) keeping the records 16-byte aligned, the block records
        (exchange_record_bytes each), then particle records."""
        torch = self._torch
        if blocks is None and parts is None:
            return None
        nbytes = 0 if blocks is None else blocks.numel()
        head = torch.tensor([nbytes, 0], dtype=torch.int64, device="cuda").view(torch.uint8)
        return torch.cat([head] + [b for b in (blocks, parts) if b is not None])

    def _unframe(self, msg):
        if msg is None or msg.numel() == 0:
            return None, None
        nbytes = int(msg[:8].view(self._torch.int64).item())
        blocks = msg[16:16 + nbytes].to("cuda")
        parts = msg[16 + nbytes:].to("cuda")
        return (blocks if nbytes else None), (parts if parts.numel() else None)

    def _exchange(self):
        """Two neighbour rounds per step: (1) partial sums of halo blocks and
        departing particles, (2) the owners' boundary-layer sums back to the
        left neighbour (which needs (1) applied first)."""
        self._torch.cuda.synchronize()
        self.sim.stream.synchronize()
        to_l = self._frame(self._pack(0), self._migrants(0))
        to_r = self._frame(self._pack(1), self._migrants(1))
        for msg in self.tr.exchange(to_l, to_r):
            blocks, parts = self._unframe(msg)
            self._unpack(blocks, False)
            if parts is not None:
                self.migrated += parts.numel() // PARTICLE_REC_BYTES
                _lib.check(self.lib.smpm_sim_accept(self._h, _lib.ptr(parts), parts.numel() // PARTICLE_REC_BYTES),
                           "accept")
        self.sim.stream.synchronize()
        _, from_r = self.tr.exchange(self._pack(2), None)
        self._unpack(from_r, True)
        self.sim.stream.synchronize()

    # -- API ------------------------------------------------------------------
    def dt_bound(self):
        if self._gvmax is None:
            self._gvmax = float(self.tr.allreduce([float(self.lib.smpm_sim_vmax(self._h))], "max")[0])
        return self.config.cfl * self.config.h / (self.sim._wave_speed + self._gvmax)

    def step(self, dt=None):
        cfg = self.config
        if dt is None:
            dt = cfg.dt if cfg.dt is not None else self.dt_bound()
        if self._replay:  # a rank's P2G outgrew its scales / capacity: all ranks redo it
            self._coordinated_prologue()
            self._exchange()
            self._replay = False
        st = self.sim.step(float(dt))
        # one collective for the step's global stats, the next dt bound and,
        # in deterministic mode, the next launch's bounds and replay flags
        b = (ctypes.c_float * 3)()
        _lib.check(self.lib.smpm_sim_p2g_bounds(self._h, 0, b), "bounds")
        extra = [*b, float(self.lib.smpm_sim_prologue_needed(self._h))]
        rows = self.tr.gather([float(self.lib.smpm_sim_vmax(self._h)), st.n_active, st.n_allocated,
                               st.mass_sum or 0.0, *(st.mom_sum if st.mom_sum is not None else (0.0, 0.0, 0.0)),
                               *extra])
        self._gvmax = float(rows[:, 0].max())
        red = rows[:, 1:7].sum(axis=0)
        glob = rows[:, 7:10].max(axis=0)
        _lib.check(self.lib.smpm_sim_p2g_bounds(self._h, 1, (ctypes.c_float * 3)(*glob)), "bounds")
        # (setting the global bounds also runs the precision check on them)
        self._replay = bool(rows[:, 10].max()) or bool(self.lib.smpm_sim_prologue_needed(self._h))
        if not self._replay:
            self._exchange()
        self.t += st.dt
        self.step_count += 1
        return StepStats(step=self.step_count, t=self.t, dt=st.dt, n_active=int(red[0]), n_allocated=int(red[1]),
                         times=dict(st.times), mass_sum=float(red[2]) if st.mass_sum is not None else None,
                         mom_sum=red[3:6] if st.mom_sum is not None else None)

    def local_particles(self):
        """(pid, x, v) of the particles this rank owns."""
        ns = int(self.lib.smpm_sim_num_stored(self._h))
        pid = np.empty(max(ns, 1), dtype=np.int64)
        x = np.empty((max(ns, 1), 3))
        v = np.empty((max(ns, 1), 3))
        n = ctypes.c_int64(0)
        _lib.check(self.lib.smpm_sim_get_local(self._h, ctypes.byref(n), pid.ctypes.data, x.ctypes.data,
                                               v.ctypes.data), "get local")
        k = int(n.value)
        return pid[:k], x[:k], v[:k]

    def gather_particles(self):
        """All ranks' (x, v) ordered by global particle id (on every rank)."""
        import torch.distributed as dist

        pid, x, v = self.local_particles()
        objs = [None] * self.tr.world
        dist.all_gather_object(objs, (pid, x, v), group=self.tr.group)
        P = np.concatenate([o[0] for o in objs])
        X = np.concatenate([o[1] for o in objs])
        V = np.concatenate([o[2] for o in objs])
        order = np.argsort(P)
        return P[order], X[order], V[order]


__all__ = ["DistributedSimulation", "partition", "slab_bounds", "subset", "base_block_x", "PHASES"]

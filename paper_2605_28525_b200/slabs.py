"""Multi-GPU slab decomposition of the sparse-MPM step.

The reference is single-process (its paper lists multi-GPU as future work,
/root/reference/PAPER.md:335-337); this module is the B200 build's
extension.  One process per GPU; the domain is cut into slabs along the
runout axis x at block boundaries.  A rank owns the particles whose base
block has block-x in [bx0, bx1) and the grid blocks in that range.

Per step, after the fused kernel (libsmpm.so, include/smpm.h), all on the
simulation's stream with one host sync per step:
  1. partial node sums of blocks outside the slab go to their owner, which
     adds them (insert-if-absent), in the same frame as the particles whose
     new base block left the slab (128-byte records, binned by the receiver;
     their P2G was already done);
  2. the owner sends the full sums of its first block layer (bx == bx0) back
     to the left neighbour, whose particles' stencils reach it -- both sides
     of an interface then hold identical bits;
  3. one all-gather of the step statistics (n_active, n_blocks, conservation
     sums, max |v| for the next CFL bound, P2G bounds, replay / overflow
     flags, frame counts), then the stream sync.
Frames have a fixed capacity with the counts in a device header, so they are
sent whole (no size round trip); capacities grow from the gathered counts.
When the particle counts drift apart by more than 10 % the slab faces move
(rebalancing).  Transport is torch.distributed point-to-point (NCCL over
NVLink on a GPU box; gloo with host staging in the CPU tests).
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

    def exchange_frames(self, send_l, send_r, recv_l, recv_r):
        """Whole fixed-size frames with both neighbours, one grouped batch, no
        size round trip.  NCCL: posted on the current (simulation) stream, which
        then waits for them -- no host sync.  gloo (CPU tests): host-staged."""
        dist = self.dist
        left = self.rank - 1 if self.rank > 0 else None
        right = self.rank + 1 if self.rank + 1 < self.world else None
        pairs = []  # (peer, send, recv)
        if left is not None:
            pairs.append((left, send_l, recv_l))
        if right is not None:
            pairs.append((right, send_r, recv_r))
        if not pairs:
            return
        if self.nccl:
            ops = []
            for peer, snd, rcv in pairs:
                if snd is not None:
                    ops.append(dist.P2POp(dist.isend, snd, peer, self.group))
                if rcv is not None:
                    ops.append(dist.P2POp(dist.irecv, rcv, peer, self.group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            return
        import torch

        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()
        ops, back = [], []
        for peer, snd, rcv in pairs:
            if snd is not None:
                ops.append(dist.P2POp(dist.isend, snd.cpu(), peer, self.group))
            if rcv is not None:
                tmp = torch.empty(rcv.numel(), dtype=rcv.dtype)
                ops.append(dist.P2POp(dist.irecv, tmp, peer, self.group))
                back.append((rcv, tmp))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for rcv, tmp in back:
            rcv.copy_(tmp, non_blocking=False)

    def all_gather_dev(self, vec, out):
        """Every rank's device vector into out (world * len), one collective on
        the current stream (NCCL) or host-staged (gloo)."""
        dist = self.dist
        if self.nccl:
            dist.all_gather_into_tensor(out, vec, group=self.group)
            return
        import torch

        parts = [torch.empty(vec.numel(), dtype=vec.dtype) for _ in range(self.world)]
        dist.all_gather(parts, vec.cpu(), group=self.group)
        out.copy_(torch.cat(parts))

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
                 migrant_capacity=None, block_capacity=None, record_conservation=False, frame_blocks=None,
                 frame_particles=None, rebalance=True, rebalance_threshold=0.10):
        torch = _lib.torch_cuda()
        self.config = config
        self.tr = _Transport(group)
        self.bounds = bounds
        n = particles.n
        # capacity: local particles + arrivals (slabs rebalance slowly)
        cap_mig = int(migrant_capacity or max(4096, n // 8))
        self._cap_mig = cap_mig
        self._cap_store = n + 4 * cap_mig  # particle storage slots (live + holes + arrivals)
        self.sim = Simulation(particles, config, materials, boundaries, record_conservation=record_conservation,
                              block_capacity=block_capacity, particle_capacity=self._cap_store,
                              slab=(int(bounds[0]), int(bounds[1]), int(pid_base), cap_mig),
                              host_sync="on_access")  # the local set changes size with migration
        self._h = self.sim._h
        self.lib = _lib.load()
        self.t = 0.0
        self.step_count = 0
        self.migrated = 0  # particles received from neighbours so far
        self._torch = torch
        self.pid_base = int(pid_base)
        self._gvmax = None  # global max |v| after the last step (next dt bound)
        # exchange frames: capacities shared by all ranks, grown from the
        # all-gathered counts (half-full -> double)
        self._cap_blocks = int(frame_blocks or 1024)
        self._cap_parts = int(frame_particles or 4096)
        self.frame_growths = 0
        self._L = int(self.lib.smpm_sim_stats_vector_len())
        dev = self.sim.stream.device
        self._vec = torch.zeros(self._L, dtype=torch.float64, device=dev)
        self._rows = torch.zeros(self.tr.world * self._L, dtype=torch.float64, device=dev)
        self._rows_host = torch.zeros(self.tr.world * self._L, dtype=torch.float64).pin_memory()
        # deterministic mode keeps the faces fixed: a rebalance reruns the P2G
        # (coordinated prologue) with freshly measured fixed-point scales, which
        # the 1-GPU run does not, so bitwise equality to 1 GPU would be lost
        self.rebalance = bool(rebalance) and not config.deterministic
        self.rebalance_threshold = float(rebalance_threshold)
        self.rebalances = 0
        self.local_counts = None
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
    def _frames(self):
        """Fixed-capacity device frames (include/smpm.h smpm_sim_frame_*): sends
        of mode 0 (to the left), 1 (to the right) and 2 (owner's layer to the
        left), and the matching receives.  Every rank holds the same capacities
        (grown from the all-gathered counts), so a frame is sent whole."""
        torch = self._torch
        key = (self._cap_blocks, self._cap_parts)
        if getattr(self, "_fkey", None) != key:
            fb = int(self.lib.smpm_sim_frame_bytes(self._h, self._cap_blocks, self._cap_parts))
            fb2 = int(self.lib.smpm_sim_frame_bytes(self._h, self._cap_blocks, 0))
            dev = self.sim.stream.device
            self._f = {k: torch.empty(fb if k[1] != "2" else fb2, dtype=torch.uint8, device=dev)
                       for k in ("s0", "s1", "s2", "r0", "r1", "r2")}
            self._fkey = key
        return self._f

    def _exchange_async(self):
        """Two neighbour rounds on the simulation's stream, no host sync:
        (1) halo partial sums + departing particles, (2) the owners' first
        block layer back to the left neighbour (which needs (1) applied)."""
        f = self._frames()
        cb, cp = self._cap_blocks, self._cap_parts
        lib, h = self.lib, self._h
        has_l, has_r = self.tr.rank > 0, self.tr.rank + 1 < self.tr.world
        if has_l:
            _lib.check(lib.smpm_sim_frame_pack(h, 0, _lib.ptr(f["s0"]), cb, cp), "frame pack")
        if has_r:
            _lib.check(lib.smpm_sim_frame_pack(h, 1, _lib.ptr(f["s1"]), cb, cp), "frame pack")
        self.tr.exchange_frames(f["s0"] if has_l else None, f["s1"] if has_r else None,
                                f["r0"] if has_l else None, f["r1"] if has_r else None)
        if has_l:  # the left neighbour's mode-1 frame
            _lib.check(lib.smpm_sim_frame_unpack(h, _lib.ptr(f["r0"]), cb, cp, 0), "frame unpack")
        if has_r:  # the right neighbour's mode-0 frame
            _lib.check(lib.smpm_sim_frame_unpack(h, _lib.ptr(f["r1"]), cb, cp, 0), "frame unpack")
        if has_l:
            _lib.check(lib.smpm_sim_frame_pack(h, 2, _lib.ptr(f["s2"]), cb, 0), "frame pack")
        self.tr.exchange_frames(f["s2"] if has_l else None, None, None, f["r2"] if has_r else None)
        if has_r:
            _lib.check(lib.smpm_sim_frame_unpack(h, _lib.ptr(f["r2"]), cb, 0, 1), "frame unpack")

    def _stats_async(self):
        """This rank's step statistics, all-gathered on the device, the next
        launch's bounds applied, and a pinned copy of the rows for the host."""
        _lib.check(self.lib.smpm_sim_stats_vector(self._h, _lib.ptr(self._vec)), "stats vector")
        self.tr.all_gather_dev(self._vec, self._rows)
        _lib.check(self.lib.smpm_sim_apply_global(self._h, _lib.ptr(self._rows), self.tr.world), "apply global")
        self._rows_host.copy_(self._rows.view(-1), non_blocking=True)

    def _settle(self, rows):
        """After the sync: mark delivered migrants, frame growth, replays."""
        L = self._L
        rk = self.tr.rank
        cb, cp = self._cap_blocks, self._cap_parts
        # my frames to the left (13, 14) and right (15, 16) arrived unless overflowed
        mask = 0
        if rows[rk, 13] <= cb and rows[rk, 14] <= cp:
            mask |= 1
        if rows[rk, 15] <= cb and rows[rk, 16] <= cp:
            mask |= 2
        _lib.check(self.lib.smpm_sim_migrants_delivered(self._h, mask), "delivered")
        need_b = float(rows[:, [13, 15, 17]].max())
        need_p = float(rows[:, [14, 16]].max())
        overflow = bool(rows[:, 19].max() > 0)
        # proactive growth at half use: identical on every rank (gathered counts)
        if need_b > cb / 2 or need_p > cp / 2:
            self._cap_blocks = max(cb, 1 << int(np.ceil(np.log2(max(2.0 * need_b, 1.0)))))
            self._cap_parts = max(cp, 1 << int(np.ceil(np.log2(max(2.0 * need_p, 1.0)))))
            self.frame_growths += 1
        # the precision check of the next launch's global bounds against this
        # launch's scales (the library makes the same decision at the sync)
        gb, sinv = rows[:, 7:10].max(axis=0), rows[0, 20:23]
        with np.errstate(divide="ignore", invalid="ignore"):  # sinv = 0: fp32 arena, no scales
            underflow = bool(np.any((gb > 0) & (sinv > 0) & (gb.astype(np.float32) / sinv < 262144.0)))
        # every input is gathered, so every rank reaches the same decision
        replay = overflow or bool(rows[:, 10].max() > 0) or underflow
        return replay, overflow

    def _sync_step(self):
        """The one host sync of a distributed step."""
        st = _lib.StepStatsC()
        _lib.check(self.lib.smpm_sim_sync(self._h, ctypes.byref(st)), "sync")
        rows = self._rows_host.numpy().reshape(self.tr.world, self._L).copy()
        return st, rows

    def _exchange(self):
        """Synchronous exchange after a coordinated prologue (construction,
        replays, rebalancing); a frame overflow grows the frames and redoes
        the prologue."""
        import torch

        for _ in range(8):
            with torch.cuda.stream(self.sim.stream):
                self._exchange_async()
                self._stats_async()
            _, rows = self._sync_step()
            replay, overflow = self._settle(rows)
            self._gvmax = float(np.sqrt(rows[:, 0].max()))
            if not overflow:
                return
            self._coordinated_prologue()
        raise RuntimeError("exchange frames did not converge")

    # -- API ------------------------------------------------------------------
    def dt_bound(self):
        return self.config.cfl * self.config.h / (self.sim._wave_speed + self._gvmax)

    def step(self, dt=None):
        """One step on every rank: fused kernels, the device-resident frame
        exchange and one all-gather of the step statistics, with a single
        host sync (the stream synchronisation before the next launch)."""
        import torch

        cfg = self.config
        if self._replay:  # a rank's P2G outgrew its scales / capacity / frames: all ranks redo it
            self._coordinated_prologue()
            self._exchange()
            self._replay = False
        if dt is None:
            dt = cfg.dt if cfg.dt is not None else self.dt_bound()
        rc = self.lib.smpm_sim_step(self._h, float(dt))
        if rc:
            self.sim._raise_status(rc, dt)
        with torch.cuda.stream(self.sim.stream):
            self._exchange_async()
            self._stats_async()
        st, rows = self._sync_step()
        replay, _ = self._settle(rows)
        self._replay = replay
        self._gvmax = float(np.sqrt(rows[:, 0].max()))
        live = rows[:, 12] - rows[:, 14] - rows[:, 16]
        self.local_counts = live
        self.migrated += int(rows[self.tr.rank, 14] + rows[self.tr.rank, 16])
        if self.rebalance and not replay and self.tr.world > 1:
            self._maybe_rebalance(live)
        self.t += st.dt
        self.step_count += 1
        rec = self.sim.record_conservation
        times = {p: 0.0 for p in PHASES}
        times["map_build"] = st.ms_map * 1e-3
        times["grid_update"] = st.ms_grid * 1e-3
        times["g2p"] = st.ms_fused * 1e-3
        return StepStats(step=self.step_count, t=self.t, dt=st.dt, n_active=int(rows[:, 1].sum()),
                         n_allocated=int(rows[:, 2].sum()) * 64, times=times,
                         mass_sum=float(rows[:, 3].sum()) if rec else None,
                         mom_sum=rows[:, 4:7].sum(axis=0) if rec else None)

    # -- rebalancing ----------------------------------------------------------
    def _maybe_rebalance(self, live):
        """Shift the slab faces when the particle counts drift apart by more
        than `rebalance_threshold`: new block-aligned
        cuts from the global block-x histogram, each face moving at most into
        its neighbours' interiors, so particles only migrate to adjacent ranks.
        The next step starts with a coordinated prologue under the new bounds:
        its P2G pass exports the particles now outside each slab and sends the
        halo sums of blocks that changed owner."""
        mean = float(live.mean())
        if mean <= 0 or float(live.max()) <= (1.0 + self.rebalance_threshold) * mean:
            return
        import torch.distributed as dist

        _, x, _ = self.local_particles()
        bx = base_block_x(x, self.config.h)
        lo = int(bx.min()) if bx.size else 0
        hist = np.bincount(bx - lo, minlength=1) if bx.size else np.zeros(0, np.int64)
        objs = [None] * self.tr.world
        stored = int(self.lib.smpm_sim_num_stored(self._h))
        dist.all_gather_object(objs, (lo, hist, tuple(self.bounds), self._cap_mig, self._cap_store, stored),
                               group=self.tr.group)
        g_lo = min(o[0] for o in objs if o[1].size)
        g_hi = max(o[0] + o[1].size for o in objs if o[1].size)
        total = np.zeros(g_hi - g_lo, dtype=np.int64)
        for o_lo, o_hist, *_ in objs:
            if o_hist.size:
                total[o_lo - g_lo:o_lo - g_lo + o_hist.size] += o_hist
        cum = np.cumsum(total)
        old = [o[2] for o in objs]
        world = self.tr.world
        cuts = []
        def left_of(f):  # particles in blocks < f
            f = np.asarray(f)
            return cum[np.clip(f - g_lo - 1, 0, cum.size - 1)] * (f > g_lo)

        for r in range(1, world):
            target = r * cum[-1] / world
            # face f: blocks < f go left; choose the f whose left count is nearest the target
            lo_lim = old[r - 1][0] + 2 if r > 1 else g_lo + 1
            hi_lim = old[r][1] - 2 if r + 1 < world else g_hi - 1
            lo_lim = max(lo_lim, cuts[-1] + 2 if cuts else lo_lim)
            faces = np.arange(lo_lim, hi_lim + 1)
            if faces.size == 0:
                cuts.append(int(old[r][0]))
                continue
            left = left_of(faces)
            # a face moves only as far as the sender's migrant buffer and the
            # receiver's particle storage allow in one step (80 % of each, so
            # the particles that drift across meanwhile still fit); a large
            # imbalance is then levelled over several steps
            moved = left - left_of(old[r][0])
            send_cap = np.where(moved > 0, objs[r][3], objs[r - 1][3])  # moved > 0: rank r -> r - 1
            recv = np.where(moved > 0, r - 1, r)
            room = np.array([objs[q][4] - objs[q][5] for q in recv], dtype=float)
            ok = (np.abs(moved) <= 0.8 * send_cap) & (np.abs(moved) <= 0.8 * room)
            if not ok.any():
                cuts.append(int(old[r][0]))
                continue
            cand = faces[ok]
            cuts.append(int(cand[np.argmin(np.abs(left[ok] - target))]))
        new = [(INT32_MIN if r == 0 else cuts[r - 1], INT32_MAX if r == world - 1 else cuts[r]) for r in range(world)]
        if new == [tuple(b) for b in old]:
            return
        self.bounds = new[self.tr.rank]
        _lib.check(self.lib.smpm_sim_set_slab(self._h, int(self.bounds[0]), int(self.bounds[1]), int(self.pid_base), 0),
                   "set slab")
        self.rebalances += 1
        self._replay = True

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

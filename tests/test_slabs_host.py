"""Host-side logic of the slab decomposition, CPU only: partitioning and the
neighbour exchange protocol over gloo with world_size 2."""

import os
import socket

import numpy as np

from paper_2605_28525_b200 import scenes, slabs


def test_partition_covers_every_particle_once():
    rng = np.random.default_rng(0)
    x = rng.uniform([0, -5, 0], [100, 5, 3], size=(200_000, 3))
    ps = scenes.rest_particles(x, np.full(len(x), 1e-3), 1500.0)

    class _Sc:
        particles = ps

    sc = _Sc()
    for world in (1, 2, 3, 4, 8):
        bounds, parts = slabs.partition(sc.particles, 0.5, world)
        assert len(bounds) == world
        allidx = np.concatenate(parts)
        assert np.array_equal(np.sort(allidx), np.arange(sc.particles.n))
        for (lo, hi), (lo2, _) in zip(bounds[:-1], bounds[1:]):
            assert hi == lo2
        for lo, hi in bounds[1:-1]:
            assert hi - lo >= 2
        if world > 1:
            sizes = np.array([len(p) for p in parts])
            assert sizes.min() > 0.5 * sc.particles.n / world


def test_base_block_matches_device_rule():
    x = np.array([[0.0, 0, 0], [0.049, 0, 0], [0.051, 0, 0], [-0.01, 0, 0], [0.45, 0, 0]])
    bx = slabs.base_block_x(x, 0.1)
    assert list(bx) == [-1, -1, 0, -1, 1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = slabs._Transport(device="cpu")
    left = torch.full((3 + rank,), 10 + rank, dtype=torch.uint8) if rank > 0 else None
    right = torch.full((5 + rank,), 20 + rank, dtype=torch.uint8) if rank + 1 < world else None
    got_l, got_r = tr.exchange(left, right)
    red = tr.allreduce([rank + 1.0], "sum")
    mx = tr.allreduce([rank + 1.0], "max")
    q.put((rank, None if got_l is None else got_l.tolist(), None if got_r is None else got_r.tolist(),
           float(red[0]), float(mx[0])))
    dist.barrier()
    dist.destroy_process_group()


def test_neighbour_exchange_gloo():
    import torch.multiprocessing as mp

    world = 3
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, gl, gr, red, mx = q.get()
        res[r] = (gl, gr, red, mx)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    # rank r receives from its left neighbour what r-1 sent right, and vice versa
    assert res[0][0] is None and res[0][1] == [11] * 4
    assert res[1][0] == [20] * 5 and res[1][1] == [12] * 5
    assert res[2][0] == [21] * 6 and res[2][1] is None
    assert all(v[2] == 6.0 and v[3] == 3.0 for v in res.values())


def _frame_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = slabs._Transport(device="cpu")
    size = 64  # fixed frame size: no size round trip
    s_l = torch.full((size,), 100 + rank, dtype=torch.uint8) if rank > 0 else None
    s_r = torch.full((size,), 200 + rank, dtype=torch.uint8) if rank + 1 < world else None
    r_l = torch.zeros(size, dtype=torch.uint8) if rank > 0 else None
    r_r = torch.zeros(size, dtype=torch.uint8) if rank + 1 < world else None
    tr.exchange_frames(s_l, s_r, r_l, r_r)
    # round 2: only leftward frames (the owners' layer sums)
    s2 = torch.full((size,), 50 + rank, dtype=torch.uint8) if rank > 0 else None
    r2 = torch.zeros(size, dtype=torch.uint8) if rank + 1 < world else None
    tr.exchange_frames(s2, None, None, r2)
    vec = torch.tensor([rank, 10.0 * rank], dtype=torch.float64)
    out = torch.zeros(2 * world, dtype=torch.float64)
    tr.all_gather_dev(vec, out)
    q.put((rank, None if r_l is None else int(r_l[0]), None if r_r is None else int(r_r[0]),
           None if r2 is None else int(r2[0]), out.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_fixed_size_frame_exchange_gloo():
    """The distributed step's transport: whole fixed-size frames with both
    neighbours in one batch (no size round trip), a leftward second round,
    and the device all-gather of the stats vector (gloo, world 3)."""
    import torch.multiprocessing as mp

    world = 3
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_frame_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, gl, gr, g2, out = q.get()
        res[r] = (gl, gr, g2, out)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res[0][0] is None and res[0][1] == 101 and res[0][2] == 51
    assert res[1][0] == 200 and res[1][1] == 102 and res[1][2] == 52
    assert res[2][0] == 201 and res[2][1] is None and res[2][2] is None
    for r in range(world):
        assert res[r][3] == [0.0, 0.0, 1.0, 10.0, 2.0, 20.0]

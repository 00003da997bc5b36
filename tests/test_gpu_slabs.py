"""Slab decomposition on 2 ranks vs 1 GPU (SURVEY section 8e gate).

Two processes share the box's single B200 and talk over gloo (host-staged
buffers); on an 8-GPU box the same code runs one rank per GPU over NCCL.
Particles are given enough x velocity to cross the slab cut, so halo sums,
the boundary-layer send-back and particle migration are all exercised."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STEPS = 8


def _scene(det=False):
    from tests.test_gpu_sim import column_scene

    ps, cfg, mats, bc = column_scene(bcs="mixed", vx=3.0, size=(1.2, 0.2, 0.3))
    cfg.deterministic = det
    return ps, cfg, mats, bc


def _dt_sequence(ps, cfg, mats, bc, steps=STEPS):
    from paper_2605_28525_b200.solver import Simulation

    sim = Simulation(ps.copy(), cfg, mats, bc, block_capacity=1 << 14)
    out = []
    for _ in range(steps):
        dt = 0.8 * sim.dt_bound()
        st = sim.step(dt)
        out.append((dt, st.n_active, st.n_allocated))
    return out, sim.particles.x.copy(), sim.particles.v.copy()


def _worker(rank, world, port, dts, outdir, det=False, threshold=0.10):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_28525_b200 import slabs

    ps, cfg, mats, bc = _scene(det)
    bounds, parts = slabs.partition(ps, cfg.h, world)
    local = slabs.subset(ps, parts[rank])
    pid_base = int(sum(len(p) for p in parts[:rank]))
    # partition keeps global order inside a slab only if particles are sorted by
    # slab; map local -> global ids explicitly through the pid base trick
    assert np.all(np.diff(parts[rank]) > 0)
    ds = slabs.DistributedSimulation(local, cfg, mats, bc, bounds[rank], pid_base, block_capacity=1 << 14,
                                     rebalance_threshold=threshold)
    stats = []
    for dt, _, _ in dts:
        st = ds.step(dt)
        stats.append((st.n_active, st.n_allocated))
    pid, x, v = ds.gather_particles()
    moved = ds.tr.allreduce([ds.migrated], "sum")
    # pid -> original index
    order = np.concatenate(parts)
    if rank == 0:
        np.savez(os.path.join(outdir, "dist.npz"), stats=np.array(stats), pid=order[pid], x=x, v=v,
                 counts=np.array([len(p) for p in parts]), moved=moved, rebalances=ds.rebalances,
                 growths=ds.frame_growths, final_counts=np.array(ds.local_counts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kernel", ["auto", "ws"])
def test_two_slabs_match_single_gpu(tmp_path, monkeypatch, kernel):
    """kernel "ws": the warp-specialised fused kernel,
    which this scene is too small to get by default, with its slab-migration
    path (departing particles copied out by the producer warps)."""
    import torch.multiprocessing as mp

    if kernel != "auto":
        monkeypatch.setenv("SMPM_FUSED", kernel)  # inherited by the spawned ranks
    ps, cfg, mats, bc = _scene()
    dts, x1, v1 = _dt_sequence(ps, cfg, mats, bc)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, dts, str(tmp_path)), nprocs=2, join=True)
    d = np.load(tmp_path / "dist.npz")
    assert d["counts"].min() > 0.3 * ps.n  # both slabs populated
    assert d["moved"][0] > 0  # particles crossed the slab cut
    stats = d["stats"]
    # step 1 is computed from identical initial positions: exact
    assert stats[0][0] == dts[0][1]
    assert stats[0][1] == dts[0][2]
    for s in range(STEPS):
        assert abs(int(stats[s][0]) - dts[s][1]) <= 2e-3 * dts[s][1], s
        assert abs(int(stats[s][1]) - dts[s][2]) <= 2e-3 * dts[s][2], s
    assert len(d["pid"]) == ps.n and np.array_equal(np.sort(d["pid"]), np.arange(ps.n))
    x = np.empty_like(d["x"])
    v = np.empty_like(d["v"])
    x[d["pid"]] = d["x"]
    v[d["pid"]] = d["v"]
    assert np.abs(x - x1).max() < 1e-6 * np.abs(x1).max()
    assert np.abs(v - v1).max() < 1e-4 * np.abs(v1).max()


def test_two_slabs_bitwise_equal_single_gpu_in_deterministic_mode(tmp_path):
    """SURVEY 8e gate, exact: with int64 fixed-point grid sums and bounds
    agreed over ranks, the 2-rank run reproduces the 1-GPU run bit for bit --
    active sets and counts every step, positions and velocities."""
    import torch.multiprocessing as mp

    ps, cfg, mats, bc = _scene(det=True)
    dts, x1, v1 = _dt_sequence(ps, cfg, mats, bc)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, dts, str(tmp_path), True), nprocs=2, join=True)
    d = np.load(tmp_path / "dist.npz")
    assert d["moved"][0] > 0
    assert [tuple(r) for r in d["stats"]] == [(a, b) for _, a, b in dts]
    x = np.empty_like(d["x"])
    v = np.empty_like(d["v"])
    x[d["pid"]] = d["x"]
    v[d["pid"]] = d["v"]
    assert np.array_equal(x, x1) and np.array_equal(v, v1)


def test_drifting_slabs_rebalance(tmp_path):
    """SURVEY 8e rebalancing: the column drifts across the cut (vx = 3 m/s),
    the particle counts drift apart and the faces move (threshold 2 % here),
    the frames grow from their minimum with the halo and migrant stream --
    without a capacity error, and the run still matches the 1-GPU run."""
    import torch.multiprocessing as mp

    ps, cfg, mats, bc = _scene(det=False)
    steps = 30
    dts, x1, v1 = _dt_sequence(ps, cfg, mats, bc, steps)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(2, port, dts, str(tmp_path), False, 0.02), nprocs=2, join=True)
    d = np.load(tmp_path / "dist.npz")
    assert int(d["rebalances"]) >= 1, "the faces never moved"
    assert d["moved"][0] > 0
    fc = d["final_counts"]
    assert fc.max() <= 1.10 * fc.mean() + 64, fc  # balanced after rebalancing
    assert len(d["pid"]) == ps.n and np.array_equal(np.sort(d["pid"]), np.arange(ps.n))
    x = np.empty_like(d["x"])
    v = np.empty_like(d["v"])
    x[d["pid"]] = d["x"]
    v[d["pid"]] = d["v"]
    assert np.abs(x - x1).max() < 1e-6 * np.abs(x1).max()
    assert np.abs(v - v1).max() < 1e-4 * np.abs(v1).max()


def _landslide_worker(rank, world, port, outdir, cap):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_28525_b200 import scenes
    from paper_2605_28525_b200.slabs import DistributedSimulation

    slab = scenes.landslide_slabs(world, fraction=0.02)[rank]
    sc = scenes.landslide(fraction=0.02, columns=(slab[2], slab[3]))
    per_col = sc.particles.n // max(1, slab[3] - slab[2])
    sim = DistributedSimulation(sc.particles, sc.config, sc.materials, sc.boundaries, (slab[0], slab[1]),
                                pid_base=slab[2] * per_col, migrant_capacity=cap)
    counts = [sc.particles.n]
    for _ in range(6):
        sim.step()
        counts.append(int(sim.local_counts[rank]))
    if rank == 0:
        np.savez(os.path.join(outdir, "ls.npz"), rebalances=sim.rebalances, counts=np.array(counts),
                 n=sum(int(c) for c in sim.local_counts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cap", [None, 2_000_000], ids=["default_buffers", "large_buffers"])
def test_imbalanced_landslide_slabs_rebalance_within_capacity(tmp_path, cap):
    """The bench's slab setup on a small release (bench.py --gpus N --scale
    0.02: 17 lattice columns on rank 0, 3 on rank 1; one block of x holds
    ~0.8M particles).  A face moves only as far as 80 % of the sender's
    migrant buffer and of the receiver's free storage allow: with the default
    buffers (n / 8) no move fits and the run continues unbalanced (it used to overflow the migrant
    buffer: a capacity error); with buffers for a block the faces move."""
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_landslide_worker, args=(2, port, str(tmp_path), cap), nprocs=2, join=True)
    d = np.load(tmp_path / "ls.npz")
    assert int(d["n"]) == 2_020_000  # nobody lost
    c = d["counts"]
    if cap is None:
        assert int(d["rebalances"]) == 0
    else:
        assert int(d["rebalances"]) >= 1
        assert c[-1] < c[0]  # rank 0 handed particles over

"""Scenario runs, the dense baseline and the CLI on the GPU (cases follow the
reference's T/test_bench.py and T/test_scenarios_io.py).  The shipped scenes
(tests/golden/scenarios/, copied from the reference package) load unchanged
and run on the GPU step; the active-node series and the dense allocation are
checked bit-exactly against the oracle."""

from pathlib import Path

import numpy as np
import pytest
import yaml
from click.testing import CliRunner

from paper_2605_28525_b200 import bench, scenarios
from paper_2605_28525_b200.cli import main as cli_main

pytestmark = pytest.mark.gpu
SCEN = Path(__file__).resolve().parent / "golden" / "scenarios"
STEMS = ("granular_collapse", "localized_flow", "sliding_box", "terrain_demo")


def _lockstep(o, sc, backend, steps):
    """GPU Simulation and the oracle in lock step, the oracle restarted from
    the GPU state each step (per-step parity, as in test_gpu_sim); returns
    [(gpu stats, oracle stats)]."""
    cfg = sc.sim
    sim = scenarios.build_simulation(sc, backend=backend)
    mats = [r.model for r in sc.materials]
    out = []
    for _ in range(steps):
        state = sim.particles.copy()
        ref = o.OracleSimulation(state, cfg.h, cfg.gravity, mats, sc.boundaries, backend=backend,
                                 deterministic=True, node_min=cfg.node_min, node_max=cfg.node_max)
        dt = 0.9 * min(sim.dt_bound(), ref.dt_bound())
        out.append((sim.step(dt), ref.step(dt)))
    return sim, out


@pytest.mark.parametrize("stem", STEMS)
def test_shipped_scene_runs_like_oracle(oracle, stem):
    sc = scenarios.load_config(SCEN / f"{stem}.yaml")
    sim, pairs = _lockstep(oracle, sc, "hash", 4)
    assert [(g.n_active, g.n_allocated) for g, _ in pairs] == [(r["n_active"], r["n_allocated"]) for _, r in pairs]
    m = bench.run(sc, backend="hash", max_steps=4)
    assert m.n_steps == 4 and m.backend == "hash" and m.n_particles == scenarios.build_particles(sc).n
    assert m.r_active == bench.sparsity_ratio(m.n_active_series, m.n_dense) > 1


def test_dense_baseline_allocates_the_domain(oracle):
    sc = scenarios.load_config(SCEN / "terrain_demo.yaml")
    sim, pairs = _lockstep(oracle, sc, "dense", 3)
    assert [(g.n_active, g.n_allocated) for g, _ in pairs] == [(r["n_active"], r["n_allocated"]) for _, r in pairs]
    assert all(g.n_allocated == sim.n_dense for g, _ in pairs)
    dense = bench.run(sc, backend="dense", max_steps=3)
    sparse = bench.run(sc, backend="hash", max_steps=3)
    assert dense.n_active_series == sparse.n_active_series
    rep = bench.compare(dense, sparse)
    assert rep.memory_reduction == dense.n_dense / sparse.peak_alloc_nodes
    assert rep.speedup > 0 and set(rep.phase_table()) == set(bench.PHASES)


def test_dense_and_hash_trajectories_agree():
    sc = scenarios.load_config(SCEN / "granular_collapse.yaml")
    a = scenarios.build_simulation(sc, backend="dense")
    b = scenarios.build_simulation(sc, backend="hash")
    for _ in range(5):
        dt = 0.8 * b.dt_bound()
        sa, sb = a.step(dt), b.step(dt)
        assert sa.n_active == sb.n_active
    xa, xb = a.particles.x, b.particles.x
    assert np.abs(xa - xb).max() <= 1e-6 * np.abs(xb).max()


def test_frames_and_metrics_output(tmp_path):
    sc = scenarios.load_config(SCEN / "terrain_demo.yaml")
    m = bench.run(sc, max_steps=6, out_dir=tmp_path, record_conservation=True)
    frames = sorted(tmp_path.glob("frame_*.csv"))
    assert frames and frames[0].name == "frame_000000.csv"
    pos, vel = scenarios.read_particles(frames[0])
    assert pos.shape == (m.n_particles, 3)
    rows, summary = scenarios.read_metrics(tmp_path / "metrics.csv")
    assert len(rows) == m.n_steps and summary["physics_hash"] == sc.physics_hash()
    assert "mass_sum_kg" in rows[0] and float(rows[0]["mass_sum_kg"]) > 0


def test_async_frames_equal_synchronous_frames(tmp_path):
    """Frames through the device snapshot + side-stream copy + writer thread
    (frames.py) are byte-identical to frames written from the host arrays at
    the same steps (deterministic mode: both runs are bitwise equal)."""
    sc = scenarios.load_config(SCEN / "granular_collapse.yaml")
    sc.fps = 200.0  # a frame every 5 ms of simulated time
    a, b = tmp_path / "async", tmp_path / "sync"
    bench.run(sc, max_steps=40, out_dir=a, deterministic=True, async_frames=True)
    bench.run(sc, max_steps=40, out_dir=b, deterministic=True, async_frames=False)
    fa, fb = sorted(a.glob("frame_*.csv")), sorted(b.glob("frame_*.csv"))
    assert len(fa) >= 2 and [f.name for f in fa] == [f.name for f in fb]
    for x, y in zip(fa, fb):
        assert x.read_bytes() == y.read_bytes(), x.name


def test_compare_rejections():
    sc = scenarios.load_config(SCEN / "terrain_demo.yaml")
    a = bench.run(sc, backend="hash", max_steps=2)
    b = bench.run(sc, backend="scan", max_steps=3)
    with pytest.raises(ValueError):
        bench.compare(a, b)
    d = bench.run(sc, backend="dense", max_steps=2)
    with pytest.raises(ValueError):
        bench.compare(d, d)
    with pytest.raises(ValueError):
        bench.compare(d, b)


def test_cli_run_and_compare(tmp_path):
    cfg = str(SCEN / "sliding_box.yaml")
    r = CliRunner().invoke(cli_main, ["run", cfg, "--backend", "hash", "--max-steps", "3", "--out", str(tmp_path)])
    assert r.exit_code == 0, r.output
    assert "sparsity ratio:" in r.output and (tmp_path / "metrics.csv").exists()
    out = tmp_path / "cmp.csv"
    r = CliRunner().invoke(cli_main, ["compare", cfg, "--sparse-backend", "hash", "--max-steps", "3",
                                      "--out", str(out)])
    assert r.exit_code == 0, r.output
    rows, summary = scenarios.read_metrics(out)
    assert {row["phase"] for row in rows} == set(bench.PHASES) and float(summary["memory_reduction"]) > 1


def test_dense_backend_raises_when_a_particle_leaves_the_domain():
    """The dense backend allocates only the declared domain: a stencil node
    outside it raises InactiveNodeError (solver.py:1053-1058); hash does not."""
    from paper_2605_28525_b200.errors import InactiveNodeError

    doc = yaml.safe_load((SCEN / "terrain_demo.yaml").read_text())
    doc["materials"][0]["region_min_m"] = [0.7, -0.15, 0.15]
    doc["materials"][0]["region_max_m"] = [0.95, 0.15, 0.45]
    doc["materials"][0]["initial_velocity_m_s"] = [20.0, 0.0, 0.0]
    sc = scenarios.parse_config(doc, base_dir=SCEN)
    sim = scenarios.build_simulation(sc, backend="dense")
    with pytest.raises(InactiveNodeError, match="outside the active grid"):
        for _ in range(200):
            sim.step()
    sim = scenarios.build_simulation(sc, backend="hash")
    for _ in range(20):
        sim.step()

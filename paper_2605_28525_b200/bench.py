"""Run harness: timed scenario runs, frame output and the dense-versus-sparse
comparison -- the reference's ``sparsempm.bench``
(/root/reference/pkg/src/sparsempm/bench.py, ``S/bench.py`` below) on the GPU
step.

Phase times are the device (CUDA-event) times of the fused pipeline, reported
under the reference's phase names (solver.PHASES: on the GPU "g2p" holds the
fused G2P + stress + P2G kernel, "grid_update" the grid kernel, "map_build"
the scan + binning); metric bookkeeping and frame IO are timed separately and
never count towards compute totals, as in the reference.  Nodal memory uses
the reference's analytic accounting (NODE_BYTES per allocated node), so
dense/sparse ratios compare like for like.  The dense baseline is the GPU
dense-allocation mode (SimConfig.backend == "dense").
"""

import math
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import ConfigError, SimulationError
from .materials import MaterialModel
from .frames import AsyncFrameWriter
from .scenarios import MaterialRegion, ScenarioConfig, build_simulation, load_config, write_metrics, write_particles
from .solver import NODE_BYTES, PHASES, BoundaryCondition, Heightfield, SimConfig

_WARMED = set()


def _warm_scenario(backend, deterministic):
    """A throwaway scene touching every kernel of a mode (plane + terrain)."""
    region = MaterialRegion(name="warm",
                            model=MaterialModel(kind="drucker_prager", density=1000.0, youngs_modulus=1e5,
                                                poisson_ratio=0.3, friction_angle_deg=30.0),
                            region_min=np.full(3, 0.4), region_max=np.full(3, 0.6), velocity=np.zeros(3))
    sim = SimConfig(h=0.1, gravity=np.array([0.0, 0.0, -9.81]), total_time=1.0, domain_min=np.zeros(3),
                    domain_max=np.ones(3), backend=backend, deterministic=deterministic)
    terrain = Heightfield(x0=-1.0, y0=-1.0, cell=2.0, data=np.full((2, 2), 0.05))
    bcs = [BoundaryCondition(kind="plane", mu=0.3), BoundaryCondition(kind="heightfield", mu=0.3, heightfield=terrain)]
    return ScenarioConfig(name="warm", sim=sim, materials=[region], boundaries=bcs, boundary_paths=[None, None])


def warm_kernels(backend="scan", deterministic=False):
    """Load the library and create the CUDA context off the timing path
    (S/bench.py:59-67; there is no JIT on the GPU build)."""
    key = (backend, bool(deterministic))
    if key in _WARMED:
        return
    sim = build_simulation(_warm_scenario(backend, deterministic))
    sim.step()
    sim.step()
    _WARMED.add(key)


@dataclass
class RunMetrics:
    """Timing and sparsity record of one run (S/bench.py:70-190)."""

    scenario: str
    backend: str
    n_threads: int
    deterministic: bool
    n_particles: int
    n_dense: int
    physics_hash: str
    steps: list = field(default_factory=list)
    io_total: float = 0.0

    @property
    def n_steps(self):
        return len(self.steps)

    @property
    def sim_time(self):
        return self.steps[-1].t if self.steps else 0.0

    @property
    def phase_totals(self):
        return {p: float(sum(s.times[p] for s in self.steps)) for p in PHASES}

    @property
    def compute_total(self):
        return sum(self.phase_totals.values())

    @property
    def metrics_total(self):
        return sum(s.times.get("metrics", 0.0) for s in self.steps)

    @property
    def peak_alloc_nodes(self):
        return max(s.n_allocated for s in self.steps)

    @property
    def peak_nodal_bytes(self):
        """Analytic peak nodal memory: allocated nodes x NODE_BYTES."""
        return self.peak_alloc_nodes * NODE_BYTES

    @property
    def n_active_series(self):
        return [s.n_active for s in self.steps]

    @property
    def r_active(self):
        return sparsity_ratio(self.n_active_series, self.n_dense)

    def step_rows(self):
        rows = []
        for s in self.steps:
            row = {"row_kind": "step", "step": s.step, "t_s": repr(s.t), "dt_s": repr(s.dt), "n_active": s.n_active,
                   "allocated_nodes": s.n_allocated}
            row.update({f"{p}_s": repr(s.times[p]) for p in PHASES})
            row["metrics_s"] = repr(s.times.get("metrics", 0.0))
            if s.mass_sum is not None:
                row["mass_sum_kg"] = repr(s.mass_sum)
                for a, name in enumerate(("mom_x", "mom_y", "mom_z")):
                    row[name] = repr(float(s.mom_sum[a]))
            rows.append(row)
        return rows

    def summary_row(self):
        have = bool(self.steps)
        row = {"row_kind": "summary", "step": self.n_steps, "t_s": repr(self.sim_time), "scenario": self.scenario,
               "backend": self.backend, "threads": self.n_threads, "deterministic": self.deterministic,
               "n_particles": self.n_particles, "n_dense": self.n_dense,
               "max_n_active": max(self.n_active_series, default=0),
               "r_active": repr(self.r_active) if have else "",
               "peak_alloc_nodes": self.peak_alloc_nodes if have else 0,
               "peak_nodal_bytes": self.peak_nodal_bytes if have else 0,
               "compute_total_s": repr(self.compute_total), "metrics_total_s": repr(self.metrics_total),
               "io_total_s": repr(self.io_total), "physics_hash": self.physics_hash}
        row.update({f"{p}_s": repr(v) for p, v in self.phase_totals.items()})
        return row


def run(scenario, backend=None, threads=None, deterministic=None, out_dir=None, max_steps=None,
        record_conservation=False, warm=True, async_frames=True):
    """Execute a scenario (ScenarioConfig or YAML path) and collect RunMetrics
    (S/bench.py:193-247).  ``out_dir`` enables frame CSVs at the configured
    cadence plus metrics.csv; ``max_steps`` truncates the run."""
    if isinstance(scenario, (str, Path)):
        scenario = load_config(scenario)
    sim = build_simulation(scenario, backend=backend, threads=threads, deterministic=deterministic,
                           record_conservation=record_conservation)
    cfg = sim.config
    if warm:
        warm_kernels(cfg.backend, cfg.deterministic)
    metrics = RunMetrics(scenario=scenario.name, backend=cfg.backend, n_threads=cfg.n_threads,
                         deterministic=cfg.deterministic, n_particles=sim.particles.n, n_dense=sim.n_dense,
                         physics_hash=scenario.physics_hash())
    out = None if out_dir is None else Path(out_dir)
    if out is not None:
        out.mkdir(parents=True, exist_ok=True)
    fps, total = scenario.fps, cfg.total_time
    frame = 0

    framed = out is not None and fps > 0
    # frames leave through a device snapshot + side-stream copy + writer
    # thread (frames.py), so stepping does not wait for the CSV text
    writer = AsyncFrameWriter(sim) if framed and async_frames else None

    def emit():
        nonlocal frame
        t0 = time.perf_counter()
        path = out / f"frame_{frame:06d}.csv"
        if writer is not None:
            writer.submit(path)
        else:
            write_particles(path, sim.particles)
        metrics.io_total += time.perf_counter() - t0
        frame += 1

    if framed:
        emit()
    while sim.t < total - 1e-12:
        if max_steps is not None and sim.step_count >= max_steps:
            break
        dt = min(cfg.dt if cfg.dt is not None else sim.dt_bound(), total - sim.t)
        metrics.steps.append(sim.step(dt))
        while framed and sim.t >= frame / fps - 1e-9 and frame / fps <= total:
            emit()
    if writer is not None:
        t0 = time.perf_counter()
        writer.close()
        metrics.io_total += time.perf_counter() - t0
    if not metrics.steps:
        raise SimulationError("run finished without taking any step")
    if out is not None:
        write_metrics(out / "metrics.csv", metrics.step_rows(), metrics.summary_row())
    return metrics


def sparsity_ratio(n_active_series, n_dense):
    """Worst-case sparsity win min_steps n_dense / n_active (S/bench.py:250-262)."""
    series = list(n_active_series)
    if not series:
        raise ValueError("sparsity ratio needs at least one step")
    if min(series) <= 0:
        raise ValueError("degenerate run: a step had zero active nodes")
    if n_dense <= 0:
        raise ValueError(f"n_dense must be positive, got {n_dense}")
    return float(n_dense) / float(max(series))


@dataclass
class ComparisonReport:
    """Dense-baseline versus sparse-backend comparison (S/bench.py:265-330)."""

    scenario: str
    dense: RunMetrics
    sparse: RunMetrics

    @property
    def speedup(self):
        return self.dense.compute_total / self.sparse.compute_total

    @property
    def memory_reduction(self):
        return self.dense.peak_nodal_bytes / self.sparse.peak_nodal_bytes

    @property
    def r_active(self):
        return self.sparse.r_active

    def phase_table(self):
        d, s = self.dense.phase_totals, self.sparse.phase_totals
        return {p: (d[p], s[p], d[p] / s[p] if s[p] > 0 else math.inf) for p in PHASES}

    def rows(self):
        return [{"row_kind": "phase", "phase": p, "dense_s": repr(d), "sparse_s": repr(s), "ratio": repr(r)}
                for p, (d, s, r) in self.phase_table().items()]

    def summary_row(self):
        return {"row_kind": "summary", "phase": "total", "scenario": self.scenario,
                "sparse_backend": self.sparse.backend, "threads": self.sparse.n_threads, "steps": self.sparse.n_steps,
                "dense_s": repr(self.dense.compute_total), "sparse_s": repr(self.sparse.compute_total),
                "speedup": repr(self.speedup), "memory_reduction": repr(self.memory_reduction),
                "r_active": repr(self.r_active), "dense_peak_nodal_bytes": self.dense.peak_nodal_bytes,
                "sparse_peak_nodal_bytes": self.sparse.peak_nodal_bytes, "n_dense": self.sparse.n_dense,
                "max_n_active": max(self.sparse.n_active_series)}


def compare(dense_metrics, sparse_metrics):
    """ComparisonReport of a dense baseline and a sparse run of the same
    physics and length (S/bench.py:333-357): ValueError on role or step-count
    mismatch, ConfigError on different scenarios."""
    if dense_metrics.backend != "dense":
        raise ValueError(f"baseline run must use the dense backend, got {dense_metrics.backend!r}")
    if sparse_metrics.backend == "dense":
        raise ValueError("comparison run must use a sparse backend")
    if dense_metrics.physics_hash != sparse_metrics.physics_hash:
        raise ConfigError(f"cannot compare runs of different scenarios "
                          f"({dense_metrics.scenario!r} vs {sparse_metrics.scenario!r})")
    if dense_metrics.n_steps != sparse_metrics.n_steps:
        raise ValueError(f"step counts differ: {dense_metrics.n_steps} dense vs {sparse_metrics.n_steps} sparse")
    return ComparisonReport(scenario=dense_metrics.scenario, dense=dense_metrics, sparse=sparse_metrics)


def write_comparison(path, report):
    """Phase table plus summary of a comparison as CSV."""
    write_metrics(path, report.rows(), report.summary_row())


def sliding_box_oracle(theta_deg, mu, g=9.81, t=1.0):
    """Rigid Coulomb slider on an incline: displacement after t
    (S/bench.py:364-380); 0 while tan(theta) <= mu."""
    theta = math.radians(theta_deg)
    if not 0 <= theta < math.pi / 2:
        raise ValueError(f"theta must lie in [0, 90) degrees, got {theta_deg}")
    if mu < 0:
        raise ValueError(f"mu must be >= 0, got {mu}")
    if math.tan(theta) <= mu:
        return 0.0
    return 0.5 * g * (math.sin(theta) - mu * math.cos(theta)) * t * t


def slide_geometry(scenario):
    """(incline angle deg, friction, |g|, downslope unit vector) implied by the
    gravity and the first plane boundary (S/bench.py:383-405)."""
    plane = next((b for b in scenario.boundaries if b.kind == "plane"), None)
    if plane is None:
        raise ConfigError("scenario has no plane boundary")
    g = scenario.sim.gravity
    gmag = float(np.linalg.norm(g))
    if gmag <= 0:
        raise ConfigError("scenario gravity is zero")
    n = plane.normal
    theta = math.degrees(math.acos(min(1.0, max(-1.0, float(np.dot(-g, n) / gmag)))))
    tang = g - np.dot(g, n) * n
    tn = float(np.linalg.norm(tang))
    return theta, float(plane.mu), gmag, (tang / tn if tn > 0 else np.zeros(3))


def runout_distance(positions, center_xy, quantile=0.99):
    """Quantile of the horizontal distance from a column axis (S/bench.py:408-415)."""
    p = np.asarray(positions, dtype=np.float64)
    dx, dy = p[:, 0] - center_xy[0], p[:, 1] - center_xy[1]
    return float(np.quantile(np.sqrt(dx * dx + dy * dy), quantile))

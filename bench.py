"""Benchmark of the fused GPU sparse-MPM step (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C4] [--scale S]

One JSON line on rank 0.  metric: particle-steps/s (BASELINE.json).  A "step"
is one Simulation.step of the whole scene (inputs resident in HBM for
`value`; through the public API from host buffers for `e2e`).  The default
workload is C4 (the 101M-particle landslide) on 1 GPU.
`--impl reference` times the CPU oracle port of the reference path (the
reference is Python/numba; oracle/ restates it in C + OpenMP) on the same
full scene, with all host threads, for the SURVEY.md 8d step budget (C4: 2
steps after 1 warm step) and reports the steps it timed.  Our line adds a
late-time point (`late`: the same simulation after --late-steps steps of
flow) and a fresh-process end-to-end figure (`e2e.cold`).
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-steps/sec"
CONFIG_NAMES = {"C1": "granular_column", "C2": "two_spheres", "C3": "incline", "C4": "landslide"}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def make_scene(cfg_name, scale):
    from paper_2605_28525_b200 import scenes

    if cfg_name == "C4":
        return scenes.landslide(fraction=scale)
    if cfg_name == "C3":
        return scenes.incline()
    if cfg_name == "C2":
        return scenes.two_spheres(box="stress")
    return scenes.granular_column()


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    (nvidia-ml-py) every 5 ms from a thread, nvidia-smi -lms as the fallback
    (its start-up can outlast a sub-second timed region)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reason bits)
        self.nvml = None
        self.stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:  # noqa: BLE001
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            nv, h = self.nvml
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._sample()  # one sample at the start even of a sub-millisecond region
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _sample(self):
        nv, h = self.nvml
        try:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((float(sm), float(self.max_mhz), int(rs)))
        except Exception:  # noqa: BLE001
            pass

    def _poll(self):
        while not self.stop.is_set():
            self._sample()
            self.stop.wait(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml:
            self.t.join(timeout=2)
            self._sample()  # and one at the end
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for s_, m_, bits in self.samples:
            sm.append(s_)
            mx.append(m_)
            reasons.update(n for n, b in self.BITS.items() if bits & b)
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


# steps the CPU port times per configuration (K = 20
# for C1/C2, 5 for C3, 2-3 for C4 -- about 10-30 s of CPU work each)
CPU_STEPS = {"C1": 20, "C2": 20, "C3": 5, "C4": 2}


def workload_config(cfg_name, sc, n, deterministic, world=1):
    """The workload description both arms print (same dict: same scene,
    particle count, resolution and time-step rule; C5 = C4 on N GPUs)."""
    label = "C5" if world > 1 and cfg_name == "C4" else cfg_name
    return {"workload": CONFIG_NAMES[cfg_name], "config": label, "n_particles": int(n), "h": sc.config.h,
            "ppc": 2, "dt": "CFL bound (cfl=0.4)", "l2": "inputs larger than L2 (state %.1f GB)" % (n * 242 / 1e9)
            if n * 242 > 126e6 else "L2 flushed between steps: no (state fits in L2)",
            "deterministic": bool(deterministic)}


def run_cpu_port(cfg_name, steps, scale=1.0, threads=None, scene=None):
    """Time the oracle port of the reference's CPU scan path on the full
    scene (S/bench.py:172-233 compute_total: stress, map_build, alloc_zero,
    p2g, grid_update, g2p), CFL time step, one untimed warm step first."""
    from oracle import oracle as o

    sc = scene if scene is not None else make_scene(cfg_name, scale)
    ps = sc.particles
    threads = threads or len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    sim = o.OracleSimulation(ps, sc.config.h, sc.config.gravity, sc.materials, sc.boundaries,
                             backend="scan", deterministic=False, threads=threads, adopt=True)
    sim.step(count_nodes=False)  # warm (page-in, first-touch of the per-step arrays)
    total = 0.0
    for _ in range(steps):
        st = sim.step(count_nodes=False)
        total += sum(st["times"][p] for p in o.COMPUTE_PHASES)
    n = ps.n
    return {"value": n * steps / total, "unit": METRIC, "cores": threads, "kind": "port",
            "sample": f"full {CONFIG_NAMES[cfg_name]} scene ({cfg_name}, {n} particles) x {steps} timed steps after "
                      f"1 warm step, scan backend, CFL dt, {threads} OpenMP threads (oracle/ C port of the "
                      f"reference's numba path)",
            "ms_per_step": 1e3 * total / steps, "n_particles": n, "steps": steps, "wall_s": time.perf_counter() - t0}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sc = make_scene(args.config, args.scale)
    n = sc.particles.n
    steps = max(1, min(args.steps, CPU_STEPS[args.config]))
    base = run_cpu_port(args.config, steps, scene=sc)
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": METRIC, "n_gpus": args.gpus,
            "steps": steps, "warmup": 1, "ms_per_step": base["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, sc, n, args.deterministic,
                                      int(os.environ.get("WORLD_SIZE", "1"))),
            "parallelism": f"cpu{base['cores']}",
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": base["value"], "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": f"requested --steps {args.steps} --warmup {args.warmup}; timed {steps} steps of the full scene "
                    f"(SURVEY.md 8d CPU budget), wall {base['wall_s']:.1f} s"}
    print(json.dumps(line), flush=True)


def _phase_means(hist):
    return {k: float(np.mean(v)) for k, v in hist.items()}


def ours(args):
    import torch

    from paper_2605_28525_b200 import _lib, scenes
    from paper_2605_28525_b200.solver import Simulation

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    dist = None
    # SMPM_FORCE_DIST=1 runs the slab code path at world size 1 (exercises the
    # NCCL plumbing on a 1-GPU box: init, all_gather, empty neighbour rounds)
    distributed = world > 1 or os.environ.get("SMPM_FORCE_DIST") == "1"
    if distributed:
        import torch.distributed as dist

        dist.init_process_group(os.environ.get("SMPM_DIST_BACKEND", "nccl"))
        if args.config != "C4":
            raise SystemExit("multi-GPU bench runs the C4 landslide (C5 = C4 on N GPUs)")
        slab = scenes.landslide_slabs(world, fraction=args.scale)[rank]
        sc = scenes.landslide(fraction=args.scale, columns=(slab[2], slab[3]))
        per_col = sc.particles.n // max(1, slab[3] - slab[2])
    else:
        sc = make_scene(args.config, args.scale)
    sc.config.deterministic = bool(args.deterministic)
    n_local = sc.particles.n

    def make_sim(ps):
        if not distributed:
            return Simulation(ps, sc.config, sc.materials, sc.boundaries)
        from paper_2605_28525_b200.slabs import DistributedSimulation

        return DistributedSimulation(ps, sc.config, sc.materials, sc.boundaries, (slab[0], slab[1]),
                                     pid_base=slab[2] * per_col)

    def max_over_ranks(x):
        if not distributed:
            return x
        t = torch.tensor([x], device="cuda" if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if not distributed:
            return x
        t = torch.tensor([x], device="cuda" if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    n = int(sum_over_ranks(n_local))
    # ---- value: device-resident state, K steps timed on the sim's stream
    sim = make_sim(sc.particles)
    inner = sim.sim if distributed else sim
    stream = inner.stream
    for _ in range(args.warmup):
        sim.step()
    hist = {"map": [], "grid": [], "fused": []}
    nalloc = []
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local % max(1, torch.cuda.device_count())) as clk:
        start.record(stream)
        for _ in range(args.steps):
            st = sim.step()
            hist["fused"].append(st.times["g2p"] * 1e3)
            hist["grid"].append(st.times["grid_update"] * 1e3)
            hist["map"].append(st.times["map_build"] * 1e3)
            nalloc.append(st.n_allocated)
        end.record(stream)
        torch.cuda.synchronize()
    ms = max_over_ranks(start.elapsed_time(end))
    value = n * args.steps / (ms * 1e-3)
    # ---- the same K steps through Simulation.run (device-side step checks,
    # one host synchronisation for the whole batch instead of one per step)
    run_leg = None
    if not distributed:
        torch.cuda.synchronize()
        start.record(stream)
        sim.run(args.steps)
        end.record(stream)
        torch.cuda.synchronize()
        ms_run = start.elapsed_time(end)
        run_leg = {"ms_per_step": ms_run / args.steps, "value": n * args.steps / (ms_run * 1e-3),
                   "scope": "Simulation.run(K): same steps, one host sync per batch (smpm_sim_run)"}
    # ---- roofline of the dominant kernel (fused g2p->stress->p2g), this rank
    dbg0 = (ctypes.c_int64 * 24)()
    _lib.check(_lib.load().smpm_sim_debug_stats(inner._h, dbg0), "debug stats")
    fused_name = {0: "k_g2p2g_f32", 1: "k_g2p2g_ws", 2: "k_g2p2g (int32)", 3: "k_g2p2g (int64 det)"}.get(
        int(dbg0[23]), "k_g2p2g")
    peak, peak_kind = measured_peaks()
    ph = _phase_means(hist)
    n_alloc_local = float(np.mean(nalloc)) if world == 1 else float(np.mean(nalloc)) / world
    fused_bytes = 204.0 * n_local + 40.0 * n_alloc_local  # SURVEY 8d per-unit figures
    achieved = fused_bytes / (ph["fused"] * 1e-3) / 1e9
    step_bytes = 204.0 * n + 80.0 * float(np.mean(nalloc))
    traffic, atomics = None, None
    tf = ROOT / "profiles" / "fused_traffic.json"
    if tf.exists() and world == 1 and args.scale == 1.0:  # the ncu capture is of the full 1-GPU workload
        try:
            prof = json.loads(tf.read_text())
            traffic, atomics = prof.get(args.config), prof.get(f"{args.config}_atomics")
        except Exception:  # noqa: BLE001
            traffic = None
    # ---- late-time point: the same simulation flowing (disordered particles,
    # larger strains: wide work-item layout, moderate-strain path), timed the
    # same way after it reached step args.late_steps
    late = None
    if not distributed and args.late_steps > 0:
        while inner.step_count < args.late_steps:
            sim.step()
        lh = {"fused": [], "map": [], "grid": []}
        lalloc = []
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            st = sim.step()
            lh["fused"].append(st.times["g2p"] * 1e3)
            lh["map"].append(st.times["map_build"] * 1e3)
            lh["grid"].append(st.times["grid_update"] * 1e3)
            lalloc.append(st.n_allocated)
        s1.record(stream)
        torch.cuda.synchronize()
        lms = s0.elapsed_time(s1)
        lph = _phase_means(lh)
        lbytes = 204.0 * n_local + 40.0 * float(np.mean(lalloc))
        dbg = (ctypes.c_int64 * 24)()
        _lib.check(_lib.load().smpm_sim_debug_stats(inner._h, dbg), "debug stats")
        late = {"after_steps": args.late_steps, "sim_time_s": round(inner.t, 4), "steps": args.steps,
                "ms_per_step": lms / args.steps, "value": n * args.steps / (lms * 1e-3),
                "phases_ms": {"map_build(scan+bin)": lph["map"], "grid_update": lph["grid"], "fused": lph["fused"]},
                "work_item_layout": "wide" if int(dbg[21]) == 1 else "narrow",
                "mean_allocated_nodes": float(np.mean(lalloc)),
                "roofline_frac": lbytes / (lph["fused"] * 1e-3) / 1e9 / peak}
    # the device-resident sim is destroyed; its buffers stay in the library's
    # device-memory cache (include/smpm.h), which the e2e sim of the same
    # configuration reuses, like any process that runs simulations back to back
    del sim, inner
    # ---- the other grid mode, same workload and timing (precise_grid=False:
    # per-particle int32 fixed-point scatter, one global scale per launch)
    alt = None
    if not distributed and not args.deterministic and not args.no_alt:
        import copy

        cfg_alt = copy.copy(sc.config)
        cfg_alt.precise_grid = not bool(getattr(sc.config, "precise_grid", True))
        sim_a = Simulation(sc.particles, cfg_alt, sc.materials, sc.boundaries)
        for _ in range(args.warmup):
            sim_a.step()
        fa = []
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(sim_a.stream)
        for _ in range(args.steps):
            fa.append(sim_a.step().times["g2p"] * 1e3)
        a1.record(sim_a.stream)
        torch.cuda.synchronize()
        ams = a0.elapsed_time(a1)
        alt = {"precise_grid": cfg_alt.precise_grid, "ms_per_step": ams / args.steps,
               "value": n * args.steps / (ams * 1e-3), "fused_ms": float(np.mean(fa)),
               "roofline_frac": fused_bytes / (float(np.mean(fa)) * 1e-3) / 1e9 / peak,
               "note": "same workload and timing with the other P2G grid mode (DESIGN.md section 4); "
                       "precise_grid=False trades light-node / contact precision for speed"}
        del sim_a
    # ---- e2e: public API from host buffers (upload + K steps + download x,v)
    host = sc.particles
    if not distributed:
        # the caller's result arrays (x, v), allocated and paged in once like
        # any persistent host buffer; fresh pages would add first-touch faults
        out_x = np.zeros_like(host.x)
        out_v = np.zeros_like(host.v)
        out_x.fill(0.0)
        out_v.fill(0.0)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    t0 = time.perf_counter()
    sim2 = make_sim(host)
    t_up = time.perf_counter()
    for _ in range(args.steps):
        sim2.step()
    t_st = time.perf_counter()
    if not distributed:
        _lib.check(_lib.load().smpm_sim_get_particles(sim2._h, out_x.ctypes.data, out_v.ctypes.data, None, None,
                                                      None, None))
    else:
        sim2.local_particles()
    t_end = time.perf_counter()
    e2e_s = max_over_ranks(t_end - t0)
    e2e_parts = {"create_upload_s": round(t_up - t0, 4), "steps_s": round(t_st - t_up, 4),
                 "download_s": round(t_end - t_st, 4)}
    stats_bytes = args.steps * (2 * 128 + 24)
    h2d = n * 128  # host-packed 128-B particle records (smpm_sim_set_particles, include/smpm.h)
    d2h = n * 36   # x (fp64) and v (fp32, as stored; widened on the host) of every particle
    e2e_value = n * args.steps / e2e_s
    sim2 = None
    # ---- cold e2e: the same public-API sequence in a fresh process (cold
    # cudaMalloc of the device state, no buffer cache, fresh pinned buffers)
    e2e_cold = None
    if not distributed and not args.no_cold:
        # the parent keeps its device memory while the child runs (the GPU has
        # room for both): freeing it first would make the child's allocations
        # wait for the driver to scrub memory another process just released,
        # which a cold start on an idle GPU does not pay
        r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--e2e-cold-child", "--config", args.config,
                            "--scale", str(args.scale), "--steps", str(args.steps)] +
                           (["--deterministic"] if args.deterministic else []),
                           capture_output=True, text=True, timeout=900)
        try:
            e2e_cold = json.loads(r.stdout.strip().splitlines()[-1])
        except (IndexError, json.JSONDecodeError):
            e2e_cold = {"error": (r.stderr or r.stdout)[-300:]}
    line = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": workload_config(args.config, sc, n, args.deterministic, world),
        "precise_grid": bool(getattr(sc.config, "precise_grid", True)),
        "parallelism": f"slab{world}" if world > 1 else "single",
        "mean_allocated_nodes": float(np.mean(nalloc)),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": f"{fused_name} (G2P+F+return map+next P2G)",
                     "peak_kind": peak_kind, "kernel_ms": ph["fused"], "atomics": atomics,
                     "step_frac": step_bytes / world / (ms / args.steps * 1e-3) / 1e9 / peak},
        "phases_ms": {"map_build(scan+bin)": ph["map"], "grid_update": ph["grid"], "fused": ph["fused"]},
        "e2e": {"value": e2e_value, "unit": METRIC,
                "h2d_bytes_per_step": int(h2d / args.steps) + 8,
                "d2h_bytes_per_step": int((d2h + stats_bytes) / args.steps), "rank0_breakdown": e2e_parts,
                "scope": "Simulation() from host fp64 arrays (create + upload), K steps, x/v download into "
                         "preallocated host arrays; device buffers reused from the value leg (library cache)",
                "cold": e2e_cold},
        "run": run_leg,
        "late": late,
        "alt_grid_mode": alt,
        "gpu_launches": 5 * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        del host, sim2
        line["cpu_baseline"] = {k: v for k, v in run_cpu_port(args.config, CPU_STEPS[args.config], scene=sc).items()
                                if k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


def e2e_cold_child(args):
    """One fresh process: create + upload + K steps + x/v download through the
    public API, nothing cached (bench.py's e2e.cold)."""
    import torch

    from paper_2605_28525_b200 import _lib

    sc = make_scene(args.config, args.scale)
    host = sc.particles
    out_x, out_v = np.zeros_like(host.x), np.zeros_like(host.v)
    out_x.fill(0.0)
    out_v.fill(0.0)
    torch.cuda.init()
    _lib.load()
    t0 = time.perf_counter()
    sim = sc.simulation()
    t_up = time.perf_counter()
    for _ in range(args.steps):
        sim.step()
    t_st = time.perf_counter()
    _lib.check(_lib.load().smpm_sim_get_particles(sim._h, out_x.ctypes.data, out_v.ctypes.data, None, None, None,
                                                  None))
    t_end = time.perf_counter()
    n = host.n
    print(json.dumps({"value": n * args.steps / (t_end - t0), "unit": METRIC,
                      "breakdown": {"create_upload_s": round(t_up - t0, 4), "steps_s": round(t_st - t_up, 4),
                                    "download_s": round(t_end - t_st, 4)},
                      "scope": "fresh process: cold cudaMalloc + pinned-buffer allocation + upload, K steps, "
                               "x/v download (process start, imports and scene generation untimed)"}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=sorted(CONFIG_NAMES))
    ap.add_argument("--scale", type=float, default=1.0, help="fraction of the C4 release columns")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cold", action="store_true", help="skip the fresh-process e2e leg")
    ap.add_argument("--no-alt", action="store_true", help="skip timing the other grid mode")
    ap.add_argument("--late-steps", type=int, default=600,
                    help="also time --steps steps after the simulation reached this step (0: skip)")
    ap.add_argument("--e2e-cold-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--deterministic", action="store_true",
                    help="bitwise run-to-run reproducible mode (int64 fixed-point grid sums)")
    args = ap.parse_args()
    if args.e2e_cold_child:
        e2e_cold_child(args)
    elif args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()

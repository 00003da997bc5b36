"""Golden outputs of the reference's scenario / IO / harness layer.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_scenarios_golden.py

Imports the unmodified reference ``sparsempm`` and records, for the shipped
scenario files (copied verbatim as data into tests/golden/scenarios/), the
resolved document, the physics hash, the seeded particles and the terrain
grid; the exact CSV text of write_particles / write_metrics; and the
closed-form harness helpers (sliding_box_oracle, slide_geometry,
runout_distance, sparsity_ratio).  -> tests/golden/scenarios.json / .npz
"""

import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
SCEN = OUT / "scenarios"

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
from sparsempm import bench, scenarios  # noqa: E402
from sparsempm.solver import ParticleSet  # noqa: E402


def main():
    doc = {"scenes": {}, "csv": {}, "oracle": {}}
    arrays = {}
    for path in sorted(SCEN.glob("*.yaml")):
        sc = scenarios.load_config(path)
        ps = scenarios.build_particles(sc)
        doc["scenes"][path.stem] = {"to_dict": sc.to_dict(), "physics_hash": sc.physics_hash(), "n": ps.n}
        for k in ("x", "v", "m", "V0", "mat_id"):
            arrays[f"{path.stem}/{k}"] = getattr(ps, k)
        for i, b in enumerate(sc.boundaries):
            if b.kind == "heightfield":
                hf = b.heightfield
                arrays[f"{path.stem}/hf{i}"] = hf.data
                doc["scenes"][path.stem][f"hf{i}"] = [hf.x0, hf.y0, hf.cell]
        if any(b.kind == "plane" for b in sc.boundaries):
            th, mu, g, down = bench.slide_geometry(sc)
            doc["scenes"][path.stem]["slide_geometry"] = [th, mu, g, [float(v) for v in down]]
    rng = np.random.default_rng(7)
    x = rng.normal(size=(5, 3)) * 1e3
    ps = ParticleSet.from_samples(x, np.ones(5), 1000.0, velocity=(0.1, -1.0 / 3.0, 2e-17))
    with tempfile.TemporaryDirectory() as td:
        scenarios.write_particles(Path(td) / "p.csv", ps)
        doc["csv"]["particles"] = (Path(td) / "p.csv").read_text()
        rows = [{"row_kind": "step", "step": 1, "t_s": repr(0.1)}, {"row_kind": "step", "step": 2, "extra": "x"}]
        scenarios.write_metrics(Path(td) / "m.csv", rows, {"row_kind": "summary", "step": 2, "r": repr(1 / 3)})
        doc["csv"]["metrics"] = (Path(td) / "m.csv").read_text()
        arrays["csv/x"] = x
    doc["oracle"]["sliding_box"] = [[th, mu, g, t, bench.sliding_box_oracle(th, mu, g=g, t=t)]
                                    for th, mu, g, t in [(35, 0.4, 9.81, 1.0), (20, 0.5, 9.81, 1.0), (45, 0.0, 3.7, 2.5)]]
    pts = rng.normal(size=(200, 3))
    doc["oracle"]["runout"] = [bench.runout_distance(pts, (0.1, -0.2), q) for q in (0.5, 0.99)]
    arrays["oracle/runout_pts"] = pts
    doc["oracle"]["sparsity"] = bench.sparsity_ratio([10, 40, 25], 1000)
    (OUT / "scenarios.json").write_text(json.dumps(doc, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "scenarios.npz", **arrays)
    print("wrote", OUT / "scenarios.json", len(arrays), "arrays")


if __name__ == "__main__":
    main()

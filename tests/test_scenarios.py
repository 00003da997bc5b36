"""Scenario layer vs the reference (CPU): the shipped YAML scenes resolve to
the same documents, physics hashes, seeded particles and terrain grids; CSV
writers produce the same text; validation names the offending field; the
closed-form harness helpers agree.  Goldens: tests/golden/make_scenarios_golden.py
(reference S/scenarios.py, S/bench.py; cases follow T/test_scenarios_io.py and
T/test_bench.py)."""

import json
from pathlib import Path

import numpy as np
import pytest
import yaml
from click.testing import CliRunner

from paper_2605_28525_b200 import bench, scenarios
from paper_2605_28525_b200.cli import main as cli_main
from paper_2605_28525_b200.errors import ConfigError
from paper_2605_28525_b200.solver import ParticleSet

GOLD = Path(__file__).resolve().parent / "golden"
SCEN = GOLD / "scenarios"
G = json.loads((GOLD / "scenarios.json").read_text())
A = np.load(GOLD / "scenarios.npz")
STEMS = sorted(G["scenes"])


@pytest.mark.parametrize("stem", STEMS)
def test_shipped_scene_matches_reference(stem):
    sc = scenarios.load_config(SCEN / f"{stem}.yaml")
    ref = G["scenes"][stem]
    assert sc.to_dict() == ref["to_dict"]
    assert sc.physics_hash() == ref["physics_hash"]
    ps = scenarios.build_particles(sc)
    assert ps.n == ref["n"]
    for k in ("x", "v", "m", "V0", "mat_id"):
        assert np.array_equal(getattr(ps, k), A[f"{stem}/{k}"]), k
    for i, b in enumerate(sc.boundaries):
        if b.kind == "heightfield":
            assert np.array_equal(b.heightfield.data, A[f"{stem}/hf{i}"])
            assert [b.heightfield.x0, b.heightfield.y0, b.heightfield.cell] == ref[f"hf{i}"]
    if "slide_geometry" in ref:
        th, mu, g, down = bench.slide_geometry(sc)
        assert [th, mu, g] == ref["slide_geometry"][:3]
        assert np.array_equal(down, np.array(ref["slide_geometry"][3]))


def test_yaml_round_trip(tmp_path):
    sc = scenarios.load_config(SCEN / "terrain_demo.yaml")
    out = tmp_path / "terrain_demo.yaml"
    scenarios.save_config(out, sc)
    (tmp_path / "terrain").mkdir()
    (tmp_path / "terrain" / "valley.asc").write_text((SCEN / "terrain" / "valley.asc").read_text())
    back = scenarios.load_config(out)
    assert back.to_dict() == sc.to_dict() and back.physics_hash() == sc.physics_hash()


def _doc():
    return {"name": "unit", "grid": {"cell_size_m": 0.05, "domain_min_m": [0, 0, 0], "domain_max_m": [1, 1, 1]},
            "time": {"total_s": 0.5}, "gravity_m_s2": [0, 0, -9.81],
            "materials": [{"model": "elastic", "density_kg_m3": 1000.0, "youngs_modulus_pa": 1e6,
                           "poisson_ratio": 0.3, "region_min_m": [0.3, 0.3, 0.3], "region_max_m": [0.7, 0.7, 0.7]}],
            "boundaries": [{"type": "plane", "point_m": [0, 0, 0.1], "normal": [0, 0, 1], "friction_coeff": 0.4}]}


def test_defaults_resolve_like_reference():
    sc = scenarios.parse_config(_doc())
    assert (sc.sim.backend, sc.sim.block_size, sc.sim.cfl, sc.sim.dt, sc.sim.n_threads) == ("scan", 4, 0.4, None, 1)
    assert sc.sim.deterministic is False and sc.ppc == 2 and sc.fps == 0.0


@pytest.mark.parametrize("mutate,needle", [
    (lambda d: d.update(typo=1), "config.typo"),
    (lambda d: d["grid"].update(cell_size_m=-1), "grid.cell_size_m"),
    (lambda d: d["grid"].pop("domain_min_m"), "grid.domain_min_m"),
    (lambda d: d["time"].update(total_s="soon"), "time.total_s"),
    (lambda d: d.update(gravity_m_s2=[0, 0]), "gravity_m_s2"),
    (lambda d: d.update(solver={"backend": "octree"}), "solver.backend"),
    (lambda d: d.update(solver={"threads": 0}), "solver.threads"),
    (lambda d: d.update(schema_version=2), "schema_version"),
    (lambda d: d["materials"][0].update(model="clay"), "materials[0].model"),
    (lambda d: d["materials"][0].update(density_kg_m3=0), "materials[0].density_kg_m3"),
    (lambda d: d["materials"][0].update(region_max_m=[0.1, 0.9, 0.9]), "region_max_m"),
    (lambda d: d["boundaries"][0].update(type="sphere"), "boundaries[0].type"),
    (lambda d: d["boundaries"][0].update(normal=[0, 0, 0]), "boundaries[0].normal"),
    (lambda d: d["boundaries"][0].update(friction_coeff=-1), "boundaries[0].friction_coeff"),
])
def test_validation_names_the_field(mutate, needle):
    d = _doc()
    mutate(d)
    with pytest.raises(ConfigError, match=needle.replace("[", r"\[").replace("]", r"\]")):
        scenarios.parse_config(d)


def test_drucker_prager_requires_friction_angle():
    d = _doc()
    d["materials"][0]["model"] = "drucker_prager"
    with pytest.raises(ConfigError, match="friction_angle_deg"):
        scenarios.parse_config(d)


def test_load_config_errors(tmp_path):
    with pytest.raises(ConfigError, match="not found"):
        scenarios.load_config(tmp_path / "nope.yaml")
    (tmp_path / "bad.yaml").write_text("a: [1,")
    with pytest.raises(ConfigError, match="not valid YAML"):
        scenarios.load_config(tmp_path / "bad.yaml")
    (tmp_path / "list.yaml").write_text("- 1\n- 2\n")
    with pytest.raises(ConfigError, match="mapping"):
        scenarios.load_config(tmp_path / "list.yaml")
    (tmp_path / "named.yaml").write_text(yaml.safe_dump({k: v for k, v in _doc().items() if k != "name"}))
    assert scenarios.load_config(tmp_path / "named.yaml").name == "named"


def test_sample_box_properties():
    pos, vol = scenarios.sample_box([0, 0, 0], [1, 0.5, 0.25], 0.1, 2)
    assert len(pos) == 20 * 10 * 5
    assert vol.sum() == pytest.approx(0.125, rel=1e-12)
    assert np.all((pos > 0) & (pos < [1, 0.5, 0.25]))
    p1, _ = scenarios.sample_box([0.0, 0.0, 0.0], [0.01, 0.01, 0.01], 0.1, 2)
    assert len(p1) == 1
    with pytest.raises(ValueError):
        scenarios.sample_box([0, 0, 0], [1, 0, 1], 0.1)


@pytest.mark.parametrize("text,needle", [
    ("ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9\n1 2\n-9 4\n", "NODATA"),
    ("ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\n1 2 3\n", "expected 4"),
    ("ncols 2\nnrows 2\nxllcorner 0\ncellsize 1\n1 2\n3 4\n", "yllcorner"),
    ("ncols 1\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\n1\n3\n", "at least 2x2"),
    ("ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\n1 2\n3 x\n", "malformed elevation"),
])
def test_heightfield_errors(tmp_path, text, needle):
    p = tmp_path / "t.asc"
    p.write_text(text)
    with pytest.raises(ConfigError, match=needle):
        scenarios.load_heightfield(p)


def test_heightfield_orientation(tmp_path):
    p = tmp_path / "t.asc"
    p.write_text("ncols 3\nnrows 2\nxllcorner 10\nyllcorner 20\ncellsize 2\n1 2 3\n4 5 6\n")
    hf = scenarios.load_heightfield(p)
    assert (hf.x0, hf.y0, hf.cell) == (11.0, 21.0, 2.0)
    assert hf.data.tolist() == [[4, 1], [5, 2], [6, 3]]  # first row is the northernmost


def test_csv_text_matches_reference(tmp_path):
    x = A["csv/x"]
    ps = ParticleSet.from_samples(x, np.ones(5), 1000.0, velocity=(0.1, -1.0 / 3.0, 2e-17))
    scenarios.write_particles(tmp_path / "p.csv", ps)
    assert (tmp_path / "p.csv").read_text() == G["csv"]["particles"]
    pos, vel = scenarios.read_particles(tmp_path / "p.csv")
    assert np.array_equal(pos, ps.x) and np.array_equal(vel, ps.v)
    rows = [{"row_kind": "step", "step": 1, "t_s": repr(0.1)}, {"row_kind": "step", "step": 2, "extra": "x"}]
    scenarios.write_metrics(tmp_path / "m.csv", rows, {"row_kind": "summary", "step": 2, "r": repr(1 / 3)})
    assert (tmp_path / "m.csv").read_text() == G["csv"]["metrics"]
    steps, summary = scenarios.read_metrics(tmp_path / "m.csv")
    assert len(steps) == 2 and summary["r"] == repr(1 / 3)


def test_empty_particle_csv(tmp_path):
    ps = ParticleSet.from_samples(np.zeros((0, 3)), np.zeros(0), 1000.0)
    scenarios.write_particles(tmp_path / "e.csv", ps)
    pos, vel = scenarios.read_particles(tmp_path / "e.csv")
    assert pos.shape == (0, 3) and vel.shape == (0, 3)


def test_closed_form_helpers_match_reference():
    for th, mu, g, t, want in G["oracle"]["sliding_box"]:
        assert bench.sliding_box_oracle(th, mu, g=g, t=t) == want
    pts = A["oracle/runout_pts"]
    assert [bench.runout_distance(pts, (0.1, -0.2), q) for q in (0.5, 0.99)] == G["oracle"]["runout"]
    assert bench.sparsity_ratio([10, 40, 25], 1000) == G["oracle"]["sparsity"]
    for bad in ([], [0, 3]):
        with pytest.raises(ValueError):
            bench.sparsity_ratio(bad, 10)
    with pytest.raises(ValueError):
        bench.sparsity_ratio([3], 0)
    for th, mu in ((-1, 0.1), (90, 0.1), (30, -0.1)):
        with pytest.raises(ValueError):
            bench.sliding_box_oracle(th, mu)


def test_cli_validate_and_oracle(tmp_path):
    r = CliRunner().invoke(cli_main, ["validate-config", str(SCEN / "sliding_box.yaml")])
    assert r.exit_code == 0
    assert yaml.safe_load(r.output) == G["scenes"]["sliding_box"]["to_dict"]
    bad = tmp_path / "bad.yaml"
    bad.write_text(yaml.safe_dump({**_doc(), "typo": 1}))
    r = CliRunner().invoke(cli_main, ["validate-config", str(bad)])
    assert r.exit_code == 2 and "config.typo" in r.output
    r = CliRunner().invoke(cli_main, ["validate-config", str(tmp_path / "missing.yaml")])
    assert r.exit_code == 2
    r = CliRunner().invoke(cli_main, ["oracle", "sliding-box", "--theta-deg", "35", "--mu", "0.4"])
    assert r.exit_code == 0 and float(r.output) == G["oracle"]["sliding_box"][0][4]
    r = CliRunner().invoke(cli_main, ["oracle", "sliding-box", "--theta-deg", "95", "--mu", "0.4"])
    assert r.exit_code == 2

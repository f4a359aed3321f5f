"""The CLI front end (paper_2007_13988_b200/cli.py) mirroring the reference CLI's hot-path
subcommands (tools/isocull_cli.cpp): scene files, the stats/bench CSV schema, exit codes; on the
GPU the bench CSV rows equal the reference's own variants on the same scenes."""
import csv
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2007_13988_b200 import abi, cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KINDS = {0: "sphere", 1: "box", 2: "capsule", 3: "torus"}


def scene_json(name, sc):
    """A reference-format scene file from the golden export (tests/golden/scenes.json)."""
    prims = []
    for p in sc["prims"]:
        d = {"kind": KINDS[p["kind"]], "center": p["center"]}
        if p["kind"] in (0, 2):
            d["radius"] = p["radius"]
        if p["kind"] == 1:
            d["half"] = p["half"]
        if p["kind"] == 2:
            d["a"], d["b"] = p["a"], p["b"]
        if p["kind"] == 3:
            d["major"], d["minor"] = p["major"], p["minor"]
        prims.append(d)
    t = sc["texture"]
    tex = {1: lambda: {"type": "constant", "color": t["color"]},
           2: lambda: {"type": "gradient", "axis": "xyz"[t["axis"]], "from": t["from"], "to": t["to"]},
           3: lambda: {"type": "per_primitive", "colors": t["colors"]}}[t["kind"]]()
    return {"name": name, "tau": sc["tau"], "primitives": prims, "texture": tex}


@pytest.fixture(scope="module")
def scene_files(tmp_path_factory):
    d = tmp_path_factory.mktemp("scenes")
    data = json.load(open(os.path.join(ROOT, "tests", "golden", "scenes.json")))
    out = {}
    for name, sc in data.items():
        p = d / f"{name}.json"
        p.write_text(json.dumps(scene_json(name, sc)))
        out[name] = str(p)
    return out


def test_scene_loader_matches_reference_export(scene_files):
    data = json.load(open(os.path.join(ROOT, "tests", "golden", "scenes.json")))
    for name, path in scene_files.items():
        nm, prims, tau, tex = cli.load_scene(path)
        assert nm == name and tau == data[name]["tau"] and len(prims) == len(data[name]["prims"])
        for p, q in zip(prims, data[name]["prims"]):
            assert p.kind == q["kind"] and list(p.center) == q["center"] and p.radius == q["radius"]
            assert list(p.inv_rotation) == q["inv_rotation"]
        assert tex["kind"] == data[name]["texture"]["kind"]


def test_rotation_and_errors(tmp_path):
    # a rotated box: inverse rotation = transpose of Ry Rx Rz (scene.hpp:216-230)
    p = tmp_path / "rot.json"
    p.write_text(json.dumps({"primitives": [{"kind": "box", "half": [0.1, 0.2, 0.3], "rotation": [30, 20, 10]}]}))
    _, prims, tau, tex = cli.load_scene(str(p))
    m = np.array(prims[0].inv_rotation).reshape(3, 3)
    assert prims[0].rotated == 1 and np.allclose(m @ m.T, np.eye(3)) and tau == 2.0 / 256.0
    assert tex["kind"] == abi.ICG_TEXTURE_NONE
    assert cli.level_for_resolution(256, 32) == 3
    with pytest.raises(ValueError):
        cli.level_for_resolution(100, 16)
    assert cli.stats_row("s", "progressive", "", 128, 10, 2.0, 1.0, 3.25) == \
        "s,progressive,,128,10,2.000000,1.000000,3.250000\n"
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"primitives": [{"kind": "cone"}]}))
    r = subprocess.run([sys.executable, "-m", "paper_2007_13988_b200.cli", "extract", "--scene", str(bad)],
                       cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 2 and "unknown primitive kind" in r.stderr  # invalid_argument -> 2


@pytest.mark.gpu
def test_bench_csv_matches_reference(scene_files, tmp_path):
    from oracle import oracle as O
    from paper_2007_13988_b200 import api
    names = ["sphere", "thin_rod"]
    args = ["bench", "--resolution", "64", "--coarsest", "16", "--out", str(tmp_path)]
    for n in names:
        args += ["--scene", scene_files[n]]
    assert cli.main(args) == 0
    rows = list(csv.DictReader(open(tmp_path / "bench.csv")))
    assert list(rows[0].keys()) == cli.STATS_HEADER.split(",")
    assert len(rows) == len(names) * (3 + 6)
    data = json.load(open(os.path.join(ROOT, "tests", "golden", "scenes.json")))
    from .conftest import load_scenes
    sc = load_scenes()
    for row in rows:
        prims, tau = sc[row["scene"]]
        rs = O.RefScene(prims=prims, tau=tau)
        v = api.VARIANTS[row["variant"]]
        thr = float(row["threshold"]) if row["threshold"] else 0.0
        r = O.ref_extract(rs.pt_fn, rs.user, 16, 2, variant=v, threshold=thr, workers=8)
        b = O.ref_extract(rs.pt_fn, rs.user, 16, 2, variant=0, workers=8)
        assert int(row["total_evals"]) == r["total_evals"], row
        assert row["accel_factor"] == "%.6f" % (b["total_evals"] / r["total_evals"])
        assert row["iou"] == "%.6f" % O.compare_iou(r["binarized"], b["binarized"])
    del data
    # render: PPM + depth map of the reference renderer
    assert cli.main(["render", "--scene", scene_files["sphere"], "--camera", "30,20,0", "--resolution", "64",
                     "--out", str(tmp_path), "--depth-dump"]) == 0
    assert (tmp_path / "render.ppm").read_bytes().startswith(b"P6\n65 65\n255\n")
    assert os.path.getsize(tmp_path / "depth.f32") == 8 + 65 * 65 * 4

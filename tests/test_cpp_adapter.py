"""The header-only C++ adapter (include/isocull_b200.hpp) and the INTEGRATION.md caller, compiled
as C++17 with g++ against the headers and linked with the product library; the CPU leg runs the
host-only surface, the GPU leg runs a frame and a config-0 extraction and must agree with the
Python face on the same seeded inputs."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "adapter_demo.cpp")
LIBDIR = os.path.join(ROOT, "paper_2007_13988_b200")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cpp") / "adapter_demo")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", LIBDIR, "-lisocull_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    # the library is named libisocull_b200.so: link it by path (no lib prefix games)
    cmd[cmd.index("-lisocull_b200")] = os.path.join(LIBDIR, "libisocull_b200.so")
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def run(exe, mode):
    r = subprocess.run([exe, mode], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr + r.stdout
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_adapter_host_surface(demo):
    d = run(demo, "cpu")
    assert d["fails"] == 0


@pytest.mark.gpu
def test_adapter_frame_matches_python_face(demo):
    from paper_2007_13988_b200 import abi, api
    d = run(demo, "gpu")
    caps = api.gen_capsules(42)
    with api.Context(0) as ctx:
        ctx.set_mlp(abi.ICG_MLP_GEOMETRY, *api.gen_mlp(7, 0))
        ctx.set_mlp(abi.ICG_MLP_TEXTURE, *api.gen_mlp(8, 1))
        f = api.PifuField(api.gen_feature_map(1000, 256, 32, 32), caps, 50.0, abi.ICG_PREC_FP32)
        ext, img = ctx.frame(f, api.AlgoConfig("progressive", 16, 2), api.CameraSpec.from_angles(90, 0), 64, 64,
                             want_grid=True)
        an = api.AnalyticField(caps, 0.02)
        p = ctx.extract(an, api.AlgoConfig("progressive", 8, 3))
        b = ctx.extract(an, api.AlgoConfig("brute", 8, 3))
        tan = api.AnalyticField(caps, 0.02, {"kind": abi.ICG_TEXTURE_CONSTANT, "color": [0.25, 0.5, 0.75]})
        rv = ctx.render_view(tan, api.CameraSpec.from_angles(30, 20), api.AlgoConfig("progressive", 8, 3))
        ot = ctx.extract(an, api.AlgoConfig("octree_threshold", 8, 3, threshold=0.12))
        mv, mt = ctx.marching_cubes(p.values)
    assert d["evals"] == ext.evals_per_level and d["total"] == ext.total_evals
    assert d["value_sum"] == pytest.approx(float(np.sum(ext.values, dtype=np.float64)), rel=1e-12)
    assert d["covered"] == img.covered_pixels
    assert d["rgb_sum"] == pytest.approx(float(np.sum(img.rgb, dtype=np.float64)), rel=1e-9)
    assert d["c0_evals"] == p.evals_per_level
    assert d["iou"] == api.compare_iou(p.binarized, b.binarized)
    assert d["accel"] == api.acceleration_factor(p, b)
    assert d["invalid_threw"] is True
    assert d["rv_covered"] == rv.covered_pixels and d["rv_calls"] == rv.oracle_calls
    assert d["octree_evals"] == ot.total_evals
    assert d["mesh_vertices"] == len(mv) and d["mesh_triangles"] == len(mt)

"""Pins the CPU oracle (oracle/isocull_oracle.c) against the UNMODIFIED
reference compiled from /root/reference (oracle/_ref/libisocull_ref.so) and
against the reference-generated golden fixtures (tests/golden/)."""
import ctypes as C
import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from paper_2007_13988_b200 import api

import os
needs_ref = pytest.mark.skipif(not (O.ref_available() and os.path.isdir("/root/reference/proj/scenes")),
                               reason="reference (oracle/_ref + /root/reference) not present")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@needs_ref
def test_rng_matches_reference():
    # random.hpp:16-43
    for seed in (0, 1, 42, 2 ** 63 + 5):
        a = np.empty(4096)
        b = np.empty(4096)
        O.orc().orc_rng_uniforms(seed, 4096, a.ctypes.data_as(C.POINTER(C.c_double)))
        O.ref().ref_rng_uniforms(seed, 4096, b.ctypes.data_as(C.POINTER(C.c_double)))
        assert np.array_equal(a, b)
        O.orc().orc_rng_normals(seed, 4096, a.ctypes.data_as(C.POINTER(C.c_double)))
        O.ref().ref_rng_normals(seed, 4096, b.ctypes.data_as(C.POINTER(C.c_double)))
        assert np.array_equal(a, b)
        # the product's input generator draws the same sequence
        assert np.array_equal(api.gen_normals(seed, 4096), b.astype(np.float32))


def test_seeded_inputs_product_equals_oracle():
    assert np.array_equal(api.capsules_array(api.gen_capsules(42)), api.capsules_array(O.gen_capsules(42)))
    for which in (0, 1):
        pw, pb = api.gen_mlp(11, which)
        ow, ob = O.gen_mlp(11, which)
        assert all(np.array_equal(a, b) for a, b in zip(pw, ow))
        assert all(np.array_equal(a, b) for a, b in zip(pb, ob))


@needs_ref
@pytest.mark.parametrize("cells", [2, 3, 5])
def test_upsample_matches_reference(cells):
    rng = np.random.default_rng(cells)
    n = cells + 1
    v = rng.choice([0.0, 1.0, 0.25, 0.7], size=n ** 3).astype(np.float32)
    s = rng.integers(1, 3, size=n ** 3).astype(np.uint8)
    fn = 2 * cells + 1
    rv, rs = np.empty(fn ** 3, np.float32), np.empty(fn ** 3, np.uint8)
    ov, os_ = np.empty(fn ** 3, np.float32), np.empty(fn ** 3, np.uint8)
    f32, u8 = C.POINTER(C.c_float), C.POINTER(C.c_uint8)
    assert O.ref().ref_upsample(0, cells, v.ctypes.data_as(f32), s.ctypes.data_as(u8), rv.ctypes.data_as(f32),
                                rs.ctypes.data_as(u8)) == 0
    O.orc().orc_upsample_interpolate(cells, v.ctypes.data_as(f32), s.ctypes.data_as(u8), ov.ctypes.data_as(f32),
                                     os_.ctypes.data_as(u8))
    assert np.array_equal(rv, ov) and np.array_equal(rs, os_)


@needs_ref
def test_dilate_and_argmax_match_reference():
    rng = np.random.default_rng(3)
    n = 9
    m = (rng.random(n ** 3) < 0.03).astype(np.uint8)
    a, b = np.empty_like(m), np.empty_like(m)
    u8 = C.POINTER(C.c_uint8)
    O.ref().ref_dilate(n, m.ctypes.data_as(u8), a.ctypes.data_as(u8))
    O.orc().orc_dilate_1ring(n, m.ctypes.data_as(u8), b.ctypes.data_as(u8))
    assert np.array_equal(a, b)
    v = rng.choice([0.0, 0.5, 1.0, 0.3], size=n ** 3).astype(np.float32)
    f32, i32 = C.POINTER(C.c_float), C.POINTER(C.c_int32)
    mv1, mi1 = np.empty(n * n, np.float32), np.empty(n * n, np.int32)
    mv2, mi2 = np.empty(n * n, np.float32), np.empty(n * n, np.int32)
    O.ref().ref_argmax_z(n - 1, v.ctypes.data_as(f32), mv1.ctypes.data_as(f32), mi1.ctypes.data_as(i32))
    O.orc().orc_argmax_z(n, v.ctypes.data_as(f32), mv2.ctypes.data_as(f32), mi2.ctypes.data_as(i32))
    assert np.array_equal(mv1, mv2) and np.array_equal(mi1, mi2)


@needs_ref
@pytest.mark.parametrize("name", ["sphere", "torus", "capsule_figure", "thin_rod", "thin_slab", "offset_slab"])
def test_progressive_matches_reference_on_bundled_scenes(name, scenes):
    prims, tau = scenes[name]
    an = O.Analytic(prims, tau)
    # the reference runs its own scene oracle, loaded by its own JSON parser
    ref_scene = O.RefScene(f"/root/reference/proj/scenes/{name}.json")
    for conflict_pass in (True, False):
        r = O.ref_extract(ref_scene.pt_fn, ref_scene.user, 16, 2, conflict_pass=conflict_pass)
        o = O.extract_progressive(an, 16, 2, conflict_pass=conflict_pass)
        assert r["evals_per_level"] == o["evals_per_level"]
        assert np.array_equal(r["values"], o["values"])
        assert np.array_equal(r["states"], o["states"])
        assert np.array_equal(r["binarized"], o["binarized"])


def test_progressive_matches_golden_fixtures(scenes, ref_golden):
    """Works without /root/reference: golden values were produced by the reference itself."""
    for name, (prims, tau) in scenes.items():
        an = O.Analytic(prims, tau)
        o = O.extract_progressive(an, 16, 2)
        g = ref_golden[f"{name}/16/2/progressive"]
        assert o["evals_per_level"] == g["evals_per_level"]
        assert sha(o["values"]) == g["sha_values"]
        assert sha(o["states"]) == g["sha_states"]
        assert sha(o["binarized"]) == g["sha_binarized"]
        nc = O.extract_progressive(an, 16, 2, conflict_pass=False)
        assert nc["evals_per_level"] == ref_golden[f"{name}/16/2/no_conflict"]["evals_per_level"]
        b = O.extract_brute(an, 16, 2)
        gb = ref_golden[f"{name}/16/2/brute"]
        assert b["total_evals"] == gb["total_evals"] == 65 ** 3
        assert sha(b["binarized"]) == gb["sha_binarized"]


def test_config0_capsules_match_golden(ref_golden):
    caps = api.gen_capsules(42)
    o = O.extract_progressive(O.Analytic(caps, 0.02, threads=4), 32, 2)
    g = ref_golden["capsules42/32/2/progressive"]
    assert o["evals_per_level"] == g["evals_per_level"]
    assert sha(o["values"]) == g["sha_values"] and sha(o["states"]) == g["sha_states"]


@needs_ref
def test_conflict_bound_and_warning_match_reference(scenes):
    prims, tau = scenes["offset_slab"]
    an = O.Analytic(prims, tau)
    ref_scene = O.RefScene(f"/root/reference/proj/scenes/offset_slab.json")
    for it in (1, 2):
        r = O.ref_extract(ref_scene.pt_fn, ref_scene.user, 16, 3, max_conflict_iters=it)
        o = O.extract_progressive(an, 16, 3, max_conflict_iters=it)
        assert r["evals_per_level"] == o["evals_per_level"]
        assert r["conflict_warning"] == o["conflict_warning"]
        assert np.array_equal(r["values"], o["values"])


@needs_ref
def test_replay_oracle_reproduces_reference_control_flow():
    """The replay oracle (lookup of a finest-level grid) drives the reference to
    the identical result with zero misses — the mechanism the GPU parity tests use."""
    caps = api.gen_capsules(7)
    an = O.Analytic(caps, 0.02)
    o = O.extract_progressive(an, 8, 3)
    rp = O.Replay(o["values"], o["states"], 64)
    r = O.ref_extract(rp.pt_fn, rp.user, 8, 3)
    assert rp.c.misses == 0
    assert r["evals_per_level"] == o["evals_per_level"]
    assert np.array_equal(r["values"], o["values"]) and np.array_equal(r["states"], o["states"])


@needs_ref
def test_camera_matches_reference():
    for yaw, pitch in ((90, 0), (0, 0), (30, -20), (450, 10)):
        rot, t = np.empty(9), np.empty(3)
        O.ref().ref_camera_from_angles(yaw, pitch, 0.25, 1.0, rot.ctypes.data_as(C.POINTER(C.c_double)),
                                       t.ctypes.data_as(C.POINTER(C.c_double)))
        oc = O.camera_from_angles(yaw, pitch, 0.25, 1.0)
        pc = api.CameraSpec.from_angles(yaw, pitch, 0.25, 1.0)
        assert np.array_equal(rot, np.array(oc.rotation[:]))
        assert np.array_equal(rot, pc.rotation.reshape(9))
        assert np.array_equal(t, pc.translation)


@needs_ref
def test_compare_iou_matches_reference():
    rng = np.random.default_rng(0)
    a = (rng.random(5000) < 0.3).astype(np.uint8)
    b = (rng.random(5000) < 0.3).astype(np.uint8)
    u8 = C.POINTER(C.c_uint8)
    r = O.ref().ref_compare_iou(a.ctypes.data_as(u8), b.ctypes.data_as(u8), a.size)
    assert r == O.compare_iou(a, b) == api.compare_iou(a, b)
    z = np.zeros(10, np.uint8)
    assert api.compare_iou(z, z) == 1.0

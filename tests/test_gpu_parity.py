"""GPU parity tests: the sm_100a library (through the C ABI) against the CPU
oracle and the reference-generated fixtures, on identical seeded inputs.

Bars (BASELINE.json north_star):
  - integer / index outputs (evaluated sets, refined cells, states, first-crossing
    indices, masks) bit-exact;
  - occupancies within 1e-4 absolute for the fp32 paths, colours within 1e-3;
  - control flow checked exactly with the replay oracle: the GPU's evaluated values
    are fed back into the reference's extract_progressive, which must request
    exactly the nodes the GPU evaluated and reproduce its grid bit-for-bit.
"""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O
from paper_2007_13988_b200 import abi, api

pytestmark = pytest.mark.gpu

OCC_TOL_FP32 = 1e-4
RGB_TOL = 1e-3


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def replay_check(res, coarsest, level):
    """Feed the GPU grid back into the reference (or the oracle restatement when
    the reference shim is absent) through a lookup oracle; require identity."""
    rp = O.Replay(res.values, res.states, coarsest << level)
    if O.ref_available():
        r = O.ref_extract(rp.pt_fn, rp.user, coarsest, level)
    else:
        r = O.extract_progressive(rp, coarsest, level)
    assert rp.c.misses == 0, "reference requested nodes the GPU never evaluated"
    assert r["evals_per_level"] == res.evals_per_level
    assert np.array_equal(r["states"], res.states)
    assert np.array_equal(r["values"], res.values)


# ---------------------------------------------------------------------------
# config 0: analytic capsule figure
# ---------------------------------------------------------------------------
def test_config0_analytic_256_matches_oracle(gpu_ctx):
    caps = api.gen_capsules(42)
    cfg = api.AlgoConfig("progressive", 32, 3)
    g = gpu_ctx.extract(api.AnalyticField(caps, 0.02), cfg)
    o = O.extract_progressive(O.Analytic(caps, 0.02, threads=8), 32, 3)
    assert g.evals_per_level == o["evals_per_level"] == [35937, 10977, 48133, 199562]
    assert g.refined_cells_per_level[1:] == o["refined_cells_per_level"][1:] == [1149, 4901, 20084]
    assert g.conflict_iters_per_level == o["conflict_iters_per_level"]
    assert np.array_equal(g.states, o["states"])
    assert np.array_equal(g.values, o["values"])
    assert np.array_equal(g.binarized, o["binarized"])
    replay_check(g, 32, 3)


def test_config0_brute_force_and_iou(gpu_ctx):
    caps = api.gen_capsules(42)
    f = api.AnalyticField(caps, 0.02)
    p = gpu_ctx.extract(f, api.AlgoConfig("progressive", 32, 3))
    b = gpu_ctx.extract(f, api.AlgoConfig("brute", 32, 3))
    assert b.total_evals == 257 ** 3 and b.evals_per_level[3] == 257 ** 3
    assert np.all(b.states == abi.ICG_STATE_EVALUATED)
    # evaluated values are bit-identical to the dense evaluation (SPEC localize invariants)
    ev = p.states == abi.ICG_STATE_EVALUATED
    assert np.array_equal(p.values[ev], b.values[ev])
    iou = gpu_ctx.compare_iou(p.binarized, b.binarized)
    assert iou == api.compare_iou(p.binarized, b.binarized) >= 0.999
    assert api.acceleration_factor(p, b) > 50


@pytest.mark.parametrize("name", ["sphere", "torus", "capsule_figure", "thin_rod", "thin_slab", "offset_slab"])
def test_bundled_scenes_match_reference_golden(gpu_ctx, scenes, ref_golden, name):
    prims, tau = scenes[name]
    f = api.AnalyticField(prims, tau)
    g = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 2))
    gold = ref_golden[f"{name}/16/2/progressive"]
    assert g.evals_per_level == gold["evals_per_level"]
    assert sha(g.states) == gold["sha_states"]
    assert sha(g.binarized) == gold["sha_binarized"]
    assert sha(g.values) == gold["sha_values"]
    nc = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 2, conflict_pass=False))
    assert nc.evals_per_level == ref_golden[f"{name}/16/2/no_conflict"]["evals_per_level"]
    b = gpu_ctx.extract(f, api.AlgoConfig("brute", 16, 2))
    assert sha(b.binarized) == ref_golden[f"{name}/16/2/brute"]["sha_binarized"]


def test_conflict_bound_warning(gpu_ctx, scenes):
    prims, tau = scenes["offset_slab"]
    f = api.AnalyticField(prims, tau)
    an = O.Analytic(prims, tau)
    for it in (1, 2):
        g = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 3, max_conflict_iters=it))
        o = O.extract_progressive(an, 16, 3, max_conflict_iters=it)
        assert g.evals_per_level == o["evals_per_level"]
        assert g.conflict_warning == o["conflict_warning"]
        assert np.array_equal(g.values, o["values"])


def test_spec_acceptance_on_gpu(gpu_ctx, scenes):
    # SPEC.md:629 acceptance 2 (sphere 256^3 <= 5% of brute; measured 260,209 evals)
    prims, tau = scenes["sphere"]
    p = gpu_ctx.extract(api.AnalyticField(prims, tau), api.AlgoConfig("progressive", 16, 4))
    assert p.total_evals == 260209
    # SPEC.md:628 acceptance 1 at 128^3: IoU >= 0.999 on the bundled scenes
    for name in ("sphere", "torus", "capsule_figure", "thin_slab"):
        pr, t = scenes[name]
        f = api.AnalyticField(pr, t)
        a = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 3))
        b = gpu_ctx.extract(f, api.AlgoConfig("brute", 16, 3))
        assert api.compare_iou(a.binarized, b.binarized) >= 0.999, name
    # SPEC.md:632 acceptance 5: conflict pass is needed on offset_slab
    pr, t = scenes["offset_slab"]
    f = api.AnalyticField(pr, t)
    full = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 3))
    abl = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 3, conflict_pass=False))
    b = gpu_ctx.extract(f, api.AlgoConfig("brute", 16, 3))
    assert api.compare_iou(full.binarized, b.binarized) == 1.0
    assert api.compare_iou(abl.binarized, b.binarized) < 0.999


def test_empty_scene_and_edge_cases(gpu_ctx, scenes):
    # a sphere far outside the cube: only level 0 is evaluated (SPEC localize example)
    prims, tau = scenes["sphere"]
    p = abi.icg_primitive()
    C = __import__("ctypes")
    C.memmove(C.byref(p), C.byref(prims[0]), C.sizeof(p))
    p.center[:] = [5.0, 5.0, 5.0]
    p.radius = 0.1
    f = api.AnalyticField([p], tau)
    r = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 3))
    assert r.evals_per_level == [17 ** 3, 0, 0, 0] and r.binarized.sum() == 0
    # invalid configs raise ValueError (validate_config, localize.hpp:47-55)
    with pytest.raises(ValueError):
        gpu_ctx.extract(f, api.AlgoConfig("progressive", 1, 2))
    with pytest.raises(ValueError):
        gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 7))
    # empty batch -> empty result
    assert gpu_ctx.occupancy_batch(f, np.zeros((0, 3))).size == 0
    # target level 0 = dense coarse grid only
    r0 = gpu_ctx.extract(f, api.AlgoConfig("progressive", 4, 0))
    assert r0.evals_per_level == [125]


# ---------------------------------------------------------------------------
# configs 1-2: PIFu field
# ---------------------------------------------------------------------------
def _pifu(gpu_ctx, inp, precision):
    gpu_ctx.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
    gpu_ctx.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
    return api.PifuField(inp["fmap"], inp["caps"], 50.0, precision)


def _oracle_model(inp):
    return O.Pifu(inp["fmap"], inp["caps"], inp["gw"], inp["gb"], inp["tw"], inp["tb"], threads=8)


PRECISIONS_FP32 = [pytest.param(abi.ICG_PREC_FP32_SIMT, id="simt_fp32"), pytest.param(abi.ICG_PREC_FP32, id="tc_bf16x3")]


@pytest.mark.parametrize("precision", PRECISIONS_FP32)
def test_pifu_occupancy_arithmetic(gpu_ctx, pifu_inputs, precision):
    f = _pifu(gpu_ctx, pifu_inputs, precision)
    m = _oracle_model(pifu_inputs)
    rng = np.random.default_rng(5)
    pts = rng.uniform(-1, 1, (3000, 3))
    # include lattice nodes and points near the surface band
    pts[:500] = np.round((pts[:500] + 1) * 128) / 128 - 1
    g = gpu_ctx.occupancy_batch(f, pts)
    o = m.occupancy(pts)
    assert np.abs(g - o).max() <= OCC_TOL_FP32
    tex_g = gpu_ctx.texture_batch(f, pts[:1000])
    tex_o = m.texture(pts[:1000])
    assert np.abs(tex_g - tex_o).max() <= RGB_TOL


@pytest.mark.parametrize("precision", PRECISIONS_FP32)
def test_pifu_localization_replay_parity(gpu_ctx, pifu_inputs, precision):
    f = _pifu(gpu_ctx, pifu_inputs, precision)
    for coarsest, level in ((8, 3), (32, 2)):
        g = gpu_ctx.extract(f, api.AlgoConfig("progressive", coarsest, level))
        replay_check(g, coarsest, level)
        ev = g.states == abi.ICG_STATE_EVALUATED
        assert int(ev.sum()) == g.total_evals  # no node evaluated twice
    # arithmetic: GPU-evaluated node values vs the oracle at the same nodes
    n = (32 << 2) + 1
    idx = np.flatnonzero(ev)
    sub = idx[:: max(1, len(idx) // 4000)]
    i, j, k = sub % n, (sub // n) % n, sub // (n * n)
    pts = np.stack([-1 + 2 * i / 128.0, -1 + 2 * j / 128.0, 1 - 2 * k / 128.0], 1)
    o = _oracle_model(pifu_inputs).occupancy(pts)
    assert np.abs(g.values[sub] - o).max() <= OCC_TOL_FP32


@pytest.mark.parametrize("precision", PRECISIONS_FP32)
def test_render_first_crossing_parity(gpu_ctx, pifu_inputs, precision):
    f = _pifu(gpu_ctx, pifu_inputs, precision)
    cfg = api.AlgoConfig("progressive", 16, 3)
    cam = api.CameraSpec.from_angles(90, 0)
    W = H = 256
    ext, img = gpu_ctx.frame(f, cfg, cam, W, H, background=(0.1, 0.2, 0.3), want_grid=True)
    m = _oracle_model(pifu_inputs)
    r = O.render_first_crossing(ext.values, 128, O.camera_from_angles(90, 0), W, H, (0.1, 0.2, 0.3), tex=m)
    assert np.array_equal(img.mask, r["mask"])
    assert np.array_equal(img.surface_k, r["surface_k"])
    assert np.array_equal(img.depth, r["depth"])
    assert img.covered_pixels == r["covered"] and img.degenerate_brackets == r["degenerate"]
    assert img.grazing_pixels == r["grazing"]
    assert img.covered_pixels > 100
    assert np.abs(img.rgb - r["rgb"]).max() <= RGB_TOL
    bg = img.mask == 0
    assert np.all(img.rgb[bg] == np.array([0.1, 0.2, 0.3], np.float32))
    assert np.all(img.depth[bg] == -2.0)


def test_render_analytic_sphere_depth(gpu_ctx, scenes):
    # front view centre depth 0.5 within 2/R; other angles agree with the oracle
    prims, tau = scenes["sphere"]
    f = api.AnalyticField(prims, tau)
    an = O.Analytic(prims, tau)
    for yaw, pitch in ((0, 0), (90, 0), (30, 20)):
        cam = api.CameraSpec.from_angles(yaw, pitch)
        ext = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 3))
        img = gpu_ctx.render_localized(f, cam, 129, 129)
        assert img.mask[64, 64] == 1 and abs(img.depth[64, 64] - 0.5) <= 2.0 / 128
        r = O.render_first_crossing(ext.values, 128, O.camera_from_angles(yaw, pitch), 129, 129)
        assert np.array_equal(img.surface_k, r["surface_k"]) and np.array_equal(img.depth, r["depth"])
    del an


def test_config2_full_size_properties(gpu_ctx, pifu_inputs):
    """BASELINE config 2 at full size (256^3 + 512^2) through one icg_frame call:
    size-independent invariants instead of a full CPU oracle run."""
    f = _pifu(gpu_ctx, pifu_inputs, abi.ICG_PREC_FP32)
    cfg = api.AlgoConfig("progressive", 32, 3)
    cam = api.CameraSpec.from_angles(90, 0)
    ext, img = gpu_ctx.frame(f, cfg, cam, 512, 512, want_grid=True)
    ev = ext.states == abi.ICG_STATE_EVALUATED
    assert int(ev.sum()) == ext.total_evals
    assert ext.evals_per_level[0] == 33 ** 3
    assert np.array_equal(ext.binarized, (ext.values >= 0.5).astype(np.uint8))
    assert not ext.conflict_warning
    assert img.texture_points == img.covered_pixels > 0
    # idempotence: a second frame on the same inputs is bit-identical
    ext2, img2 = gpu_ctx.frame(f, cfg, cam, 512, 512, want_grid=True)
    assert np.array_equal(ext.values, ext2.values) and np.array_equal(img.rgb, img2.rgb)
    # the node values the oracle would produce at a sample of evaluated nodes
    m = _oracle_model(pifu_inputs)
    idx = np.flatnonzero(ev)[::997]
    n = 257
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    pts = np.stack([-1 + 2 * i / 256.0, -1 + 2 * j / 256.0, 1 - 2 * k / 256.0], 1)
    assert np.abs(ext.values[idx] - m.occupancy(pts)).max() <= OCC_TOL_FP32


@pytest.mark.gpu
@pytest.mark.parametrize("yaw,pitch", [(0, 0), (30, 20), (135, -40), (90, 0), (270, 75)])
def test_render_general_cameras_exact(gpu_ctx, pifu_inputs, yaw, pitch):
    """Empty-space skipping in the ray pass must not change a single crossing,
    depth bit, or the grazing / degenerate counters, for oblique rays too."""
    f = _pifu(gpu_ctx, pifu_inputs, abi.ICG_PREC_FP32)
    cfg = api.AlgoConfig("progressive", 16, 3)
    cam = api.CameraSpec.from_angles(yaw, pitch)
    W, H = 200, 150
    ext, img = gpu_ctx.frame(f, cfg, cam, W, H, want_grid=True)
    r = O.render_first_crossing(ext.values, 128, O.camera_from_angles(yaw, pitch), W, H)
    assert np.array_equal(img.mask, r["mask"])
    assert np.array_equal(img.surface_k, r["surface_k"])
    assert np.array_equal(img.depth, r["depth"])
    assert img.covered_pixels == r["covered"] and img.degenerate_brackets == r["degenerate"]
    assert img.grazing_pixels == r["grazing"]


@pytest.mark.gpu
@pytest.mark.parametrize("max_iters", [1, 2, 5])
def test_pifu_conflict_bound_replay(gpu_ctx, pifu_inputs, max_iters):
    """A conflict-iteration bound (AlgoConfig.max_conflict_iters, localize.hpp:343-346) cuts the
    loop wherever it is running -- CTA-pair kernels or the persistent tail -- exactly where the
    reference cuts it; the warning flag agrees."""
    f = _pifu(gpu_ctx, pifu_inputs, abi.ICG_PREC_FP32)
    coarsest, level = 16, 3
    g = gpu_ctx.extract(f, api.AlgoConfig("progressive", coarsest, level, max_conflict_iters=max_iters))
    rp = O.Replay(g.values, g.states, coarsest << level)
    if O.ref_available():
        r = O.ref_extract(rp.pt_fn, rp.user, coarsest, level, max_conflict_iters=max_iters)
    else:
        r = O.extract_progressive(rp, coarsest, level, max_conflict_iters=max_iters)
    assert rp.c.misses == 0
    assert r["evals_per_level"] == g.evals_per_level
    assert np.array_equal(r["states"], g.states)
    assert np.array_equal(r["values"], g.values)
    assert r["conflict_warning"] == g.conflict_warning


@pytest.mark.gpu
def test_frame_graph_replay_identical(gpu_ctx, pifu_inputs):
    """Frames of the same shape run eagerly, then warm, then are captured as a CUDA graph and
    replayed (fixed pinned output buffers keep the shape): every output bit is identical."""
    import ctypes as C
    f = _pifu(gpu_ctx, pifu_inputs, abi.ICG_PREC_FP32)
    cfg = api.AlgoConfig("progressive", 16, 3)
    cam = api.CameraSpec.from_angles(90, 0)
    W, H = 128, 96
    npx = W * H
    sizes = {"depth": npx * 4, "rgb": npx * 12, "mask": npx, "sk": npx * 4}
    ptrs = {k: api.host_alloc(b) for k, b in sizes.items()}
    img = abi.icg_image()
    img.mem = abi.ICG_MEM_HOST
    img.depth = C.cast(C.c_void_p(ptrs["depth"]), abi.f32p)
    img.rgb = C.cast(C.c_void_p(ptrs["rgb"]), abi.f32p)
    img.mask = C.cast(C.c_void_p(ptrs["mask"]), abi.u8p)
    img.surface_k = C.cast(C.c_void_p(ptrs["sk"]), abi.i32p)

    def view(k, dt, n):
        return np.ctypeslib.as_array((C.c_uint8 * (n * np.dtype(dt).itemsize)).from_address(ptrs[k])).view(dt).copy()

    outs = []
    for _ in range(5):
        ext, im = gpu_ctx.frame_raw(f, cfg, cam, W, H, img)
        outs.append((list(ext.evals_per_level[:4]), im.covered_pixels, im.grazing_pixels,
                     view("rgb", np.float32, npx * 3), view("depth", np.float32, npx), view("sk", np.int32, npx)))
    for o in outs[1:]:
        assert o[0] == outs[0][0] and o[1] == outs[0][1] and o[2] == outs[0][2]
        for a, b in zip(o[3:], outs[0][3:]):
            assert np.array_equal(a, b)
    for p_ in ptrs.values():
        api.host_free(p_)


@pytest.mark.gpu
def test_concurrent_contexts_match_serial(pifu_inputs):
    """Distinct contexts driven from concurrent host threads (several frames in flight on one
    GPU, as bench.py does) give exactly the results of running the frames one at a time."""
    import threading
    inp = pifu_inputs
    cfg = api.AlgoConfig("progressive", 16, 3)
    cam = api.CameraSpec.from_angles(90, 0)
    fmaps = [inp["fmap"], np.ascontiguousarray(inp["fmap"][:, ::-1, :]), np.ascontiguousarray(inp["fmap"] * 0.5)]
    ctxs = []
    for _ in fmaps:
        c = api.Context(0)
        c.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
        c.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
        ctxs.append(c)
    serial = []
    for c, fm in zip(ctxs, fmaps):
        serial.append(c.frame(api.PifuField(fm, inp["caps"], 50.0, abi.ICG_PREC_FP32), cfg, cam, 96, 96,
                              want_grid=True))
    results = [None] * len(ctxs)

    def run(k):
        out = None
        for _ in range(3):
            out = ctxs[k].frame(api.PifuField(fmaps[k], inp["caps"], 50.0, abi.ICG_PREC_FP32), cfg, cam, 96, 96,
                                want_grid=True)
        results[k] = out

    ths = [threading.Thread(target=run, args=(k,)) for k in range(len(ctxs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for (es, is_), (ec, ic) in zip(serial, results):
        assert np.array_equal(es.values, ec.values) and np.array_equal(es.states, ec.states)
        assert np.array_equal(is_.rgb, ic.rgb) and np.array_equal(is_.surface_k, ic.surface_k)
    for c in ctxs:
        c.close()


# ---------------------------------------------------------------------------
# config 3: bf16 weights / activations with fp32 accumulation
# ---------------------------------------------------------------------------
OCC_TOL_BF16 = 1e-2
RGB_TOL_BF16 = 1e-2  # bf16 texture network (config 3); the fp32 configs hold 1e-3


@pytest.mark.gpu
def test_bf16_occupancy_and_texture(gpu_ctx, pifu_inputs):
    f = _pifu(gpu_ctx, pifu_inputs, abi.ICG_PREC_BF16)
    m = _oracle_model(pifu_inputs)
    rng = np.random.default_rng(11)
    pts = rng.uniform(-1, 1, (3000, 3))
    pts[:500] = np.round((pts[:500] + 1) * 128) / 128 - 1
    assert np.abs(gpu_ctx.occupancy_batch(f, pts) - m.occupancy(pts)).max() <= OCC_TOL_BF16
    assert np.abs(gpu_ctx.texture_batch(f, pts[:1000]) - m.texture(pts[:1000])).max() <= RGB_TOL_BF16


@pytest.mark.gpu
def test_bf16_localization_replay_and_render(gpu_ctx, pifu_inputs):
    """Config 3 at test scale: the control flow is exact (replay through the reference), node
    values within the bf16 tolerance, first crossings exact against the oracle renderer on the
    GPU's own grid."""
    f = _pifu(gpu_ctx, pifu_inputs, abi.ICG_PREC_BF16)
    cfg = api.AlgoConfig("progressive", 16, 3)
    cam = api.CameraSpec.from_angles(90, 0)
    ext, img = gpu_ctx.frame(f, cfg, cam, 200, 200, want_grid=True)
    replay_check(ext, 16, 3)
    ev = np.flatnonzero(ext.states == abi.ICG_STATE_EVALUATED)
    sub = ev[:: max(1, len(ev) // 3000)]
    n = 129
    i, j, k = sub % n, (sub // n) % n, sub // (n * n)
    pts = np.stack([-1 + 2 * i / 128.0, -1 + 2 * j / 128.0, 1 - 2 * k / 128.0], 1)
    m = _oracle_model(pifu_inputs)
    assert np.abs(ext.values[sub] - m.occupancy(pts)).max() <= OCC_TOL_BF16
    r = O.render_first_crossing(ext.values, 128, O.camera_from_angles(90, 0), 200, 200, tex=m)
    assert np.array_equal(img.surface_k, r["surface_k"]) and np.array_equal(img.depth, r["depth"])
    assert np.abs(img.rgb - r["rgb"]).max() <= RGB_TOL_BF16


@pytest.mark.gpu
def test_config3_full_size_properties(gpu_ctx):
    """BASELINE config 3 at full size (512^3 with the 32->512 hierarchy, feature map 256x256x256,
    1024x1024 render, bf16): size-independent invariants and sampled node values."""
    caps = api.gen_capsules(42)
    fmap = api.gen_feature_map(1000, 256, 256, 256)
    gw, gb = api.gen_mlp(7, 0)
    tw, tb = api.gen_mlp(8, 1)
    gpu_ctx.set_mlp(abi.ICG_MLP_GEOMETRY, gw, gb)
    gpu_ctx.set_mlp(abi.ICG_MLP_TEXTURE, tw, tb)
    f = api.PifuField(fmap, caps, 50.0, abi.ICG_PREC_BF16)
    cfg = api.AlgoConfig("progressive", 32, 4)
    cam = api.CameraSpec.from_angles(90, 0)
    ext, img = gpu_ctx.frame(f, cfg, cam, 1024, 1024, want_grid=True)
    ev = np.flatnonzero(ext.states == abi.ICG_STATE_EVALUATED)
    assert len(ev) == ext.total_evals and ext.evals_per_level[0] == 33 ** 3
    assert len(ext.evals_per_level) == 5 and all(e > 0 for e in ext.evals_per_level)
    assert np.array_equal(ext.binarized, (ext.values >= 0.5).astype(np.uint8))
    assert img.texture_points == img.covered_pixels > 0
    ext2, img2 = gpu_ctx.frame(f, cfg, cam, 1024, 1024)
    assert ext2.evals_per_level == ext.evals_per_level and np.array_equal(img.rgb, img2.rgb)
    m = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=8)
    sub = ev[:: max(1, len(ev) // 2000)]
    n = 513
    i, j, k = sub % n, (sub // n) % n, sub // (n * n)
    pts = np.stack([-1 + 2 * i / 512.0, -1 + 2 * j / 512.0, 1 - 2 * k / 512.0], 1)
    assert np.abs(ext.values[sub] - m.occupancy(pts)).max() <= OCC_TOL_BF16


@pytest.mark.gpu
def test_chain_prediction_alternating_inputs(pifu_inputs):
    """One context alternates between feature maps whose conflict chains differ (size classes
    per iteration, tail hand-over): every frame equals the same frame on a fresh context, i.e.
    mispredicted evaluator sets are caught on device and replayed."""
    inp = pifu_inputs
    cfg = api.AlgoConfig("progressive", 32, 3)
    cam = api.CameraSpec.from_angles(90, 0)
    fmaps = [api.gen_feature_map(2000 + s) for s in range(3)]

    def ctx_new():
        c = api.Context(0)
        c.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
        c.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
        return c

    ref = []
    for fm in fmaps:
        c = ctx_new()
        e, i = c.frame(api.PifuField(fm, inp["caps"], 50.0, abi.ICG_PREC_FP32), cfg, cam, 128, 128, want_grid=True)
        ref.append((e.evals_per_level, e.values.copy(), i.surface_k.copy()))
        c.close()
    c = ctx_new()
    for rep in range(3):
        for s, fm in enumerate(fmaps):
            e, i = c.frame(api.PifuField(fm, inp["caps"], 50.0, abi.ICG_PREC_FP32), cfg, cam, 128, 128,
                           want_grid=True)
            assert e.evals_per_level == ref[s][0]
            assert np.array_equal(e.values, ref[s][1]) and np.array_equal(i.surface_k, ref[s][2])
    c.close()


@pytest.mark.gpu
def test_render_empty_space_skip_identical(pifu_inputs, monkeypatch):
    """Rays along grid x skip the samples whose cell corners are all exactly zero (per-x-line
    nonzero extents): every output bit and counter equals the walk over all samples."""
    inp = pifu_inputs
    cfg = api.AlgoConfig("progressive", 32, 3)
    cams = [api.CameraSpec.from_angles(90, 0), api.CameraSpec.from_angles(-90, 0, dist=0.3, scale=1.3),
            api.CameraSpec.from_angles(90, 0, scale=0.7)]
    outs = {}
    for skip in (True, False):
        monkeypatch.setenv("ICG_NO_XEXT", "0" if skip else "1")
        c = api.Context(0)
        c.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
        c.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
        f = api.PifuField(inp["fmap"], inp["caps"], 50.0, abi.ICG_PREC_FP32)
        outs[skip] = [c.frame(f, cfg, cam, 300, 200)[1] for cam in cams]
        c.close()
    for a, b in zip(outs[True], outs[False]):
        assert a.covered_pixels > 0
        assert (a.covered_pixels, a.degenerate_brackets, a.grazing_pixels, a.texture_points) == \
            (b.covered_pixels, b.degenerate_brackets, b.grazing_pixels, b.texture_points)
        for x, y in ((a.depth, b.depth), (a.rgb, b.rgb), (a.mask, b.mask), (a.surface_k, b.surface_k)):
            assert np.array_equal(x, y)


@pytest.mark.gpu
def test_texture_colour_error_wide_sample(gpu_ctx, pifu_inputs):
    """The texture kernel keeps one fp16 copy of every weight and operand (fp32 accumulation):
    colours over a wide random sample stay within the 1e-3 bar (fp64 model: 5.2e-4 max)."""
    f = _pifu(gpu_ctx, pifu_inputs, abi.ICG_PREC_FP32)
    m = _oracle_model(pifu_inputs)
    pts = np.random.default_rng(11).uniform(-0.9, 0.9, (20000, 3))
    err = np.abs(gpu_ctx.texture_batch(f, pts) - m.texture(pts)).max()
    print(f"max colour error {err:.3e}")
    assert err <= RGB_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("chain_fact", ["1", "0"])
def test_points_in_m_factored_pass_matches(pifu_inputs, monkeypatch, chain_fact):
    """config 2 (256^3) through the points-in-M factored kernel (k_fact2, also taking the level-3
    conflict batches above 9472 nodes when chain_fact=1) against k_mlp_pair<FACT> and the
    full-network chain kernels: identical evaluated sets, states and counts, values within 1e-5,
    and both within the oracle bar on a sample."""
    inp = pifu_inputs
    cfg = api.AlgoConfig("progressive", 32, 3)
    out = {}
    for f2 in ("1", "0"):
        monkeypatch.setenv("ICG_FACT2", f2)
        monkeypatch.setenv("ICG_CHAIN_FACT", chain_fact)
        c = api.Context(0)
        c.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
        c.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
        f = api.PifuField(inp["fmap"], inp["caps"], 50.0, abi.ICG_PREC_FP32)
        out[f2] = c.extract(f, cfg)
        c.close()
    a, b = out["1"], out["0"]
    assert a.total_evals == b.total_evals and list(a.evals_per_level) == list(b.evals_per_level)
    assert list(a.conflict_iters_per_level) == list(b.conflict_iters_per_level)
    assert np.array_equal(a.states, b.states)
    assert np.abs(a.values - b.values).max() <= 1e-5
    m = _oracle_model(inp)
    idx = np.flatnonzero(a.states == abi.ICG_STATE_EVALUATED)[::1499]
    n = 257
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    pts = np.stack([-1 + 2 * i / 256.0, -1 + 2 * j / 256.0, 1 - 2 * k / 256.0], 1)
    assert np.abs(a.values[idx] - m.occupancy(pts)).max() <= OCC_TOL_FP32


@pytest.mark.gpu
def test_level_sets_config0_match_oracle(gpu_ctx):
    """icg_level_set: per-level refined-cell and evaluated-node sets of the
    config-0 extraction equal the oracle's (which records them while localizing), for the
    progressive and the brute-force variants, host and device outputs."""
    caps = api.gen_capsules(42)
    f = api.AnalyticField(caps, 0.02)
    g = gpu_ctx.extract(f, api.AlgoConfig("progressive", 32, 3, keep_level_sets=True))
    o = O.extract_progressive(O.Analytic(caps, 0.02, threads=8), 32, 3, level_sets=True)
    for l in range(4):
        ev = gpu_ctx.level_set(l, "evaluated")
        rf = gpu_ctx.level_set(l, "refined")
        assert np.array_equal(ev, o["evaluated_sets"][l]), l
        assert np.array_equal(rf, o["refined_sets"][l]), l
        assert len(ev) == g.evals_per_level[l] and len(rf) == g.refined_cells_per_level[l]
    # capacity handling and device output through the raw ABI
    import ctypes as C
    n = C.c_size_t()
    lib = abi.lib()
    small = np.empty(4, np.uint32)
    assert lib.icg_level_set(gpu_ctx.h, 3, abi.ICG_SET_EVALUATED_NODES, abi.ICG_MEM_HOST,
                             small.ctypes.data_as(C.POINTER(C.c_uint32)), 4, C.byref(n)) == abi.ICG_ECAPACITY
    assert n.value == g.evals_per_level[3]
    dptr = gpu_ctx.device_alloc(4 * n.value)
    assert lib.icg_level_set(gpu_ctx.h, 3, abi.ICG_SET_EVALUATED_NODES, abi.ICG_MEM_DEVICE,
                             C.cast(C.c_void_p(dptr), C.POINTER(C.c_uint32)), n.value, C.byref(n)) == abi.ICG_OK
    back = np.empty(n.value, np.uint32)
    gpu_ctx.memcpy(back.ctypes.data, dptr, 4 * n.value, abi.ICG_MEM_HOST, abi.ICG_MEM_DEVICE)
    gpu_ctx.device_free(dptr)
    assert np.array_equal(back, o["evaluated_sets"][3])
    # brute force: every node at the target level, nothing refined
    gpu_ctx.extract(f, api.AlgoConfig("brute", 8, 2, keep_level_sets=True))
    assert np.array_equal(gpu_ctx.level_set(2, "evaluated"), np.arange(33 ** 3, dtype=np.uint32))
    assert len(gpu_ctx.level_set(2, "refined")) == 0 and len(gpu_ctx.level_set(0, "evaluated")) == 0
    # an extraction without keep_level_sets drops them
    gpu_ctx.extract(f, api.AlgoConfig("progressive", 8, 2))
    with pytest.raises(ValueError):
        gpu_ctx.level_set(1, "evaluated")


@pytest.mark.gpu
def test_frame_graph_survives_shape_changes(pifu_inputs):
    """A captured frame graph must not be replayed after the context's work buffers moved
    (a larger grid / image / feature map in between).  Frame A runs with FIXED pinned output
    buffers (grid + image), so the second and later calls replay its CUDA graph; a larger frame B
    and a larger extraction then grow the buffers; frame A again must equal a fresh context's."""
    import ctypes as C
    inp = pifu_inputs
    ctx = api.Context(0)
    ctx.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
    ctx.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
    fa = api.PifuField(np.ascontiguousarray(inp["fmap"][:, :64, :64]), inp["caps"], 50.0, abi.ICG_PREC_FP32)
    fb = api.PifuField(inp["fmap"], inp["caps"], 50.0, abi.ICG_PREC_FP32)
    cam = api.CameraSpec.from_angles(90, 0)
    ca, cb = api.AlgoConfig("progressive", 16, 2), api.AlgoConfig("progressive", 16, 3)
    W = H = 64
    n3 = 65 ** 3
    sizes = {"depth": W * H * 4, "rgb": W * H * 12, "mask": W * H, "sk": W * H * 4, "v": n3 * 4, "s": n3}
    ptrs = {k: api.host_alloc(b) for k, b in sizes.items()}
    img = abi.icg_image()
    img.mem = abi.ICG_MEM_HOST
    img.depth = C.cast(C.c_void_p(ptrs["depth"]), abi.f32p)
    img.rgb = C.cast(C.c_void_p(ptrs["rgb"]), abi.f32p)
    img.mask = C.cast(C.c_void_p(ptrs["mask"]), abi.u8p)
    img.surface_k = C.cast(C.c_void_p(ptrs["sk"]), abi.i32p)
    ext = abi.icg_extraction()
    ext.mem = abi.ICG_MEM_HOST
    ext.values = C.cast(C.c_void_p(ptrs["v"]), abi.f32p)
    ext.states = C.cast(C.c_void_p(ptrs["s"]), abi.u8p)

    def view(k, dt, n):
        return np.ctypeslib.as_array((C.c_uint8 * (n * np.dtype(dt).itemsize)).from_address(ptrs[k])).view(dt).copy()

    def frame_a():
        e, im = ctx.frame_raw(fa, ca, cam, W, H, img, ext)
        return (e.cells, view("v", np.float32, n3), view("s", np.uint8, n3), view("rgb", np.float32, W * H * 3),
                view("sk", np.int32, W * H))

    outs = [frame_a() for _ in range(4)]  # eager, warm, captured, replayed
    ctx.frame(fb, cb, cam, 256, 256)      # larger grid / image: buffers grow
    ctx.extract(fb, api.AlgoConfig("progressive", 32, 3))
    outs += [frame_a() for _ in range(4)]
    ctx.close()
    for p_ in ptrs.values():
        api.host_free(p_)
    with api.Context(0) as fresh:
        fresh.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
        fresh.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
        ref_e, ref_i = fresh.frame(fa, ca, cam, W, H, want_grid=True)
    for cells, v, st, rgb, sk in outs:
        assert cells == 64
        assert np.array_equal(v, ref_e.values) and np.array_equal(st, ref_e.states)
        assert np.array_equal(rgb, ref_i.rgb.reshape(-1)) and np.array_equal(sk, ref_i.surface_k.reshape(-1))


@pytest.mark.gpu
@pytest.mark.parametrize("precision", PRECISIONS_FP32)
def test_input_camera_phi_projection(gpu_ctx, pifu_inputs, precision):
    """icg_field.input_camera: Phi sampled at the input view's world_to_view(P).xy,
    depth feature its z, against the oracle with the same camera; the localization runs the
    per-point path (no column sharing) and replays exactly through the reference."""
    inp = pifu_inputs
    gpu_ctx.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
    gpu_ctx.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
    cam = api.CameraSpec.from_angles(30, 20, 0.1, 0.9)
    f = api.PifuField(inp["fmap"], inp["caps"], 50.0, precision, input_camera=cam)
    m = O.Pifu(inp["fmap"], inp["caps"], inp["gw"], inp["gb"], inp["tw"], inp["tb"], threads=8,
               input_camera=(cam.rotation, cam.translation, cam.scale))
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1, 1, (2000, 3))
    assert np.abs(gpu_ctx.occupancy_batch(f, pts) - m.occupancy(pts)).max() <= OCC_TOL_FP32
    assert np.abs(gpu_ctx.texture_batch(f, pts[:500]) - m.texture(pts[:500])).max() <= RGB_TOL
    # the camera changes the field (not the identity by accident)
    m_id = _oracle_model(inp)
    assert np.abs(m_id.occupancy(pts[:200]) - m.occupancy(pts[:200])).max() > 1e-2
    g = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 2))
    replay_check(g, 16, 2)
    ev = np.flatnonzero(g.states == abi.ICG_STATE_EVALUATED)
    n = 65
    i, j, k = ev % n, (ev // n) % n, ev // (n * n)
    nodes = np.stack([-1 + 2 * i / 64.0, -1 + 2 * j / 64.0, 1 - 2 * k / 64.0], 1)
    assert np.abs(g.values[ev] - m.occupancy(nodes)).max() <= OCC_TOL_FP32


@pytest.mark.gpu
def test_on_device_feature_producer(gpu_ctx, pifu_inputs):
    """icg_gen_feature_map_device against the oracle restatement (fp64 Box-Muller rounded to fp32:
    device and host libm may differ by an ulp), and a frame on the device-generated map equals the
    frame on the same map uploaded from the host."""
    m = gpu_ctx.gen_feature_map(1234, 256, 64, 64)
    o = O.feature_normals(1234, 256, 64, 64)
    assert np.abs(m - o).max() <= 1e-6 * max(1.0, float(np.abs(o).max()))
    n = 256 * 64 * 64
    dp = gpu_ctx.device_alloc(4 * n)
    gpu_ctx.gen_feature_map(1234, 256, 64, 64, device_out=dp)
    inp = pifu_inputs
    gpu_ctx.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
    gpu_ctx.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
    fd = api.PifuField(None, inp["caps"], 50.0, abi.ICG_PREC_FP32, device_ptr=dp, shape=(256, 64, 64))
    fh = api.PifuField(m, inp["caps"], 50.0, abi.ICG_PREC_FP32)
    cfg, cam = api.AlgoConfig("progressive", 16, 2), api.CameraSpec.from_angles(90, 0)
    e1, i1 = gpu_ctx.frame(fd, cfg, cam, 64, 64, want_grid=True)
    e2, i2 = gpu_ctx.frame(fh, cfg, cam, 64, 64, want_grid=True)
    gpu_ctx.device_free(dp)
    assert np.array_equal(e1.values, e2.values) and np.array_equal(i1.rgb, i2.rgb)


@pytest.mark.gpu
@pytest.mark.parametrize("switch", ["ICG_TEX_PAIR", "ICG_COLS_PAIR"])
def test_alternate_kernels_match_default(pifu_inputs, monkeypatch, switch):
    """The reference paths kept behind switches -- the fused pair texture kernel (ICG_TEX_PAIR=1)
    and the pair kernel's column pass (ICG_COLS_PAIR=1) -- against the default texture GEMM chain
    and column GEMM on a config-2 frame (256^3, 512^2): identical geometry and first crossings,
    grid values within 1e-5 (so bracket depths within 1e-5), colours within 1e-3 of each other."""
    inp = pifu_inputs
    cfg = api.AlgoConfig("progressive", 32, 3)
    cam = api.CameraSpec.from_angles(90, 0)
    out = {}
    for v in ("0", "1"):
        monkeypatch.setenv(switch, v)
        c = api.Context(0)
        c.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
        c.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
        f = api.PifuField(inp["fmap"], inp["caps"], 50.0, abi.ICG_PREC_FP32)
        out[v] = c.frame(f, cfg, cam, 512, 512, want_grid=True)
        c.close()
    (ea, ia), (eb, ib) = out["0"], out["1"]
    assert np.array_equal(ea.states, eb.states)
    assert np.abs(ea.values - eb.values).max() <= 1e-5
    assert np.array_equal(ia.mask, ib.mask) and np.array_equal(ia.surface_k, ib.surface_k)
    cov = ia.mask.astype(bool)
    assert np.array_equal(ia.depth[~cov], ib.depth[~cov])
    assert np.abs(ia.depth[cov] - ib.depth[cov]).max() <= 1e-5
    assert cov.sum() > 1000
    assert np.abs(ia.rgb[cov] - ib.rgb[cov]).max() <= RGB_TOL


@pytest.mark.gpu
def test_odd_feature_map_shape(gpu_ctx, pifu_inputs):
    """A feature map whose H x W is not a multiple of 64 (the 32 x 32-tile transpose instead of the
    64 x 64 one) through the per-point and the column-factored paths, against the oracle."""
    inp = pifu_inputs
    gpu_ctx.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
    gpu_ctx.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
    fmap = api.gen_feature_map(77, 256, 20, 21)
    f = api.PifuField(fmap, inp["caps"], 50.0, abi.ICG_PREC_FP32)
    m = O.Pifu(fmap, inp["caps"], inp["gw"], inp["gb"], inp["tw"], inp["tb"], threads=8)
    pts = np.random.default_rng(11).uniform(-1, 1, (1500, 3))
    assert np.abs(gpu_ctx.occupancy_batch(f, pts) - m.occupancy(pts)).max() <= OCC_TOL_FP32
    g = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 2))
    ev = np.flatnonzero(g.states == abi.ICG_STATE_EVALUATED)
    n = 65
    i, j, k = ev % n, (ev // n) % n, ev // (n * n)
    node_pts = np.stack([-1 + 2 * i / 64.0, -1 + 2 * j / 64.0, 1 - 2 * k / 64.0], 1)
    assert np.abs(g.values[ev] - m.occupancy(node_pts)).max() <= OCC_TOL_FP32


@pytest.mark.gpu
@pytest.mark.parametrize("cfg_args", [(32, 2), (16, 3)])
def test_frame_kept_extents_equal_render_of_grid(gpu_ctx, pifu_inputs, cfg_args):
    """icg_frame keeps the final grid's x-line extents during the extraction (level pass + every
    evaluation epilogue); rendering the same extracted grid afterwards recomputes them with
    k_xline_extents.  Both must give identical images, crossing indices and counters."""
    inp = pifu_inputs
    gpu_ctx.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
    gpu_ctx.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
    f = api.PifuField(inp["fmap"], inp["caps"], 50.0, abi.ICG_PREC_FP32)
    cfg = api.AlgoConfig("progressive", *cfg_args)
    cam = api.CameraSpec.from_angles(90, 0)
    ext, img = gpu_ctx.frame(f, cfg, cam, 192, 160, want_grid=True)
    img2 = gpu_ctx.render_localized(f, cam, 192, 160)
    assert img.covered_pixels == img2.covered_pixels > 0
    assert np.array_equal(img.surface_k, img2.surface_k)
    assert np.array_equal(img.mask, img2.mask)
    assert np.array_equal(img.depth, img2.depth)
    assert np.array_equal(img.rgb, img2.rgb)

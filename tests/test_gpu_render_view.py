"""The reference's own mesh-free renderer on the GPU (icg_render_view / icg_surface_depth_map,
render.hpp:89-280: view-space progressive localization, shadow culling, candidate and bracket
evaluation, per-pixel depth, texture at covered pixels) against the UNMODIFIED reference
(oracle/_ref render_view) on the same fields: bit-exact for the analytic scenes (fp64 field,
fp64 depth), within the north-star tolerances for the PIFu field."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2007_13988_b200 import abi, api

from .conftest import load_scene_textures

pytestmark = pytest.mark.gpu

CAMERAS = [(90, 0), (30, 20), (0, 0), (200, -35)]


@pytest.fixture(scope="module")
def textures():
    return load_scene_textures()


def ref_scene(prims, tau, tex):
    return O.RefScene(prims=prims, tau=tau, texture=tex)


@pytest.mark.parametrize("name", ["sphere", "torus", "capsule_figure", "thin_rod", "thin_slab", "offset_slab"])
def test_render_view_analytic_scenes_bit_exact(gpu_ctx, scenes, textures, name):
    prims, tau = scenes[name]
    f = api.AnalyticField(prims, tau, textures[name])
    rs = ref_scene(prims, tau, textures[name])
    cfg = api.AlgoConfig("progressive", 16, 2)
    for yaw, pitch in CAMERAS:
        img = gpu_ctx.render_view(f, api.CameraSpec.from_angles(yaw, pitch), cfg, background=(0.1, 0.2, 0.3))
        r = O.ref_render_view(rs, yaw, pitch, 16, 2, bg=(0.1, 0.2, 0.3), workers=8)
        assert img.oracle_calls == r["oracle_calls"], (yaw, pitch)
        assert img.degenerate_brackets == r["degenerate"] and img.grazing_pixels == r["grazing"]
        assert np.array_equal(img.mask, r["mask"]), (yaw, pitch)
        assert np.array_equal(img.depth, r["depth"].astype(np.float32)), (yaw, pitch)
        assert np.array_equal(img.rgb, r["rgb"].astype(np.float32)), (yaw, pitch)
        assert img.covered_pixels == int(r["mask"].sum()) == img.texture_points


def test_surface_depth_map_and_errors(gpu_ctx, scenes, textures):
    prims, tau = scenes["capsule_figure"]
    f = api.AnalyticField(prims, tau, textures["capsule_figure"])
    cam = api.CameraSpec.from_angles(30, 20)
    cfg = api.AlgoConfig("progressive", 16, 2)
    full = gpu_ctx.render_view(f, cam, cfg)
    dm = api.surface_depth_map(gpu_ctx, api.AnalyticField(prims, tau), cam, cfg)  # no texture needed
    assert np.array_equal(dm.depth, full.depth) and np.array_equal(dm.mask, full.mask)
    assert dm.oracle_calls == full.oracle_calls and dm.texture_points == full.covered_pixels
    with pytest.raises(ValueError):  # render_view requires a texture (render.hpp:247)
        gpu_ctx.render_view(api.AnalyticField(prims, tau), cam, cfg)
    with pytest.raises(ValueError):  # depth_pass requires progressive, target level >= 1 (render.hpp:91-94)
        gpu_ctx.render_view(f, cam, api.AlgoConfig("brute", 16, 2))
    with pytest.raises(ValueError):
        gpu_ctx.render_view(f, cam, api.AlgoConfig("progressive", 16, 0))
    # composite (render.hpp:284-291)
    back = np.full((65, 65, 3), 0.5, np.float32)
    comp = api.composite(full, back)
    assert np.array_equal(comp[full.mask == 1], full.rgb[full.mask == 1]) and np.all(comp[full.mask == 0] == 0.5)
    with pytest.raises(ValueError):
        api.composite(full, back[:64])


def test_spec_acceptance_6_shadow_culled_render(gpu_ctx, scenes, textures):
    """sphere, centre depth 0.5 within 2/R, and >= 40 % fewer oracle calls than a full-L
    localization of the view-space field (the reference measures 55.8 %)."""
    prims, tau = scenes["sphere"]
    f = api.AnalyticField(prims, tau, textures["sphere"])
    cfg = api.AlgoConfig("progressive", 16, 4)
    img = gpu_ctx.render_view(f, api.CameraSpec.from_angles(0, 0), cfg)
    n = 257
    assert img.mask[n // 2, n // 2] == 1 and abs(img.depth[n // 2, n // 2] - 0.5) <= 2.0 / 256
    full = gpu_ctx.extract(f, api.AlgoConfig("progressive", 16, 4))  # identity view: same field
    saving = 1.0 - img.oracle_calls / full.total_evals
    assert saving >= 0.40, saving
    r = O.ref_render_view(ref_scene(prims, tau, textures["sphere"]), 0, 0, 16, 4, workers=8)
    assert img.oracle_calls == r["oracle_calls"]
    assert np.array_equal(img.depth, r["depth"].astype(np.float32))


@pytest.mark.parametrize("precision", [abi.ICG_PREC_FP32, abi.ICG_PREC_FP32_SIMT])
def test_render_view_pifu_against_reference(gpu_ctx, pifu_inputs, precision):
    """The PIFu field through the reference's render_view (per-point FieldOracle callbacks of the
    fp64 oracle) against icg_render_view: identical control flow (coverage, oracle calls), depth
    within 1e-4, colours within 1e-3."""
    inp = pifu_inputs
    gpu_ctx.set_mlp(abi.ICG_MLP_GEOMETRY, inp["gw"], inp["gb"])
    gpu_ctx.set_mlp(abi.ICG_MLP_TEXTURE, inp["tw"], inp["tb"])
    f = api.PifuField(inp["fmap"], inp["caps"], 50.0, precision)
    m = O.Pifu(inp["fmap"], inp["caps"], inp["gw"], inp["gb"], inp["tw"], inp["tb"], threads=1)
    for yaw, pitch in ((90, 0), (30, 20)):
        img = gpu_ctx.render_view(f, api.CameraSpec.from_angles(yaw, pitch), api.AlgoConfig("progressive", 16, 2))
        r = O.ref_render_view(m, yaw, pitch, 16, 2, workers=os.cpu_count() or 8)
        assert img.oracle_calls == r["oracle_calls"]
        assert np.array_equal(img.mask, r["mask"])
        cov = img.mask == 1
        assert np.abs(img.depth[cov] - r["depth"][cov]).max() <= 1e-4
        assert np.abs(img.rgb[cov] - r["rgb"][cov]).max() <= 1e-3

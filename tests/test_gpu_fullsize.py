"""Parity at the EXACT configurations bench.py times (BASELINE.json configs[2] and [3]),
through the C ABI, against the reference and the CPU oracle on the same seeded inputs.

For each config, one GPU frame (progressive localization + first-crossing render + texture)
is checked four ways:
  1. control flow, exactly: the GPU's evaluated values are replayed through the REFERENCE's
     extract_progressive (oracle/_ref, localize.hpp:315-363) — it must request only nodes the
     GPU evaluated and reproduce the grid, states and evals_per_level bit for bit; the
     per-level refined-cell and evaluated-node sets (icg_level_set) must equal the oracle
     restatement's on the same replay;
  2. arithmetic, every node: every evaluated node's occupancy against the fp64 oracle
     (1e-4 for the fp32 config, 1e-2 for the bf16 config);
  3. render, exactly: mask, first-crossing index and depth bit-exact against the oracle
     renderer on the GPU's grid; every covered pixel's colour within 1e-3 (1e-2 bf16);
  4. an independent fp64 oracle localization of the same field, compared with the GPU's
     refined-cell and evaluated-node sets and first crossings under the north-star
     tolerance-halo rule (tests/halo.py).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2007_13988_b200 import abi, api

from . import halo as H

pytestmark = pytest.mark.gpu

CONFIGS = {
    # name: (coarsest, level, fmap (C, H, W), render, precision, occ tol, rgb tol)
    "config2": (32, 3, (256, 128, 128), 512, abi.ICG_PREC_FP32, 1e-4, 1e-3),
    "config3": (32, 4, (256, 256, 256), 1024, abi.ICG_PREC_BF16, 1e-2, 1e-2),
}


def node_points(idx, cells):
    n = cells + 1
    i, j, k = idx % n, (idx // n) % n, idx // (n * n)
    return np.stack([-1 + 2 * i / cells, -1 + 2 * j / cells, 1 - 2 * k / cells], 1)


@pytest.fixture(scope="module", params=sorted(CONFIGS))
def frame(request):
    name = request.param
    r0, L, (c, h, w), res, prec, occ_tol, rgb_tol = CONFIGS[name]
    caps = api.gen_capsules(42)
    fmap = api.gen_feature_map(1000, c, h, w)
    gw, gb = api.gen_mlp(7, abi.ICG_MLP_GEOMETRY)
    tw, tb = api.gen_mlp(8, abi.ICG_MLP_TEXTURE)
    ctx = api.Context(0)
    ctx.set_mlp(abi.ICG_MLP_GEOMETRY, gw, gb)
    ctx.set_mlp(abi.ICG_MLP_TEXTURE, tw, tb)
    f = api.PifuField(fmap, caps, 50.0, prec)
    cfg = api.AlgoConfig("progressive", r0, L, keep_level_sets=True)
    cam = api.CameraSpec.from_angles(90, 0)
    ext, img = ctx.frame(f, cfg, cam, res, res, want_grid=True)
    sets = {"evaluated": [ctx.level_set(l, "evaluated") for l in range(L + 1)],
            "refined": [ctx.level_set(l, "refined") for l in range(L + 1)]}
    ctx.close()
    model = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=os.cpu_count() or 8)
    yield dict(name=name, r0=r0, L=L, res=res, occ_tol=occ_tol, rgb_tol=rgb_tol, ext=ext, img=img,
               sets=sets, model=model)


def test_replay_through_reference_exact(frame):
    ext, r0, L = frame["ext"], frame["r0"], frame["L"]
    cells = r0 << L
    ev = ext.states == abi.ICG_STATE_EVALUATED
    assert int(ev.sum()) == ext.total_evals  # no node evaluated twice
    assert np.array_equal(ext.binarized, (ext.values >= 0.5).astype(np.uint8))
    assert not ext.conflict_warning
    rp = O.Replay(ext.values, ext.states, cells)
    assert O.ref_available(), "oracle/_ref (the reference compiled in place) must travel with the repo"
    r = O.ref_extract(rp.pt_fn, rp.user, r0, L, workers=8)
    assert rp.c.misses == 0, "the reference requested nodes the GPU never evaluated"
    assert r["evals_per_level"] == ext.evals_per_level
    assert np.array_equal(r["states"], ext.states)
    assert np.array_equal(r["values"], ext.values)
    # per-level sets: the restatement's replay records them (its control flow is pinned to the
    # reference by tests/test_oracle_vs_reference.py and by the identical grid above)
    rp2 = O.Replay(ext.values, ext.states, cells)
    o = O.extract_progressive(rp2, r0, L, level_sets=True)
    assert rp2.c.misses == 0
    for l in range(L + 1):
        assert np.array_equal(frame["sets"]["evaluated"][l], o["evaluated_sets"][l]), f"evaluated set, level {l}"
        assert np.array_equal(frame["sets"]["refined"][l], o["refined_sets"][l]), f"refined set, level {l}"
        assert len(frame["sets"]["evaluated"][l]) == ext.evals_per_level[l]
        assert len(frame["sets"]["refined"][l]) == ext.refined_cells_per_level[l]


def test_every_evaluated_node_against_oracle(frame):
    ext = frame["ext"]
    cells = frame["r0"] << frame["L"]
    idx = np.flatnonzero(ext.states == abi.ICG_STATE_EVALUATED)
    o = frame["model"].occupancy(node_points(idx, cells))
    err = np.abs(ext.values[idx].astype(np.float64) - o)
    assert err.max() <= frame["occ_tol"], f"max |docc| {err.max():.3e} over {len(idx)} nodes"


def test_render_exact_on_gpu_grid(frame):
    ext, img, res = frame["ext"], frame["img"], frame["res"]
    cells = frame["r0"] << frame["L"]
    r = O.render_first_crossing(ext.values, cells, O.camera_from_angles(90, 0), res, res, tex=frame["model"])
    assert np.array_equal(img.mask, r["mask"])
    assert np.array_equal(img.surface_k, r["surface_k"])
    assert np.array_equal(img.depth, r["depth"])
    assert img.covered_pixels == r["covered"] > 0
    assert img.degenerate_brackets == r["degenerate"] and img.grazing_pixels == r["grazing"]
    cov = img.mask == 1
    err = np.abs(img.rgb[cov] - r["rgb"][cov]).max()
    assert err <= frame["rgb_tol"], f"max colour error {err:.3e} over {int(cov.sum())} covered pixels"
    assert np.array_equal(img.rgb[~cov], r["rgb"][~cov])


def test_independent_oracle_under_tolerance_halo(frame):
    """The fp64 oracle localizes the same field on its own; sets and first crossings must match
    the GPU's exactly outside the north-star tolerance halo."""
    r0, L, res = frame["r0"], frame["L"], frame["res"]
    cells = r0 << L
    o = O.extract_progressive(frame["model"], r0, L, level_sets=True)
    gs = frame["sets"]
    tol = frame["occ_tol"]
    halo = H.build_halo(gs["evaluated"], o["evaluated_sets"], frame["ext"].values, o["values"], L, r0, tol)
    stats = H.compare_outside_halo(gs["evaluated"], o["evaluated_sets"], gs["refined"], o["refined_sets"], halo, L,
                                   r0)
    r = O.render_first_crossing(o["values"], cells, O.camera_from_angles(90, 0), res, res)
    img = frame["img"]
    outside = ~H.ray_touches_halo_yaw90(halo, res, res)
    assert np.array_equal(img.mask[outside], r["mask"][outside])
    assert np.array_equal(img.surface_k[outside], r["surface_k"][outside])
    print(f"{frame['name']}: halo {stats}, pixels inside halo {int((~outside).sum())}")

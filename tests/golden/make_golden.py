"""Regenerates the committed golden fixtures in tests/golden/.

Run in the build container (needs /root/reference for the reference shim):
    python tests/golden/make_golden.py

Fixtures:
  scenes.json        bundled reference scenes (proj/scenes/*.json) exported as
                     union-of-primitive lists through the reference's own loader
                     (scene.hpp:302-333, ref_scene_export)
  ref_extract.json   reference extract_progressive / brute results (evals per
                     level, totals, sha256 of grid values / states / binarized)
                     computed by the UNMODIFIED reference (oracle/_ref)
  pifu_points.npz    PIFu field at fixed points: oracle (C, fp64) and an
                     independent numpy fp64 restatement — the only pin the
                     unhoused PIFu arithmetic has
"""
import glob
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from tests.pifu_numpy import pifu_numpy  # noqa: E402
from paper_2007_13988_b200 import api  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SCENE_DIR = "/root/reference/proj/scenes"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def prim_to_dict(p):
    return dict(kind=p.kind, rotated=p.rotated, center=list(p.center), a=list(p.a), b=list(p.b), radius=p.radius,
                half=list(p.half), major=p.major, minor=p.minor, inv_rotation=list(p.inv_rotation))


def main():
    scenes = {}
    for path in sorted(glob.glob(os.path.join(SCENE_DIR, "*.json"))):
        name = os.path.splitext(os.path.basename(path))[0]
        sc = O.RefScene(path)
        prims, tau, has_tex = sc.export()
        scenes[name] = dict(tau=tau, has_texture=has_tex, prims=[prim_to_dict(p) for p in prims],
                            texture=sc.texture())
    json.dump(scenes, open(os.path.join(OUT, "scenes.json"), "w"), indent=1)

    runs = {}
    cases = [(name, 16, 2) for name in scenes] + [("sphere", 16, 3)]
    for name, r0, lv in cases:
        sc = O.RefScene(os.path.join(SCENE_DIR, name + ".json"))
        for variant, vname in ((3, "progressive"), (0, "brute")):
            r = O.ref_extract(sc.pt_fn, sc.user, r0, lv, variant=variant)
            runs[f"{name}/{r0}/{lv}/{vname}"] = dict(
                evals_per_level=r["evals_per_level"], total_evals=r["total_evals"],
                oracle_calls=r["oracle_calls"], inside=int(r["binarized"].sum()),
                sha_values=sha(r["values"]), sha_states=sha(r["states"]), sha_binarized=sha(r["binarized"]))
        r = O.ref_extract(sc.pt_fn, sc.user, r0, lv, conflict_pass=False)
        runs[f"{name}/{r0}/{lv}/no_conflict"] = dict(evals_per_level=r["evals_per_level"],
                                                     sha_binarized=sha(r["binarized"]))
    # config-0 capsule figure (seed 42), 32 -> 128
    caps = api.gen_capsules(42)
    rs = O.RefScene(capsules=caps, tau=0.02)
    r = O.ref_extract(rs.pt_fn, rs.user, 32, 2)
    runs["capsules42/32/2/progressive"] = dict(evals_per_level=r["evals_per_level"], total_evals=r["total_evals"],
                                              inside=int(r["binarized"].sum()), sha_values=sha(r["values"]),
                                              sha_states=sha(r["states"]), sha_binarized=sha(r["binarized"]))
    json.dump(runs, open(os.path.join(OUT, "ref_extract.json"), "w"), indent=1)

    # PIFu field at fixed points
    fmap = api.gen_feature_map(1000, 256, 32, 32)
    gw, gb = api.gen_mlp(7, 0)
    tw, tb = api.gen_mlp(8, 1)
    rng = np.random.default_rng(1234)
    pts = rng.uniform(-1.0, 1.0, (256, 3))
    pts[:32] = (np.round((pts[:32] + 1) * 32) / 32 - 1)  # some lattice nodes
    m = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=1)
    occ, logit, tex = m.occupancy(pts), m.logit(pts), m.texture(pts)
    n_occ, n_logit, n_tex = pifu_numpy(fmap, api.capsules_array(caps), gw, gb, tw, tb, pts)
    np.savez_compressed(os.path.join(OUT, "pifu_points.npz"), points=pts, occupancy=occ, logit=logit, texture=tex,
                        np_occupancy=n_occ, np_logit=n_logit, np_texture=n_tex,
                        seeds=np.array([42, 1000, 7, 8]), fmap_shape=np.array([256, 32, 32]))
    print("max |oracle - numpy| logit", np.abs(logit - n_logit).max(), "tex", np.abs(tex - n_tex).max())


if __name__ == "__main__":
    main()

import sys, numpy as np
sys.path.insert(0, '.')
from tests.conftest import load_scenes, load_scene_textures
from oracle import oracle as O
from paper_2007_13988_b200 import api
sc = load_scenes(); tx = load_scene_textures()
ctx = api.Context(0)
for name in ["torus", "capsule_figure"]:
    prims, tau = sc[name]
    f = api.AnalyticField(prims, tau, tx[name])
    for yaw, pitch in [(0, 0), (90, 0)]:
        img = ctx.render_view(f, api.CameraSpec.from_angles(yaw, pitch), api.AlgoConfig("progressive", 16, 2))
        r = O.ref_render_view(O.RefScene(prims=prims, tau=tau, texture=tx[name]), yaw, pitch, 16, 2, workers=8)
        d = img.depth.astype(np.float64) - r["depth"].astype(np.float32).astype(np.float64)
        bad = np.argwhere(np.abs(d) > 0)
        print(name, yaw, pitch, "ndiff", len(bad), "max", np.abs(d).max(), "calls", img.oracle_calls, r["oracle_calls"])
        for (row, col) in bad[:5]:
            print("   px", row, col, "gpu %.9g" % img.depth[row, col], "ref %.17g" % r["depth"][row, col], "k", img.surface_k[row, col])

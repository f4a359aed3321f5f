"""Column-factored vs full geometry field on one config-2 frame: values, evaluated sets, device time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2007_13988_b200 import abi, api
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
prec = abi.ICG_PREC_BF16 if len(sys.argv) > 1 and sys.argv[1] == "bf16" else abi.ICG_PREC_FP32
res = {}
for fact in (False, True):
    os.environ["ICG_NO_FACT"] = "0" if fact else "1"
    ctx = api.Context(0); ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
    f = api.PifuField(fmap, caps, 50.0, prec)
    cfg = api.AlgoConfig("progressive", 32, 3); cam = api.CameraSpec.from_angles(90, 0)
    for i in range(3):
        ext, img = ctx.frame(f, cfg, cam, 512, 512, want_grid=True)
    ts = []
    for i in range(5):
        e2, i2 = ctx.frame(f, cfg, cam, 512, 512)
        ts.append(i2.wall_seconds * 1e3)
    res[fact] = (ext, img)
    print("fact" if fact else "full", "evals", ext.evals_per_level, "frame ms", np.round(ts, 3), flush=True)
    ctx.close() if hasattr(ctx, "close") else None
(e0, i0), (e1, i1) = res[False], res[True]
ev0 = e0.states == abi.ICG_STATE_EVALUATED
ev1 = e1.states == abi.ICG_STATE_EVALUATED
both = ev0 & ev1
print("evaluated sets equal:", bool((ev0 == ev1).all()), "sym diff", int((ev0 != ev1).sum()))
print("max |dv| at common evaluated nodes:", float(np.abs(e0.values[both] - e1.values[both]).max()))
print("surface_k equal:", bool(np.array_equal(i0.surface_k, i1.surface_k)), "max |drgb|", float(np.abs(i0.rgb - i1.rgb).max()))

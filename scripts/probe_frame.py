"""Quick timing probe of one frame with a per-stage device-time breakdown (dev tool).

usage: probe_frame.py [simt|fp32|bf16] [config2|config3]
"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2007_13988_b200 import abi, api
prec = {"simt": abi.ICG_PREC_FP32_SIMT, "fp32": abi.ICG_PREC_FP32, "bf16": abi.ICG_PREC_BF16}[sys.argv[1] if len(sys.argv) > 1 else "simt"]
cfgname = sys.argv[2] if len(sys.argv) > 2 else "config2"
r0, lv, (C, H, W), res = {"config2": (32, 3, (256, 128, 128), 512), "config3": (32, 4, (256, 256, 256), 1024)}[cfgname]
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000, C, H, W)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
ctx = api.Context(0)
ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
f = api.PifuField(fmap, caps, 50.0, prec)
cfg = api.AlgoConfig("progressive", r0, lv); cam = api.CameraSpec.from_angles(90, 0)
for i in range(3):
    t = time.time(); ext, img = ctx.frame(f, cfg, cam, res, res); dt = time.time() - t
    print(f"frame {i}: host {dt*1e3:.1f} ms device {img.wall_seconds*1e3:.1f} ms evals {ext.evals_per_level} total {ext.total_evals} "
          f"iters {ext.conflict_iters_per_level} covered {img.covered_pixels} deg {img.degenerate_brackets} graz {img.grazing_pixels}")
ctx.profile(True)
ext, img = ctx.frame(f, cfg, cam, res, res)
p = ctx.profile_get()
ctx.profile(False)
print("profile:", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in p.items()})
if cfgname == "config2":
    a = api.AnalyticField(caps, 0.02)
    for i in range(2):
        t = time.time(); e = ctx.extract(a, cfg, want_grid=False); print(f"analytic extract: host {(time.time()-t)*1e3:.2f} ms device {e.wall_seconds*1e3:.3f} ms {e.evals_per_level}")

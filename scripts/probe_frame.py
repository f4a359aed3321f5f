"""Quick timing probe of one config-2 frame (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2007_13988_b200 import abi, api
prec = {"simt": abi.ICG_PREC_FP32_SIMT, "fp32": abi.ICG_PREC_FP32, "bf16": abi.ICG_PREC_BF16}[sys.argv[1] if len(sys.argv) > 1 else "simt"]
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
ctx = api.Context(0)
ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
f = api.PifuField(fmap, caps, 50.0, prec)
cfg = api.AlgoConfig("progressive", 32, 3); cam = api.CameraSpec.from_angles(90, 0)
for i in range(3):
    t = time.time(); ext, img = ctx.frame(f, cfg, cam, 512, 512); dt = time.time() - t
    print(f"frame {i}: host {dt*1e3:.1f} ms device {img.wall_seconds*1e3:.1f} ms evals {ext.evals_per_level} total {ext.total_evals} "
          f"iters {ext.conflict_iters_per_level} covered {img.covered_pixels} deg {img.degenerate_brackets} graz {img.grazing_pixels}")
a = api.AnalyticField(caps, 0.02)
for i in range(3):
    t = time.time(); e = ctx.extract(a, cfg, want_grid=False); print(f"analytic extract: host {(time.time()-t)*1e3:.2f} ms device {e.wall_seconds*1e3:.3f} ms {e.evals_per_level}")

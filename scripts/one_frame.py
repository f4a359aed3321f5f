"""Runs W warm-up frames then one frame (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_13988_b200 import abi, api
prec = {"simt": abi.ICG_PREC_FP32_SIMT, "fp32": abi.ICG_PREC_FP32, "bf16": abi.ICG_PREC_BF16}[sys.argv[1]]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
ctx = api.Context(0); ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
f = api.PifuField(fmap, caps, 50.0, prec)
cfg = api.AlgoConfig("progressive", 32, 3); cam = api.CameraSpec.from_angles(90, 0)
for i in range(warm + 1):
    ext, img = ctx.frame(f, cfg, cam, 512, 512)
print("device ms", img.wall_seconds * 1e3)

"""Runs W warm-up frames then one frame of a bench config (for ncu launch lists / captures):
python scripts/one_frame.py [config2|config3] [W]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_13988_b200 import abi, api  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "config2"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 2
r0, lv, (c, h, w), res, prec = {"config2": (32, 3, (256, 128, 128), 512, abi.ICG_PREC_FP32),
                                 "config3": (32, 4, (256, 256, 256), 1024, abi.ICG_PREC_BF16)}[cfg_name]
caps = api.gen_capsules(42)
fmap = api.gen_feature_map(1000, c, h, w)
gw, gb = api.gen_mlp(7, 0)
tw, tb = api.gen_mlp(8, 1)
ctx = api.Context(0)
ctx.set_mlp(0, gw, gb)
ctx.set_mlp(1, tw, tb)
f = api.PifuField(fmap, caps, 50.0, prec)
cfg = api.AlgoConfig("progressive", r0, lv)
cam = api.CameraSpec.from_angles(90, 0)
for i in range(warm + 1):
    ext, img = ctx.frame(f, cfg, cam, res, res)
print("device ms", img.wall_seconds * 1e3, "evals", ext.total_evals)

"""Per-level evaluation counts of one config-2 frame and the level-3 E0 / chain split
(ICG_CHAIN_TRACE prints the chain batches): python scripts/e0_count.py [config2|config3]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_13988_b200 import abi, api  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "config2"
r0, lv, (c, h, w), prec = {"config2": (32, 3, (256, 128, 128), abi.ICG_PREC_FP32),
                           "config3": (32, 4, (256, 256, 256), abi.ICG_PREC_BF16)}[cfg_name]
ctx = api.Context(0)
gw, gb = api.gen_mlp(7, 0)
ctx.set_mlp(0, gw, gb)
f = api.PifuField(api.gen_feature_map(1000, c, h, w), api.gen_capsules(42), 50.0, prec)
ext = ctx.extract(f, api.AlgoConfig("progressive", r0, lv))
print("evals_per_level", list(ext.evals_per_level), "total", ext.total_evals)

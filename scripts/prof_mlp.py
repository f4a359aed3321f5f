"""Isolated fused-MLP launches for ncu: warm-up, then one 64-point batch and one 300k-point batch."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2007_13988_b200 import abi, api
prec = {"fp32": abi.ICG_PREC_FP32, "bf16": abi.ICG_PREC_BF16}[sys.argv[1] if len(sys.argv) > 1 else "fp32"]
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
ctx = api.Context(0); ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
f = api.PifuField(fmap, caps, 50.0, prec)
rng = np.random.default_rng(0)
small = rng.uniform(-1, 1, (64, 3)); big = rng.uniform(-1, 1, (300000, 3))
ctx.occupancy_batch(f, small); ctx.occupancy_batch(f, big)      # warm-up (2 launches)
ctx.occupancy_batch(f, small)                                    # launch 3: single tile
ctx.occupancy_batch(f, big)                                      # launch 4: 4688 tiles
print("ok")

"""Device time of the geometry field on fixed batches (CUDA events via the library profiler)."""
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
for n in (64, 128, 9472, 300000):
    pts = rng.uniform(-1, 1, (n, 3))
    ctx.occupancy_batch(f, pts)
    ctx.profile(True, reset=True)
    for _ in range(3): ctx.occupancy_batch(f, pts)
    pr = ctx.profile_get(); ms = pr["geo_mlp_ms"] / 3
    print(f"{sys.argv[1] if len(sys.argv)>1 else 'fp32'} n={n:7d}: {ms*1e3:9.1f} us  -> {n*2363906/(ms/1e3)/1e12:7.1f} TFLOP/s alg")
    ctx.profile(False)

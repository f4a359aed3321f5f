import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2007_13988_b200 import abi, api
from oracle import oracle as O
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
ctx = api.Context(0); ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
f = api.PifuField(fmap, caps, 50.0, abi.ICG_PREC_FP32_SIMT)
rng = np.random.default_rng(5); pts = rng.uniform(-1, 1, (64, 3))
m = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=4)
o = m.occupancy(pts); lo = m.logit(pts)
a = ctx.occupancy_batch(f, pts); b = ctx.occupancy_batch(f, pts)
print("repeat equal:", np.array_equal(a, b))
singles = np.array([ctx.occupancy_batch(f, p[None])[0] for p in pts])
print("single vs batch max diff", np.abs(singles - a).max())
la = np.log(a) - np.log1p(-a.astype(np.float64)); 
print("logit gpu vs oracle:", np.c_[la[:12], lo[:12]])
print("max occ diff", np.abs(a - o).max(), "singles", np.abs(singles - o).max())
# zero feature map -> isolates gather
f0 = api.PifuField(np.zeros_like(fmap), caps, 50.0, abi.ICG_PREC_FP32_SIMT)
m0 = O.Pifu(np.zeros_like(fmap), caps, gw, gb, tw, tb, threads=4)
a0 = ctx.occupancy_batch(f0, pts); print("zero fmap max diff", np.abs(a0 - m0.occupancy(pts)).max())

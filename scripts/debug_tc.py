import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2007_13988_b200 import abi, api
from oracle import oracle as O
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
ctx = api.Context(0); ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
m = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=8)
rng = np.random.default_rng(5); pts = rng.uniform(-1, 1, (1000, 3))
o = m.occupancy(pts); lo = m.logit(pts)
for name, prec in (("simt", abi.ICG_PREC_FP32_SIMT), ("tc_x3", abi.ICG_PREC_FP32), ("tc_bf16", abi.ICG_PREC_BF16)):
    f = api.PifuField(fmap, caps, 50.0, prec)
    t = time.time(); a = ctx.occupancy_batch(f, pts); dt = time.time() - t
    la = np.log(np.maximum(a, 1e-30)) - np.log1p(-np.minimum(a.astype(np.float64), 1 - 1e-7))
    print(name, "occ max diff %.3e" % np.abs(a - o).max(), "logit diff (|l|<10) %.3e" % np.abs(la - lo)[np.abs(lo) < 10].max() if (np.abs(lo) < 10).any() else "", "%.1f ms" % (dt * 1e3))
    print("   first logits", np.c_[la[:4], lo[:4]].ravel())
    tx = ctx.texture_batch(f, pts[:256]); to = m.texture(pts[:256])
    print("   tex max diff %.3e" % np.abs(tx - to).max())

import sys, os
sys.path.insert(0, "/root/repo")
from paper_2007_13988_b200 import abi, api
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
ctx = api.Context(0); ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
f = api.PifuField(fmap, caps, 50.0, abi.ICG_PREC_FP32)
g = ctx.extract(f, api.AlgoConfig("progressive", 8, 3))
print("ok", g.total_evals)

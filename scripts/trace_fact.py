"""One big column-factored batch (config-2 L3 sized) with the pair-kernel event trace (dev tool):
ICG_TC_TRACE=1 ICG_TC_EVENTS=1 python scripts/trace_fact.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_13988_b200 import abi, api
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
ctx = api.Context(0); ctx.set_mlp(0, gw, gb); ctx.set_mlp(1, tw, tb)
f = api.PifuField(fmap, caps, 50.0, abi.ICG_PREC_FP32)
ext = ctx.extract(f, api.AlgoConfig("brute", 64, 0))
print("evals", ext.total_evals)

"""One big column-factored batch (a dense 65^3 grid, 274,625 points) with the k_fact2 wait trace
(dev tool): ICG_TC_TRACE=1 python scripts/trace_fact.py [fp32|bf16]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_13988_b200 import abi, api  # noqa: E402

prec = {"fp32": abi.ICG_PREC_FP32, "bf16": abi.ICG_PREC_BF16}[sys.argv[1] if len(sys.argv) > 1 else "fp32"]
caps = api.gen_capsules(42)
fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0)
ctx = api.Context(0)
ctx.set_mlp(0, gw, gb)
f = api.PifuField(fmap, caps, 50.0, prec)
for _ in range(2):
    ext = ctx.extract(f, api.AlgoConfig("brute", 64, 0))
print("evals", ext.total_evals, "ms", ext.wall_seconds * 1e3)

"""k_fact2 against k_mlp_pair<FACT> on the fp32 512^3 hierarchy (dev tool)."""
import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_2007_13988_b200 import abi, api
caps = api.gen_capsules(42); fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0); tw, tb = api.gen_mlp(8, 1)
out = {}
for f2 in ("1", "0"):
    os.environ["ICG_FACT2"] = f2
    c = api.Context(0); c.set_mlp(0, gw, gb); c.set_mlp(1, tw, tb)
    f = api.PifuField(fmap, caps, 50.0, abi.ICG_PREC_FP32)
    e = c.extract(f, api.AlgoConfig("progressive", 32, 4))
    out[f2] = (e.total_evals, e.states.copy(), e.values.copy(), e.wall_seconds)
    c.close()
a, b = out["1"], out["0"]
print("evals", a[0], b[0], "states equal", bool(np.array_equal(a[1], b[1])), "max|dv| %.3e" % np.abs(a[2] - b[2]).max(),
      "ms %.2f vs %.2f" % (a[3] * 1e3, b[3] * 1e3))

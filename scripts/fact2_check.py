"""Swapped-operand factored pass (k_fact2.cu, ICG_FACT2=1) against k_mlp_pair<FACT> (dev tool):
values, states and counts of the same extractions."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_13988_b200 import abi, api

caps = api.gen_capsules(42)
fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0)
tw, tb = api.gen_mlp(8, 1)


def ctx(f2):
    os.environ["ICG_FACT2"] = "1" if f2 else "0"
    c = api.Context(0)
    c.set_mlp(0, gw, gb)
    c.set_mlp(1, tw, tb)
    return c


ca, cb = ctx(False), ctx(True)
f = api.PifuField(fmap, caps, 50.0, abi.ICG_PREC_FP32)
for cfg in (api.AlgoConfig("brute", 64, 0), api.AlgoConfig("progressive", 16, 3), api.AlgoConfig("progressive", 32, 3)):
    ea, eb = ca.extract(f, cfg), cb.extract(f, cfg)
    ev = ea.states == 2
    d = np.abs(ea.values - eb.values)
    print(cfg.variant, cfg.coarsest_cells, cfg.target_level, "evals", ea.total_evals, eb.total_evals,
          "max|dv| %.3e" % d.max(), "states equal", bool(np.array_equal(ea.states, eb.states)),
          "evaluated-set equal", bool(np.array_equal(ev, eb.states == 2)))
for c, name in ((ca, "FACT"), (cb, "FACT2")):
    cfg = api.AlgoConfig("progressive", 32, 3)
    for _ in range(3):
        c.extract(f, cfg)
    t = time.time()
    for _ in range(10):
        e = c.extract(f, cfg)
    print(name, "extract wall ms %.3f" % ((time.time() - t) * 100), "device ms %.3f" % (e.wall_seconds * 1e3))

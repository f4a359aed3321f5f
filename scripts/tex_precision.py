"""Texture-kernel precision model (dev tool): colour error of fp16 operand schemes against fp64.
Every layer input (Phi, hidden activations, h3) is rounded to one fp16 copy, as the texture kernel
stores them; weights are fp16 hi + lo (2 MMAs per K step, the shipped scheme) or one fp16 copy
(1 MMA per K step); products accumulate in fp32-or-better; the z column enters in fp32."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_13988_b200 import api
from tests.pifu_numpy import _phi

f16 = lambda a: a.astype(np.float16).astype(np.float64)


def wsplit(w, single):
    hi = f16(w)
    return hi if single else hi + f16(w - hi)


def mlp(ws, bs, skip_main, z, upto, single, quant, slope=0.02):
    h = None
    for l in range(upto):
        w = ws[l].astype(np.float64)
        x = skip_main if h is None else np.concatenate([h, skip_main], 1)
        wm, wz = w[:, :-1], w[:, -1]
        if quant:
            acc = f16(x) @ wsplit(wm, single).T
        else:
            acc = x @ wm.T
        h = acc + z[:, None] * wz + bs[l].astype(np.float64)
        if l < 4:
            h = np.where(h < 0, h * slope, h)
    return h


caps = api.gen_capsules(42)
fmap = api.gen_feature_map(1000)
gw, gb = api.gen_mlp(7, 0)
tw, tb = api.gen_mlp(8, 1)
rng = np.random.default_rng(3)
pts = rng.uniform(-0.8, 0.8, size=(20000, 3))
phi = _phi(fmap, pts)
z = pts[:, 2]
for name, single in (("fp16 hi+lo weights", False), ("fp16 single weights", True)):
    out = {}
    for quant in (False, True):
        h3 = mlp(gw, gb, phi, z, 3, single, quant)
        t = 1.0 / (1.0 + np.exp(-mlp(tw, tb, np.concatenate([phi, h3], 1), z, 5, single, quant)))
        out[quant] = t
    err = np.abs(out[True] - out[False])
    print(f"{name}: max |d rgb| {err.max():.2e}  p99.9 {np.quantile(err, 0.999):.2e}  mean {err.mean():.2e}")
for name, sp, st in (("prefix hi+lo, texture single", False, True), ("prefix single, texture hi+lo", True, False)):
    h3q = mlp(gw, gb, phi, z, 3, sp, True)
    tq = 1.0 / (1.0 + np.exp(-mlp(tw, tb, np.concatenate([phi, h3q], 1), z, 5, st, True)))
    h3 = mlp(gw, gb, phi, z, 3, sp, False)
    t = 1.0 / (1.0 + np.exp(-mlp(tw, tb, np.concatenate([phi, h3], 1), z, 5, st, False)))
    err = np.abs(tq - t)
    print(f"{name}: max |d rgb| {err.max():.2e}  p99.9 {np.quantile(err, 0.999):.2e}")

"""Independent numpy fp64 restatement of the PIFu field (test-only).

Written separately from oracle/isocull_oracle.c (vectorised over points,
different loop structure) so the two pin each other: the PIFu arithmetic has
no reference implementation, BASELINE.json configs[1-3] define it.
"""
import numpy as np


def _capsule_sdf(caps, p):
    d = None
    for row in caps:
        a, b, r = row[0:3], row[3:6], row[6]
        pa, ba = p - a, b - a
        den = ba @ ba
        h = np.clip((pa @ ba) / den, 0.0, 1.0) if den > 0 else np.zeros(len(p))
        v = pa - h[:, None] * ba
        di = np.sqrt((v * v).sum(1)) - r
        d = di if d is None else np.minimum(d, di)
    return d


def _phi(fmap, p):
    C, H, W = fmap.shape
    u = np.clip((p[:, 0] + 1.0) * 0.5 * (W - 1), 0, W - 1)
    v = np.clip((1.0 - p[:, 1]) * 0.5 * (H - 1), 0, H - 1)
    x0 = np.minimum(np.floor(u).astype(int), W - 2)
    y0 = np.minimum(np.floor(v).astype(int), H - 2)
    ax, ay = u - x0, v - y0
    f = fmap.astype(np.float64)
    return ((1 - ax) * (1 - ay))[:, None] * f[:, y0, x0].T + (ax * (1 - ay))[:, None] * f[:, y0, x0 + 1].T + \
        ((1 - ax) * ay)[:, None] * f[:, y0 + 1, x0].T + (ax * ay)[:, None] * f[:, y0 + 1, x0 + 1].T


def _mlp(ws, bs, skip, upto, slope=0.02):
    h = None
    for l in range(upto):
        x = skip if h is None else np.concatenate([h, skip], 1)
        h = x @ ws[l].astype(np.float64).T + bs[l].astype(np.float64)
        if l < 4:
            h = np.where(h < 0, h * slope, h)
    return h


def pifu_numpy(fmap, caps, gw, gb, tw, tb, pts, sdf_scale=50.0):
    pts = np.asarray(pts, np.float64)
    phi = _phi(fmap, pts)
    skip = np.concatenate([phi, pts[:, 2:3]], 1)
    out = _mlp(gw, gb, skip, 5)[:, 0]
    logit = out - sdf_scale * _capsule_sdf(caps, pts)
    occ = 1.0 / (1.0 + np.exp(-logit))
    h3 = _mlp(gw, gb, skip, 3)
    tskip = np.concatenate([phi, h3, pts[:, 2:3]], 1)
    tex = 1.0 / (1.0 + np.exp(-_mlp(tw, tb, tskip, 5)))
    return occ, logit, tex

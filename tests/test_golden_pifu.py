"""PIFu field restatement pins: the C oracle against the committed golden
vectors and against an independent numpy fp64 restatement (tests/pifu_numpy.py)."""
import os

import numpy as np

from oracle import oracle as O
from paper_2007_13988_b200 import api
from tests.pifu_numpy import pifu_numpy

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pifu_points.npz")


def _model():
    g = np.load(GOLD)
    cs, fs, gs, ts = (int(x) for x in g["seeds"])
    c, h, w = (int(x) for x in g["fmap_shape"])
    caps = api.gen_capsules(cs)
    fmap = api.gen_feature_map(fs, c, h, w)
    gw, gb = api.gen_mlp(gs, 0)
    tw, tb = api.gen_mlp(ts, 1)
    return g, caps, fmap, gw, gb, tw, tb


def test_oracle_matches_golden_vectors():
    g, caps, fmap, gw, gb, tw, tb = _model()
    m = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=2)
    pts = g["points"]
    assert np.array_equal(m.logit(pts), g["logit"])
    assert np.array_equal(m.occupancy(pts), g["occupancy"])
    assert np.array_equal(m.texture(pts), g["texture"])


def test_oracle_matches_independent_numpy():
    g, caps, fmap, gw, gb, tw, tb = _model()
    occ, logit, tex = pifu_numpy(fmap, api.capsules_array(caps), gw, gb, tw, tb, g["points"])
    assert np.abs(logit - g["logit"]).max() < 1e-10
    assert np.abs(occ - g["occupancy"]).max() < 1e-12
    assert np.abs(tex - g["texture"]).max() < 1e-12


def test_field_properties():
    g, caps, fmap, gw, gb, tw, tb = _model()
    occ, tex = g["occupancy"], g["texture"]
    assert np.all((occ >= 0) & (occ <= 1)) and np.all((tex >= 0) & (tex <= 1))
    # batching independence: per-point evaluation equals the batch
    m = O.Pifu(fmap, caps, gw, gb, tw, tb, threads=1)
    one = np.array([m.logit(p[None])[0] for p in g["points"][:8]])
    assert np.array_equal(one, g["logit"][:8])

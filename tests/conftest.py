import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")
    config.addinivalue_line("markers", "slow: long-running")


def load_scenes():
    from paper_2007_13988_b200 import abi
    data = json.load(open(os.path.join(GOLDEN, "scenes.json")))
    out = {}
    for name, sc in data.items():
        prims = []
        for d in sc["prims"]:
            p = abi.icg_primitive()
            p.kind, p.rotated = d["kind"], d["rotated"]
            p.center[:] = d["center"]
            p.a[:] = d["a"]
            p.b[:] = d["b"]
            p.radius = d["radius"]
            p.half[:] = d["half"]
            p.major, p.minor = d["major"], d["minor"]
            p.inv_rotation[:] = d["inv_rotation"]
            prims.append(p)
        out[name] = (prims, sc["tau"])
    return out


def load_scene_textures():
    """Texture rules of the bundled scenes as the reference parsed them (scene.hpp:272-298)."""
    data = json.load(open(os.path.join(GOLDEN, "scenes.json")))
    return {name: sc.get("texture", {"kind": 0}) for name, sc in data.items()}


@pytest.fixture(scope="session")
def scenes():
    return load_scenes()


@pytest.fixture(scope="session")
def ref_golden():
    return json.load(open(os.path.join(GOLDEN, "ref_extract.json")))


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2007_13988_b200 import api
    ctx = api.Context(0)
    yield ctx
    ctx.close()


@pytest.fixture(scope="session")
def pifu_inputs():
    """Seeded PIFu inputs at test scale: capsules(42), fmap(1000) 256x128x128, weights(7, 8)."""
    from paper_2007_13988_b200 import api
    caps = api.gen_capsules(42)
    fmap = api.gen_feature_map(1000)
    gw, gb = api.gen_mlp(7, 0)
    tw, tb = api.gen_mlp(8, 1)
    return dict(caps=caps, fmap=fmap, gw=gw, gb=gb, tw=tw, tb=tb)

"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares; host-side helpers and argument validation work without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2007_13988_b200 import abi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "isocull_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(icg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(abi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    bound = {name for name, _, _ in abi.SIGNATURES}
    assert set(syms) == bound


def test_abi_version_and_struct_sizes():
    lib = abi.lib()
    assert lib.icg_abi_version() == abi.ICG_ABI_VERSION == 4
    # spot-check layouts against the C compiler's view
    assert C.sizeof(abi.icg_primitive) == 8 + 8 * 24
    assert C.sizeof(abi.icg_algo_config) == 32
    assert C.sizeof(abi.icg_camera) == 13 * 8
    assert C.sizeof(abi.icg_profile) == 30 * 8


def test_no_device_is_reported_not_faked():
    n = C.c_int(-1)
    assert abi.lib().icg_device_count(C.byref(n)) == abi.ICG_OK
    if n.value == 0:
        with pytest.raises(RuntimeError):
            api.Context(0)


def test_host_helpers():
    outs, ins, skip, nw, nb = api.mlp_shape(abi.ICG_MLP_GEOMETRY)
    assert outs == [1024, 512, 256, 128, 1] and ins == [257, 1281, 769, 513, 385] and skip == 257
    assert nw == 1183874 - 1665 + 0 or nw == sum(o * i for o, i in zip(outs, ins))
    assert sum(o * i for o, i in zip(outs, ins)) == 1181953  # MACs per point
    outs, ins, skip, nw, nb = api.mlp_shape(abi.ICG_MLP_TEXTURE)
    assert ins == [513, 1537, 1025, 769, 641] and nw == 1675011
    cam = api.CameraSpec.from_angles(90, 0)
    # yaw 90: view x = world z, view z = -world x (render.hpp:36-45)
    assert np.allclose(cam.rotation @ np.array([1.0, 0, 0]), [0, 0, -1])
    assert np.allclose(cam.rotation @ np.array([0, 0, 1.0]), [1, 0, 0])


def test_config_validation_errors_without_gpu():
    # validate_config, localize.hpp:47-55 -> ValueError (invalid_argument)
    with pytest.raises(ValueError):
        api.AlgoConfig(variant="octree_magic").to_c()
    assert api.acceleration_factor(api.ExtractionResult(0, None, None, None, [], 10, [], [], False, 0.0),
                                   api.ExtractionResult(0, None, None, None, [], 100, [], [], False, 0.0)) == 10.0
    with pytest.raises(ValueError):
        api.compare_iou(np.zeros(3, np.uint8), np.zeros(4, np.uint8))


def test_argument_validation_without_gpu():
    lib = abi.lib()
    a = np.ones(8, np.uint8)
    out = C.c_double()
    p = a.ctypes.data_as(abi.u8p)
    # device arrays need a context (no host dereference of device pointers); unknown mem is rejected
    assert lib.icg_compare_iou(None, p, p, 8, abi.ICG_MEM_DEVICE, C.byref(out)) == abi.ICG_EINVAL
    assert lib.icg_compare_iou(None, p, p, 8, 7, C.byref(out)) == abi.ICG_EINVAL
    assert lib.icg_compare_iou(None, p, p, 8, abi.ICG_MEM_HOST, C.byref(out)) == abi.ICG_OK and out.value == 1.0
    n = C.c_size_t(5)
    assert lib.icg_level_set(None, 0, abi.ICG_SET_EVALUATED_NODES, abi.ICG_MEM_HOST, None, 0,
                             C.byref(n)) == abi.ICG_EINVAL
    assert lib.icg_memcpy(None, None, None, 0, 0, 0) == abi.ICG_EINVAL

"""Output formats: write_ppm / write_float_map / dump_grid
are byte-identical to the reference's own writers (image.hpp:18-48,
grid.hpp:199-222, run through oracle/_ref), and load_grid_dump round-trips."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2007_13988_b200 import api  # noqa: E402
from oracle import oracle as O  # noqa: E402

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference shim not built")


def _rgb(w, h, seed=3):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-0.2, 1.2, (h, w, 3))
    # exact half-way bytes, clamp edges
    a.reshape(-1)[:8] = [0.5 / 255, 1.5 / 255, 254.5 / 255, 0.0, 1.0, -0.0, 0.5, 127.5 / 255]
    return a


@needs_ref
def test_ppm_bytes_match_reference(tmp_path):
    w, h = 37, 23
    rgb = _rgb(w, h)
    mine, ref = str(tmp_path / "a.ppm"), str(tmp_path / "b.ppm")
    api.write_ppm(mine, w, h, rgb)
    flat = np.ascontiguousarray(rgb.reshape(-1))
    assert O.ref().ref_write_ppm(ref.encode(), w, h, flat.ctypes.data_as(O.f64p)) == 0
    assert open(mine, "rb").read() == open(ref, "rb").read()


@needs_ref
def test_float_map_bytes_match_reference(tmp_path):
    w, h = 19, 11
    v = np.random.default_rng(5).normal(size=w * h)
    v[:3] = [-2.0, 1e-40, 3.4e38]
    mine, ref = str(tmp_path / "a.f32"), str(tmp_path / "b.f32")
    api.write_float_map(mine, w, h, v)
    assert O.ref().ref_write_float_map(ref.encode(), w, h, v.ctypes.data_as(O.f64p)) == 0
    assert open(mine, "rb").read() == open(ref, "rb").read()


@needs_ref
def test_grid_dump_bytes_match_reference_and_round_trip(tmp_path):
    import ctypes as C
    cells, level = 8, 2
    v = np.random.default_rng(9).uniform(0, 1, (cells + 1) ** 3).astype(np.float32)
    mine, ref = str(tmp_path / "a.grid"), str(tmp_path / "b.grid")
    api.dump_grid(mine, level, cells, v)
    assert O.ref().ref_dump_grid(ref.encode(), level, cells, v.ctypes.data_as(C.POINTER(C.c_float))) == 0
    assert open(mine, "rb").read() == open(ref, "rb").read()
    lv, R, back = api.load_grid_dump(ref)
    assert (lv, R) == (level, cells) and np.array_equal(back, v)


def test_format_errors(tmp_path):
    with pytest.raises(ValueError):
        api.write_ppm(str(tmp_path / "x.ppm"), 4, 4, np.zeros(5))
    with pytest.raises(ValueError):
        api.write_float_map(str(tmp_path / "x.f32"), 4, 4, np.zeros(5))
    p = tmp_path / "short.grid"
    p.write_bytes(b"\x00\x00")
    with pytest.raises(RuntimeError):
        api.load_grid_dump(str(p))


@needs_ref
def test_c_abi_writers_match_reference(tmp_path):
    """The C-ABI stream writers (icg_write_ppm / icg_write_float_map / icg_dump_grid /
    icg_load_grid_dump) on fp32 buffers: byte-identical to the reference writers fed the same
    values; host-only, no GPU."""
    import ctypes as C
    from paper_2007_13988_b200 import abi
    lib = abi.lib()
    w, h = 29, 13
    rgb = _rgb(w, h).astype(np.float32)
    d64 = np.ascontiguousarray(rgb.astype(np.float64).reshape(-1))
    a, b = str(tmp_path / "a.ppm"), str(tmp_path / "b.ppm")
    assert lib.icg_write_ppm(a.encode(), w, h, np.ascontiguousarray(rgb).ctypes.data_as(abi.f32p)) == 0
    assert O.ref().ref_write_ppm(b.encode(), w, h, d64.ctypes.data_as(O.f64p)) == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    v = np.random.default_rng(2).normal(size=w * h).astype(np.float32)
    a, b = str(tmp_path / "a.f32"), str(tmp_path / "b.f32")
    assert lib.icg_write_float_map(a.encode(), w, h, v.ctypes.data_as(abi.f32p)) == 0
    v64 = v.astype(np.float64)
    assert O.ref().ref_write_float_map(b.encode(), w, h, v64.ctypes.data_as(O.f64p)) == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    g = np.random.default_rng(4).uniform(0, 1, 9 ** 3).astype(np.float32)
    a, b = str(tmp_path / "a.grid"), str(tmp_path / "b.grid")
    assert lib.icg_dump_grid(a.encode(), 1, 8, g.ctypes.data_as(abi.f32p)) == 0
    assert O.ref().ref_dump_grid(b.encode(), 1, 8, g.ctypes.data_as(C.POINTER(C.c_float))) == 0
    assert open(a, "rb").read() == open(b, "rb").read()
    lv, cells = C.c_int32(), C.c_int32()
    back = np.empty(9 ** 3, np.float32)
    small = np.empty(10, np.float32)
    assert lib.icg_load_grid_dump(b.encode(), C.byref(lv), C.byref(cells), small.ctypes.data_as(abi.f32p), 10) == \
        abi.ICG_ECAPACITY
    assert lib.icg_load_grid_dump(b.encode(), C.byref(lv), C.byref(cells), back.ctypes.data_as(abi.f32p),
                                  back.size) == 0
    assert (lv.value, cells.value) == (1, 8) and np.array_equal(back, g)
    assert lib.icg_load_grid_dump(str(tmp_path / "missing").encode(), C.byref(lv), C.byref(cells), None, 0) == \
        abi.ICG_ERUNTIME


def test_feature_producer_restatement_statistics():
    """The oracle's restatement of the on-device feature producer: N(0,1) statistics, seed- and
    index-determined (any prefix of a longer map is the shorter map)."""
    a = O.feature_normals(1000, 4, 64, 64)
    b = O.feature_normals(1000, 8, 64, 64)
    assert np.array_equal(a.reshape(-1), b.reshape(-1)[: a.size])
    assert abs(float(b.mean())) < 0.02 and abs(float(b.std()) - 1.0) < 0.02
    assert not np.array_equal(a, O.feature_normals(1001, 4, 64, 64))

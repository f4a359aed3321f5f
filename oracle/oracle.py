"""CPU ORACLE bindings — TEST INFRASTRUCTURE ONLY.

Loads oracle/liborc.so (the C restatement, isocull_oracle.c) and
oracle/_ref/libisocull_ref.so (the unmodified reference headers behind
ref_shim.cpp).  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
use this module, and only as the checker / the CPU baseline; the product
package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libisocull_ref.so")


# Plain-data struct layouts of include/isocull_b200.h (the C oracle includes that header for its
# types; nothing of the product package is imported here).
class icg_primitive(C.Structure):
    _fields_ = [("kind", C.c_int32), ("rotated", C.c_int32), ("center", C.c_double * 3), ("a", C.c_double * 3),
                ("b", C.c_double * 3), ("radius", C.c_double), ("half", C.c_double * 3), ("major", C.c_double),
                ("minor", C.c_double), ("inv_rotation", C.c_double * 9)]


class icg_camera(C.Structure):
    _fields_ = [("rotation", C.c_double * 9), ("translation", C.c_double * 3), ("scale", C.c_double)]


def _as(cls, obj):
    """obj as an instance of the oracle's struct `cls` (the product's ctypes structs have the
    same layout: copied by value)."""
    if isinstance(obj, cls):
        return obj
    if C.sizeof(type(obj)) != C.sizeof(cls):
        raise TypeError(f"{type(obj).__name__} does not have the layout of {cls.__name__}")
    return cls.from_buffer_copy(bytes(obj))

f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class orc_mlp(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("skip_dim", C.c_int), ("out_dims", C.c_int * 5), ("in_dims", C.c_int * 5),
                ("w", f32p * 5), ("b", f32p * 5), ("slope", C.c_double)]


class orc_pifu(C.Structure):
    _fields_ = [("fmap", f32p), ("C", C.c_int), ("H", C.c_int), ("W", C.c_int),
                ("prims", C.POINTER(icg_primitive)), ("n_prims", C.c_int), ("sdf_scale", C.c_double),
                ("geo", orc_mlp), ("tex", orc_mlp), ("has_texture", C.c_int), ("has_cam", C.c_int),
                ("cam_rot", C.c_double * 9), ("cam_t", C.c_double * 3), ("cam_scale", C.c_double)]


class orc_pifu_cb(C.Structure):
    _fields_ = [("model", C.POINTER(orc_pifu)), ("threads", C.c_int)]


class orc_analytic(C.Structure):
    _fields_ = [("prims", C.POINTER(icg_primitive)), ("n_prims", C.c_int), ("tau", C.c_double),
                ("threads", C.c_int)]


class orc_replay(C.Structure):
    _fields_ = [("values", f32p), ("states", u8p), ("cells", C.c_int), ("misses", C.c_uint64),
                ("calls", C.c_uint64)]


class orc_extract_out(C.Structure):
    _fields_ = [("values", f32p), ("states", u8p), ("binarized", u8p), ("evals_per_level", C.c_uint64 * 16),
                ("total_evals", C.c_uint64), ("refined_cells_per_level", C.c_uint64 * 16),
                ("conflict_iters_per_level", C.c_uint32 * 16), ("conflict_warning", C.c_int),
                ("wall_seconds", C.c_double), ("eval_level", u8p), ("refined_cells", u8p * 16)]


class orc_render_out(C.Structure):
    _fields_ = [("depth", f32p), ("rgb", f32p), ("mask", u8p), ("surface_k", i32p), ("surface_pts", f64p),
                ("covered", C.c_uint64), ("degenerate", C.c_uint64), ("grazing", C.c_uint64)]


_ORC = None
_REF = None


def orc() -> C.CDLL:
    global _ORC
    if _ORC is None:
        if not os.path.exists(ORC_PATH):
            raise ImportError(f"oracle not built: {ORC_PATH} (run make -C oracle)")
        lib = C.CDLL(ORC_PATH)
        lib.orc_rng_uniforms.argtypes = [C.c_uint64, C.c_size_t, f64p]
        lib.orc_rng_normals.argtypes = [C.c_uint64, C.c_size_t, f64p]
        lib.orc_feature_normals.argtypes = [C.c_uint64, C.c_size_t, f32p]
        lib.orc_scene_sdf.restype = C.c_double
        lib.orc_scene_sdf.argtypes = [C.POINTER(icg_primitive), C.c_int, f64p]
        lib.orc_analytic_occupancy_batch.argtypes = [C.POINTER(icg_primitive), C.c_int, C.c_double, f64p,
                                                     C.c_size_t, f64p, C.c_int]
        for n in ("orc_pifu_occupancy_batch", "orc_pifu_logit_batch", "orc_pifu_texture_batch"):
            getattr(lib, n).argtypes = [C.POINTER(orc_pifu), f64p, C.c_size_t, f64p, C.c_int]
        lib.orc_sample_features.argtypes = [C.POINTER(orc_pifu), f64p, f64p]
        lib.orc_extract_progressive.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                                C.POINTER(orc_extract_out)]
        lib.orc_extract_brute.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(orc_extract_out)]
        lib.orc_compare_iou.restype = C.c_double
        lib.orc_compare_iou.argtypes = [u8p, u8p, C.c_size_t]
        lib.orc_upsample_interpolate.argtypes = [C.c_int, f32p, u8p, f32p, u8p]
        lib.orc_dilate_1ring.argtypes = [C.c_int, u8p, u8p]
        lib.orc_argmax_z.argtypes = [C.c_int, f32p, f32p, i32p]
        lib.orc_render_first_crossing.argtypes = [f32p, C.c_int, C.POINTER(icg_camera), C.c_int, C.c_int, f32p,
                                                  C.c_void_p, C.c_void_p, C.POINTER(orc_render_out)]
        lib.orc_camera_from_angles.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double,
                                               C.POINTER(icg_camera)]
        lib.orc_gen_capsules.argtypes = [C.c_uint64, C.c_int, C.POINTER(icg_primitive)]
        lib.orc_gen_mlp.argtypes = [C.c_uint64, C.c_int, f32p, f32p]
        lib.orc_pt_replay.restype = C.c_double
        _ORC = lib
    return _ORC


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref() -> C.CDLL:
    global _REF
    if _REF is None:
        if not ref_available():
            raise ImportError(f"reference shim not built: {REF_PATH}")
        lib = C.CDLL(REF_PATH)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_write_ppm.argtypes = [C.c_char_p, C.c_int, C.c_int, f64p]
        lib.ref_write_float_map.argtypes = [C.c_char_p, C.c_int, C.c_int, f64p]
        lib.ref_dump_grid.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_float)]
        lib.ref_extract.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, f32p, u8p, u8p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_int), C.POINTER(C.c_double)]
        lib.ref_render_view.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_int, C.c_int, f64p, C.c_int, f64p, f64p, u8p,
                                        C.POINTER(C.c_uint64), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]
        lib.ref_occupancy_batch.restype = C.c_uint64
        lib.ref_occupancy_batch.argtypes = [C.c_void_p, C.c_void_p, f64p, C.c_size_t, C.c_int, f64p]
        lib.ref_texture_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, f64p, C.c_size_t, C.c_int, f64p]
        lib.ref_camera_from_angles.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, f64p, f64p]
        lib.ref_scene_load.restype = C.c_void_p
        lib.ref_scene_load.argtypes = [C.c_char_p]
        lib.ref_scene_capsules.restype = C.c_void_p
        lib.ref_scene_capsules.argtypes = [C.POINTER(icg_primitive), C.c_int, C.c_double]
        lib.ref_scene_free.argtypes = [C.c_void_p]
        lib.ref_marching_cubes.argtypes = [f32p, C.c_int, C.c_double, f64p, C.c_int, i32p, C.c_int,
                                           C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.ref_export_obj.argtypes = [C.c_char_p, f64p, C.c_int, i32p, C.c_int]
        lib.ref_scene_make.restype = C.c_void_p
        lib.ref_scene_make.argtypes = [C.POINTER(icg_primitive), C.c_int, C.c_double, C.c_int, C.c_int, f64p, f64p,
                                       f64p, f64p]
        lib.ref_scene_texture.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), f64p, f64p, f64p,
                                          f64p, C.c_int]
        lib.ref_scene_export.argtypes = [C.c_void_p, C.POINTER(icg_primitive), C.c_int, f64p, C.POINTER(C.c_int)]
        lib.ref_scene_occ.restype = C.c_double
        lib.ref_scene_occ.argtypes = [C.c_void_p, f64p]
        lib.ref_scene_sdf.restype = C.c_double
        lib.ref_scene_sdf.argtypes = [C.c_void_p, f64p]
        lib.ref_upsample.argtypes = [C.c_int, C.c_int, f32p, u8p, f32p, u8p]
        lib.ref_binarize.argtypes = [C.c_size_t, f32p, f32p]
        lib.ref_boundary_candidates.argtypes = [C.c_int, f32p, u8p]
        lib.ref_dilate.argtypes = [C.c_int, u8p, u8p]
        lib.ref_argmax_z.argtypes = [C.c_int, f32p, f32p, i32p]
        lib.ref_compare_iou.restype = C.c_double
        lib.ref_compare_iou.argtypes = [u8p, u8p, C.c_size_t]
        lib.ref_rng_uniforms.argtypes = [C.c_uint64, C.c_size_t, f64p]
        lib.ref_rng_normals.argtypes = [C.c_uint64, C.c_size_t, f64p]
        _REF = lib
    return _REF


def fnptr(lib: C.CDLL, name: str) -> int:
    return C.cast(getattr(lib, name), C.c_void_p).value


# ---------------------------------------------------------------------------
# Fields
# ---------------------------------------------------------------------------
def prim_array(prims):
    arr = (icg_primitive * max(1, len(prims)))(*[_as(icg_primitive, p) for p in prims])
    return arr


class Analytic:
    """Analytic union-of-primitives field (field.hpp:81-91)."""

    def __init__(self, prims, tau: float, threads: int = 1):
        self.prims = prim_array(prims)
        self.c = orc_analytic(C.cast(self.prims, C.POINTER(icg_primitive)), len(prims), tau, threads)
        self.batch_fn = fnptr(orc(), "orc_cb_analytic")
        self.pt_fn = fnptr(orc(), "orc_pt_analytic")
        self.user = C.addressof(self.c)

    def occupancy(self, pts: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        out = np.empty(len(pts))
        orc().orc_analytic_occupancy_batch(self.c.prims, self.c.n_prims, self.c.tau, _p(pts, C.c_double),
                                           len(pts), _p(out, C.c_double), self.c.threads)
        return out


class Pifu:
    """CPU restatement of the PIFu field: Phi + f_O (+ f_T), fp64."""

    def __init__(self, fmap: np.ndarray, caps, geo_w, geo_b, tex_w=None, tex_b=None, sdf_scale=50.0,
                 threads: int = 1, input_camera=None):
        """input_camera: (rotation 3x3, translation 3, scale) of the PIFu input view, or None."""
        self.keep = []
        self.fmap = np.ascontiguousarray(fmap, np.float32)
        self.prims = prim_array(caps)
        m = orc_pifu()
        m.fmap = _p(self.fmap, C.c_float)
        m.C, m.H, m.W = self.fmap.shape
        m.prims = C.cast(self.prims, C.POINTER(icg_primitive))
        m.n_prims = len(caps)
        m.sdf_scale = sdf_scale
        self._fill(m.geo, geo_w, geo_b, 257)
        if tex_w is not None:
            self._fill(m.tex, tex_w, tex_b, 513)
            m.has_texture = 1
        if input_camera is not None:
            rot, t, sc = input_camera
            m.has_cam = 1
            m.cam_rot[:] = [float(x) for x in np.asarray(rot, np.float64).reshape(9)]
            m.cam_t[:] = [float(x) for x in np.asarray(t, np.float64).reshape(3)]
            m.cam_scale = float(sc)
        self.m = m
        self.cb = orc_pifu_cb(C.pointer(self.m), threads)
        self.user = C.addressof(self.cb)
        self.batch_fn = fnptr(orc(), "orc_cb_pifu_occ")
        self.tex_fn = fnptr(orc(), "orc_cb_pifu_tex")
        self.pt_fn = fnptr(orc(), "orc_pt_pifu_occ")
        self.pt_tex_fn = fnptr(orc(), "orc_pt_pifu_tex")
        self.threads = threads

    def _fill(self, net: orc_mlp, ws, bs, skip):
        net.n_layers = 5
        net.skip_dim = skip
        net.slope = 0.02
        prev = 0
        for l in range(5):
            w = np.ascontiguousarray(ws[l], np.float32)
            b = np.ascontiguousarray(bs[l], np.float32)
            self.keep += [w, b]
            net.out_dims[l] = w.shape[0]
            net.in_dims[l] = w.shape[1]
            assert w.shape[1] == prev + skip
            prev = w.shape[0]
            net.w[l] = _p(w, C.c_float)
            net.b[l] = _p(b, C.c_float)

    def _run(self, name, pts, width):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        out = np.empty(len(pts) * width)
        getattr(orc(), name)(C.byref(self.m), _p(pts, C.c_double), len(pts), _p(out, C.c_double), self.threads)
        return out if width == 1 else out.reshape(-1, width)

    def occupancy(self, pts):
        return self._run("orc_pifu_occupancy_batch", pts, 1)

    def logit(self, pts):
        return self._run("orc_pifu_logit_batch", pts, 1)

    def texture(self, pts):
        return self._run("orc_pifu_texture_batch", pts, 3)

    def features(self, p):
        out = np.empty(self.m.C)
        pp = np.ascontiguousarray(p, np.float64)
        orc().orc_sample_features(C.byref(self.m), _p(pp, C.c_double), _p(out, C.c_double))
        return out


class Replay:
    """Lookup oracle over a finest-level grid (values/states) — exact control-flow replay."""

    def __init__(self, values: np.ndarray, states: np.ndarray, cells: int):
        self.v = np.ascontiguousarray(values, np.float32)
        self.s = np.ascontiguousarray(states, np.uint8)
        self.c = orc_replay(_p(self.v, C.c_float), _p(self.s, C.c_uint8), cells, 0, 0)
        self.user = C.addressof(self.c)
        self.batch_fn = fnptr(orc(), "orc_cb_replay")
        self.pt_fn = fnptr(orc(), "orc_pt_replay")


# ---------------------------------------------------------------------------
# Operators (restatement)
# ---------------------------------------------------------------------------
def _new_out(cells):
    n = (cells + 1) ** 3
    vals = np.empty(n, np.float32)
    sts = np.empty(n, np.uint8)
    binz = np.empty(n, np.uint8)
    o = orc_extract_out()
    o.values, o.states, o.binarized = _p(vals, C.c_float), _p(sts, C.c_uint8), _p(binz, C.c_uint8)
    return o, vals, sts, binz


def _result(o, L, vals, sts, binz):
    return dict(values=vals, states=sts, binarized=binz,
                evals_per_level=[int(o.evals_per_level[l]) for l in range(L + 1)],
                total_evals=int(o.total_evals),
                refined_cells_per_level=[int(o.refined_cells_per_level[l]) for l in range(L + 1)],
                conflict_iters_per_level=[int(o.conflict_iters_per_level[l]) for l in range(L + 1)],
                conflict_warning=bool(o.conflict_warning), wall_seconds=o.wall_seconds)


def extract_progressive(fld, coarsest: int, level: int, max_conflict_iters: int = 0, conflict_pass: bool = True,
                        level_sets: bool = False):
    """level_sets: also return r["evaluated_sets"][l] (ascending node indices of the level-l grid
    evaluated at level l) and r["refined_sets"][l] (ascending cell indices of the level-(l-1) grid
    whose binarized corners disagree; empty at l = 0)."""
    o, vals, sts, binz = _new_out(coarsest << level)
    keep = []
    if level_sets:
        n = (coarsest << level) + 1
        ev = np.empty(n ** 3, np.uint8)
        o.eval_level = _p(ev, C.c_uint8)
        keep.append(ev)
        for l in range(1, level + 1):
            rc_ = coarsest << (l - 1)
            a = np.zeros(rc_ ** 3, np.uint8)
            o.refined_cells[l] = _p(a, C.c_uint8)
            keep.append(a)
    rc = orc().orc_extract_progressive(fld.batch_fn, fld.user, coarsest, level, max_conflict_iters,
                                       1 if conflict_pass else 0, C.byref(o))
    if rc:
        raise ValueError("orc_extract_progressive: invalid config")
    r = _result(o, level, vals, sts, binz)
    if level_sets:
        n = (coarsest << level) + 1
        r["evaluated_sets"] = []
        for l in range(level + 1):
            f = np.flatnonzero(ev == l)
            s = level - l
            nl = (coarsest << l) + 1
            i, j, k = (f % n) >> s, ((f // n) % n) >> s, (f // (n * n)) >> s
            r["evaluated_sets"].append((i + nl * (j + nl * k)).astype(np.uint32))
        r["refined_sets"] = [np.zeros(0, np.uint32)] + [np.flatnonzero(a).astype(np.uint32) for a in keep[1:]]
    return r


def extract_brute(fld, coarsest: int, level: int):
    o, vals, sts, binz = _new_out(coarsest << level)
    rc = orc().orc_extract_brute(fld.batch_fn, fld.user, coarsest, level, C.byref(o))
    if rc:
        raise ValueError("orc_extract_brute: invalid config")
    return _result(o, level, vals, sts, binz)


def camera_from_angles(yaw, pitch, dist=0.0, scale=1.0) -> icg_camera:
    cam = icg_camera()
    orc().orc_camera_from_angles(yaw, pitch, dist, scale, C.byref(cam))
    return cam


def render_first_crossing(values: np.ndarray, cells: int, cam: icg_camera, width: int, height: int,
                          background=(0.0, 0.0, 0.0), tex: Optional[Pifu] = None, want_points=False):
    npx = width * height
    out = orc_render_out()
    depth = np.empty(npx, np.float32)
    rgb = np.empty(npx * 3, np.float32)
    mask = np.empty(npx, np.uint8)
    sk = np.empty(npx, np.int32)
    spts = np.full(npx * 3, np.nan) if want_points else None
    out.depth, out.rgb, out.mask, out.surface_k = _p(depth, C.c_float), _p(rgb, C.c_float), _p(mask, C.c_uint8), \
        _p(sk, C.c_int32)
    if spts is not None:
        out.surface_pts = _p(spts, C.c_double)
    bg = np.asarray(background, np.float32)
    v = np.ascontiguousarray(values, np.float32)
    cam = _as(icg_camera, cam)
    rc = orc().orc_render_first_crossing(_p(v, C.c_float), cells, C.byref(cam), width, height, _p(bg, C.c_float),
                                         tex.tex_fn if tex else None, tex.user if tex else None, C.byref(out))
    if rc:
        raise ValueError("render: invalid arguments")
    res = dict(depth=depth.reshape(height, width), rgb=rgb.reshape(height, width, 3),
               mask=mask.reshape(height, width), surface_k=sk.reshape(height, width),
               covered=int(out.covered), degenerate=int(out.degenerate), grazing=int(out.grazing))
    if spts is not None:
        res["surface_pts"] = spts.reshape(height, width, 3)
    return res


def compare_iou(a, b) -> float:
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    return orc().orc_compare_iou(_p(a, C.c_uint8), _p(b, C.c_uint8), a.size)


def gen_capsules(seed: int, n: int = 15):
    arr = (icg_primitive * n)()
    orc().orc_gen_capsules(seed, n, arr)
    return list(arr)


def gen_feature_map(seed: int, c: int = 256, h: int = 128, w: int = 128) -> np.ndarray:
    """C x H x W float32 map of Rng(seed) normals in generation order (the product's
    icg_gen_normals draws the same sequence)."""
    out = np.empty(c * h * w)
    orc().orc_rng_normals(seed, out.size, _p(out, C.c_double))
    return out.astype(np.float32).reshape(c, h, w)


def feature_normals(seed: int, c: int, h: int, w: int) -> np.ndarray:
    """Restatement of the product's on-device feature producer (icg_gen_feature_map_device)."""
    out = np.empty(c * h * w, np.float32)
    orc().orc_feature_normals(C.c_uint64(seed), C.c_size_t(out.size), _p(out, C.c_float))
    return out.reshape(c, h, w)


def gen_mlp(seed: int, which: int):
    outs = (1024, 512, 256, 128, 1) if which == 0 else (1024, 512, 256, 128, 3)
    skip = 257 if which == 0 else 513
    ins = [(outs[l - 1] if l else 0) + skip for l in range(5)]
    nw = sum(o * i for o, i in zip(outs, ins))
    w = np.empty(nw, np.float32)
    b = np.empty(sum(outs), np.float32)
    orc().orc_gen_mlp(seed, which, _p(w, C.c_float), _p(b, C.c_float))
    ws, bs, wo, bo = [], [], 0, 0
    for o, i in zip(outs, ins):
        ws.append(w[wo:wo + o * i].reshape(o, i))
        bs.append(b[bo:bo + o])
        wo += o * i
        bo += o
    return ws, bs


# ---------------------------------------------------------------------------
# Reference (oracle/_ref) operators
# ---------------------------------------------------------------------------
def ref_extract(pt_fn: int, user: int, coarsest: int, level: int, variant: int = 3, threshold: float = 0.0,
                max_conflict_iters: int = 0, conflict_pass: bool = True, workers: int = 1):
    cells = coarsest << level
    n = (cells + 1) ** 3
    vals = np.empty(n, np.float32)
    sts = np.empty(n, np.uint8)
    binz = np.empty(n, np.uint8)
    evals = (C.c_uint64 * 16)()
    total, calls = C.c_uint64(), C.c_uint64()
    warn, wall = C.c_int(), C.c_double()
    rc = ref().ref_extract(pt_fn, user, variant, threshold, coarsest, level, max_conflict_iters,
                           1 if conflict_pass else 0, workers, _p(vals, C.c_float), _p(sts, C.c_uint8),
                           _p(binz, C.c_uint8), evals, C.byref(total), C.byref(calls), C.byref(warn), C.byref(wall))
    if rc == 2:
        raise ValueError(ref().ref_last_error().decode())
    if rc:
        raise RuntimeError(ref().ref_last_error().decode())
    return dict(values=vals, states=sts, binarized=binz, evals_per_level=[int(evals[l]) for l in range(level + 1)],
                total_evals=int(total.value), oracle_calls=int(calls.value), conflict_warning=bool(warn.value),
                wall_seconds=wall.value)


def ref_occupancy_batch(pt_fn: int, user: int, pts: np.ndarray, workers: int = 1) -> np.ndarray:
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    out = np.empty(len(pts))
    ref().ref_occupancy_batch(pt_fn, user, _p(pts, C.c_double), len(pts), workers, _p(out, C.c_double))
    return out


def ref_texture_batch(pt_fn: int, tex_fn: int, user: int, pts: np.ndarray, workers: int = 1) -> np.ndarray:
    pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    out = np.empty((len(pts), 3))
    ref().ref_texture_batch(pt_fn, tex_fn, user, _p(pts, C.c_double), len(pts), workers, _p(out, C.c_double))
    return out


class RefScene:
    """A reference SceneSpec: loaded from a scene JSON by the reference's parser, built from capsules,
    or built from (prims, tau, texture dict) data (ref_scene_make, validated by validate_scene)."""

    def __init__(self, path: Optional[str] = None, capsules=None, tau: float = 0.02, prims=None, texture=None):
        if path is not None:
            self.h = ref().ref_scene_load(path.encode())
            if not self.h:
                raise ValueError(ref().ref_last_error().decode())
        elif prims is not None:
            arr = prim_array(prims)
            t = texture or {"kind": 0}
            vec = lambda k: np.ascontiguousarray(t.get(k, [0.0, 0.0, 0.0]), np.float64)
            col, fr, to = vec("color"), vec("from"), vec("to")
            cols = np.ascontiguousarray(t.get("colors", [[0.0] * 3] * max(1, len(prims))), np.float64)
            self.h = ref().ref_scene_make(C.cast(arr, C.POINTER(icg_primitive)), len(prims), tau, int(t["kind"]),
                                          int(t.get("axis", 2)), _p(col, C.c_double), _p(fr, C.c_double),
                                          _p(to, C.c_double), _p(cols, C.c_double))
            if not self.h:
                raise ValueError(ref().ref_last_error().decode())
        else:
            arr = prim_array(capsules)
            self.h = ref().ref_scene_capsules(C.cast(arr, C.POINTER(icg_primitive)), len(capsules), tau)
        self.pt_fn = fnptr(ref(), "ref_scene_occ")
        self.tex_fn = fnptr(ref(), "ref_scene_tex")
        self.user = self.h

    def export(self):
        arr = (icg_primitive * 64)()
        tau = C.c_double()
        has_tex = C.c_int()
        n = ref().ref_scene_export(self.h, arr, 64, C.byref(tau), C.byref(has_tex))
        if n < 0:
            raise ValueError("scene is not a plain union")
        return list(arr[:n]), tau.value, bool(has_tex.value)

    def texture(self) -> dict:
        """The scene's TextureRule as the reference parsed it: kind (ICG_TEXTURE_*), axis, color,
        from, to, colors (per primitive)."""
        kind, axis = C.c_int(), C.c_int()
        col, fr, to = np.zeros(3), np.zeros(3), np.zeros(3)
        cols = np.zeros(64 * 3)
        n = ref().ref_scene_texture(self.h, C.byref(kind), C.byref(axis), _p(col, C.c_double), _p(fr, C.c_double),
                                    _p(to, C.c_double), _p(cols, C.c_double), 64)
        return {"kind": kind.value, "axis": axis.value, "color": col.tolist(), "from": fr.tolist(), "to": to.tolist(),
                "colors": cols[:3 * n].reshape(n, 3).tolist()}

    def sdf(self, p):
        pp = np.ascontiguousarray(p, np.float64)
        return ref().ref_scene_sdf(self.h, _p(pp, C.c_double))

    def __del__(self):
        try:
            ref().ref_scene_free(self.h)
        except Exception:
            pass


def ref_marching_cubes(values: np.ndarray, cells: int, iso: float = 0.5):
    """The reference's marching_cubes (mesh.hpp:75-156): (vertices (n,3), triangles (m,3))."""
    v = np.ascontiguousarray(values, np.float32).reshape(-1)
    nv, nt = C.c_int(), C.c_int()
    rc = ref().ref_marching_cubes(_p(v, C.c_float), cells, iso, None, 0, None, 0, C.byref(nv), C.byref(nt))
    if rc:
        raise ValueError(ref().ref_last_error().decode())
    V = np.empty((nv.value, 3))
    T = np.empty((nt.value, 3), np.int32)
    ref().ref_marching_cubes(_p(v, C.c_float), cells, iso, _p(V, C.c_double), nv.value, _p(T, C.c_int32), nt.value,
                             C.byref(nv), C.byref(nt))
    return V, T


def ref_render_view(scene: RefScene, yaw, pitch, coarsest, level, bg=(0.0, 0.0, 0.0), workers=1, dist=0.0,
                    scale=1.0):
    n = (coarsest << level) + 1
    depth = np.empty(n * n)
    rgb = np.empty(n * n * 3)
    mask = np.empty(n * n, np.uint8)
    calls = C.c_uint64()
    deg, graz, size = C.c_int(), C.c_int(), C.c_int()
    b = np.asarray(bg, np.float64)
    # a RefScene (per-point occ / tex of the reference SceneSpec) or a Pifu model (per-point callbacks)
    tex_fn = scene.pt_tex_fn if hasattr(scene, "pt_tex_fn") else scene.tex_fn
    rc = ref().ref_render_view(scene.pt_fn, tex_fn, scene.user, yaw, pitch, dist, scale, coarsest, level,
                               _p(b, C.c_double), workers, _p(depth, C.c_double), _p(rgb, C.c_double),
                               _p(mask, C.c_uint8), C.byref(calls), C.byref(deg), C.byref(graz), C.byref(size))
    if rc:
        raise ValueError(ref().ref_last_error().decode())
    return dict(depth=depth.reshape(n, n), rgb=rgb.reshape(n, n, 3), mask=mask.reshape(n, n),
                oracle_calls=int(calls.value), degenerate=deg.value, grazing=graz.value)

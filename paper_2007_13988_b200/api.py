"""Reference-shaped host API over the C ABI (the Python face of the drop-in).

Mirrors the reference's operator surface (/root/reference/proj/include/isocull):

  reference                                   here
  ------------------------------------------  ------------------------------------------
  FieldOracle (field.hpp:22-77)               AnalyticField / PifuField (device data)
  AlgoConfig, validate_config (localize:36)   AlgoConfig (same fields, same errors)
  ExtractionResult (localize.hpp:57-64)       ExtractionResult
  extract / extract_progressive /             extract / extract_progressive /
    extract_brute_force (localize:181-373)      extract_brute_force
  compare_iou, acceleration_factor            compare_iou, acceleration_factor
  CameraSpec::from_angles (render.hpp:36)     CameraSpec.from_angles
  render_view -> RenderedImage (render:244)   render_view -> RenderedImage (the reference's
                                                view-aligned renderer, icg_render_view)
  surface_depth_map -> DepthMap (render:219)  surface_depth_map
  composite (render.hpp:284)                  composite
  (north-star renderer)     render_frame / Context.frame: localize + first-crossing
                                                render through the localized world grid

Errors follow the reference: std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError.  All work runs in the sm_100a library.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import abi

GEO_OUT = (1024, 512, 256, 128, 1)
TEX_OUT = (1024, 512, 256, 128, 3)
GEO_SKIP, TEX_SKIP = 257, 513


def _check(rc: int) -> None:
    if rc == abi.ICG_OK:
        return
    msg = abi.lib().icg_last_error().decode(errors="replace")
    if rc == abi.ICG_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"isocull_b200 error {rc}: {msg}")


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ---------------------------------------------------------------------------
# Fields (FieldOracle surrogates)
# ---------------------------------------------------------------------------
def capsule_prims(caps: np.ndarray) -> list:
    """caps: (n, 7) array of a.xyz, b.xyz, r."""
    out = []
    for row in np.asarray(caps, dtype=np.float64):
        p = abi.icg_primitive()
        p.kind = abi.ICG_PRIM_CAPSULE
        p.a[:] = row[0:3]
        p.b[:] = row[3:6]
        p.radius = row[6]
        p.inv_rotation[0] = p.inv_rotation[4] = p.inv_rotation[8] = 1.0
        out.append(p)
    return out


class _Field:
    def __init__(self):
        self._prims = None
        self._fmap = None
        self.c = abi.icg_field()

    def _set_prims(self, prims: Sequence[abi.icg_primitive], tau: float):
        arr = (abi.icg_primitive * max(1, len(prims)))(*prims)
        self._prims = arr
        self.c.scene.prims = C.cast(arr, C.POINTER(abi.icg_primitive))
        self.c.scene.n_prims = len(prims)
        self.c.scene.tau = tau


class AnalyticField(_Field):
    """O(P) = 1/(1+exp(sdf(P)/tau)) over a union of primitives (build_oracle, field.hpp:83-91), with
    an optional TextureRule (scene.hpp:48-55): dict kind (ICG_TEXTURE_*), axis, color, from, to,
    colors (per primitive) -- the layout of tests/golden/scenes.json."""

    def __init__(self, prims: Sequence[abi.icg_primitive], tau: float, texture: Optional[dict] = None):
        super().__init__()
        self.c.kind = abi.ICG_FIELD_ANALYTIC
        self._set_prims(prims, tau)
        if texture and texture.get("kind", 0):
            t = self.c.scene.texture
            t.kind = int(texture["kind"])
            t.axis = int(texture.get("axis", 2))
            t.color[:] = [float(x) for x in texture.get("color", [1.0, 1.0, 1.0])]
            t.from_[:] = [float(x) for x in texture.get("from", [0.0, 0.0, 0.0])]
            t.to[:] = [float(x) for x in texture.get("to", [1.0, 1.0, 1.0])]
            cols = np.ascontiguousarray(texture.get("colors") or [[0.0, 0.0, 0.0]], dtype=np.float64).reshape(-1)
            self._colors = cols
            t.colors = _ptr(cols, C.c_double)


class PifuField(_Field):
    """O(P) = sigmoid(f_O(Phi(P_xy), P_z) - sdf_scale * sdf(P)) (BASELINE configs 1-4)."""

    def __init__(self, feature_map, capsules: Sequence[abi.icg_primitive], sdf_scale: float = 50.0,
                 precision: int = abi.ICG_PREC_FP32, device_ptr: Optional[int] = None,
                 shape: Optional[tuple] = None, input_camera: Optional["CameraSpec"] = None):
        """input_camera: the view the feature map was encoded from (Phi at its world_to_view x, y; depth
        feature its z); None = orthographic identity."""
        super().__init__()
        if input_camera is not None:
            self.c.has_input_camera = 1
            self.c.input_camera = input_camera.to_c()
        self.c.kind = abi.ICG_FIELD_PIFU
        self._set_prims(capsules, 0.02)
        self.c.sdf_scale = sdf_scale
        self.c.precision = precision
        if device_ptr is not None:
            ch, hh, ww = shape
            self.c.feature_map = C.cast(C.c_void_p(device_ptr), abi.f32p)
            self.c.fmap_mem = abi.ICG_MEM_DEVICE
        else:
            fm = np.ascontiguousarray(feature_map, dtype=np.float32)
            self._fmap = fm
            ch, hh, ww = fm.shape
            self.c.feature_map = _ptr(fm, C.c_float)
            self.c.fmap_mem = abi.ICG_MEM_HOST
        self.c.fmap_c, self.c.fmap_h, self.c.fmap_w = ch, hh, ww


# ---------------------------------------------------------------------------
# Config / results
# ---------------------------------------------------------------------------
VARIANTS = {"brute": abi.ICG_VARIANT_BRUTE, "octree_binarized": abi.ICG_VARIANT_OCTREE_BINARIZED,
            "octree_threshold": abi.ICG_VARIANT_OCTREE_THRESHOLD, "progressive": abi.ICG_VARIANT_PROGRESSIVE}


@dataclass
class AlgoConfig:
    variant: str = "progressive"
    coarsest_cells: int = 16
    target_level: int = 3
    max_conflict_iters: int = 0
    conflict_pass: bool = True
    keep_level_sets: bool = False  # keep per-level refined-cell / evaluated-node sets (Context.level_set)
    threshold: float = 0.0  # octree_threshold only, in (0, 0.5)

    def target_cells(self) -> int:
        return self.coarsest_cells << self.target_level

    def to_c(self) -> abi.icg_algo_config:
        v = VARIANTS.get(self.variant)
        if v is None:  # variant_from_name, localize.hpp:29-34
            raise ValueError(f"unknown variant '{self.variant}'")
        return abi.icg_algo_config(v, self.coarsest_cells, self.target_level, self.max_conflict_iters,
                                   1 if self.conflict_pass else 0, 1 if self.keep_level_sets else 0,
                                   float(self.threshold))


@dataclass
class ExtractionResult:
    cells: int
    values: Optional[np.ndarray]
    states: Optional[np.ndarray]
    binarized: Optional[np.ndarray]
    evals_per_level: list
    total_evals: int
    refined_cells_per_level: list
    conflict_iters_per_level: list
    conflict_warning: bool
    wall_seconds: float


@dataclass
class CameraSpec:
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    scale: float = 1.0

    @staticmethod
    def from_angles(yaw_deg: float, pitch_deg: float, dist: float = 0.0, scale: float = 1.0) -> "CameraSpec":
        cam = abi.icg_camera()
        _check(abi.lib().icg_camera_from_angles(yaw_deg, pitch_deg, dist, scale, C.byref(cam)))
        return CameraSpec(np.array(cam.rotation[:]).reshape(3, 3), np.array(cam.translation[:]), cam.scale)

    def to_c(self) -> abi.icg_camera:
        c = abi.icg_camera()
        c.rotation[:] = [float(x) for x in np.asarray(self.rotation, dtype=np.float64).reshape(9)]
        c.translation[:] = [float(x) for x in np.asarray(self.translation, dtype=np.float64).reshape(3)]
        c.scale = float(self.scale)
        return c


@dataclass
class RenderedImage:
    width: int
    height: int
    rgb: np.ndarray          # (H, W, 3) float32
    depth: np.ndarray        # (H, W) float32, -2 where uncovered
    mask: np.ndarray         # (H, W) uint8
    surface_k: np.ndarray    # (H, W) int32, -1 where uncovered
    covered_pixels: int
    degenerate_brackets: int
    grazing_pixels: int
    texture_points: int
    wall_seconds: float
    oracle_calls: int = 0  # render_view / surface_depth_map: occupancy evaluations of the depth pass


# ---------------------------------------------------------------------------
# Context and operators
# ---------------------------------------------------------------------------
class Context:
    """One per GPU (icg_create / icg_destroy)."""

    def __init__(self, device: int = 0):
        self._lib = abi.lib()
        h = C.c_void_p()
        _check(self._lib.icg_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self._lib.icg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # weights -----------------------------------------------------------------
    def set_mlp(self, which: int, weights: Sequence[np.ndarray], biases: Sequence[np.ndarray], slope: float = 0.02):
        outs = GEO_OUT if which == abi.ICG_MLP_GEOMETRY else TEX_OUT
        skip = GEO_SKIP if which == abi.ICG_MLP_GEOMETRY else TEX_SKIP
        d = abi.icg_mlp_desc()
        d.which, d.n_layers, d.skip_dim = which, 5, skip
        keep = []
        for l in range(5):
            w = np.ascontiguousarray(weights[l], dtype=np.float32)
            b = np.ascontiguousarray(biases[l], dtype=np.float32)
            keep += [w, b]
            d.out_dims[l] = outs[l]
            d.weights[l] = _ptr(w, C.c_float)
            d.biases[l] = _ptr(b, C.c_float)
        d.leaky_slope = slope
        _check(self._lib.icg_set_mlp(self.h, C.byref(d)))

    # operators -----------------------------------------------------------------
    def extract(self, fld: _Field, cfg: AlgoConfig, want_grid: bool = True) -> ExtractionResult:
        n = cfg.target_cells() + 1
        out = abi.icg_extraction()
        out.mem = abi.ICG_MEM_HOST
        vals = sts = binz = None
        if want_grid and cfg.target_cells() <= 1024:
            vals = np.empty(n ** 3, np.float32)
            sts = np.empty(n ** 3, np.uint8)
            binz = np.empty(n ** 3, np.uint8)
            out.values, out.states, out.binarized = _ptr(vals, C.c_float), _ptr(sts, C.c_uint8), _ptr(binz, C.c_uint8)
        cc = cfg.to_c()
        _check(self._lib.icg_extract(self.h, C.byref(fld.c), C.byref(cc), C.byref(out)))
        return _extraction(out, cfg, vals, sts, binz)

    def render_localized(self, fld: _Field, camera: CameraSpec, width: int, height: int,
                         background=(0.0, 0.0, 0.0)) -> RenderedImage:
        img, bufs = _image_bufs(width, height)
        bg = np.asarray(background, dtype=np.float32)
        cam = camera.to_c()
        _check(self._lib.icg_render_localized(self.h, C.byref(fld.c), C.byref(cam), width, height,
                                              _ptr(bg, C.c_float), C.byref(img)))
        return _image(img, width, height, bufs)

    def frame(self, fld: _Field, cfg: AlgoConfig, camera: CameraSpec, width: int, height: int,
              background=(0.0, 0.0, 0.0), want_grid: bool = False):
        n = cfg.target_cells() + 1
        ext = abi.icg_extraction()
        ext.mem = abi.ICG_MEM_HOST
        vals = sts = binz = None
        if want_grid:
            vals = np.empty(n ** 3, np.float32)
            sts = np.empty(n ** 3, np.uint8)
            binz = np.empty(n ** 3, np.uint8)
            ext.values, ext.states, ext.binarized = _ptr(vals, C.c_float), _ptr(sts, C.c_uint8), _ptr(binz, C.c_uint8)
        img, bufs = _image_bufs(width, height)
        bg = np.asarray(background, dtype=np.float32)
        cam = camera.to_c()
        cc = cfg.to_c()
        _check(self._lib.icg_frame(self.h, C.byref(fld.c), C.byref(cc), C.byref(cam), width, height,
                                   _ptr(bg, C.c_float), C.byref(ext), C.byref(img)))
        return _extraction(ext, cfg, vals, sts, binz), _image(img, width, height, bufs)

    def level_set(self, level: int, which: str) -> np.ndarray:
        """Ascending u32 list of a per-level set of the last extraction that ran with
        keep_level_sets: which = "evaluated" (node indices of the level-l grid evaluated at level l)
        or "refined" (cell indices of the level-(l-1) grid whose 8 binarized corners disagree)."""
        w = {"evaluated": abi.ICG_SET_EVALUATED_NODES, "refined": abi.ICG_SET_REFINED_CELLS}.get(which)
        if w is None:
            raise ValueError(f"unknown level set '{which}'")
        n = C.c_size_t()
        _check(self._lib.icg_level_set(self.h, level, w, abi.ICG_MEM_HOST, None, 0, C.byref(n)))
        out = np.empty(n.value, np.uint32)
        if n.value:
            _check(self._lib.icg_level_set(self.h, level, w, abi.ICG_MEM_HOST, _ptr(out, C.c_uint32), n.value,
                                           C.byref(n)))
        return out

    def render_view(self, fld: _Field, camera: CameraSpec, cfg: AlgoConfig, background=(0.0, 0.0, 0.0),
                    depth_only: bool = False) -> RenderedImage:
        """render_view (render.hpp:244-280) / surface_depth_map (depth_only, :219-240): the reference's
        view-aligned renderer, (R_L+1)^2 pixels."""
        n = cfg.target_cells() + 1
        img, bufs = _image_bufs(n, n)
        cam = camera.to_c()
        cc = cfg.to_c()
        if depth_only:
            _check(self._lib.icg_surface_depth_map(self.h, C.byref(fld.c), C.byref(cam), C.byref(cc), C.byref(img)))
        else:
            bg = np.asarray(background, dtype=np.float32)
            _check(self._lib.icg_render_view(self.h, C.byref(fld.c), C.byref(cam), C.byref(cc), _ptr(bg, C.c_float),
                                             C.byref(img)))
        out = _image(img, n, n, bufs)
        out.oracle_calls = int(img.oracle_calls)
        return out

    def gen_feature_map(self, seed: int, c: int = 256, h: int = 128, w: int = 128, device_out: Optional[int] = None):
        """On-device feature producer (icg_gen_feature_map_device): a seeded C x H x W N(0,1) map
        generated on this GPU, into the device buffer `device_out` (returns it) or to the host."""
        if device_out is not None:
            _check(self._lib.icg_gen_feature_map_device(self.h, seed, c, h, w, abi.ICG_MEM_DEVICE,
                                                        C.cast(C.c_void_p(device_out), abi.f32p)))
            return device_out
        out = np.empty((c, h, w), np.float32)
        _check(self._lib.icg_gen_feature_map_device(self.h, seed, c, h, w, abi.ICG_MEM_HOST, _ptr(out, C.c_float)))
        return out

    def marching_cubes(self, values: Optional[np.ndarray] = None, iso: float = 0.5):
        """marching_cubes(grid, iso) (mesh.hpp:75-156) on the GPU: (vertices (n, 3) float64,
        triangles (m, 3) int32).  values: a (R+1)^3 grid (host), or None for the grid the last
        extraction on this context localized."""
        cells = 0
        vp = None
        if values is not None:
            vals = np.ascontiguousarray(values, dtype=np.float32).reshape(-1)
            cells = int(round(vals.size ** (1.0 / 3.0))) - 1
            if (cells + 1) ** 3 != vals.size:
                raise ValueError("marching_cubes: values must hold (R+1)^3 nodes")
            vp = _ptr(vals, C.c_float)
        m = abi.icg_mesh()
        rc = self._lib.icg_marching_cubes(self.h, vp, cells, abi.ICG_MEM_HOST, iso, C.byref(m))
        if rc != abi.ICG_ECAPACITY:
            _check(rc)
        V = np.empty((m.n_vertices, 3), np.float64)
        T = np.empty((m.n_triangles, 3), np.int32)
        m.vertices, m.vertex_capacity = _ptr(V, C.c_double), m.n_vertices
        m.triangles, m.triangle_capacity = _ptr(T, C.c_int32), m.n_triangles
        _check(self._lib.icg_marching_cubes(self.h, vp, cells, abi.ICG_MEM_HOST, iso, C.byref(m)))
        return V, T

    def occupancy_batch(self, fld: _Field, points: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        out = np.empty(len(pts), np.float32)
        _check(self._lib.icg_occupancy_batch(self.h, C.byref(fld.c), _ptr(pts, C.c_double), len(pts),
                                             abi.ICG_MEM_HOST, _ptr(out, C.c_float)))
        return out

    def texture_batch(self, fld: _Field, points: np.ndarray) -> np.ndarray:
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        out = np.empty((len(pts), 3), np.float32)
        _check(self._lib.icg_texture_batch(self.h, C.byref(fld.c), _ptr(pts, C.c_double), len(pts),
                                           abi.ICG_MEM_HOST, _ptr(out, C.c_float)))
        return out

    def compare_iou(self, a: np.ndarray, b: np.ndarray) -> float:
        return compare_iou(a, b, self)

    # instrumentation ------------------------------------------------------------
    def profile(self, on: bool = True, reset: bool = True):
        _check(self._lib.icg_profile_enable(self.h, 1 if on else 0))
        if reset:
            _check(self._lib.icg_profile_reset(self.h))

    def profile_get(self) -> dict:
        p = abi.icg_profile()
        _check(self._lib.icg_profile_get(self.h, C.byref(p)))
        return {name: getattr(p, name) for name, _ in abi.icg_profile._fields_}

    # raw buffers (pinned host / device) for end-to-end and device-resident runs
    def device_alloc(self, nbytes: int) -> int:
        ptr = C.c_void_p()
        _check(self._lib.icg_device_alloc(self.h, nbytes, C.byref(ptr)))
        return ptr.value

    def device_free(self, ptr: int):
        _check(self._lib.icg_device_free(self.h, C.c_void_p(ptr)))

    def memcpy(self, dst: int, src: int, nbytes: int, dst_mem: int, src_mem: int):
        _check(self._lib.icg_memcpy(self.h, C.c_void_p(dst), C.c_void_p(src), nbytes, dst_mem, src_mem))

    def memset(self, dst: int, value: int, nbytes: int):
        """Device bytes set on the context's stream (returns when done)."""
        _check(self._lib.icg_memset(self.h, C.c_void_p(dst), value, nbytes))

    def frame_raw(self, fld: "_Field", cfg: AlgoConfig, camera: CameraSpec, width: int, height: int,
                  img: "abi.icg_image", ext: Optional["abi.icg_extraction"] = None, background=(0.0, 0.0, 0.0)):
        """icg_frame with caller-owned output structs (host or device buffers)."""
        bg = np.asarray(background, dtype=np.float32)
        cam = camera.to_c()
        cc = cfg.to_c()
        if ext is None:
            ext = abi.icg_extraction()
            ext.mem = abi.ICG_MEM_HOST
        _check(self._lib.icg_frame(self.h, C.byref(fld.c), C.byref(cc), C.byref(cam), width, height,
                                   _ptr(bg, C.c_float), C.byref(ext), C.byref(img)))
        return ext, img


def span_begin(ctxs) -> None:
    """Start a device-timed span over contexts of one device (see icg_span_begin)."""
    arr = (abi.ctx_p * len(ctxs))(*[c.h for c in ctxs])
    _check(abi.lib().icg_span_begin(arr, len(ctxs)))


def span_end(ctxs) -> float:
    """Milliseconds from span_begin to the last context's completion (icg_span_end)."""
    arr = (abi.ctx_p * len(ctxs))(*[c.h for c in ctxs])
    ms = C.c_float()
    _check(abi.lib().icg_span_end(arr, len(ctxs), C.byref(ms)))
    return ms.value


def host_alloc(nbytes: int) -> int:
    ptr = C.c_void_p()
    _check(abi.lib().icg_host_alloc(nbytes, C.byref(ptr)))
    return ptr.value


def host_free(ptr: int):
    _check(abi.lib().icg_host_free(C.c_void_p(ptr)))


def _extraction(out, cfg, vals, sts, binz) -> ExtractionResult:
    L = cfg.target_level
    return ExtractionResult(
        cells=out.cells, values=vals, states=sts, binarized=binz,
        evals_per_level=[int(out.evals_per_level[l]) for l in range(L + 1)],
        total_evals=int(out.total_evals),
        refined_cells_per_level=[int(out.refined_cells_per_level[l]) for l in range(L + 1)],
        conflict_iters_per_level=[int(out.conflict_iters_per_level[l]) for l in range(L + 1)],
        conflict_warning=bool(out.conflict_warning), wall_seconds=out.wall_seconds)


def _image_bufs(w, h):
    img = abi.icg_image()
    img.mem = abi.ICG_MEM_HOST
    bufs = dict(depth=np.empty(w * h, np.float32), rgb=np.empty(w * h * 3, np.float32),
                mask=np.empty(w * h, np.uint8), surface_k=np.empty(w * h, np.int32))
    img.depth = _ptr(bufs["depth"], C.c_float)
    img.rgb = _ptr(bufs["rgb"], C.c_float)
    img.mask = _ptr(bufs["mask"], C.c_uint8)
    img.surface_k = _ptr(bufs["surface_k"], C.c_int32)
    return img, bufs


def _image(img, w, h, bufs) -> RenderedImage:
    return RenderedImage(w, h, bufs["rgb"].reshape(h, w, 3), bufs["depth"].reshape(h, w),
                         bufs["mask"].reshape(h, w), bufs["surface_k"].reshape(h, w), int(img.covered_pixels),
                         int(img.degenerate_brackets), int(img.grazing_pixels), int(img.texture_points),
                         img.wall_seconds)


def extract(ctx: Context, fld: _Field, cfg: AlgoConfig) -> ExtractionResult:
    """extract(oracle, cfg, workers), localize.hpp:365-373."""
    return ctx.extract(fld, cfg)


def extract_progressive(ctx: Context, fld: _Field, cfg: AlgoConfig) -> ExtractionResult:
    cfg = AlgoConfig("progressive", cfg.coarsest_cells, cfg.target_level, cfg.max_conflict_iters, cfg.conflict_pass,
                     cfg.keep_level_sets)
    return ctx.extract(fld, cfg)


def extract_brute_force(ctx: Context, fld: _Field, cfg: AlgoConfig) -> ExtractionResult:
    cfg = AlgoConfig("brute", cfg.coarsest_cells, cfg.target_level)
    return ctx.extract(fld, cfg)


def extract_octree_binarized(ctx: Context, fld: _Field, cfg: AlgoConfig) -> ExtractionResult:
    """extract_octree_binarized, localize.hpp:199-260 (Fig. 4 baseline)."""
    cfg = AlgoConfig("octree_binarized", cfg.coarsest_cells, cfg.target_level, keep_level_sets=cfg.keep_level_sets)
    return ctx.extract(fld, cfg)


def extract_octree_threshold(ctx: Context, fld: _Field, cfg: AlgoConfig) -> ExtractionResult:
    """extract_octree_threshold, localize.hpp:265-306 (Fig. 4 baseline); cfg.threshold in (0, 0.5)."""
    cfg = AlgoConfig("octree_threshold", cfg.coarsest_cells, cfg.target_level, keep_level_sets=cfg.keep_level_sets,
                     threshold=cfg.threshold)
    return ctx.extract(fld, cfg)


def render_view(ctx: Context, fld: _Field, camera: CameraSpec, cfg: AlgoConfig,
                background=(0.0, 0.0, 0.0)) -> RenderedImage:
    """render_view(oracle, camera, cfg, background, workers), render.hpp:244-280 (icg_render_view)."""
    return ctx.render_view(fld, camera, cfg, background)


def surface_depth_map(ctx: Context, fld: _Field, camera: CameraSpec, cfg: AlgoConfig) -> RenderedImage:
    """surface_depth_map(oracle, camera, cfg, workers), render.hpp:219-240 (depth + mask)."""
    return ctx.render_view(fld, camera, cfg, depth_only=True)


def render_frame(ctx: Context, fld: _Field, camera: CameraSpec, cfg: AlgoConfig, width: int, height: int,
                 background=(0.0, 0.0, 0.0)) -> RenderedImage:
    """North-star renderer: localize (progressive) then first-crossing render through the localized
    grid (one icg_frame call)."""
    return ctx.frame(fld, cfg, camera, width, height, background)[1]


def compare_iou(a: np.ndarray, b: np.ndarray, ctx: Optional[Context] = None) -> float:
    """compare_iou, localize.hpp:377-387 (dimension mismatch -> ValueError)."""
    a = np.ascontiguousarray(a, dtype=np.uint8).reshape(-1)
    b = np.ascontiguousarray(b, dtype=np.uint8).reshape(-1)
    if a.size != b.size:
        raise ValueError("compare_iou: dimension mismatch")
    out = C.c_double()
    _check(abi.lib().icg_compare_iou(ctx.h if ctx else None, _ptr(a, C.c_uint8), _ptr(b, C.c_uint8), a.size,
                                     abi.ICG_MEM_HOST, C.byref(out)))
    return out.value


def composite(image: RenderedImage, backdrop) -> np.ndarray:
    """composite(image, backdrop), render.hpp:284-291: covered pixels from the image, the rest from
    the backdrop ((H, W, 3) or (n, 3) floats; size mismatch -> ValueError)."""
    rgb = np.ascontiguousarray(image.rgb, dtype=np.float32).reshape(-1)
    mask = np.ascontiguousarray(image.mask, dtype=np.uint8).reshape(-1)
    bd = np.ascontiguousarray(backdrop, dtype=np.float32)
    shape = bd.shape
    bd = bd.reshape(-1)
    out = np.empty_like(bd)
    _check(abi.lib().icg_composite(_ptr(rgb, C.c_float), _ptr(mask, C.c_uint8), mask.size, _ptr(bd, C.c_float),
                                   bd.size // 3, _ptr(out, C.c_float)))
    return out.reshape(shape)


def acceleration_factor(result: ExtractionResult, brute: ExtractionResult) -> float:
    """acceleration_factor, localize.hpp:389-393."""
    if result.total_evals == 0 or brute.total_evals == 0:
        raise ValueError("acceleration_factor: zero evaluation count")
    return brute.total_evals / result.total_evals


# ---------------------------------------------------------------------------
# Output formats (image.hpp:18-48, grid.hpp:199-222), byte-identical
# ---------------------------------------------------------------------------
def write_ppm(path: str, width: int, height: int, rgb) -> None:
    """Binary P6, 8-bit; byte = lround(255 * clamp(v, 0, 1)) (image.hpp:18-33)."""
    a = np.asarray(rgb, dtype=np.float64).reshape(-1)
    if a.size != 3 * width * height:
        raise ValueError("write_ppm: buffer size mismatch")
    x = 255.0 * np.clip(a, 0.0, 1.0)
    b = np.floor(x + 0.5).astype(np.uint8)  # lround for non-negative values (half away from zero)
    with open(path, "wb") as f:
        f.write(f"P6\n{width} {height}\n255\n".encode())
        f.write(b.tobytes())


def write_float_map(path: str, width: int, height: int, values) -> None:
    """int32 width, height, then float32 values, little-endian (image.hpp:37-48)."""
    a = np.asarray(values, dtype=np.float64).reshape(-1)
    if a.size != width * height:
        raise ValueError("write_float_map: buffer size mismatch")
    with open(path, "wb") as f:
        f.write(np.array([width, height], dtype="<i4").tobytes())
        f.write(a.astype("<f4").tobytes())


def write_obj(path: str, vertices, triangles) -> None:
    """export_obj (mesh.hpp:159-172) through the C ABI (icg_write_obj)."""
    V = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
    T = np.ascontiguousarray(triangles, dtype=np.int32).reshape(-1, 3)
    _check(abi.lib().icg_write_obj(path.encode(), _ptr(V, C.c_double), len(V), _ptr(T, C.c_int32), len(T)))


def mc_case(case_bits: int):
    """The generated triangulation of one cube case: a list of (e0, e1, e2) edge triples."""
    e = (C.c_int8 * 16)()
    n = C.c_int()
    _check(abi.lib().icg_mc_case(case_bits, e, C.byref(n)))
    return [tuple(e[3 * t:3 * t + 3]) for t in range(n.value)]


def dump_grid(path: str, level: int, cells: int, values) -> None:
    """int32 level, int32 R, then float32 node values x-fastest (grid.hpp:199-209)."""
    a = np.asarray(values, dtype=np.float32).reshape(-1)
    if a.size != (cells + 1) ** 3:
        raise ValueError("dump_grid: value count does not match (R+1)^3")
    with open(path, "wb") as f:
        f.write(np.array([level, cells], dtype="<i4").tobytes())
        f.write(a.astype("<f4").tobytes())


def load_grid_dump(path: str):
    """Inverse of dump_grid (grid.hpp:211-222): returns (level, cells, values)."""
    with open(path, "rb") as f:
        hdr = f.read(8)
        if len(hdr) < 8:
            raise RuntimeError(f"load_grid_dump: short header in {path}")
        level, cells = (int(v) for v in np.frombuffer(hdr, dtype="<i4"))
        n = (cells + 1) ** 3
        data = f.read(4 * n)
        if len(data) < 4 * n:
            raise RuntimeError(f"load_grid_dump: short data in {path}")
    return level, cells, np.frombuffer(data, dtype="<f4").copy()


# ---------------------------------------------------------------------------
# Seeded synthetic inputs (host helpers in the library)
# ---------------------------------------------------------------------------
def gen_capsules(seed: int, n: int = 15) -> list:
    arr = (abi.icg_primitive * n)()
    _check(abi.lib().icg_gen_capsules(seed, n, arr))
    return list(arr)


def capsules_array(prims) -> np.ndarray:
    return np.array([[*p.a, *p.b, p.radius] for p in prims], dtype=np.float64)


def gen_normals(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float32)
    _check(abi.lib().icg_gen_normals(seed, n, _ptr(out, C.c_float)))
    return out


def gen_feature_map(seed: int, c: int = 256, h: int = 128, w: int = 128) -> np.ndarray:
    return gen_normals(seed, c * h * w).reshape(c, h, w)


def mlp_shape(which: int):
    outs = (C.c_int32 * 5)()
    ins = (C.c_int32 * 5)()
    skip = C.c_int32()
    nw, nb = C.c_size_t(), C.c_size_t()
    _check(abi.lib().icg_mlp_shape(which, outs, ins, C.byref(skip), C.byref(nw), C.byref(nb)))
    return list(outs), list(ins), skip.value, nw.value, nb.value


def gen_mlp(seed: int, which: int):
    """Kaiming-uniform weights (list of [out][in] float32) and biases."""
    outs, ins, _, nw, nb = mlp_shape(which)
    w = np.empty(nw, np.float32)
    b = np.empty(nb, np.float32)
    _check(abi.lib().icg_gen_mlp(seed, which, _ptr(w, C.c_float), _ptr(b, C.c_float)))
    ws, bs, wo, bo = [], [], 0, 0
    for o, i in zip(outs, ins):
        ws.append(w[wo:wo + o * i].reshape(o, i))
        bs.append(b[bo:bo + o])
        wo += o * i
        bo += o
    return ws, bs

"""ctypes mirror of the C ABI in include/isocull_b200.h.

Loads the in-tree sm_100a library ``libisocull_b200.so``.  There is no Python,
PyTorch or CPU fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ICG_LIB") or os.path.join(HERE, "libisocull_b200.so")  # ICG_LIB: dev builds

# ---- constants (include/isocull_b200.h) ----------------------------------
ICG_OK, ICG_ERUNTIME, ICG_EINVAL, ICG_ECAPACITY, ICG_ENODEV = 0, 1, 2, 3, 4
ICG_MAX_LEVELS = 16
ICG_MAX_PRIMS = 64
ICG_MEM_HOST, ICG_MEM_DEVICE = 0, 1
ICG_STATE_UNKNOWN, ICG_STATE_INTERPOLATED, ICG_STATE_EVALUATED, ICG_STATE_SHADOW = 0, 1, 2, 3
ICG_PRIM_SPHERE, ICG_PRIM_BOX, ICG_PRIM_CAPSULE, ICG_PRIM_TORUS = 0, 1, 2, 3
ICG_FIELD_ANALYTIC, ICG_FIELD_PIFU = 0, 1
ICG_PREC_FP32, ICG_PREC_BF16, ICG_PREC_FP32_SIMT = 0, 1, 2
ICG_MLP_GEOMETRY, ICG_MLP_TEXTURE = 0, 1
ICG_MLP_LAYERS = 5
ICG_VARIANT_BRUTE, ICG_VARIANT_OCTREE_BINARIZED, ICG_VARIANT_OCTREE_THRESHOLD, ICG_VARIANT_PROGRESSIVE = 0, 1, 2, 3
ICG_SET_EVALUATED_NODES, ICG_SET_REFINED_CELLS = 0, 1
ICG_ABI_VERSION = 4

f32p = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class icg_primitive(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("rotated", C.c_int32),
        ("center", C.c_double * 3),
        ("a", C.c_double * 3),
        ("b", C.c_double * 3),
        ("radius", C.c_double),
        ("half", C.c_double * 3),
        ("major", C.c_double),
        ("minor", C.c_double),
        ("inv_rotation", C.c_double * 9),
    ]


ICG_TEXTURE_NONE, ICG_TEXTURE_CONSTANT, ICG_TEXTURE_GRADIENT, ICG_TEXTURE_PER_PRIMITIVE = 0, 1, 2, 3


class icg_texture_rule(C.Structure):
    _fields_ = [("kind", C.c_int32), ("axis", C.c_int32), ("color", C.c_double * 3), ("from_", C.c_double * 3),
                ("to", C.c_double * 3), ("colors", C.POINTER(C.c_double))]


class icg_scene(C.Structure):
    _fields_ = [("prims", C.POINTER(icg_primitive)), ("n_prims", C.c_int32), ("tau", C.c_double),
                ("texture", icg_texture_rule)]


class icg_camera(C.Structure):
    _fields_ = [("rotation", C.c_double * 9), ("translation", C.c_double * 3), ("scale", C.c_double)]


class icg_field(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("scene", icg_scene),
        ("sdf_scale", C.c_double),
        ("feature_map", f32p),
        ("fmap_c", C.c_int32),
        ("fmap_h", C.c_int32),
        ("fmap_w", C.c_int32),
        ("fmap_mem", C.c_int32),
        ("precision", C.c_int32),
        ("has_input_camera", C.c_int32),
        ("input_camera", icg_camera),
    ]


class icg_mlp_desc(C.Structure):
    _fields_ = [
        ("which", C.c_int32),
        ("n_layers", C.c_int32),
        ("skip_dim", C.c_int32),
        ("out_dims", C.c_int32 * 5),
        ("weights", f32p * 5),
        ("biases", f32p * 5),
        ("leaky_slope", C.c_float),
    ]


class icg_algo_config(C.Structure):
    _fields_ = [
        ("variant", C.c_int32),
        ("coarsest_cells", C.c_int32),
        ("target_level", C.c_int32),
        ("max_conflict_iters", C.c_int32),
        ("conflict_pass", C.c_int32),
        ("keep_level_sets", C.c_int32),
        ("threshold", C.c_double),
    ]


class icg_extraction(C.Structure):
    _fields_ = [
        ("mem", C.c_int32),
        ("values", f32p),
        ("states", u8p),
        ("binarized", u8p),
        ("cells", C.c_int32),
        ("levels", C.c_int32),
        ("evals_per_level", C.c_uint64 * ICG_MAX_LEVELS),
        ("total_evals", C.c_uint64),
        ("refined_cells_per_level", C.c_uint64 * ICG_MAX_LEVELS),
        ("conflict_iters_per_level", C.c_uint32 * ICG_MAX_LEVELS),
        ("conflict_warning", C.c_int32),
        ("wall_seconds", C.c_double),
    ]


class icg_image(C.Structure):
    _fields_ = [
        ("mem", C.c_int32),
        ("depth", f32p),
        ("rgb", f32p),
        ("mask", u8p),
        ("surface_k", i32p),
        ("covered_pixels", C.c_uint64),
        ("degenerate_brackets", C.c_uint64),
        ("grazing_pixels", C.c_uint64),
        ("texture_points", C.c_uint64),
        ("wall_seconds", C.c_double),
        ("oracle_calls", C.c_uint64),
    ]


class icg_mesh(C.Structure):
    _fields_ = [("vertices", f64p), ("vertex_capacity", C.c_uint64), ("triangles", i32p),
                ("triangle_capacity", C.c_uint64), ("n_vertices", C.c_uint64), ("n_triangles", C.c_uint64)]


class icg_profile(C.Structure):
    _fields_ = [
        ("kernel_launches", C.c_uint64),
        ("geo_mlp_launches", C.c_uint64),
        ("geo_points", C.c_uint64),
        ("geo_mlp_ms", C.c_double),
        ("tex_mlp_launches", C.c_uint64),
        ("tex_points", C.c_uint64),
        ("tex_mlp_ms", C.c_double),
        ("dense_launches", C.c_uint64),
        ("dense_ms", C.c_double),
        ("dense_bytes", C.c_uint64),
        ("render_launches", C.c_uint64),
        ("render_ms", C.c_double),
        ("render_bytes", C.c_uint64),
        ("frame_ms", C.c_double),
        ("frames", C.c_uint64),
        ("fact_launches", C.c_uint64),
        ("fact_points", C.c_uint64),
        ("fact_ms", C.c_double),
        ("chain_launches", C.c_uint64),
        ("chain_points", C.c_uint64),
        ("chain_ms", C.c_double),
        ("gather_launches", C.c_uint64),
        ("gather_points", C.c_uint64),
        ("gather_ms", C.c_double),
        ("gather_bytes", C.c_uint64),
        ("expand_launches", C.c_uint64),
        ("expand_ms", C.c_double),
        ("last_level_launches", C.c_uint64),
        ("last_level_ms", C.c_double),
        ("last_level_bytes", C.c_uint64),
    ]


ctx_p = C.c_void_p

# (name, restype, argtypes) for every symbol the header declares
SIGNATURES = [
    ("icg_abi_version", C.c_int, []),
    ("icg_last_error", C.c_char_p, []),
    ("icg_device_count", C.c_int, [C.POINTER(C.c_int)]),
    ("icg_create", C.c_int, [C.c_int, C.POINTER(ctx_p)]),
    ("icg_destroy", C.c_int, [ctx_p]),
    ("icg_set_mlp", C.c_int, [ctx_p, C.POINTER(icg_mlp_desc)]),
    ("icg_extract", C.c_int, [ctx_p, C.POINTER(icg_field), C.POINTER(icg_algo_config), C.POINTER(icg_extraction)]),
    ("icg_render_localized", C.c_int,
     [ctx_p, C.POINTER(icg_field), C.POINTER(icg_camera), C.c_int, C.c_int, f32p, C.POINTER(icg_image)]),
    ("icg_render_view", C.c_int,
     [ctx_p, C.POINTER(icg_field), C.POINTER(icg_camera), C.POINTER(icg_algo_config), f32p, C.POINTER(icg_image)]),
    ("icg_surface_depth_map", C.c_int,
     [ctx_p, C.POINTER(icg_field), C.POINTER(icg_camera), C.POINTER(icg_algo_config), C.POINTER(icg_image)]),
    ("icg_frame", C.c_int,
     [ctx_p, C.POINTER(icg_field), C.POINTER(icg_algo_config), C.POINTER(icg_camera), C.c_int, C.c_int, f32p,
      C.POINTER(icg_extraction), C.POINTER(icg_image)]),
    ("icg_level_set", C.c_int,
     [ctx_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint32), C.c_size_t, C.POINTER(C.c_size_t)]),
    ("icg_occupancy_batch", C.c_int, [ctx_p, C.POINTER(icg_field), f64p, C.c_size_t, C.c_int, f32p]),
    ("icg_texture_batch", C.c_int, [ctx_p, C.POINTER(icg_field), f64p, C.c_size_t, C.c_int, f32p]),
    ("icg_compare_iou", C.c_int, [ctx_p, u8p, u8p, C.c_size_t, C.c_int, f64p]),
    ("icg_composite", C.c_int, [f32p, u8p, C.c_size_t, f32p, C.c_size_t, f32p]),
    ("icg_marching_cubes", C.c_int, [ctx_p, f32p, C.c_int, C.c_int, C.c_double, C.POINTER(icg_mesh)]),
    ("icg_mc_case", C.c_int, [C.c_int, C.POINTER(C.c_int8), C.POINTER(C.c_int)]),
    ("icg_write_obj", C.c_int, [C.c_char_p, f64p, C.c_uint64, i32p, C.c_uint64]),
    ("icg_profile_enable", C.c_int, [ctx_p, C.c_int]),
    ("icg_profile_reset", C.c_int, [ctx_p]),
    ("icg_profile_get", C.c_int, [ctx_p, C.POINTER(icg_profile)]),
    ("icg_span_begin", C.c_int, [C.POINTER(ctx_p), C.c_int]),
    ("icg_span_end", C.c_int, [C.POINTER(ctx_p), C.c_int, C.POINTER(C.c_float)]),
    ("icg_host_alloc", C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    ("icg_host_free", C.c_int, [C.c_void_p]),
    ("icg_device_alloc", C.c_int, [ctx_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    ("icg_device_free", C.c_int, [ctx_p, C.c_void_p]),
    ("icg_memcpy", C.c_int, [ctx_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int]),
    ("icg_memset", C.c_int, [ctx_p, C.c_void_p, C.c_int, C.c_size_t]),
    ("icg_gen_capsules", C.c_int, [C.c_uint64, C.c_int, C.POINTER(icg_primitive)]),
    ("icg_gen_normals", C.c_int, [C.c_uint64, C.c_size_t, f32p]),
    ("icg_gen_mlp", C.c_int, [C.c_uint64, C.c_int, f32p, f32p]),
    ("icg_mlp_shape", C.c_int,
     [C.c_int, i32p, i32p, i32p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    ("icg_camera_from_angles", C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(icg_camera)]),
    ("icg_gen_feature_map_device", C.c_int, [ctx_p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, f32p]),
    ("icg_write_ppm", C.c_int, [C.c_char_p, C.c_int, C.c_int, f32p]),
    ("icg_write_float_map", C.c_int, [C.c_char_p, C.c_int, C.c_int, f32p]),
    ("icg_dump_grid", C.c_int, [C.c_char_p, C.c_int, C.c_int, f32p]),
    ("icg_load_grid_dump", C.c_int, [C.c_char_p, i32p, i32p, f32p, C.c_size_t]),
]


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"isocull_b200: CUDA extension not built ({path} missing); run `make` or "
            "__graft_entry__.build() — there is no CPU fallback")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB

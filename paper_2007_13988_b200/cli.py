"""Command-line front end over the C ABI, mirroring the reference CLI's hot-path subcommands
(tools/isocull_cli.cpp) so its outputs are drop-in:

  python -m paper_2007_13988_b200.cli extract --scene S.json [--variant V --threshold T
                                              --resolution R --coarsest C --out DIR --dump-grid]
  python -m paper_2007_13988_b200.cli bench --scene S.json [--scene ...] [--variant ...]
                                            [--threshold ...] [--resolution ...] [--coarsest C] [--out DIR]
  python -m paper_2007_13988_b200.cli render --scene S.json [--camera yaw,pitch,dist --projection ortho|weak
                                             --scale s --background r,g,b --resolution R --coarsest C
                                             --out DIR --depth-dump]

CSV schema (isocull_cli.cpp:52-59): scene,variant,threshold,R_L,total_evals,accel_factor,iou,wall_ms
with %.6f doubles; `bench` writes DIR/bench.csv (one brute-force reference per scene and
resolution, every variant and threshold, :134-172), `extract` writes the GPU marching-cubes mesh
DIR/<scene>_<variant>.obj and appends to DIR/stats.csv (:82-119; --dump-grid also dumps the
localized grid), `render` writes DIR/render.ppm and optionally DIR/depth.f32 (:188-218).  Exit codes: invalid_argument -> 2, other errors -> 1 (:358-364).

Scene files use the reference's JSON format (scene.hpp:204-321) for union scenes: primitives
sphere / box / capsule / torus with optional center and rotation (yaw, pitch, roll degrees,
R = Ry Rx Rz), tau, texture constant / gradient / per_primitive.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from typing import List, Optional

from . import abi, api

STATS_HEADER = "scene,variant,threshold,R_L,total_evals,accel_factor,iou,wall_ms"


def csv_double(v: float) -> str:
    return "%.6f" % v


def stats_row(scene, variant, threshold, resolution, evals, accel, iou, wall_ms) -> str:
    return f"{scene},{variant},{threshold},{resolution},{evals},{csv_double(accel)},{csv_double(iou)},{csv_double(wall_ms)}\n"


def level_for_resolution(resolution: int, coarsest: int) -> int:
    """isocull_cli.cpp:31-44"""
    if coarsest < 2:
        raise ValueError("coarsest must be >= 2")
    level, r = 0, coarsest
    while r < resolution and level < 16:
        r *= 2
        level += 1
    if r != resolution:
        raise ValueError(f"resolution must be coarsest * 2^L, got {resolution} with coarsest {coarsest}")
    return level


# ---- scene JSON (union scenes) -------------------------------------------------------------
def _vec3(j, what):
    if not isinstance(j, list) or len(j) != 3:
        raise ValueError(f"scene: {what} must be a 3-array")
    v = [float(x) for x in j]
    if not all(math.isfinite(x) for x in v):
        raise ValueError(f"scene: {what} not finite")
    return v


def _mat_mul(a, b):
    """Mat3 operator* (geom.hpp:75-84): s = 0; s += a[i][k] b[k][j] in k order."""
    out = []
    for i in range(3):
        for j in range(3):
            acc = 0.0
            for k in range(3):
                acc += a[3 * i + k] * b[3 * k + j]
            out.append(acc)
    return out


def _rotation(angles):
    """yaw (about y), pitch (about x), roll (about z), degrees: Ry * Rx * Rz (scene.hpp:216-221)."""
    y, p, r = (a * math.pi / 180.0 for a in angles)  # deg_to_rad, geom.hpp:11
    cy, sy, cp, sp, cr, sr = math.cos(y), math.sin(y), math.cos(p), math.sin(p), math.cos(r), math.sin(r)
    ry = [cy, 0.0, sy, 0.0, 1.0, 0.0, -sy, 0.0, cy]
    rx = [1.0, 0.0, 0.0, 0.0, cp, -sp, 0.0, sp, cp]
    rz = [cr, -sr, 0.0, sr, cr, 0.0, 0.0, 0.0, 1.0]
    return _mat_mul(_mat_mul(ry, rx), rz)


def load_scene(path: str):
    """(name, prims, tau, texture dict) of a union scene file."""
    try:
        j = json.load(open(path))
    except OSError:
        raise ValueError(f"scene: cannot open {path}")
    except json.JSONDecodeError as e:
        raise ValueError(f"scene: {path}: {e}")
    if "csg" in j:
        raise ValueError("scene: only union scenes (no csg tree) are supported")
    prims = []
    kinds = {"sphere": abi.ICG_PRIM_SPHERE, "box": abi.ICG_PRIM_BOX, "capsule": abi.ICG_PRIM_CAPSULE,
             "torus": abi.ICG_PRIM_TORUS}
    for pj in j["primitives"]:
        p = abi.icg_primitive()
        kind = pj["kind"]
        if kind not in kinds:
            raise ValueError(f"scene: unknown primitive kind '{kind}'")
        p.kind = kinds[kind]
        if "center" in pj:
            p.center[:] = _vec3(pj["center"], "center")
        p.inv_rotation[:] = [1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0]
        if "rotation" in pj:
            m = _rotation(_vec3(pj["rotation"], "rotation"))
            p.inv_rotation[:] = [m[0], m[3], m[6], m[1], m[4], m[7], m[2], m[5], m[8]]  # transposed
            p.rotated = 1
        if kind in ("sphere", "capsule"):
            p.radius = float(pj["radius"])
        if kind == "box":
            p.half[:] = _vec3(pj["half"], "half")
        if kind == "capsule":
            p.a[:] = _vec3(pj["a"], "a")
            p.b[:] = _vec3(pj["b"], "b")
        if kind == "torus":
            p.major, p.minor = float(pj["major"]), float(pj["minor"])
        prims.append(p)
    tex = {"kind": abi.ICG_TEXTURE_NONE}
    if "texture" in j:
        t = j["texture"]
        typ = t["type"]
        if typ == "constant":
            tex = {"kind": abi.ICG_TEXTURE_CONSTANT, "color": _vec3(t["color"], "color")}
        elif typ == "gradient":
            axis = {"x": 0, "y": 1, "z": 2}.get(t["axis"])
            if axis is None:
                raise ValueError("scene: gradient axis must be x, y or z")
            tex = {"kind": abi.ICG_TEXTURE_GRADIENT, "axis": axis, "from": _vec3(t["from"], "from"),
                   "to": _vec3(t["to"], "to")}
        elif typ == "per_primitive":
            tex = {"kind": abi.ICG_TEXTURE_PER_PRIMITIVE, "colors": [_vec3(c, "color") for c in t["colors"]]}
            if len(tex["colors"]) != len(prims):
                raise ValueError("scene: per_primitive texture needs one color per primitive")
        else:
            raise ValueError(f"scene: unknown texture type '{typ}'")
    name = j.get("name", "scene")
    tau = float(j.get("tau", 2.0 / 256.0))
    if not prims:
        raise ValueError("scene: no primitives")
    if not tau > 0.0:
        raise ValueError("scene: tau must be > 0")
    return name, prims, tau, tex


# ---- subcommands ---------------------------------------------------------------------------
def make_config(variant: str, threshold: float, resolution: int, coarsest: int) -> api.AlgoConfig:
    if variant not in api.VARIANTS:
        raise ValueError(f"unknown variant '{variant}'")
    return api.AlgoConfig(variant, coarsest, level_for_resolution(resolution, coarsest), threshold=threshold)


def cmd_extract(a, ctx: api.Context) -> int:
    name, prims, tau, tex = load_scene(a.scene)
    cfg = make_config(a.variant, a.threshold, a.resolution, a.coarsest)
    f = api.AnalyticField(prims, tau, tex)
    res = ctx.extract(f, cfg)
    accel = iou = 1.0
    if a.variant != "brute":
        brute = ctx.extract(f, api.AlgoConfig("brute", a.coarsest, cfg.target_level))
        accel = api.acceleration_factor(res, brute)
        iou = api.compare_iou(res.binarized, brute.binarized, ctx)
    os.makedirs(a.out, exist_ok=True)
    V, T = ctx.marching_cubes(res.values)
    obj = os.path.join(a.out, f"{name}_{a.variant}.obj")
    api.write_obj(obj, V, T)
    path = os.path.join(a.out, "stats.csv")
    fresh = not os.path.exists(path)
    with open(path, "a") as fcsv:
        if fresh:
            fcsv.write(STATS_HEADER + "\n")
        fcsv.write(stats_row(name, a.variant, csv_double(a.threshold) if a.variant == "octree_threshold" else "",
                             a.resolution, res.total_evals, accel, iou, res.wall_seconds * 1e3))
    if a.dump_grid:
        api.dump_grid(os.path.join(a.out, f"{name}_{a.variant}.grid"), cfg.target_level, res.cells, res.values)
    print(f"extract: {name} ({a.variant}, {a.resolution}^3, tau={tau:g}): evals={res.total_evals} "
          f"accel={csv_double(accel)} iou={csv_double(iou)} -> {obj}", file=sys.stderr)
    if res.conflict_warning:
        print("extract: warning: conflict pass hit its iteration bound", file=sys.stderr)
    return 0


def cmd_bench(a, ctx: api.Context) -> int:
    os.makedirs(a.out, exist_ok=True)
    path = os.path.join(a.out, "bench.csv")
    with open(path, "w") as fcsv:
        fcsv.write(STATS_HEADER + "\n")
        for sp in a.scene:
            name, prims, tau, tex = load_scene(sp)
            f = api.AnalyticField(prims, tau, tex)
            print(f"bench: scene {name} tau={tau:g}", file=sys.stderr)
            for resolution in a.resolution:
                base = make_config("brute", 0.12, resolution, a.coarsest)
                brute = ctx.extract(f, base)
                for variant in a.variant:
                    thresholds = a.threshold if variant == "octree_threshold" else [0.0]
                    for t in thresholds:
                        res = brute if variant == "brute" else ctx.extract(
                            f, make_config(variant, t, resolution, a.coarsest))
                        fcsv.write(stats_row(name, variant, csv_double(t) if variant == "octree_threshold" else "",
                                             resolution, res.total_evals, api.acceleration_factor(res, brute),
                                             api.compare_iou(res.binarized, brute.binarized, ctx),
                                             res.wall_seconds * 1e3))
    print(f"bench: wrote {path}", file=sys.stderr)
    return 0


def cmd_render(a, ctx: api.Context) -> int:
    name, prims, tau, tex = load_scene(a.scene)
    if tex["kind"] == abi.ICG_TEXTURE_NONE:
        raise ValueError("render: scene has no texture")
    if len(a.camera) != 3:
        raise ValueError("render: --camera wants yaw,pitch,dist")
    if len(a.background) != 3:
        raise ValueError("render: --background wants r,g,b")
    if a.projection not in ("ortho", "weak"):
        raise ValueError("render: projection must be ortho or weak")
    cfg = make_config("progressive", 0.12, a.resolution, a.coarsest)
    scale = a.scale if a.projection == "weak" else 1.0
    cam = api.CameraSpec.from_angles(a.camera[0], a.camera[1], a.camera[2], scale)
    img = ctx.render_view(api.AnalyticField(prims, tau, tex), cam, cfg, tuple(a.background))
    os.makedirs(a.out, exist_ok=True)
    ppm = os.path.join(a.out, "render.ppm")
    api.write_ppm(ppm, img.width, img.height, img.rgb)
    if a.depth_dump:
        api.write_float_map(os.path.join(a.out, "depth.f32"), img.width, img.height, img.depth)
    print(f"render: {name} {img.width}x{img.height} oracle_calls={img.oracle_calls} "
          f"degenerate={img.degenerate_brackets} grazing={img.grazing_pixels} -> {ppm}", file=sys.stderr)
    return 0


def _floats(s: str) -> List[float]:
    return [float(x) for x in s.split(",")]


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="isocull_b200")
    ap.add_argument("--device", type=int, default=0)
    sub = ap.add_subparsers(dest="cmd", required=True)
    ex = sub.add_parser("extract", help="surface localization of one scene")
    ex.add_argument("--scene", required=True)
    ex.add_argument("--variant", default="progressive")
    ex.add_argument("--threshold", type=float, default=0.12)
    ex.add_argument("--resolution", type=int, default=128)
    ex.add_argument("--coarsest", type=int, default=16)
    ex.add_argument("--out", default="out")
    ex.add_argument("--dump-grid", action="store_true")
    be = sub.add_parser("bench", help="benchmark extraction variants")
    be.add_argument("--scene", action="append", required=True)
    be.add_argument("--variant", action="append")
    be.add_argument("--threshold", action="append", type=float)
    be.add_argument("--resolution", action="append", type=int)
    be.add_argument("--coarsest", type=int, default=16)
    be.add_argument("--out", default="out")
    re_ = sub.add_parser("render", help="mesh-free novel-view render")
    re_.add_argument("--scene", required=True)
    re_.add_argument("--camera", type=_floats, default=[0.0, 0.0, 0.0])
    re_.add_argument("--projection", default="ortho")
    re_.add_argument("--scale", type=float, default=1.0)
    re_.add_argument("--background", type=_floats, default=[0.0, 0.0, 0.0])
    re_.add_argument("--resolution", type=int, default=128)
    re_.add_argument("--coarsest", type=int, default=16)
    re_.add_argument("--out", default="out")
    re_.add_argument("--depth-dump", action="store_true")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    if a.cmd == "bench":  # CLI11 defaults of cmd_bench (isocull_cli.cpp:122-131)
        a.variant = a.variant or ["brute", "octree_binarized", "octree_threshold", "progressive"]
        a.threshold = a.threshold or [0.05, 0.08, 0.12, 0.2, 0.3, 0.4]
        a.resolution = a.resolution or [128]
    try:
        for sp in a.scene if isinstance(a.scene, list) else [a.scene]:
            load_scene(sp)  # scene errors are invalid_argument (exit 2) before any device work
        with api.Context(a.device) as ctx:
            return {"extract": cmd_extract, "bench": cmd_bench, "render": cmd_render}[a.cmd](a, ctx)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 -- the reference CLI maps every other error to exit 1
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/isocull/*.hpp, compiled read-only where they
// lie; nothing is copied into this repo).  Built by oracle/Makefile into
// oracle/_ref/libisocull_ref.so.  It lets the tests (and bench.py's
// --impl reference arm) run the reference's own operators:
//   extract / extract_progressive / extract_brute_force ... localize.hpp:181-373
//   render_view (view-aligned reference renderer) ........... render.hpp:244-280
//   grid primitives ......................................... grid.hpp:87-197
//   Rng ..................................................... random.hpp:16-43
//   scene JSON loading ...................................... scene.hpp:302-333
//   output formats (PPM, float map, grid dump) .............. image.hpp:18-48, grid.hpp:199-222
// with the field supplied as a C callback wrapped in the reference's own
// FieldOracle (field.hpp:22-77), so the reference's call counter and
// parallel_for drive evaluation exactly as they do in the reference.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "isocull/field.hpp"
#include "isocull/grid.hpp"
#include "isocull/image.hpp"
#include "isocull/localize.hpp"
#include "isocull/mesh.hpp"
#include "isocull/random.hpp"
#include "isocull/render.hpp"
#include "isocull/scene.hpp"

#include "../include/isocull_b200.h"

using namespace isocull;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}
}  // namespace

extern "C" {

typedef double (*ref_pt_occ_fn)(void* user, const double* p);
typedef void (*ref_pt_tex_fn)(void* user, const double* p, double* rgb);

const char* ref_last_error() { return g_err.c_str(); }

static FieldOracle make_oracle(ref_pt_occ_fn occ, ref_pt_tex_fn tex, void* user) {
    FieldOracle::OccupancyFn o = [occ, user](const Vec3& p) {
        double q[3] = {p.x, p.y, p.z};
        return occ(user, q);
    };
    FieldOracle::TextureFn t;
    if (tex)
        t = [tex, user](const Vec3& p) {
            double q[3] = {p.x, p.y, p.z}, c[3];
            tex(user, q, c);
            return Vec3{c[0], c[1], c[2]};
        };
    return FieldOracle(std::move(o), std::move(t));
}

// extract(oracle, cfg, workers), localize.hpp:365-373
int ref_extract(ref_pt_occ_fn occ, void* user, int variant, double threshold, int coarsest, int level,
                int max_conflict_iters, int conflict_pass, int workers, float* values, uint8_t* states,
                uint8_t* binarized, uint64_t* evals_per_level, uint64_t* total_evals, uint64_t* oracle_calls,
                int* conflict_warning, double* wall_seconds) {
    try {
        FieldOracle oracle = make_oracle(occ, nullptr, user);
        AlgoConfig cfg;
        cfg.variant = static_cast<Variant>(variant);
        cfg.threshold = threshold;
        cfg.coarsest_cells = coarsest;
        cfg.target_level = level;
        cfg.max_conflict_iters = max_conflict_iters;
        cfg.conflict_pass = conflict_pass != 0;
        ExtractionResult r = extract(oracle, cfg, workers);
        if (values) std::memcpy(values, r.grid.values.data(), r.grid.values.size() * sizeof(float));
        if (states) std::memcpy(states, r.grid.states.data(), r.grid.states.size());
        if (binarized) std::memcpy(binarized, r.binarized.data(), r.binarized.size());
        for (std::size_t l = 0; l < r.evals_per_level.size() && l < 16; ++l) evals_per_level[l] = r.evals_per_level[l];
        *total_evals = r.total_evals;
        *oracle_calls = oracle.calls();
        *conflict_warning = r.conflict_warning ? 1 : 0;
        *wall_seconds = r.wall_seconds;
        return ICG_OK;
    } catch (const std::invalid_argument& e) {
        return fail(e, ICG_EINVAL);
    } catch (const std::exception& e) {
        return fail(e, ICG_ERUNTIME);
    }
}

// render_view(oracle, camera, cfg, background, workers), render.hpp:244-280
int ref_render_view(ref_pt_occ_fn occ, ref_pt_tex_fn tex, void* user, double yaw, double pitch, double dist,
                    double scale, int coarsest, int level, const double* bg, int workers, double* depth,
                    double* rgb, uint8_t* mask, uint64_t* oracle_calls, int* degenerate, int* grazing,
                    int* size) {
    try {
        FieldOracle oracle = make_oracle(occ, tex, user);
        AlgoConfig cfg;
        cfg.variant = Variant::progressive;
        cfg.coarsest_cells = coarsest;
        cfg.target_level = level;
        CameraSpec cam = CameraSpec::from_angles(yaw, pitch, dist, scale);
        RenderedImage img = render_view(oracle, cam, cfg, Vec3{bg[0], bg[1], bg[2]}, workers);
        std::size_t n = img.depth.size();
        if (depth) std::memcpy(depth, img.depth.data(), n * sizeof(double));
        if (mask) std::memcpy(mask, img.mask.data(), n);
        if (rgb)
            for (std::size_t i = 0; i < n; ++i) {
                rgb[3 * i] = img.rgb[i].x;
                rgb[3 * i + 1] = img.rgb[i].y;
                rgb[3 * i + 2] = img.rgb[i].z;
            }
        *oracle_calls = img.oracle_calls;
        *degenerate = img.degenerate_brackets;
        *grazing = img.grazing_pixels;
        *size = img.width;
        return ICG_OK;
    } catch (const std::invalid_argument& e) {
        return fail(e, ICG_EINVAL);
    } catch (const std::exception& e) {
        return fail(e, ICG_ERUNTIME);
    }
}

// FieldOracle::occupancy_batch / texture_batch (field.hpp:41-47, 56-63): the
// reference's own batched evaluation (parallel_for over `workers` threads,
// one std::function call per point).  Returns the call counter.
uint64_t ref_occupancy_batch(ref_pt_occ_fn occ, void* user, const double* pts, std::size_t n, int workers,
                             double* out) {
    FieldOracle oracle = make_oracle(occ, nullptr, user);
    std::vector<Vec3> p(n);
    for (std::size_t i = 0; i < n; ++i) p[i] = Vec3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    std::vector<double> v = oracle.occupancy_batch(p, workers);
    std::memcpy(out, v.data(), n * sizeof(double));
    return oracle.calls();
}

void ref_texture_batch(ref_pt_occ_fn occ, ref_pt_tex_fn tex, void* user, const double* pts, std::size_t n,
                       int workers, double* rgb) {
    FieldOracle oracle = make_oracle(occ, tex, user);
    std::vector<Vec3> p(n);
    for (std::size_t i = 0; i < n; ++i) p[i] = Vec3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    std::vector<Vec3> v = oracle.texture_batch(p, workers);
    for (std::size_t i = 0; i < n; ++i) {
        rgb[3 * i] = v[i].x;
        rgb[3 * i + 1] = v[i].y;
        rgb[3 * i + 2] = v[i].z;
    }
}

// CameraSpec::from_angles, render.hpp:36-45
void ref_camera_from_angles(double yaw, double pitch, double dist, double scale, double* rot9, double* t3) {
    CameraSpec c = CameraSpec::from_angles(yaw, pitch, dist, scale);
    for (int i = 0; i < 9; ++i) rot9[i] = c.rotation.m[i];
    t3[0] = c.translation.x;
    t3[1] = c.translation.y;
    t3[2] = c.translation.z;
}

// ---- scenes (scene.hpp) ----------------------------------------------------
struct RefScene {
    SceneSpec spec;
};

void* ref_scene_load(const char* path) {
    try {
        return new RefScene{load_scene(path)};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void* ref_scene_capsules(const icg_primitive* prims, int n, double tau) {
    auto* s = new RefScene;
    for (int i = 0; i < n; ++i) {
        Primitive p;
        p.kind = PrimitiveKind::capsule;
        p.capsule_a = {prims[i].a[0], prims[i].a[1], prims[i].a[2]};
        p.capsule_b = {prims[i].b[0], prims[i].b[1], prims[i].b[2]};
        p.radius = prims[i].radius;
        s->spec.primitives.push_back(p);
        CsgNode leaf;
        leaf.prim = i;
        s->spec.csg.children.push_back(leaf);
    }
    s->spec.csg.op = CsgOp::union_op;
    s->spec.tau = tau;
    return s;
}

// A union scene built from C-ABI primitives and a texture rule (parse_scene's default union tree,
// scene.hpp:302-321, with the fields parse_primitive / parse_texture fill), validated by the
// reference's validate_scene: the GPU box rebuilds the bundled scenes from tests/golden/scenes.json.
void* ref_scene_make(const icg_primitive* prims, int n, double tau, int tex_kind, int axis, const double* color,
                     const double* from, const double* to, const double* colors) {
    try {
        auto* s = new RefScene;
        for (int i = 0; i < n; ++i) {
            const icg_primitive& q = prims[i];
            Primitive p;
            p.kind = static_cast<PrimitiveKind>(q.kind);
            p.center = {q.center[0], q.center[1], q.center[2]};
            p.capsule_a = {q.a[0], q.a[1], q.a[2]};
            p.capsule_b = {q.b[0], q.b[1], q.b[2]};
            p.radius = q.radius;
            p.half = {q.half[0], q.half[1], q.half[2]};
            p.major = q.major;
            p.minor = q.minor;
            p.rotated = q.rotated != 0;
            for (int k = 0; k < 9; ++k) p.inv_rotation.m[k] = q.inv_rotation[k];
            s->spec.primitives.push_back(p);
            CsgNode leaf;
            leaf.prim = i;
            s->spec.csg.children.push_back(leaf);
        }
        s->spec.csg.op = CsgOp::union_op;
        s->spec.tau = tau;
        TextureRule& t = s->spec.texture;
        t.kind = static_cast<TextureKind>(tex_kind);
        if (color) t.color = {color[0], color[1], color[2]};
        t.axis = axis;
        if (from) t.from = {from[0], from[1], from[2]};
        if (to) t.to = {to[0], to[1], to[2]};
        if (tex_kind == static_cast<int>(TextureKind::per_primitive))
            for (int i = 0; i < n; ++i) t.colors.push_back({colors[3 * i], colors[3 * i + 1], colors[3 * i + 2]});
        validate_scene(s->spec);
        return s;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// The scene's texture rule (after the reference's own JSON parsing): kind, axis, color, from, to,
// per-primitive colors (room for max primitives).  Returns the number of per-primitive colors.
int ref_scene_texture(void* handle, int* kind, int* axis, double* color, double* from, double* to, double* colors,
                      int max) {
    const TextureRule& t = static_cast<RefScene*>(handle)->spec.texture;
    *kind = static_cast<int>(t.kind);
    *axis = t.axis;
    color[0] = t.color.x, color[1] = t.color.y, color[2] = t.color.z;
    from[0] = t.from.x, from[1] = t.from.y, from[2] = t.from.z;
    to[0] = t.to.x, to[1] = t.to.y, to[2] = t.to.z;
    int n = static_cast<int>(t.colors.size());
    for (int i = 0; i < n && i < max; ++i)
        colors[3 * i] = t.colors[i].x, colors[3 * i + 1] = t.colors[i].y, colors[3 * i + 2] = t.colors[i].z;
    return n;
}

void ref_scene_free(void* s) { delete static_cast<RefScene*>(s); }

// marching_cubes(grid, iso) (mesh.hpp:75-156) on a (cells+1)^3 grid; outputs up to the capacities
int ref_marching_cubes(const float* values, int cells, double iso, double* vertices, int vcap, int32_t* triangles,
                       int tcap, int* nv, int* nt) {
    try {
        LevelGrid g = LevelGrid::make(0, cells, NodeState::evaluated);
        std::memcpy(g.values.data(), values, g.values.size() * sizeof(float));
        TriangleMesh m = marching_cubes(g, iso);
        *nv = static_cast<int>(m.vertices.size());
        *nt = static_cast<int>(m.triangles.size());
        for (int i = 0; i < *nv && i < vcap; ++i) {
            vertices[3 * i] = m.vertices[i].x;
            vertices[3 * i + 1] = m.vertices[i].y;
            vertices[3 * i + 2] = m.vertices[i].z;
        }
        for (int i = 0; i < *nt && i < tcap; ++i)
            for (int c = 0; c < 3; ++c) triangles[3 * i + c] = m.triangles[i][c];
        return ICG_OK;
    } catch (const std::invalid_argument& e) {
        return fail(e, ICG_EINVAL);
    } catch (const std::exception& e) {
        return fail(e, ICG_ERUNTIME);
    }
}

// export_obj (mesh.hpp:159-172)
int ref_export_obj(const char* path, const double* vertices, int nv, const int32_t* triangles, int nt) {
    try {
        TriangleMesh m;
        for (int i = 0; i < nv; ++i) m.vertices.push_back({vertices[3 * i], vertices[3 * i + 1], vertices[3 * i + 2]});
        for (int i = 0; i < nt; ++i) m.triangles.push_back({triangles[3 * i], triangles[3 * i + 1], triangles[3 * i + 2]});
        export_obj(m, path);
        return ICG_OK;
    } catch (const std::exception& e) {
        return fail(e, ICG_ERUNTIME);
    }
}

// Exports the (union-only) primitive list in the C ABI layout; returns -1 if
// the scene uses a non-union CSG tree.
int ref_scene_export(void* handle, icg_primitive* out, int max, double* tau, int* has_texture) {
    auto* s = static_cast<RefScene*>(handle);
    const SceneSpec& sc = s->spec;
    if (sc.csg.prim >= 0 || sc.csg.op != CsgOp::union_op) return -1;
    for (const auto& c : sc.csg.children)
        if (c.prim < 0) return -1;
    int n = static_cast<int>(sc.primitives.size());
    if (n > max) return -1;
    for (int i = 0; i < n; ++i) {
        const Primitive& p = sc.primitives[i];
        icg_primitive& o = out[i];
        std::memset(&o, 0, sizeof(o));
        o.kind = static_cast<int32_t>(p.kind);
        o.rotated = p.rotated ? 1 : 0;
        o.center[0] = p.center.x, o.center[1] = p.center.y, o.center[2] = p.center.z;
        o.a[0] = p.capsule_a.x, o.a[1] = p.capsule_a.y, o.a[2] = p.capsule_a.z;
        o.b[0] = p.capsule_b.x, o.b[1] = p.capsule_b.y, o.b[2] = p.capsule_b.z;
        o.radius = p.radius;
        o.half[0] = p.half.x, o.half[1] = p.half.y, o.half[2] = p.half.z;
        o.major = p.major, o.minor = p.minor;
        for (int k = 0; k < 9; ++k) o.inv_rotation[k] = p.inv_rotation.m[k];
    }
    *tau = sc.tau;
    *has_texture = sc.has_texture() ? 1 : 0;
    return n;
}

// FieldOracle-shaped callbacks over a loaded scene (build_oracle, field.hpp:83-91)
double ref_scene_occ(void* handle, const double* p) {
    auto* s = static_cast<RefScene*>(handle);
    return occupancy_from_distance(s->spec.signed_distance(Vec3{p[0], p[1], p[2]}), s->spec.tau);
}

void ref_scene_tex(void* handle, const double* p, double* rgb) {
    auto* s = static_cast<RefScene*>(handle);
    Vec3 c = s->spec.texture_color(Vec3{p[0], p[1], p[2]});
    rgb[0] = c.x, rgb[1] = c.y, rgb[2] = c.z;
}

double ref_scene_sdf(void* handle, const double* p) {
    return static_cast<RefScene*>(handle)->spec.signed_distance(Vec3{p[0], p[1], p[2]});
}

// ---- grid primitives (grid.hpp) --------------------------------------------
int ref_upsample(int level, int cells, const float* values, const uint8_t* states, float* out_values,
                 uint8_t* out_states) {
    try {
        LevelGrid g = LevelGrid::make(level, cells);
        std::memcpy(g.values.data(), values, g.values.size() * sizeof(float));
        std::memcpy(g.states.data(), states, g.states.size());
        LevelGrid f = upsample_interpolate(g);
        std::memcpy(out_values, f.values.data(), f.values.size() * sizeof(float));
        std::memcpy(out_states, f.states.data(), f.states.size());
        return ICG_OK;
    } catch (const std::invalid_argument& e) {
        return fail(e, ICG_EINVAL);
    }
}

void ref_binarize(std::size_t n, const float* in, float* out) {
    for (std::size_t i = 0; i < n; ++i) out[i] = binarize_value(in[i]);
}

void ref_boundary_candidates(int cells, const float* values, uint8_t* mask) {
    LevelGrid g = LevelGrid::make(0, cells, NodeState::evaluated);
    std::memcpy(g.values.data(), values, g.values.size() * sizeof(float));
    NodeMask m = boundary_candidates(g);
    std::memcpy(mask, m.bits.data(), m.bits.size());
}

void ref_dilate(int nodes, const uint8_t* in, uint8_t* out) {
    NodeMask m = NodeMask::make(nodes);
    std::memcpy(m.bits.data(), in, m.bits.size());
    NodeMask d = dilate_1ring(m);
    std::memcpy(out, d.bits.data(), d.bits.size());
}

void ref_argmax_z(int cells, const float* values, float* max_value, int* max_index) {
    LevelGrid g = LevelGrid::make(0, cells, NodeState::evaluated);
    std::memcpy(g.values.data(), values, g.values.size() * sizeof(float));
    ArgmaxZ a = argmax_z(g);
    std::memcpy(max_value, a.max_value.data(), a.max_value.size() * sizeof(float));
    std::memcpy(max_index, a.max_index.data(), a.max_index.size() * sizeof(int));
}

double ref_compare_iou(const uint8_t* a, const uint8_t* b, std::size_t n) {
    return compare_iou(std::span<const uint8_t>(a, n), std::span<const uint8_t>(b, n));
}

// ---- Rng (random.hpp) --------------------------------------------------------
void ref_rng_uniforms(uint64_t seed, std::size_t n, double* out) {
    Rng r(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = r.uniform();
}

void ref_rng_normals(uint64_t seed, std::size_t n, double* out) {
    Rng r(seed);
    for (std::size_t i = 0; i < n; ++i) out[i] = r.normal();
}

// ---- output formats (image.hpp, grid.hpp) ----------------------------------------
int ref_write_ppm(const char* path, int w, int h, const double* rgb) {
    try {
        std::vector<Vec3> px((std::size_t)w * h);
        for (std::size_t i = 0; i < px.size(); ++i) px[i] = Vec3{rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
        write_ppm(path, w, h, px);
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, ICG_EINVAL);
    } catch (const std::exception& e) {
        return fail(e, ICG_ERUNTIME);
    }
}

int ref_write_float_map(const char* path, int w, int h, const double* values) {
    try {
        write_float_map(path, w, h, std::span<const double>(values, (std::size_t)w * h));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, ICG_EINVAL);
    } catch (const std::exception& e) {
        return fail(e, ICG_ERUNTIME);
    }
}

int ref_dump_grid(const char* path, int level, int cells, const float* values) {
    try {
        LevelGrid g = LevelGrid::make(level, cells, NodeState::evaluated);
        std::memcpy(g.values.data(), values, g.values.size() * sizeof(float));
        dump_grid(g, path);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, ICG_ERUNTIME);
    }
}

}  // extern "C"

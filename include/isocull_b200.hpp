/*
 * isocull_b200.hpp — header-only C++ adapter over the C ABI (isocull_b200.h).
 *
 * Reproduces the reference's operator shapes (namespace isocull in
 * /root/reference/proj/include/isocull) so a reference-style caller switches
 * CPU <-> B200 by changing one include and one namespace:
 *
 *   reference                                     here
 *   AlgoConfig, Variant (localize.hpp:16-45)      AlgoConfig, Variant (same fields)
 *   validate_config (localize.hpp:47-55)          validate_config (same messages)
 *   LevelGrid, NodeState (grid.hpp:15-60)         LevelGrid, NodeState
 *   ExtractionResult (localize.hpp:57-64)         ExtractionResult (+ refined_cells_per_level)
 *   extract / extract_progressive /               extract / extract_progressive /
 *     extract_brute_force (localize.hpp:181-373)    extract_brute_force  (Context instead of workers)
 *   compare_iou, acceleration_factor (:377-393)   compare_iou, acceleration_factor
 *   CameraSpec (render.hpp:19-46)                 CameraSpec (same maps, from_angles)
 *   RenderedImage (render.hpp:50-59)              RenderedImage
 *   render_view (render.hpp:244-280)              render_view (view-aligned, shadow-culled)
 *   surface_depth_map (render.hpp:219-240)        surface_depth_map
 *   (north-star renderer)       render_localized / frame: first-crossing render
 *                                                   through the localized world grid
 *   composite (render.hpp:284-291)                composite
 *
 * Errors are thrown like the reference: ICG_EINVAL -> std::invalid_argument,
 * anything else -> std::runtime_error (the reference CLI maps them to exit 2 / 1,
 * tools/isocull_cli.cpp:358-364).  Link libisocull_b200.so.
 */
#ifndef ISOCULL_B200_HPP
#define ISOCULL_B200_HPP

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "isocull_b200.h"

namespace isocull_b200 {

inline void check(int rc) {
    if (rc == ICG_OK) return;
    const std::string msg = icg_last_error();
    if (rc == ICG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("isocull_b200 error " + std::to_string(rc) + ": " + msg);
}

struct Vec3 {
    double x = 0.0, y = 0.0, z = 0.0;
};

enum class NodeState : std::uint8_t { unknown = 0, interpolated = 1, evaluated = 2, shadow = 3 };
enum class Variant { brute, octree_binarized, octree_threshold, progressive };

struct AlgoConfig {
    Variant variant = Variant::progressive;
    double threshold = 0.0;
    int coarsest_cells = 16;
    int target_level = 3;
    int max_conflict_iters = 0;
    bool conflict_pass = true;
    bool keep_level_sets = false;  // keep per-level refined-cell / evaluated-node sets (level_set)

    int target_cells() const { return coarsest_cells << target_level; }

    icg_algo_config to_c() const {
        icg_algo_config c{};
        c.variant = variant == Variant::brute ? ICG_VARIANT_BRUTE
                    : variant == Variant::progressive ? ICG_VARIANT_PROGRESSIVE
                    : variant == Variant::octree_binarized ? ICG_VARIANT_OCTREE_BINARIZED
                                                           : ICG_VARIANT_OCTREE_THRESHOLD;
        c.threshold = threshold;
        c.coarsest_cells = coarsest_cells;
        c.target_level = target_level;
        c.max_conflict_iters = max_conflict_iters;
        c.conflict_pass = conflict_pass ? 1 : 0;
        c.keep_level_sets = keep_level_sets ? 1 : 0;
        return c;
    }
};

inline void validate_config(const AlgoConfig& cfg) {
    if (cfg.coarsest_cells < 2) throw std::invalid_argument("config: coarsest cells must be >= 2");
    if (cfg.target_level < 0) throw std::invalid_argument("config: target level must be >= 0");
    if (cfg.target_level > 10 || cfg.target_cells() > 1024)
        throw std::invalid_argument("config: target resolution exceeds 1024 cells per axis");
    if (cfg.variant == Variant::octree_threshold && !(cfg.threshold > 0.0 && cfg.threshold < 0.5))
        throw std::invalid_argument("config: threshold must lie in (0, 0.5)");
}

struct LevelGrid {
    int level = 0;
    int cells = 0;
    std::vector<float> values;
    std::vector<NodeState> states;

    int nodes() const { return cells + 1; }
    std::size_t node_count() const {
        const std::size_t n = static_cast<std::size_t>(cells) + 1;
        return n * n * n;
    }
    std::size_t index(int i, int j, int k) const {
        const std::size_t n = static_cast<std::size_t>(nodes());
        return static_cast<std::size_t>(i) + n * (static_cast<std::size_t>(j) + n * static_cast<std::size_t>(k));
    }
    Vec3 node_position(int i, int j, int k) const {
        const double r = static_cast<double>(cells);
        return {-1.0 + 2.0 * i / r, -1.0 + 2.0 * j / r, 1.0 - 2.0 * k / r};
    }
};

struct ExtractionResult {
    LevelGrid grid;
    std::vector<std::uint8_t> binarized;
    std::vector<std::uint64_t> evals_per_level;
    std::uint64_t total_evals = 0;
    double wall_seconds = 0.0;
    bool conflict_warning = false;
    std::vector<std::uint64_t> refined_cells_per_level;  // new output
};

struct CameraSpec {
    double rotation[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    Vec3 translation{};
    double scale = 1.0;

    Vec3 world_to_view(const Vec3& w) const {
        const double* m = rotation;
        const Vec3 v{m[0] * w.x + m[1] * w.y + m[2] * w.z + translation.x,
                     m[3] * w.x + m[4] * w.y + m[5] * w.z + translation.y,
                     m[6] * w.x + m[7] * w.y + m[8] * w.z + translation.z};
        return {scale * v.x, scale * v.y, v.z};
    }
    Vec3 view_to_world(const Vec3& p) const {
        const double* m = rotation;
        const Vec3 v{p.x / scale - translation.x, p.y / scale - translation.y, p.z - translation.z};
        return {m[0] * v.x + m[3] * v.y + m[6] * v.z, m[1] * v.x + m[4] * v.y + m[7] * v.z,
                m[2] * v.x + m[5] * v.y + m[8] * v.z};
    }
    static CameraSpec from_angles(double yaw_deg, double pitch_deg, double dist = 0.0, double scale = 1.0) {
        icg_camera c{};
        check(icg_camera_from_angles(yaw_deg, pitch_deg, dist, scale, &c));
        return from_c(c);
    }
    static CameraSpec from_c(const icg_camera& c) {
        CameraSpec s;
        for (int i = 0; i < 9; ++i) s.rotation[i] = c.rotation[i];
        s.translation = {c.translation[0], c.translation[1], c.translation[2]};
        s.scale = c.scale;
        return s;
    }
    icg_camera to_c() const {
        icg_camera c{};
        for (int i = 0; i < 9; ++i) c.rotation[i] = rotation[i];
        c.translation[0] = translation.x;
        c.translation[1] = translation.y;
        c.translation[2] = translation.z;
        c.scale = scale;
        return c;
    }
};

struct RenderedImage {
    int width = 0, height = 0;
    std::vector<Vec3> rgb;
    std::vector<double> depth;  // -2 where uncovered (render.hpp:72)
    std::vector<std::uint8_t> mask;
    std::vector<std::int32_t> surface_k;  // first-crossing sample index, -1 where uncovered
    Vec3 background{};
    std::uint64_t oracle_calls = 0;  // texture evaluations (covered pixels)
    int degenerate_brackets = 0;
    int grazing_pixels = 0;
};

// The field as data (a std::function cannot run on the GPU): an analytic
// union-of-primitives scene (build_oracle, field.hpp:83-91) or the PIFu field.
class Field {
  public:
    // texture: TextureRule (scene.hpp:48-55); per-primitive colors, n_prims x 3, in `colors`
    static Field analytic(std::vector<icg_primitive> prims, double tau, icg_texture_rule texture = {},
                          std::vector<double> colors = {}) {
        Field f;
        f.prims_ = std::move(prims);
        f.colors_ = std::move(colors);
        f.c_.kind = ICG_FIELD_ANALYTIC;
        f.c_.scene.tau = tau;
        f.c_.scene.texture = texture;
        f.bind();
        return f;
    }
    // feature map C x H x W fp32 (host memory, copied by every call); capsules bias the logit
    static Field pifu(const float* fmap, int c, int h, int w, std::vector<icg_primitive> capsules,
                      double sdf_scale = 50.0, int precision = ICG_PREC_FP32) {
        Field f;
        f.prims_ = std::move(capsules);
        f.c_.kind = ICG_FIELD_PIFU;
        f.c_.scene.tau = 0.02;
        f.c_.sdf_scale = sdf_scale;
        f.c_.feature_map = fmap;
        f.c_.fmap_c = c;
        f.c_.fmap_h = h;
        f.c_.fmap_w = w;
        f.c_.fmap_mem = ICG_MEM_HOST;
        f.c_.precision = precision;
        f.bind();
        return f;
    }
    Field(const Field& o) : prims_(o.prims_), colors_(o.colors_), c_(o.c_) { bind(); }
    Field& operator=(const Field& o) {
        prims_ = o.prims_;
        colors_ = o.colors_;
        c_ = o.c_;
        bind();
        return *this;
    }
    void set_input_camera(const CameraSpec& cam) {
        c_.has_input_camera = 1;
        c_.input_camera = cam.to_c();
    }
    const icg_field* get() const { return &c_; }

  private:
    Field() = default;
    void bind() {
        c_.scene.prims = prims_.empty() ? nullptr : prims_.data();
        c_.scene.n_prims = static_cast<std::int32_t>(prims_.size());
        c_.scene.texture.colors = colors_.empty() ? nullptr : colors_.data();
    }
    std::vector<icg_primitive> prims_;
    std::vector<double> colors_;
    icg_field c_{};
};

// One context per GPU (icg_create / icg_destroy); not copyable, movable.
class Context {
  public:
    explicit Context(int device = 0) { check(icg_create(device, &h_)); }
    ~Context() {
        if (h_) icg_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    Context(Context&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    Context& operator=(Context&& o) noexcept {
        if (this != &o) {
            if (h_) icg_destroy(h_);
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    icg_context* get() const { return h_; }

    // weights[l]: row-major [out][prev_out + skip] fp32, biases[l]: [out]
    void set_mlp(int which, const std::vector<std::vector<float>>& weights, const std::vector<std::vector<float>>& biases,
                 float leaky_slope = 0.02f) {
        if (weights.size() != ICG_MLP_LAYERS || biases.size() != ICG_MLP_LAYERS)
            throw std::invalid_argument("set_mlp: the PIFu MLPs have 5 layers");
        icg_mlp_desc d{};
        std::int32_t outs[5], ins[5], skip = 0;
        check(icg_mlp_shape(which, outs, ins, &skip, nullptr, nullptr));
        d.which = which;
        d.n_layers = ICG_MLP_LAYERS;
        d.skip_dim = skip;
        for (int l = 0; l < ICG_MLP_LAYERS; ++l) {
            if (weights[l].size() != static_cast<std::size_t>(outs[l]) * ins[l] || biases[l].size() != (std::size_t)outs[l])
                throw std::invalid_argument("set_mlp: layer size mismatch");
            d.out_dims[l] = outs[l];
            d.weights[l] = weights[l].data();
            d.biases[l] = biases[l].data();
        }
        d.leaky_slope = leaky_slope;
        check(icg_set_mlp(h_, &d));
    }

    // ascending per-level set of the last extraction with cfg.keep_level_sets (icg_level_set)
    std::vector<std::uint32_t> level_set(int level, int which) const {
        std::size_t n = 0;
        check(icg_level_set(h_, level, which, ICG_MEM_HOST, nullptr, 0, &n));
        std::vector<std::uint32_t> out(n);
        if (n) check(icg_level_set(h_, level, which, ICG_MEM_HOST, out.data(), n, &n));
        return out;
    }

  private:
    icg_context* h_ = nullptr;
};

namespace detail {
inline ExtractionResult to_result(const icg_extraction& e, const AlgoConfig& cfg, std::vector<float>&& values,
                                  std::vector<std::uint8_t>&& states, std::vector<std::uint8_t>&& binarized) {
    ExtractionResult r;
    r.grid.level = cfg.target_level;
    r.grid.cells = e.cells;
    r.grid.values = std::move(values);
    r.grid.states.resize(states.size());
    for (std::size_t i = 0; i < states.size(); ++i) r.grid.states[i] = static_cast<NodeState>(states[i]);
    r.binarized = std::move(binarized);
    for (int l = 0; l <= cfg.target_level; ++l) {
        r.evals_per_level.push_back(e.evals_per_level[l]);
        r.refined_cells_per_level.push_back(e.refined_cells_per_level[l]);
    }
    r.total_evals = e.total_evals;
    r.wall_seconds = e.wall_seconds;
    r.conflict_warning = e.conflict_warning != 0;
    return r;
}
}  // namespace detail

// extract(oracle, cfg, workers), localize.hpp:365-373 (variant progressive or brute)
inline ExtractionResult extract(Context& ctx, const Field& field, const AlgoConfig& cfg) {
    validate_config(cfg);
    const std::size_t n = static_cast<std::size_t>(cfg.target_cells() + 1);
    std::vector<float> values(n * n * n);
    std::vector<std::uint8_t> states(values.size()), bin(values.size());
    icg_extraction e{};
    e.mem = ICG_MEM_HOST;
    e.values = values.data();
    e.states = states.data();
    e.binarized = bin.data();
    const icg_algo_config c = cfg.to_c();
    check(icg_extract(ctx.get(), field.get(), &c, &e));
    return detail::to_result(e, cfg, std::move(values), std::move(states), std::move(bin));
}

inline ExtractionResult extract_progressive(Context& ctx, const Field& field, AlgoConfig cfg) {
    cfg.variant = Variant::progressive;
    return extract(ctx, field, cfg);
}

inline ExtractionResult extract_brute_force(Context& ctx, const Field& field, AlgoConfig cfg) {
    cfg.variant = Variant::brute;
    return extract(ctx, field, cfg);
}

// compare_iou, localize.hpp:377-387
inline double compare_iou(const std::vector<std::uint8_t>& a, const std::vector<std::uint8_t>& b) {
    if (a.size() != b.size()) throw std::invalid_argument("compare_iou: dimension mismatch");
    double iou = 1.0;
    check(icg_compare_iou(nullptr, a.data(), b.data(), a.size(), ICG_MEM_HOST, &iou));
    return iou;
}

// acceleration_factor, localize.hpp:389-393
inline double acceleration_factor(const ExtractionResult& result, const ExtractionResult& brute) {
    if (result.total_evals == 0 || brute.total_evals == 0)
        throw std::invalid_argument("acceleration_factor: zero evaluation count");
    return static_cast<double>(brute.total_evals) / static_cast<double>(result.total_evals);
}

namespace detail {
inline RenderedImage to_image(const icg_image& im, int w, int h, const Vec3& bg, const std::vector<float>& rgb,
                              const std::vector<float>& depth, std::vector<std::uint8_t>&& mask,
                              std::vector<std::int32_t>&& sk) {
    RenderedImage r;
    r.width = w;
    r.height = h;
    r.background = bg;
    r.rgb.resize(static_cast<std::size_t>(w) * h);
    r.depth.resize(r.rgb.size());
    for (std::size_t i = 0; i < r.rgb.size(); ++i) {
        r.rgb[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
        r.depth[i] = depth[i];
    }
    r.mask = std::move(mask);
    r.surface_k = std::move(sk);
    r.oracle_calls = im.texture_points;
    r.degenerate_brackets = static_cast<int>(im.degenerate_brackets);
    r.grazing_pixels = static_cast<int>(im.grazing_pixels);
    return r;
}
}  // namespace detail

// North-star renderer: first crossing through the grid the last extract() on this context
// localized, texture at covered pixels (conventions of render.hpp:140-206, 244-280)
inline RenderedImage render_localized(Context& ctx, const Field& field, const CameraSpec& camera, int width,
                                      int height, const Vec3& background = {}) {
    const std::size_t npx = static_cast<std::size_t>(width) * static_cast<std::size_t>(height);
    std::vector<float> rgb(3 * npx), depth(npx);
    std::vector<std::uint8_t> mask(npx);
    std::vector<std::int32_t> sk(npx);
    icg_image im{};
    im.mem = ICG_MEM_HOST;
    im.rgb = rgb.data();
    im.depth = depth.data();
    im.mask = mask.data();
    im.surface_k = sk.data();
    const icg_camera cam = camera.to_c();
    const float bg[3] = {(float)background.x, (float)background.y, (float)background.z};
    check(icg_render_localized(ctx.get(), field.get(), &cam, width, height, bg, &im));
    return detail::to_image(im, width, height, background, rgb, depth, std::move(mask), std::move(sk));
}

// localize (progressive) + render through the localized grid in one call (icg_frame)
inline std::pair<ExtractionResult, RenderedImage> frame(Context& ctx, const Field& field, const AlgoConfig& cfg,
                                                        const CameraSpec& camera, int width, int height,
                                                        const Vec3& background = {}) {
    validate_config(cfg);
    const std::size_t n = static_cast<std::size_t>(cfg.target_cells() + 1);
    std::vector<float> values(n * n * n);
    std::vector<std::uint8_t> states(values.size()), bin(values.size());
    icg_extraction e{};
    e.mem = ICG_MEM_HOST;
    e.values = values.data();
    e.states = states.data();
    e.binarized = bin.data();
    const std::size_t npx = static_cast<std::size_t>(width) * static_cast<std::size_t>(height);
    std::vector<float> rgb(3 * npx), depth(npx);
    std::vector<std::uint8_t> mask(npx);
    std::vector<std::int32_t> sk(npx);
    icg_image im{};
    im.mem = ICG_MEM_HOST;
    im.rgb = rgb.data();
    im.depth = depth.data();
    im.mask = mask.data();
    im.surface_k = sk.data();
    const icg_algo_config c = cfg.to_c();
    const icg_camera cam = camera.to_c();
    const float bg[3] = {(float)background.x, (float)background.y, (float)background.z};
    check(icg_frame(ctx.get(), field.get(), &c, &cam, width, height, bg, &e, &im));
    return {detail::to_result(e, cfg, std::move(values), std::move(states), std::move(bin)),
            detail::to_image(im, width, height, background, rgb, depth, std::move(mask), std::move(sk))};
}

namespace detail {
inline RenderedImage view_render(Context& ctx, const Field& field, const CameraSpec& camera, const AlgoConfig& cfg,
                                 const Vec3& background, bool texture) {
    validate_config(cfg);
    const int n = cfg.target_cells() + 1;
    const std::size_t npx = static_cast<std::size_t>(n) * n;
    std::vector<float> rgb(3 * npx), depth(npx);
    std::vector<std::uint8_t> mask(npx);
    std::vector<std::int32_t> sk(npx);
    icg_image im{};
    im.mem = ICG_MEM_HOST;
    im.rgb = rgb.data();
    im.depth = depth.data();
    im.mask = mask.data();
    im.surface_k = sk.data();
    const icg_algo_config c = cfg.to_c();
    const icg_camera cam = camera.to_c();
    const float bg[3] = {(float)background.x, (float)background.y, (float)background.z};
    if (texture)
        check(icg_render_view(ctx.get(), field.get(), &cam, &c, bg, &im));
    else
        check(icg_surface_depth_map(ctx.get(), field.get(), &cam, &c, &im));
    RenderedImage r = to_image(im, n, n, background, rgb, depth, std::move(mask), std::move(sk));
    r.oracle_calls = im.oracle_calls;
    return r;
}
}  // namespace detail

// render_view(oracle, camera, cfg, background, workers), render.hpp:244-280: view-space
// localization, shadow culling, (R_L+1)^2 pixels; oracle_calls = occupancy evaluations
inline RenderedImage render_view(Context& ctx, const Field& field, const CameraSpec& camera, const AlgoConfig& cfg,
                                 const Vec3& background = {}) {
    return detail::view_render(ctx, field, camera, cfg, background, true);
}

// surface_depth_map(oracle, camera, cfg, workers), render.hpp:219-240 (rgb = background)
inline RenderedImage surface_depth_map(Context& ctx, const Field& field, const CameraSpec& camera,
                                       const AlgoConfig& cfg) {
    return detail::view_render(ctx, field, camera, cfg, {}, false);
}

struct TriangleMesh {  // mesh.hpp:22-27
    std::vector<Vec3> vertices;
    std::vector<std::array<int, 3>> triangles;
    bool empty() const { return triangles.empty(); }
};

// marching_cubes(grid, iso), mesh.hpp:75-156, on the GPU (generated triangulation: the vertex set
// is the reference's, the triangles of a cube may differ); grid = the result of extract()
inline TriangleMesh marching_cubes(Context& ctx, const LevelGrid& grid, double iso = 0.5) {
    icg_mesh m{};
    int rc = icg_marching_cubes(ctx.get(), grid.values.data(), grid.cells, ICG_MEM_HOST, iso, &m);
    if (rc != ICG_ECAPACITY) check(rc);
    std::vector<double> v(3 * m.n_vertices);
    std::vector<std::int32_t> t(3 * m.n_triangles);
    m.vertices = v.data();
    m.vertex_capacity = m.n_vertices;
    m.triangles = t.data();
    m.triangle_capacity = m.n_triangles;
    check(icg_marching_cubes(ctx.get(), grid.values.data(), grid.cells, ICG_MEM_HOST, iso, &m));
    TriangleMesh out;
    for (std::uint64_t i = 0; i < m.n_vertices; ++i) out.vertices.push_back({v[3 * i], v[3 * i + 1], v[3 * i + 2]});
    for (std::uint64_t i = 0; i < m.n_triangles; ++i) out.triangles.push_back({t[3 * i], t[3 * i + 1], t[3 * i + 2]});
    return out;
}

// export_obj, mesh.hpp:159-172
inline void export_obj(const TriangleMesh& mesh, const std::string& path) {
    std::vector<double> v;
    std::vector<std::int32_t> t;
    for (const Vec3& p : mesh.vertices) v.insert(v.end(), {p.x, p.y, p.z});
    for (const auto& tr : mesh.triangles) t.insert(t.end(), {tr[0], tr[1], tr[2]});
    check(icg_write_obj(path.c_str(), v.data(), mesh.vertices.size(), t.data(), mesh.triangles.size()));
}

// composite, render.hpp:284-291
inline std::vector<Vec3> composite(const RenderedImage& image, const std::vector<Vec3>& backdrop) {
    if (backdrop.size() != image.rgb.size()) throw std::invalid_argument("composite: dimension mismatch");
    std::vector<Vec3> out(backdrop);
    for (std::size_t i = 0; i < out.size(); ++i)
        if (image.mask[i]) out[i] = image.rgb[i];
    return out;
}

}  // namespace isocull_b200

#endif  // ISOCULL_B200_HPP

/*
 * isocull_b200.h — C ABI of the B200-native accelerated PIFu inference path.
 *
 * This is the drop-in boundary for the reference's hot path.
 * The reference (/root/reference/proj/include/isocull) is a header-only C++20
 * library; its operators take a `FieldOracle` (std::function plugin) and return
 * results by value.  A std::function cannot run on a GPU, so the field is
 * described here by data (primitives, feature map, MLP weights) and the
 * operators run as hand-written sm_100a kernels behind these entry points.
 *
 * Every entry point below names the reference interface it replaces.
 * Conventions that hold for all of them:
 *   - plain pointers and sizes only; no C++ or torch types cross the ABI;
 *   - errors never throw: each call returns an ICG_* status and leaves a
 *     thread-local message readable through icg_last_error();
 *   - ICG_EINVAL  ≙ std::invalid_argument (reference CLI exit code 2,
 *                   tools/isocull_cli.cpp:358-364),
 *     ICG_ERUNTIME ≙ std::runtime_error   (reference CLI exit code 1);
 *   - calls are synchronous with respect to the host, like the reference
 *     operators (results are complete when the call returns);
 *   - one host thread drives one context at a time; distinct contexts (one per
 *     GPU) may be driven concurrently (reference operators are re-entrant).
 */
#ifndef ISOCULL_B200_H
#define ISOCULL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ICG_ABI_VERSION 4

/* ---- status codes ------------------------------------------------------ */
#define ICG_OK 0
#define ICG_ERUNTIME 1 /* runtime_error: CUDA failure, I/O (isocull_cli.cpp:362-364) */
#define ICG_EINVAL 2   /* invalid_argument: bad config / field (isocull_cli.cpp:358-361) */
#define ICG_ECAPACITY 3 /* a device work list overflowed its capacity */
#define ICG_ENODEV 4   /* no CUDA device / extension unusable */

/* ---- limits ------------------------------------------------------------ */
#define ICG_MAX_LEVELS 16      /* AlgoConfig target_level bound (cells <= 1024, localize.hpp:50) */
#define ICG_MAX_PRIMS 64
#define ICG_MAX_TARGET_CELLS 1024 /* validate_config, localize.hpp:50-51 */

/* ---- memory locations for caller-provided buffers ----------------------- */
#define ICG_MEM_HOST 0
#define ICG_MEM_DEVICE 1

/* ---- node states: NodeState, grid.hpp:15 -------------------------------- */
#define ICG_STATE_UNKNOWN 0
#define ICG_STATE_INTERPOLATED 1
#define ICG_STATE_EVALUATED 2
#define ICG_STATE_SHADOW 3

/* ---- analytic scene: SceneSpec / Primitive, scene.hpp:27-103 ------------ */
#define ICG_PRIM_SPHERE 0
#define ICG_PRIM_BOX 1
#define ICG_PRIM_CAPSULE 2
#define ICG_PRIM_TORUS 3

typedef struct icg_primitive {
    int32_t kind;             /* ICG_PRIM_* (PrimitiveKind, scene.hpp:25) */
    int32_t rotated;          /* nonzero: apply inv_rotation to (p - center) */
    double center[3];         /* sphere / box / torus */
    double a[3], b[3];        /* capsule segment endpoints, world coordinates */
    double radius;            /* sphere / capsule */
    double half[3];           /* box half extents */
    double major, minor;      /* torus radii (ring in the local xz plane) */
    double inv_rotation[9];   /* row-major world->local (Primitive::inv_rotation) */
} icg_primitive;

/* TextureRule (scene.hpp:48-55, texture_color :105-127): the analytic field's T(P) */
#define ICG_TEXTURE_NONE 0
#define ICG_TEXTURE_CONSTANT 1      /* color */
#define ICG_TEXTURE_GRADIENT 2      /* lerp(from, to, (P[axis] + 1) / 2) */
#define ICG_TEXTURE_PER_PRIMITIVE 3 /* colors[nearest primitive] (first minimum) */

typedef struct icg_texture_rule {
    int32_t kind;              /* ICG_TEXTURE_* */
    int32_t axis;              /* gradient: 0 = x, 1 = y, 2 = z */
    double color[3];
    double from[3], to[3];
    const double* colors;      /* per primitive: n_prims x 3 (host memory) */
} icg_texture_rule;

/* Union-only CSG of primitives (the default tree of parse_scene,
 * scene.hpp:308-317; every bundled scene and the config-0 capsule figure use
 * it).  signed_distance = min over primitives (scene.hpp:130-146). */
typedef struct icg_scene {
    const icg_primitive* prims;
    int32_t n_prims;
    double tau; /* occupancy_from_distance(d, tau) = 1/(1+exp(d/tau)), field.hpp:81 */
    icg_texture_rule texture;  /* analytic field: T(P) for render_view / texture_batch */
} icg_scene;

/* ---- camera: CameraSpec, render.hpp:19-46 -------------------------------- */
typedef struct icg_camera {
    double rotation[9];        /* row-major world->view */
    double translation[3];
    double scale;              /* weak-perspective x,y scale; 1 = orthographic */
} icg_camera;

/* ---- field descriptor: replaces FieldOracle (field.hpp:22-77) ------------ */
#define ICG_FIELD_ANALYTIC 0 /* O(P) = 1/(1+exp(sdf(P)/tau)) on device (config 0) */
#define ICG_FIELD_PIFU 1     /* O(P) = sigmoid(f_O(Phi(P_xy), P_z) - sdf_scale*sdf(P)) (configs 1-4) */

#define ICG_PREC_FP32 0      /* tcgen05 bf16x3 split products, fp32 accumulation (configs 1, 2, 4) */
#define ICG_PREC_BF16 1      /* tcgen05 bf16 operands, fp32 accumulation (config 3) */
#define ICG_PREC_FP32_SIMT 2 /* CUDA-core fp32 FFMA path (correctness cross-check) */

typedef struct icg_field {
    int32_t kind;              /* ICG_FIELD_* */
    icg_scene scene;           /* analytic field, or the capsule figure biasing the PIFu logit */
    double sdf_scale;          /* PIFu: logit += -sdf_scale * sdf(P)   (50 in BASELINE configs 1-4) */
    const float* feature_map;  /* PIFu: C x H x W fp32, channel-major (g_O(I)) */
    int32_t fmap_c, fmap_h, fmap_w;
    int32_t fmap_mem;          /* ICG_MEM_HOST (copied H2D inside the call) or ICG_MEM_DEVICE */
    int32_t precision;         /* ICG_PREC_* */
    /* PIFu input view: Phi is sampled at q.xy and the depth feature is q.z,
     * q = input_camera.world_to_view(P) = (s (R P + t).x, s (R P + t).y, (R P + t).z)
     * (CameraSpec, render.hpp:19-46).  0 = orthographic identity (q = P, BASELINE configs 1-4;
     * the column-factored fast path applies); otherwise every node takes the per-point path. */
    int32_t has_input_camera;
    icg_camera input_camera;
} icg_field;

/* ---- MLP weights (f_O / f_T; not in the reference) */
#define ICG_MLP_GEOMETRY 0 /* 257->1024->512->256->128->1, skip-concat of the 257-d input */
#define ICG_MLP_TEXTURE 1  /* 513->1024->512->256->128->3, skip-concat of the 513-d input */
#define ICG_MLP_LAYERS 5

/* weights[l]: fp32 row-major [out_dims[l]][in_dims[l]] where in_dims[l] =
 * (l==0 ? 0 : out_dims[l-1]) + skip_dim; the previous layer's activations come
 * first, the skip input last.  biases[l]: fp32 [out_dims[l]].  Host memory. */
typedef struct icg_mlp_desc {
    int32_t which;             /* ICG_MLP_* */
    int32_t n_layers;          /* must be ICG_MLP_LAYERS */
    int32_t skip_dim;          /* 257 (geometry) or 513 (texture) */
    int32_t out_dims[ICG_MLP_LAYERS];
    const float* weights[ICG_MLP_LAYERS];
    const float* biases[ICG_MLP_LAYERS];
    float leaky_slope;         /* 0.02 */
} icg_mlp_desc;

/* ---- algorithm config: AlgoConfig, localize.hpp:36-45 -------------------- */
#define ICG_VARIANT_BRUTE 0
#define ICG_VARIANT_OCTREE_BINARIZED 1 /* extract_octree_binarized, localize.hpp:199-260 (Fig. 4 baseline) */
#define ICG_VARIANT_OCTREE_THRESHOLD 2 /* extract_octree_threshold, localize.hpp:265-306 (Fig. 4 baseline) */
#define ICG_VARIANT_PROGRESSIVE 3 /* Variant enum order, localize.hpp:16 */

typedef struct icg_algo_config {
    int32_t variant;           /* ICG_VARIANT_* */
    int32_t coarsest_cells;    /* R_0 (>= 2) */
    int32_t target_level;      /* L; R_L = R_0 * 2^L <= 1024 */
    int32_t max_conflict_iters;/* 0 = one axis length per level (localize.hpp:339) */
    int32_t conflict_pass;     /* 0 = ablation (localize.hpp:42, 335-336) */
    int32_t keep_level_sets;   /* nonzero: keep every level's refined-cell and evaluated-node sets
                                  on the context for icg_level_set (one extra bitset pass per level) */
    double threshold;          /* octree_threshold only, in (0, 0.5) (AlgoConfig::threshold) */
} icg_algo_config;

/* ---- extraction result: ExtractionResult, localize.hpp:57-64 ------------- */
typedef struct icg_extraction {
    /* caller-provided output buffers; NULL = not requested.  All (R_L+1)^3,
     * x-fastest (grid.hpp:45-48). */
    int32_t mem;               /* ICG_MEM_HOST or ICG_MEM_DEVICE for the arrays below */
    float* values;             /* LevelGrid::values at level L */
    uint8_t* states;           /* LevelGrid::states (ICG_STATE_*) */
    uint8_t* binarized;        /* value >= 0.5f (binarized_volume, localize.hpp:154-158) */
    /* always filled (host scalars) */
    int32_t cells;             /* R_L */
    int32_t levels;            /* L + 1 */
    uint64_t evals_per_level[ICG_MAX_LEVELS];
    uint64_t total_evals;
    uint64_t refined_cells_per_level[ICG_MAX_LEVELS]; /* coarse cells of level l-1 whose 8 binarized corners disagree */
    uint32_t conflict_iters_per_level[ICG_MAX_LEVELS];
    int32_t conflict_warning;  /* conflict pass hit its bound (localize.hpp:343-346) */
    double wall_seconds;       /* device time of the whole extraction */
} icg_extraction;

/* ---- rendered image: RenderedImage, render.hpp:50-59 --------------------- */
typedef struct icg_image {
    int32_t mem;               /* ICG_MEM_HOST or ICG_MEM_DEVICE for the arrays below */
    float* depth;              /* W*H view z; -2 where uncovered (render.hpp:72) */
    float* rgb;                /* W*H*3, clamp01(T(P)) or background */
    uint8_t* mask;             /* W*H coverage */
    int32_t* surface_k;        /* W*H first-crossing sample index, -1 where uncovered */
    /* always filled */
    uint64_t covered_pixels;
    uint64_t degenerate_brackets; /* equal-occupancy brackets clamped to the occupied sample */
    uint64_t grazing_pixels;      /* fractional samples that never reach 0.5 */
    uint64_t texture_points;      /* texture-MLP evaluations (= covered pixels) */
    double wall_seconds;
    uint64_t oracle_calls;        /* icg_render_view / icg_surface_depth_map: occupancy evaluations of
                                     the depth pass (RenderedImage::oracle_calls, render.hpp:55) */
} icg_image;

/* ======================================================================== */
/* Context lifecycle                                                         */
/* ======================================================================== */
typedef struct icg_context icg_context;

int icg_abi_version(void);
const char* icg_last_error(void);
int icg_device_count(int* count);
int icg_create(int device, icg_context** out);
int icg_destroy(icg_context* ctx);

/* Weight upload (library-owned device copies; packed for tcgen05 and SIMT). */
int icg_set_mlp(icg_context* ctx, const icg_mlp_desc* desc);

/* ======================================================================== */
/* Operators                                                                 */
/* ======================================================================== */

/* extract(oracle, cfg, workers) -> ExtractionResult (localize.hpp:365-373):
 * progressive localization (extract_progressive, localize.hpp:315-363) or
 * dense brute force (extract_brute_force, localize.hpp:181-193).  The final
 * grid also stays resident in the context for icg_render_localized. */
int icg_extract(icg_context* ctx, const icg_field* field, const icg_algo_config* cfg,
                icg_extraction* out);

/* Per-level sets of the last extraction / frame on this context that ran with
 * cfg.keep_level_sets (the reference keeps them
 * implicitly: the `to_eval` / conflict-neighbour lists of localize.hpp:331-353
 * and the cells binarize+upsample refine, grid.hpp:133-140):
 *   ICG_SET_EVALUATED_NODES: node indices i + n(j + n k) of the level-l grid
 *     (n = R_l + 1) whose occupancy was evaluated at level l (level 0: every
 *     node; the E0 list and every conflict-loop batch of localize.hpp:331-353);
 *   ICG_SET_REFINED_CELLS: level l >= 1: cell indices ci + Rc(cj + Rc ck) of
 *     the level-(l-1) grid (Rc = R_{l-1}) whose 8 binarized corners disagree
 *     (the cells the level refines); level 0: empty.
 * Sets are returned as ascending u32 lists.  *count is always set; out may be
 * NULL (count only); capacity < count returns ICG_ECAPACITY. */
#define ICG_SET_EVALUATED_NODES 0
#define ICG_SET_REFINED_CELLS 1
int icg_level_set(icg_context* ctx, int level, int which, int mem, uint32_t* out, size_t capacity,
                  size_t* count);

/* Mesh-free render through the grid localized by the last icg_extract on this
 * context (north-star renderer, following the
 * argmax/bracket/depth conventions of render.hpp:140-206 and the texture
 * lookup of render_view, render.hpp:244-280).  background: 3 floats. */
int icg_render_localized(icg_context* ctx, const icg_field* field, const icg_camera* camera,
                         int width, int height, const float* background, icg_image* out);

/* render_view(oracle, camera, cfg, background, workers) -> RenderedImage (render.hpp:244-280):
 * the reference's own mesh-free renderer.  The field is evaluated in view space
 * (O(camera.view_to_world(p)), render.hpp:98-99): progressive localization to level L-1
 * (cfg: progressive, target_level >= 1), then at level L shadow culling behind columns whose
 * tentative maximum is 1, evaluation of the surviving fractional candidates and of the bracket
 * nodes, and per-pixel depth 1 - 2 (k1 - 1 + s) / R (render.hpp:105-206); covered pixels take the
 * texture at their surface point (clamp01), the rest the background.  The image is square,
 * width = height = R_L + 1 (one pixel per grid column; row 0 = view y +1); the caller's buffers
 * hold (R_L+1)^2 pixels.  Field: analytic with a texture rule, or PIFu with texture weights
 * (else ICG_EINVAL, "render_view: scene has no texture"). */
int icg_render_view(icg_context* ctx, const icg_field* field, const icg_camera* camera,
                    const icg_algo_config* cfg, const float* background, icg_image* out);

/* surface_depth_map(oracle, camera, cfg, workers) -> DepthMap (render.hpp:219-240): the same
 * depth pass without texture; out->depth / mask / surface_k filled, out->rgb ignored. */
int icg_surface_depth_map(icg_context* ctx, const icg_field* field, const icg_camera* camera,
                          const icg_algo_config* cfg, icg_image* out);

/* One frame = icg_extract + icg_render_localized in a single call
 * (BASELINE configs 2-4).  Either output may be NULL. */
int icg_frame(icg_context* ctx, const icg_field* field, const icg_algo_config* cfg,
              const icg_camera* camera, int width, int height, const float* background,
              icg_extraction* ext_out, icg_image* img_out);

/* Direct field evaluation: FieldOracle::occupancy_batch (field.hpp:41-47) and
 * texture_batch (field.hpp:56-63).  points: n x 3 doubles (NDC).  Outputs are
 * host or device per `mem`; occupancy as fp32 (the value the grid stores,
 * localize.hpp:86), rgb as fp32 n x 3 (unclamped sigmoid output). */
int icg_occupancy_batch(icg_context* ctx, const icg_field* field, const double* points,
                        size_t n, int mem, float* out);
int icg_texture_batch(icg_context* ctx, const icg_field* field, const double* points,
                      size_t n, int mem, float* out_rgb);

/* composite (render.hpp:284-291): out[i] = mask[i] ? image_rgb[i] : backdrop[i], 3 floats per
 * pixel; n_image != n_backdrop -> ICG_EINVAL ("composite: dimension mismatch").  Host arrays;
 * out may alias backdrop. */
int icg_composite(const float* image_rgb, const uint8_t* mask, size_t n_image, const float* backdrop,
                  size_t n_backdrop, float* out);

/* marching_cubes(grid, iso) -> TriangleMesh (mesh.hpp:75-156) on the GPU: crossed edges, vertex
 * interpolation, welding of bit-identical positions, degenerate-triangle removal and first-use
 * vertex order as the reference; the triangulation of each cube case is generated (face-walk,
 * see csrc/k_mc.cu), not the reference's Bourke table, so triangles may differ while the vertex
 * set and the surface agree.  values: (cells+1)^3 fp32 (host or device per `mem`), or NULL for
 * the grid the last extraction / frame on this context localized (cells ignored).  Outputs are
 * host arrays; *_capacity too small -> ICG_ECAPACITY with n_vertices / n_triangles set (call
 * again with room).  cells <= 1023. */
typedef struct icg_mesh {
    double* vertices;          /* n_vertices x 3 */
    uint64_t vertex_capacity;
    int32_t* triangles;        /* n_triangles x 3, 0-based vertex indices */
    uint64_t triangle_capacity;
    uint64_t n_vertices, n_triangles;
} icg_mesh;
int icg_marching_cubes(icg_context* ctx, const float* values, int cells, int mem, double iso, icg_mesh* out);

/* The generated triangulation of one cube case (bit c set: Bourke corner c below iso): up to 5
 * triangles as edge indices (Bourke edge numbering, mesh.hpp:42-46), -1 terminated.  Host only. */
int icg_mc_case(int case_bits, int8_t* edges16, int* n_triangles);

/* export_obj (mesh.hpp:159-172): "# isocull mesh: ..." header, "v %.9f %.9f %.9f", 1-based "f a b c". */
int icg_write_obj(const char* path, const double* vertices, uint64_t n_vertices, const int32_t* triangles,
                  uint64_t n_triangles);

/* compare_iou (localize.hpp:377-387) on device or host arrays of n bytes. */
int icg_compare_iou(icg_context* ctx, const uint8_t* a, const uint8_t* b, size_t n, int mem,
                    double* iou);

/* ======================================================================== */
/* Instrumentation (CUDA events on the context stream around every kernel    */
/* class; counters accumulate until icg_profile_reset).                      */
/* ======================================================================== */
typedef struct icg_profile {
    uint64_t kernel_launches;      /* all library kernel launches (incl. early-exit ones) */
    uint64_t geo_mlp_launches;     /* geometry-field evaluation launches */
    uint64_t geo_points;           /* points evaluated by them */
    double geo_mlp_ms;             /* summed device time of those launches */
    uint64_t tex_mlp_launches;
    uint64_t tex_points;
    double tex_mlp_ms;
    uint64_t dense_launches;       /* per-level dense passes + compaction (conflict expansion: ABI 4, below) */
    double dense_ms;
    uint64_t dense_bytes;          /* algorithmic bytes of the dense passes */
    uint64_t render_launches;
    double render_ms;
    uint64_t render_bytes;
    double frame_ms;               /* summed device time of whole frames / extractions */
    uint64_t frames;
    /* breakdown of the geometry launches above (column-factored PIFu field):  */
    uint64_t fact_launches;        /* bulk batches (dense L0 + each level's E0): column pass + factored pass */
    uint64_t fact_points;
    double fact_ms;
    uint64_t chain_launches;       /* conflict-loop batches (CTA-pair kernels + persistent tail) */
    uint64_t chain_points;
    double chain_ms;
    /* the texture field's Phi gather (bilinear taps of the H x W x C map at the surface points;
       part of tex_mlp_ms above): algorithmic bytes = 4 taps x C x 4 B per point (ABI 3) */
    uint64_t gather_launches;
    uint64_t gather_points;
    double gather_ms;
    uint64_t gather_bytes;
    /* ABI 4: the conflict loop's neighbour expansions (k_conflict_expand; counted in dense_* before
       ABI 4), and the target level's dense pass alone (also in dense_*): binarize + mixed cells +
       upsample / carry / candidates + E0 compaction at full size, its SURVEY §8(d) bytes */
    uint64_t expand_launches;
    double expand_ms;
    uint64_t last_level_launches;
    double last_level_ms;
    uint64_t last_level_bytes;
} icg_profile;

int icg_profile_enable(icg_context* ctx, int on);
int icg_profile_reset(icg_context* ctx);
int icg_profile_get(icg_context* ctx, icg_profile* out);

/* Device-timed span over n contexts of ONE device (several frames in flight,
 * one host thread per context).  icg_span_begin records a start event on
 * ctxs[0]'s stream and makes every context's stream wait for it;
 * icg_span_end records an end event on every stream, waits, and returns the
 * milliseconds from the start event to the last stream's end event. */
int icg_span_begin(icg_context* const* ctxs, int n);
int icg_span_end(icg_context* const* ctxs, int n, float* ms);

/* ======================================================================== */
/* Host helpers                                                              */
/* ======================================================================== */

/* Pinned host buffers for end-to-end (host-buffer) calls. */
int icg_host_alloc(size_t bytes, void** ptr);
int icg_host_free(void* ptr);
int icg_device_alloc(icg_context* ctx, size_t bytes, void** ptr);
int icg_device_free(icg_context* ctx, void* ptr);
int icg_memcpy(icg_context* ctx, void* dst, const void* src, size_t bytes, int dst_mem, int src_mem);
/* bytes of device memory set to `value` on the context's stream (returns when done; e.g. an L2 flush) */
int icg_memset(icg_context* ctx, void* dst, int value, size_t bytes);

/* Seeded synthetic inputs; Rng = mt19937_64 with the
 * reference's hand-rolled uniform / Box-Muller (random.hpp:16-43). */
/* 15-capsule stick figure: per capsule a.xyz, b.xyz ~ U[-0.5,0.5], r ~ U[0.03,0.08]. */
int icg_gen_capsules(uint64_t seed, int n, icg_primitive* out);
/* n standard normals in generation order. */
int icg_gen_normals(uint64_t seed, size_t n, float* out);
/* Kaiming-uniform MLP: per layer W ~ U(-g*sqrt(3/fan_in), +), g = sqrt(2/(1+slope^2)),
 * then b ~ U(-1/sqrt(fan_in), +).  weights_out / biases_out hold room for
 * sum(out*in) / sum(out) floats; layer l starts where l-1 ends. */
int icg_gen_mlp(uint64_t seed, int which, float* weights_out, float* biases_out);
/* Sizes for icg_gen_mlp and icg_set_mlp: fills out_dims/in_dims and totals. */
int icg_mlp_shape(int which, int32_t* out_dims, int32_t* in_dims, int32_t* skip_dim,
                  size_t* n_weights, size_t* n_biases);

/* On-device feature producer (the encoder stand-in of a frame stream): n = c*h*w seeded N(0,1)
 * values written to device (mem = ICG_MEM_DEVICE) or host memory, generated on the context's
 * GPU.  Counter-based (Philox4x32-10 + the reference's Box-Muller form, random.hpp:32-37): a
 * different stream from icg_gen_normals' host Rng. */
int icg_gen_feature_map_device(icg_context* ctx, uint64_t seed, int c, int h, int w, int mem, float* out);

/* Stream I/O, byte-identical to the reference writers: write_ppm (image.hpp:18-33, rgb w*h*3),
 * write_float_map (image.hpp:37-48), dump_grid / load_grid_dump (grid.hpp:199-222; values may be
 * NULL to read the header only).  Host buffers. */
int icg_write_ppm(const char* path, int width, int height, const float* rgb);
int icg_write_float_map(const char* path, int width, int height, const float* values);
int icg_dump_grid(const char* path, int level, int cells, const float* values);
int icg_load_grid_dump(const char* path, int* level, int* cells, float* values, size_t capacity);

/* Camera from angles, CameraSpec::from_angles (render.hpp:36-45). */
int icg_camera_from_angles(double yaw_deg, double pitch_deg, double dist, double scale,
                           icg_camera* out);

#ifdef __cplusplus
}
#endif
#endif /* ISOCULL_B200_H */

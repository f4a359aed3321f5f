/*
 * isocull_oracle.h — CPU ORACLE: TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C (fp64 / IEEE fp32, no FMA contraction) restatement of the
 * reference's hot path, used as the checker for the CUDA product.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product (paper_2007_13988_b200) never
 * links, imports or calls anything here.
 *
 * What is restated, and from where (file:line into /root/reference/proj):
 *   - Rng: mt19937_64 + uniform/normal ............ include/isocull/random.hpp:16-43
 *   - analytic SDFs, union, occupancy ............. include/isocull/scene.hpp:60-103,130-146,
 *                                                     include/isocull/field.hpp:81
 *   - progressive localization .................... include/isocull/localize.hpp:76-177,315-363
 *   - brute force, compare_iou .................... include/isocull/localize.hpp:181-193,377-387
 *   - first-crossing depth / bracket / texture .... include/isocull/render.hpp:140-206,244-280
 *     applied to the world grid along camera rays
 *   - PIFu field (feature sampler Phi, f_O, f_T): NOT in the reference
 *     ("deliberately unhoused"); restated from BASELINE.json
 *     configs[1-3] and PAPER.md:157-177,468.  Parity for this part is pinned
 *     only by this restatement and its golden fixtures (tests/golden/).
 *
 * Pins: the localization / grid / Rng restatement is checked against the
 * reference itself, compiled from /root/reference by oracle/Makefile into
 * oracle/_ref/libisocull_ref.so (tests/test_oracle_vs_reference.py), and
 * against the SPEC known-answer examples (tests/test_oracle_kat.py).
 */
#ifndef ISOCULL_ORACLE_H
#define ISOCULL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/isocull_b200.h" /* plain struct layouts only (icg_primitive, icg_camera) */

#ifdef __cplusplus
extern "C" {
#endif

/* ---- Rng (random.hpp:16-43) -------------------------------------------- */
typedef struct orc_rng {
    uint64_t mt[312];
    int idx;
} orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_raw(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_normal(orc_rng* r);
void orc_rng_uniforms(uint64_t seed, size_t n, double* out);
void orc_rng_normals(uint64_t seed, size_t n, double* out);

/* ---- analytic field (scene.hpp / field.hpp) ---------------------------- */
double orc_scene_sdf(const icg_primitive* prims, int n, const double p[3]);
double orc_occupancy_from_distance(double d, double tau);
void orc_analytic_occupancy_batch(const icg_primitive* prims, int n, double tau,
                                  const double* pts, size_t npts, double* out, int threads);

/* ---- PIFu field (restated; no reference) ------------------------------- */
typedef struct orc_mlp {
    int n_layers;          /* 5 */
    int skip_dim;          /* 257 / 513 */
    int out_dims[5];
    int in_dims[5];
    const float* w[5];     /* [out][in], in = prev_out + skip */
    const float* b[5];
    double slope;          /* 0.02 */
} orc_mlp;

typedef struct orc_pifu {
    const float* fmap;     /* C x H x W fp32 */
    int C, H, W;
    const icg_primitive* prims;
    int n_prims;
    double sdf_scale;      /* 50 */
    orc_mlp geo;
    orc_mlp tex;
    int has_texture;
    /* input view (icg_field.input_camera): Phi at q.xy, depth feature q.z with
     * q = world_to_view(P) (render.hpp:23-26); has_cam = 0: q = P */
    int has_cam;
    double cam_rot[9], cam_t[3], cam_scale;
} orc_pifu;

/* Phi: bilinear sample of all C channels at P_xy (align corners,
 * u=(x+1)/2*(W-1), v=(1-y)/2*(H-1)); out[C]. */
void orc_sample_features(const orc_pifu* m, const double p[3], double* out);
/* occupancy O(P) for n points; optional h3_out (n x 256) = geometry layer-3 activations. */
void orc_pifu_occupancy_batch(const orc_pifu* m, const double* pts, size_t n, double* out,
                              int threads);
/* geometry logit before the sigmoid (MLP output + bias - sdf_scale*sdf) */
void orc_pifu_logit_batch(const orc_pifu* m, const double* pts, size_t n, double* out,
                          int threads);
void orc_pifu_texture_batch(const orc_pifu* m, const double* pts, size_t n, double* rgb,
                            int threads);

/* ---- generic field callback (FieldOracle surrogate, field.hpp:22-77) ---- */
typedef void (*orc_occ_batch_fn)(void* user, const double* pts, size_t n, double* out);
typedef void (*orc_tex_batch_fn)(void* user, const double* pts, size_t n, double* rgb);
/* ready-made callbacks; user = orc_pifu* / orc_analytic* */
typedef struct orc_analytic {
    const icg_primitive* prims;
    int n_prims;
    double tau;
    int threads;
} orc_analytic;
void orc_cb_analytic(void* user, const double* pts, size_t n, double* out);
typedef struct orc_pifu_cb {
    const orc_pifu* model;
    int threads;
} orc_pifu_cb;
void orc_cb_pifu_occ(void* user, const double* pts, size_t n, double* out);
void orc_cb_pifu_tex(void* user, const double* pts, size_t n, double* rgb);
/* single-point adapters in the FieldOracle shape (double(const Vec3&)) used
 * by the reference shim: user = orc_analytic* / orc_pifu_cb* */
double orc_pt_analytic(void* user, const double* p);
double orc_pt_pifu_occ(void* user, const double* p);
void orc_pt_pifu_tex(void* user, const double* p, double* rgb);
/* replay oracle: looks up fp32 values of a finest-level grid by position;
 * counts misses (positions that were never evaluated there). */
typedef struct orc_replay {
    const float* values;
    const uint8_t* states;
    int cells;             /* finest R */
    uint64_t misses;       /* incremented (atomically) when a looked-up node is not evaluated */
    uint64_t calls;
} orc_replay;
void orc_cb_replay(void* user, const double* pts, size_t n, double* out);
double orc_pt_replay(void* user, const double* p);

/* ---- localization (localize.hpp) --------------------------------------- */
typedef struct orc_extract_out {
    float* values;                 /* (R_L+1)^3, caller-allocated */
    uint8_t* states;
    uint8_t* binarized;            /* optional */
    uint64_t evals_per_level[16];
    uint64_t total_evals;
    uint64_t refined_cells_per_level[16];
    uint32_t conflict_iters_per_level[16];
    int conflict_warning;
    double wall_seconds;
    /* optional per-level sets (NULL = not requested):
     * eval_level: (R_L+1)^3 bytes over the FINAL grid; the level at which the node at that
     *   position was evaluated (each physical node is evaluated at most once), 0xFF = never;
     * refined_cells[l], l >= 1: R_{l-1}^3 bytes over the level-(l-1) cells, 1 = the cell's 8
     *   binarized corners disagree (the cells level l refines). */
    uint8_t* eval_level;
    uint8_t* refined_cells[16];
} orc_extract_out;

int orc_extract_progressive(orc_occ_batch_fn occ, void* user, int coarsest_cells,
                            int target_level, int max_conflict_iters, int conflict_pass,
                            orc_extract_out* out);
int orc_extract_brute(orc_occ_batch_fn occ, void* user, int coarsest_cells, int target_level,
                      orc_extract_out* out);
double orc_compare_iou(const uint8_t* a, const uint8_t* b, size_t n);

/* grid primitives (grid.hpp:87-197), exposed for known-answer tests */
void orc_upsample_interpolate(int coarse_cells, const float* cv, const uint8_t* cs, float* fv,
                              uint8_t* fs);
void orc_dilate_1ring(int nodes, const uint8_t* mask, uint8_t* out);
void orc_argmax_z(int nodes, const float* values, float* max_value, int* max_index);

/* ---- render (row 19b) -------------------------------------------------- */
typedef struct orc_render_out {
    float* depth;      /* W*H */
    float* rgb;        /* W*H*3 */
    uint8_t* mask;     /* W*H */
    int32_t* surface_k;/* W*H */
    double* surface_pts; /* optional: W*H*3 world points of covered pixels (others untouched) */
    uint64_t covered, degenerate, grazing;
} orc_render_out;

/* First-crossing render through a localized world grid (values, R cells).
 * tex may be NULL (depth only; rgb = background at covered pixels too). */
int orc_render_first_crossing(const float* values, int cells, const icg_camera* cam, int width,
                              int height, const float* background, orc_tex_batch_fn tex,
                              void* tex_user, orc_render_out* out);

/* CameraSpec::from_angles (render.hpp:36-45) */
void orc_camera_from_angles(double yaw_deg, double pitch_deg, double dist, double scale,
                            icg_camera* out);

/* The product's on-device feature producer (icg_gen_feature_map_device) restated: element e =
 * Philox4x32-10 at counter (e, 0, 0, 0), key (seed lo, hi); 53-bit uniforms a, b from words
 * (0, 1) and (2, 3); sqrt(-2 ln a) cos(2 pi b) (random.hpp:32-37) rounded to float. */
void orc_feature_normals(uint64_t seed, size_t n, float* out);

/* ---- seeded inputs (same draw order as the product's icg_gen_*) --------- */
void orc_gen_capsules(uint64_t seed, int n, icg_primitive* out);
void orc_gen_mlp(uint64_t seed, int which, float* w, float* b);

#ifdef __cplusplus
}
#endif
#endif

// icg_internal.h — shared declarations of the B200 product library
// (host runtime in icg_host.cu, kernels in k_*.cu).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>

#include "../../include/isocull_b200.h"

namespace icg {

// Once-per-device initialisation (cudaFuncSetAttribute and friends are per device, and several
// host threads may drive contexts on several devices at once): `run(f)` calls f() the first time
// it is reached on the current device, under a lock; a failure is not recorded as done.
struct PerDeviceOnce {
    std::atomic<unsigned long long> done{0};
    std::mutex m;
    template <class F>
    int run(F&& f) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return ICG_ERUNTIME;
        const unsigned long long bit = 1ull << (dev & 63);
        if (done.load(std::memory_order_acquire) & bit) return ICG_OK;
        std::lock_guard<std::mutex> g(m);
        if (done.load(std::memory_order_relaxed) & bit) return ICG_OK;
        int r = f();
        if (r == ICG_OK) done.fetch_or(bit, std::memory_order_release);
        return r;
    }
};

// ---------------------------------------------------------------------------
// Error plumbing: no exceptions cross the C ABI.
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
struct Status {
    int code = ICG_OK;
    std::string msg;
};

#define ICG_CUDA_TRY(expr)                                                                     \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess) {                                                               \
            ::icg::set_error(std::string(#expr) + " (" + __FILE__ + ":" + std::to_string(__LINE__) + "): " + \
                             cudaGetErrorString(_e));                                            \
            return ICG_ERUNTIME;                                                               \
        }                                                                                      \
    } while (0)

// ---------------------------------------------------------------------------
// Device-side counters of one extraction / render (one struct in HBM).
// ---------------------------------------------------------------------------
constexpr int kPredIters = 48;  // conflict-loop iterations with size-class prediction
struct DevCounters {
    unsigned int list_count;          // E0 compaction result
    unsigned int cf_count[2];         // conflict lists (ping-pong by iteration)
    unsigned int nx_count[2];         // conflict-neighbour lists (ping-pong)
    unsigned int warning;             // conflict bound hit
    unsigned int unroll_exhausted;    // bit l: level l ran out of unrolled conflict iterations
    unsigned int overflow;            // a work list overflowed
    unsigned long long evals[ICG_MAX_LEVELS];
    unsigned long long refined[ICG_MAX_LEVELS];
    unsigned int conflict_iters[ICG_MAX_LEVELS];
    unsigned int ncols;               // column-factored field: distinct columns of the current batch
    unsigned int ncols_base;          // ncols before the current conflict-loop batch claimed its columns
    unsigned int e0[ICG_MAX_LEVELS];  // size of each level's E0 list (the bulk batch)
    unsigned int tail_start[ICG_MAX_LEVELS];  // 1 + host iteration at which k_tail took over (0: never)
    // conflict-loop size classes (1: 128-point pair tiles, 2: 64-point pair tiles, 4: tail) seen per
    // level and host iteration, and the levels where a batch met no launched evaluator
    uint8_t cls[ICG_MAX_LEVELS][kPredIters];
    unsigned int mispredict;
    // render counters (cleared per render: everything from `covered` to the end)
    unsigned long long covered, degenerate, grazing;
    unsigned int surface_count;
};

// Analytic scene in constant-friendly form (union of primitives).
struct DevPrim {
    int kind, rotated;
    double c[3], a[3], b[3];
    double radius, half[3], major, minor, inv[9];
};

// fp32 mirror of the scene for the PIFu capsule bias inside the MLP kernels
// (tolerance-bound; the exact fp64 form above serves the analytic field)
struct FPrim {
    int kind, rotated;
    float c[3], a[3], b[3];
    float radius, half[3], major, minor, inv[9];
};
struct FScene {
    FPrim prims[ICG_MAX_PRIMS];
    int n_prims;
    float sdf_scale;
};

struct DevScene {
    DevPrim prims[ICG_MAX_PRIMS];
    int n_prims;
    double tau;
    double sdf_scale;
    // TextureRule (scene.hpp:48-55) of the analytic field
    int tex_kind, tex_axis;
    double tex_color[3], tex_from[3], tex_to[3];
    double tex_colors[ICG_MAX_PRIMS][3];
};

// Fixed PIFu architecture (BASELINE.json configs[1-3]).
constexpr int kC = 256;           // feature channels
constexpr int kGeoSkip = 257;     // [Phi(256), z]
constexpr int kTexSkip = 513;     // [Phi(256), h3(256), z]
constexpr int kGeoOut[5] = {1024, 512, 256, 128, 1};
constexpr int kTexOut[5] = {1024, 512, 256, 128, 3};

// Weights of one MLP in the SIMT layout: per layer Wt[K][O] (O contiguous),
// K = prev_out + skip (prev activations first).
struct SimtMlp {
    const float* wt[5];
    const float* b[5];
    int out[5];
    int in[5];
    int skip;
    float slope;
};

// fp32 epilogue operands of one MLP shared by the tensor-core kernels (mlp_pack.cu).
struct TcMlp {
    const float* bias;        // concatenated fp32 biases
    const float* w_last;      // final layer fp32 [out][prev+skip]
    int bias_off[5];
    int valid;
};

// Where the evaluated points come from and where results go.
// One layer of the texture-field GEMM chain (k_texgemm.cu): A = `hid_chunks` 64-wide chunks of the
// hidden input, then skip chunks [skip_c0, skip_c1); fused epilogue acc + b + w_z z, leaky-ReLU.
constexpr int kTgW5Stride = 644;  // padded row of the fp32 texture output layer [h4 | Phi | h3 | z]
struct TgLayer {
    const unsigned* count;
    unsigned n_static;
    int n_out;
    int hid_chunks, skip_c0, skip_c1;
    const float* bias;  // [b (n_out), w_z (n_out)]
    const float* z;
    float slope;
    __half* out;        // fp16 activations (nullptr: no store)
    int ldo, out_col;
    const float* w5;    // output-layer terms of this layer's features (nullptr: none)
    int w5_off;
    float* sdot;
    int final_layer;
    float* rgb;
    const uint32_t* out_pixel;
    int pdl;  // launched as a programmatic dependent of the previous layer
};

struct EvalJob {
    // source: node list of a level grid, or explicit points
    const uint32_t* list;         // node indices (nullptr with list_count==nullptr: dense 0..n^3-1)
    const unsigned int* count;    // device count (nullptr: use n_static)
    unsigned int n_static;
    int cells;                    // level R
    const double* points;         // explicit points (n x 3), when list and count are null
    // grid epilogue
    float* values;
    uint8_t* states;
    const uint32_t* tentbin;      // conflict detection (nullptr: none)
    uint32_t* conflicts;
    unsigned int* conflict_count;
    unsigned int conflict_cap;
    unsigned long long* evals;    // += count (block 0)
    unsigned int* iters;          // += (count > 0) (block 0)
    unsigned int* overflow;
    unsigned int min_count;       // tensor-core kernel: leave batches below this to the latency path
    unsigned int max_count;       // ... and above this (nonzero) to the large-tile kernel
    const unsigned int* base;     // k_mlp_pair COLS: list window start read on device (nullptr: 0), entries [*base, *count)
    // point epilogue
    float* out;                   // occupancy per point (or rgb x3 for texture)
    const uint32_t* out_pixel;    // texture: pixel index per point (out = rgb image)
    float out_clamp;              // texture: clamp01 when nonzero
    // nonzero extents of the grid's x-lines kept by the grid epilogue (the frame path's renderer
    // skips k_xline_extents; nullptr: none): an evaluated nonzero value widens its line's extent
    int2* xext;
};

struct FieldDev {
    int kind;                 // ICG_FIELD_*
    int precision;
    const DevScene* scene;    // device pointer
    const FScene* fscene;     // device pointer, fp32 mirror
    const float* fmap_hwc;    // H x W x C fp32
    int C, H, W;
    // view-space field of render_view (render.hpp:98-99): grid nodes are view points, evaluated at
    // camera.view_to_world(p) (fp64, reference operation order); 0 = world grid
    int view;
    double vr[9], vt[3], vs;
    // PIFu input camera (icg_field.input_camera): Phi sampled at world_to_view(P).xy, depth feature
    // world_to_view(P).z; rows [s R0 | s t0], [s R1 | s t1], [R2 | t2]; 0 = orthographic identity
    int icam;
    float ic[12];
};

// ---- kernel launchers (k_*.cu) -------------------------------------------
int launch_analytic_eval(const FieldDev& f, const EvalJob& job, unsigned int max_points, cudaStream_t s);
int launch_analytic_texture(const FieldDev& f, const EvalJob& job, unsigned int max_points, cudaStream_t s);
int launch_pifu_simt_eval(const FieldDev& f, const SimtMlp& geo, const EvalJob& job,
                          unsigned int max_points, cudaStream_t s);
int launch_pifu_simt_texture(const FieldDev& f, const SimtMlp& geo, const SimtMlp& tex,
                             const EvalJob& job, unsigned int max_points, cudaStream_t s);
size_t pair_stream_bytes(int which, bool x3);
// f16skip: skip-input items as fp16 hi/lo (the texture kernel's streams, geometry prefix included)
int pair_pack(int which, const float* const* w, uint8_t* stream_x3, uint8_t* stream_hi, bool f16skip = false);
int pair_make_tmap(const void* dev_stream, size_t bytes, void* tmap_out, unsigned box_rows = 256);
// column-factored geometry field (k_mlp_pair.cu, modes COLS / FACT): part 0 = FACT stream
// (hidden-input items of layers 2-4), part 1 = COLS stream (Phi items of layers 1-4)
constexpr int kColRecord = 1936;  // floats per column record
size_t pair_fact_stream_bytes(int part, bool x3);
int pair_pack_factored(const float* const* w, int part, uint8_t* stream_x3, uint8_t* stream_hi);
// 2D tiled tensor map (k_texgemm.cu): dtype = CUtensorMapDataType, swizzle = CUtensorMapSwizzle
int make_tmap_2d(const void* base, int dtype, size_t rows, size_t cols, size_t row_bytes, unsigned box_cols,
                 unsigned box_rows, int swizzle, void* out);
// column pass as one GEMM (k_texgemm.cu, namespace cg)
int cg_pack_weights(const float* const* w, __nv_bfloat16* hi, __nv_bfloat16* lo);
int cg_make_tmap(const void* base, size_t rows, size_t cols, size_t row_bytes, unsigned box_cols, unsigned box_rows,
                 bool f32, void* out);
int launch_cols_gemm(const FieldDev& f, const EvalJob& cj, const float* wlast, __nv_bfloat16* ah, __nv_bfloat16* al,
                     float* records, const void* mapAh, const void* mapAl, const void* mapWh, const void* mapWl,
                     const void* mapR, unsigned max_cols, bool x3, cudaStream_t s);
// texture-field GEMM chain (k_texgemm.cu)
int tg_make_tmap(const void* base, size_t rows, size_t cols, unsigned box_rows, void* out);
size_t tg_weight_elems();
int tg_pack_weights(const float* const* gw, const float* const* tw, __half* dst, size_t* off);
int launch_tex_gather(const FieldDev& f, const EvalJob& job, unsigned max_points, __half* skip, float* z, float* sdot,
                      const float* w5, const float* b5, cudaStream_t s);
int launch_tex_layer(const void* mapH, const void* mapS, const void* mapW, const void* mapO, const TgLayer& L,
                     unsigned max_points, cudaStream_t s);

int launch_pifu_pair_cols(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& cols, float* records,
                          unsigned max_cols, bool x3, cudaStream_t s);
// geometry field with 64-point pair tiles (twice the pairs busy on mid-size batches)
int launch_pifu_pair_eval_small(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& job,
                                unsigned max_points, bool x3, cudaStream_t s);
// k_fact2.cu: the same pass with activations as the A operand (M = 256 points), weights as B
// x3: bf16x3 (the FACT x3 stream in 128-row hi / lo stages); else bf16 (the hi stream, 128-row stages)
int launch_pifu_fact2(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& job, const float* records,
                      const int* cmap, unsigned max_points, bool x3, cudaStream_t s);
int launch_pifu_pair_fact(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& job,
                          const float* records, const int* cmap, unsigned max_points, bool x3, cudaStream_t s);
int launch_pifu_pair_eval(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& job,
                          unsigned max_points, bool x3, cudaStream_t s);
int launch_pifu_pair_texture(const FieldDev& f, const TcMlp& geo, const TcMlp& tex, const void* tmap_geo,
                             const void* tmap_tex, const EvalJob& job, unsigned max_points, bool x3,
                             cudaStream_t s);
int launch_fmap_chw_to_hwc(const float* chw, float* hwc, int C, int H, int W, cudaStream_t s);
int launch_feature_normals(uint64_t seed, size_t n, float* out, cudaStream_t s);
// marching cubes (k_mc.cu): generated triangulation table, per-cell count / emit, weld, filter
int mc_init_tables();
int mc_table_row(int cs, int8_t* out16, int* ntri);
int launch_mc_count(const float* v, int cells, double iso, uint32_t* block_tris, unsigned nblocks, cudaStream_t s);
int launch_mc_emit(const float* v, int cells, double iso, const uint32_t* block_off, unsigned nblocks,
                   uint32_t* tri_keys, uint32_t* key_bits, cudaStream_t s);
int launch_mc_filter(const uint32_t* tri_keys, unsigned ntri, const uint32_t* keys, unsigned nkeys, const float* v,
                     int cells, double iso, uint32_t* tri_ids, uint32_t* keep, uint32_t* first_use, cudaStream_t s);
int launch_mc_mark_first(const uint32_t* first_use, unsigned nkeys, uint32_t* slot_bits, cudaStream_t s);
int launch_mc_vertices(const uint32_t* slots, unsigned nv, const uint32_t* tri_ids, const uint32_t* keys,
                       const float* v, int cells, double iso, uint32_t* new_id, double* out_v, cudaStream_t s);
int launch_mc_triangles(const uint32_t* tri_list, unsigned nt, const uint32_t* tri_ids, const uint32_t* new_id,
                        int32_t* out_t, cudaStream_t s);
int launch_exclusive_scan(uint32_t* counts, unsigned n, unsigned* total, cudaStream_t s);

// grid kernels (k_grid.cu)
struct LevelBufs {
    const float* cv;  const uint8_t* cs;   // coarse grid
    float* fv;        uint8_t* fs;         // fine grid
    uint32_t* cbin;                         // coarse binarized bits (flat)
    uint32_t* mixed;                        // coarse cell bits (flat over Rc^3)
    uint32_t* tentbin;                      // fine bits
    uint32_t* sel;                          // fine bits (flagged & !evaluated)
    uint32_t* queued;                       // fine bits
    uint32_t* block_counts;                 // per 1024-node block
    uint32_t* list;                         // E0 output
    int rc;                                 // coarse cells
    int2* xext;                             // k_fine_rows: each fine x-line's nonzero extent (nullptr: none)
};
int launch_level_classify(const LevelBufs& b, DevCounters* ctr, int level, cudaStream_t s);
int launch_level_carry(const LevelBufs& b, DevCounters* ctr, int level, cudaStream_t s);
// one level of the octree baselines (mode 0 binarized, 1 threshold): cell marks -> b.mixed (count
// in ctr->refined[level]), fine values / states -> b.fv / b.fs, nodes to evaluate -> b.sel;
// iface: scratch bitset over the coarse nodes (mode 0)
int launch_octree_level(const LevelBufs& b, uint32_t* iface, int mode, double threshold, DevCounters* ctr, int level,
                        cudaStream_t s);
// render_view's view-space depth pass at level L (k_depth.cu, render.hpp:105-206)
struct DepthJob {
    const uint32_t* cbin;  // coarse (level L-1) binarized bits
    int rc;                // coarse cells
    float* fv;             // level-L values / states (carry of the coarse grid)
    uint8_t* fs;
    uint32_t* sel;         // fine bitset (cleared by the caller)
    int* colk;             // per column: k1 of the binarized argmax before the bracket evaluation
    // final pass
    const FieldDev* fd;    // (host copy; the kernels get the camera below)
    double vr[9], vt[3], vs;  // CameraSpec (view_to_world of the surface points)
    float bg[3];
    float* depth;
    float* rgb;
    uint8_t* mask;
    int32_t* surface_k;
    double* surface_pts;
    uint32_t* surface_px;
    DevCounters* ctr;
};
int launch_depth_shadow(const DepthJob& j, cudaStream_t s);
int launch_depth_bracket(const DepthJob& j, cudaStream_t s);
int launch_depth_final(const DepthJob& j, cudaStream_t s);
// size classes of a conflict batch: which evaluator takes n nodes (0: empty)
struct ChainClasses {
    unsigned tail_max, mid_max;
    int level;
    int prev_mask;     // classes launched for the previous iteration (-1: no check)
    unsigned big_max;  // above this: the column-factored class 8 (0: no such class)
};
int launch_conflict_expand_cls(uint32_t* fine_queued, const uint8_t* fs, int fcells, const uint32_t* conflicts,
                               DevCounters* ctr, int iter, int max_iters, uint32_t* next_list, unsigned cap,
                               const ChainClasses& cc, cudaStream_t s);
int launch_unroll_check_cls(DevCounters* ctr, int iter_parity, int level, const ChainClasses& cc, int last_iter,
                            cudaStream_t s);
int launch_conflict_expand(uint32_t* fine_queued, const uint8_t* fs, int fcells, const uint32_t* conflicts,
                           DevCounters* ctr, int iter, int max_iters, uint32_t* next_list,
                           unsigned int cap, cudaStream_t s);
int launch_unroll_check(DevCounters* ctr, int iter_parity, int level, cudaStream_t s);
// persistent conflict-loop tail (k_tail.cu)
struct TailParams {
    FieldDev f;
    int cells, level, it0, max_iters;
    unsigned cap, max_start;
    float* fv;
    uint8_t* fs;
    const uint32_t* tentbin;
    uint32_t* queued;
    uint32_t* cf[2];
    uint32_t* nx[2];
    DevCounters* ctr;
    float* colrec;
    int* cmap;
    uint32_t* collist;
    const float* w[4];      // geometry layers 1-4, row-major [out][in] fp32
    const float* bias;      // tc layout: per layer [b, wz], then b5
    const float* wlast;     // final layer [128 + 257]
    float slope;
    // scratch (launch_tail carves it)
    float *h1, *h2, *h3, *h4, *pz, *phi;
    int* pslot;
    unsigned *newcols, *nnew;
    unsigned cap_pts, cap_new;
    unsigned long long* trace;  // ICG_TAIL_TRACE=1: phase times of block 0
    int2* xext;                 // x-line extents kept by the grid epilogue (EvalJob::xext)
};
size_t tail_smem_bytes();
size_t tail_scratch_bytes(unsigned cap_pts, unsigned cap_new, unsigned max_cols);
int launch_tail(TailParams p, uint8_t* scratch, unsigned cap_pts, unsigned cap_new, unsigned max_cols, cudaStream_t s,
                bool wide);

// column-factored field: give every distinct column (i + n j) of a node list a record slot
// (cmap[col] = slot, collist[slot] = col, ctr->ncols = number of slots); cmap must be all -1
int launch_col_claim(const uint32_t* list, const unsigned* count, int cells, int* cmap, uint32_t* collist,
                     DevCounters* ctr, unsigned max_points, cudaStream_t s, unsigned min_count = 0);
// counting sort of a node list by column record (so a point tile spans few columns); cnt holds
// one u32 per possible column and is cleared here
// bsum: (plane + 8191) / 8192 scratch words (chunk sums of the slot scan)
int launch_sort_by_column(const uint32_t* list, const unsigned* count, int cells, const int* cmap, uint32_t* cnt,
                          DevCounters* ctr, uint32_t* sorted, unsigned* bsum, unsigned max_points, cudaStream_t s,
                          unsigned min_count = 0);
// node list of a dense (cells+1)^3 grid in column order: t -> node (t / n1) + plane * (t % n1)
int launch_dense_column_list(int cells, uint32_t* list, cudaStream_t s);
int launch_binarize(const float* v, uint8_t* out, size_t n, cudaStream_t s);
// per-level sets (icg_level_set): nodes evaluated during a level (fine states vs the coarse states
// the even nodes carried), every bit set, and the ascending list of a bitset's set bits
int launch_level_eval_bits(const uint8_t* fs, const uint8_t* cs, int rc, uint32_t* bits, cudaStream_t s);
int launch_all_bits(uint32_t* bits, size_t nbits, cudaStream_t s);
size_t bits_to_list_scratch_words(size_t nbits);
int launch_bits_to_list(const uint32_t* bits, size_t nbits, uint32_t* scratch, uint32_t* list, unsigned* total,
                        cudaStream_t s);
int launch_iou(const uint8_t* a, const uint8_t* b, size_t n, unsigned long long* inter_union, cudaStream_t s);
int launch_fill_states(uint8_t* s, size_t n, uint8_t v, cudaStream_t st);

// render (k_render.cu)
struct RenderJob {
    const float* values;
    int cells;
    double rot[9], trans[3], scale;
    int width, height;
    float bg[3];
    float* depth;
    float* rgb;
    uint8_t* mask;
    int32_t* surface_k;
    double* surface_pts;     // world points of covered pixels (compacted)
    uint32_t* surface_px;    // pixel index per surface point
    DevCounters* ctr;
    const int2* xext;        // per grid x-line (j, k): first / last i with a nonzero value (nullptr: none)
    double* tab;             // scratch of render_tab_doubles(W, H, R) doubles (k_render_setup)
};
inline size_t render_tab_doubles(int W, int H, int R) { return (size_t)W + H + 3 * ((size_t)R + 1); }
int launch_render_first_crossing(const RenderJob& r, cudaStream_t s);
// extents of the nonzero values along every x-line of the (R+1)^3 grid (render empty-space skipping)
int launch_xline_extents(const float* values, int cells, int2* ext, cudaStream_t s);

int tc_pack_epilogue(int which, const float* const* w, const float* const* b, float* host_bias, float* host_wlast);
size_t tc_bias_floats(int which);
size_t tc_wlast_floats(int which);

}  // namespace icg

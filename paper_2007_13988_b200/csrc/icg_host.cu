// icg_host.cu — host runtime behind the C ABI (include/isocull_b200.h).
//
// One icg_context per GPU: a stream, library-owned weight copies (SIMT and
// tcgen05 layouts), grow-only device work buffers sized for the finest level,
// and the grid of the last extraction (for the renderer).  The per-level
// control flow of extract_progressive (localize.hpp:315-363) is issued as a
// fixed sequence of kernels that read their work sizes from device counters,
// so a whole extraction needs one host synchronisation (at the end).  The
// conflict loop is unrolled `unroll` times per level; if a level still had
// conflicts after the last unrolled iteration the device raises
// `unroll_exhausted` and the extraction is replayed with twice the unroll
// (results are identical; only the launch count changes).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <atomic>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "icg_internal.h"

namespace icg {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

static int einval(const std::string& m) {
    set_error(m);
    return ICG_EINVAL;
}

// Bumped by every device (re)allocation of a work buffer: a captured frame graph bakes the
// buffer addresses into its launches, so it is only replayed while this is unchanged.
static std::atomic<unsigned long long> g_alloc_gen{0};

struct DBuf {
    void* p = nullptr;
    size_t n = 0;
    int ensure(size_t bytes) {
        if (bytes <= n) return ICG_OK;
        g_alloc_gen.fetch_add(1, std::memory_order_relaxed);
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        size_t b = bytes < 256 ? 256 : bytes;
        ICG_CUDA_TRY(cudaMalloc(&p, b));
        n = b;
        return ICG_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace icg

using namespace icg;

struct icg_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEvent_t span_start = nullptr, span_end = nullptr;  // icg_span_begin / icg_span_end
    // CUDA graph of one frame's device work (icg_frame), keyed by everything its launches capture
    struct FrameKey {
        icg_algo_config cfg;
        icg_camera cam;
        unsigned long long alloc_gen;  // no work buffer moved since the capture (g_alloc_gen)
        int fmap_c, fmap_h, fmap_w;    // feature-map shape baked into the field kernels' parameters
        int W, H, kind, precision, img_mem;
        float bg[3];
        void* img_ptr[4];
        int unroll[ICG_MAX_LEVELS];
        uint8_t pred[ICG_MAX_LEVELS][kPredIters];
        uint8_t pred_valid[ICG_MAX_LEVELS];
        uint8_t tail_wide;
        bool operator==(const FrameKey& o) const { return std::memcmp(this, &o, sizeof(FrameKey)) == 0; }
    };
    // one slot per tail width, so a context alternating between alone / shared frames keeps both graphs
    struct GraphSlot {
        FrameKey graph_key{}, warm_key{};
        bool graph_valid = false, warm_valid = false;
        cudaGraphExec_t graph_exec = nullptr;
        uint64_t graph_launches = 0;
    } gslot[2];
    bool use_graph = true;
    // weights
    bool has_geo = false, has_tex = false;
    DBuf geo_wt[5], geo_b[5], tex_wt[5], tex_b[5], geo_wrow[5];
    const float* geo_rows[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    SimtMlp geo_simt{}, tex_simt{};
    DBuf geo_bias, geo_wlast, tex_bias, tex_wlast;
    TcMlp geo_tc{}, tex_tc{};
    DBuf geo_pair_stream, tex_pair_stream, geo_pair_hi, tex_pair_hi;
    // TMA descriptors of the pair streams: [0] bf16x3 (hi, lo), [1] bf16 (hi only)
    alignas(64) unsigned char geo_pair_tmap[2][128] = {};
    alignas(64) unsigned char tex_pair_tmap[2][128] = {};
    DBuf geo_pair_f16, geo_pair_f16_hi;  // geometry stream with fp16 skip items (texture kernel prefix)
    alignas(64) unsigned char geo_pair_f16_tmap[2][128] = {};
    bool geo_pair = false, tex_pair = false;
    // texture field as a per-layer GEMM chain (k_texgemm.cu): fp16 weights [g1 g2 g3 t1 t2 t3 t4],
    // padded fp32 output layer, per-point activations (capacity tg_cap points)
    std::vector<float> host_w[2][5];  // fp32 weights of each network as set (the chain packs both)
    bool host_w_set[2] = {false, false};
    DBuf tg_w, tg_w5, tg_skip, tg_h1, tg_h2, tg_h3, tg_z, tg_sdot;
    size_t tg_off[7] = {};
    unsigned tg_cap = 0;
    int tg_C = 0;  // channels of the last texture gather (profile bytes)
    bool tg_ready = false, use_tg = true;  // ICG_TEX_PAIR=1: the fused pair kernel instead
    bool tg_pdl = true;                    // ICG_TG_PDL=0: layers launched without programmatic dependence
    alignas(64) unsigned char tg_mapW[7][128] = {};
    alignas(64) unsigned char tg_mapS[128] = {};
    alignas(64) unsigned char tg_mapH[3][128] = {};  // h1 (1024 wide), h2 (512), h3 (256)
    alignas(64) unsigned char tg_mapO[4][128] = {};  // output boxes (64 x 32): h1, h2, h3, skip
    // column pass as one GEMM: bf16 Phi rows (hi, lo) of up to cg_cap columns, W_Phi (hi, lo)
    DBuf cg_ah, cg_al, cg_w;
    size_t cg_cap = 0;
    const void* cg_rec = nullptr;  // the records buffer cg_mapR describes (pointer, bytes)
    size_t cg_rec_n = 0;
    bool cg_ready = false, use_cg = true;  // ICG_COLS_PAIR=1: k_mlp_pair<COLS> instead
    alignas(64) unsigned char cg_mapA[2][128] = {};
    alignas(64) unsigned char cg_mapW[2][128] = {};
    alignas(64) unsigned char cg_mapR[128] = {};
    // column-factored geometry field (FACT / COLS streams, [part][x3 ? 0 : 1])
    DBuf geo_fact_stream[2][2];
    alignas(64) unsigned char geo_fact_tmap[2][2][128] = {};
    alignas(64) unsigned char geo_fact2_tmap[2][128] = {};  // k_fact2: the FACT [x3, hi] streams in 16 KB boxes
    bool geo_fact = false, use_fact = true;
    bool fact_used = false;  // the last extraction ran its bulk batches column-factored
    DBuf colrec, cmap, collist, colcnt, sorted, tail_scratch, scan_bsum;
    DBuf xext;  // render: nonzero extent of every grid x-line
    DBuf rtab;  // render: per-column / per-row / per-sample view_to_world terms
    bool use_xext = true;  // ICG_NO_XEXT=1: rays along grid x walk every sample
    bool use_tail = true;
    bool chain_trace = false;  // ICG_CHAIN_TRACE=1
    bool chain_fact = true;    // large conflict-loop batches column-factored (ICG_CHAIN_FACT=0: CTA-pair GEO)
    // ... above this many nodes (ICG_CHAIN_FACT_MIN; 0 = by precision: bf16x3 74 x 64 -- the 128-point
    // pair class then never runs, 427 vs 411 frames/s at 4 in flight -- bf16 74 x 128)
    unsigned chain_fact_min = 0;
    bool use_fact2 = true;     // bulk factored pass with swapped operands (k_fact2.cu); ICG_FACT2=0: k_mlp_pair<FACT>
    bool tail_wide = true;  // this frame is alone on its device: the tail kernel takes every SM
    unsigned tail_max = 128;  // conflict batches up to this size start the persistent tail kernel
    // field
    DBuf scene;
    DevScene* h_scene = nullptr;  // pinned staging
    FScene* h_fscene = nullptr;
    DBuf fscene;
    DBuf fmap_chw, fmap_hwc;
    // grids and work lists
    DBuf vals[2], sts[2];
    DBuf cbin, mixed, tentbin, sel, queued, block_counts;
    DBuf list_e0, cf[2], nx[2];
    DBuf ctr;
    DevCounters* h_ctr = nullptr;  // pinned
    DBuf binar, pts, outv;
    // render
    DBuf depth, rgb, mask, surfk, spts, spx;
    // last extraction
    int last_cells = 0, last_buf = -1;
    // per-level sets kept by an extraction with cfg.keep_level_sets (icg_level_set):
    // [0][l] nodes evaluated at level l, [1][l] refined cells of level l (bitsets)
    DBuf lvl_bits[2][ICG_MAX_LEVELS];
    bool kept_valid = false;
    icg_algo_config kept_cfg{};
    DBuf set_scratch, set_list, set_total, set_bits;
    // marching cubes scratch (icg_marching_cubes)
    DBuf mc_grid, mc_blocks, mc_total, mc_tri_keys, mc_key_bits, mc_keys, mc_tri_ids, mc_keep, mc_first, mc_slot_bits,
        mc_slots, mc_tri_list, mc_new_id, mc_out_v, mc_out_t;
    // instrumentation
    struct Mark {
        int kind;  // 0 geo mlp, 1 tex mlp, 2 dense, 3 render
        int slot;
    };
    bool prof_on = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<Mark> marks;
    int ev_used = 0;
    icg_profile prof{};
    uint64_t launches = 0;
    // device-side conflict-loop depth per level, adapted from the previous frame
    int unroll[ICG_MAX_LEVELS] = {4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4};
    int unroll_seen[ICG_MAX_LEVELS] = {};  // deepest adapted depth so far (grow-only)
    // conflict-loop size classes per level and host iteration (union over frames; invalid: all)
    uint8_t pred[ICG_MAX_LEVELS][kPredIters] = {};
    bool pred_valid[ICG_MAX_LEVELS] = {};
    bool pred_all[ICG_MAX_LEVELS] = {};  // the last frame mispredicted this level: launch everything
};

namespace {

size_t nodes3(int cells) {
    size_t n = (size_t)cells + 1;
    return n * n * n;
}
size_t words(size_t bits) { return (bits + 31) / 32; }

// frames in flight per device (contexts driven from concurrent host threads): a frame alone on
// its device lets latency-bound kernels (the conflict-loop tail) take every SM
std::atomic<int> g_inflight[64];
struct InflightGuard {
    int dev;
    bool alone;
    explicit InflightGuard(int d) : dev(d & 63) { alone = g_inflight[dev].fetch_add(1) == 0; }
    ~InflightGuard() { g_inflight[dev].fetch_sub(1); }
};
bool job_is_grid_host(const EvalJob& j) { return j.points == nullptr && j.values != nullptr; }

// ---- instrumentation ----------------------------------------------------------
int prof_begin(icg_context* c, int kind) {
    if (!c->prof_on) return -1;
    if (c->ev_used + 2 > (int)c->ev_pool.size()) {
        for (int i = 0; i < 64; ++i) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) return -1;
            c->ev_pool.push_back(e);
        }
    }
    int slot = c->ev_used;
    c->ev_used += 2;
    cudaEventRecord(c->ev_pool[slot], c->stream);
    c->marks.push_back({kind, slot});
    return slot;
}
void prof_end(icg_context* c, int slot) {
    if (slot >= 0) cudaEventRecord(c->ev_pool[slot + 1], c->stream);
}
void prof_discard(icg_context* c) {
    c->marks.clear();
    c->ev_used = 0;
}
// after a stream sync: fold the recorded intervals into the totals
void prof_collect(icg_context* c) {
    if (!c->prof_on) return;
    for (const auto& m : c->marks) {
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, c->ev_pool[m.slot], c->ev_pool[m.slot + 1]);
        switch (m.kind) {
            case 0: c->prof.geo_mlp_ms += ms; c->prof.geo_mlp_launches++; break;
            case 4:  // column-factored bulk batch (also a geometry launch)
                c->prof.geo_mlp_ms += ms; c->prof.geo_mlp_launches++;
                c->prof.fact_ms += ms; c->prof.fact_launches++;
                break;
            case 5:  // conflict-loop batch on the pair kernels + tail
                c->prof.geo_mlp_ms += ms; c->prof.geo_mlp_launches++;
                c->prof.chain_ms += ms; c->prof.chain_launches++;
                break;
            case 1: c->prof.tex_mlp_ms += ms; c->prof.tex_mlp_launches++; break;
            case 2: c->prof.dense_ms += ms; c->prof.dense_launches++; break;
            case 3: c->prof.render_ms += ms; c->prof.render_launches++; break;
            case 6: c->prof.gather_ms += ms; c->prof.gather_launches++; break;  // (inside a kind-1 interval)
            case 7: c->prof.expand_ms += ms; c->prof.expand_launches++; break;
            case 8:  // the target level's dense pass (also a dense pass)
                c->prof.dense_ms += ms; c->prof.dense_launches++;
                c->prof.last_level_ms += ms; c->prof.last_level_launches++;
                break;
        }
    }
    prof_discard(c);
}

int ensure_grid(icg_context* c, int cells) {
    size_t N = nodes3(cells);
    size_t nc = nodes3(cells / 2 > 0 ? cells / 2 : 1);
    size_t ncell = (size_t)(cells / 2) * (cells / 2) * (cells / 2) + 1;
    for (int b = 0; b < 2; ++b) {
        if (int r = c->vals[b].ensure(N * 4)) return r;
        if (int r = c->sts[b].ensure(N)) return r;
        if (int r = c->cf[b].ensure(N * 4)) return r;
        if (int r = c->nx[b].ensure(N * 4)) return r;
    }
    if (int r = c->cbin.ensure(words(nc) * 4 + 16)) return r;
    if (int r = c->mixed.ensure(words(ncell) * 4 + 16)) return r;
    if (int r = c->tentbin.ensure(words(N) * 4 + 16)) return r;
    if (int r = c->sel.ensure(words(N) * 4 + 16)) return r;
    if (int r = c->queued.ensure(words(N) * 4 + 16)) return r;
    const size_t fn = (size_t)cells + 1;  // row counts (fn^2) + per-1024 group sums
    if (int r = c->block_counts.ensure((fn * fn + fn * fn / 1024 + 64) * 4)) return r;
    if (int r = c->list_e0.ensure(N * 4)) return r;
    return ICG_OK;
}

int validate_algo(const icg_algo_config* cfg) {
    // validate_config, localize.hpp:47-55
    if (!cfg) return einval("config: null");
    if (cfg->variant < ICG_VARIANT_BRUTE || cfg->variant > ICG_VARIANT_PROGRESSIVE)
        return einval("config: unknown variant");
    if (cfg->coarsest_cells < 2) return einval("config: coarsest cells must be >= 2");
    if (cfg->target_level < 0) return einval("config: target level must be >= 0");
    if (cfg->target_level > 10 || ((long)cfg->coarsest_cells << cfg->target_level) > ICG_MAX_TARGET_CELLS)
        return einval("config: target resolution exceeds 1024 cells per axis");
    if (cfg->variant == ICG_VARIANT_OCTREE_THRESHOLD && !(cfg->threshold > 0.0 && cfg->threshold < 0.5))
        return einval("config: threshold must lie in (0, 0.5)");
    return ICG_OK;
}

int prepare_field(icg_context* c, const icg_field* f, FieldDev& fd) {
    if (!f) return einval("field: null");
    if (f->kind != ICG_FIELD_ANALYTIC && f->kind != ICG_FIELD_PIFU) return einval("field: unknown kind");
    const icg_scene& s = f->scene;
    if (s.n_prims < 0 || s.n_prims > ICG_MAX_PRIMS) return einval("scene: too many primitives");
    if (f->kind == ICG_FIELD_ANALYTIC) {
        if (s.n_prims == 0) return einval("scene: no primitives");  // validate_scene, scene.hpp:191
        if (!(s.tau > 0.0)) return einval("scene: tau must be > 0");
    }
    if (s.n_prims && !s.prims) return einval("scene: null primitive array");
    DevScene* h = c->h_scene;
    std::memset(h, 0, sizeof(DevScene));
    for (int i = 0; i < s.n_prims; ++i) {
        const icg_primitive& p = s.prims[i];
        if (p.kind < ICG_PRIM_SPHERE || p.kind > ICG_PRIM_TORUS) return einval("scene: unknown primitive kind");
        DevPrim& d = h->prims[i];
        d.kind = p.kind;
        d.rotated = p.rotated ? 1 : 0;
        for (int k = 0; k < 3; ++k) {
            d.c[k] = p.center[k];
            d.a[k] = p.a[k];
            d.b[k] = p.b[k];
            d.half[k] = p.half[k];
        }
        d.radius = p.radius;
        d.major = p.major;
        d.minor = p.minor;
        for (int k = 0; k < 9; ++k) d.inv[k] = p.inv_rotation[k];
    }
    h->n_prims = s.n_prims;
    h->tau = s.tau;
    h->sdf_scale = f->sdf_scale;
    // TextureRule (scene.hpp:48-55; validate_scene's per-primitive rule, scene.hpp:199-201)
    const icg_texture_rule& tr = s.texture;
    if (tr.kind < ICG_TEXTURE_NONE || tr.kind > ICG_TEXTURE_PER_PRIMITIVE) return einval("scene: unknown texture kind");
    if (tr.kind == ICG_TEXTURE_GRADIENT && (tr.axis < 0 || tr.axis > 2)) return einval("scene: gradient axis must be x, y or z");
    if (tr.kind == ICG_TEXTURE_PER_PRIMITIVE && !tr.colors)
        return einval("scene: per_primitive texture needs one color per primitive");
    h->tex_kind = tr.kind;
    h->tex_axis = tr.axis;
    for (int k = 0; k < 3; ++k) {
        h->tex_color[k] = tr.color[k];
        h->tex_from[k] = tr.from[k];
        h->tex_to[k] = tr.to[k];
    }
    if (tr.kind == ICG_TEXTURE_PER_PRIMITIVE)
        for (int i = 0; i < s.n_prims; ++i)
            for (int k = 0; k < 3; ++k) h->tex_colors[i][k] = tr.colors[3 * i + k];
    if (int r = c->scene.ensure(sizeof(DevScene))) return r;
    ICG_CUDA_TRY(cudaMemcpyAsync(c->scene.p, h, sizeof(DevScene), cudaMemcpyHostToDevice, c->stream));
    FScene* hf = c->h_fscene;
    std::memset(hf, 0, sizeof(FScene));
    for (int i = 0; i < s.n_prims; ++i) {
        const DevPrim& d = h->prims[i];
        FPrim& q = hf->prims[i];
        q.kind = d.kind;
        q.rotated = d.rotated;
        for (int k = 0; k < 3; ++k) {
            q.c[k] = (float)d.c[k];
            q.a[k] = (float)d.a[k];
            q.b[k] = (float)d.b[k];
            q.half[k] = (float)d.half[k];
        }
        q.radius = (float)d.radius;
        q.major = (float)d.major;
        q.minor = (float)d.minor;
        for (int k = 0; k < 9; ++k) q.inv[k] = (float)d.inv[k];
    }
    hf->n_prims = s.n_prims;
    hf->sdf_scale = (float)f->sdf_scale;
    if (int r = c->fscene.ensure(sizeof(FScene))) return r;
    ICG_CUDA_TRY(cudaMemcpyAsync(c->fscene.p, hf, sizeof(FScene), cudaMemcpyHostToDevice, c->stream));
    fd = FieldDev{};
    fd.kind = f->kind;
    fd.precision = f->precision;
    fd.scene = c->scene.as<DevScene>();
    fd.fscene = c->fscene.as<FScene>();
    if (f->kind == ICG_FIELD_PIFU) {
        if (!c->has_geo) return einval("field: PIFu field needs geometry MLP weights (icg_set_mlp)");
        if (f->precision != ICG_PREC_FP32 && f->precision != ICG_PREC_BF16 && f->precision != ICG_PREC_FP32_SIMT)
            return einval("field: unknown precision");
        if (f->precision != ICG_PREC_FP32_SIMT && !c->geo_tc.valid)
            return einval("field: tensor-core weights not packed");
        if (!f->feature_map) return einval("field: null feature map");
        if (f->fmap_c != kC) return einval("field: feature map must have 256 channels");
        if (f->fmap_h < 2 || f->fmap_w < 2) return einval("field: feature map must be at least 2x2");
        size_t n = (size_t)f->fmap_c * f->fmap_h * f->fmap_w;
        const float* chw = f->feature_map;
        if (f->fmap_mem == ICG_MEM_HOST) {
            if (int r = c->fmap_chw.ensure(n * 4)) return r;
            ICG_CUDA_TRY(cudaMemcpyAsync(c->fmap_chw.p, f->feature_map, n * 4, cudaMemcpyHostToDevice, c->stream));
            chw = c->fmap_chw.as<float>();
        } else if (f->fmap_mem != ICG_MEM_DEVICE) {
            return einval("field: fmap_mem must be ICG_MEM_HOST or ICG_MEM_DEVICE");
        }
        if (int r = c->fmap_hwc.ensure(n * 4)) return r;
        if (int r = launch_fmap_chw_to_hwc(chw, c->fmap_hwc.as<float>(), f->fmap_c, f->fmap_h, f->fmap_w, c->stream))
            return r;
        c->launches += 1;
        fd.fmap_hwc = c->fmap_hwc.as<float>();
        fd.C = f->fmap_c;
        fd.H = f->fmap_h;
        fd.W = f->fmap_w;
        if (f->has_input_camera) {
            const icg_camera& ic = f->input_camera;
            if (!(ic.scale != 0.0) || !std::isfinite(ic.scale)) return einval("field: input camera scale must be nonzero");
            fd.icam = 1;
            for (int r = 0; r < 3; ++r) {
                const double s = r < 2 ? ic.scale : 1.0;
                for (int k = 0; k < 3; ++k) fd.ic[4 * r + k] = (float)(s * ic.rotation[3 * r + k]);
                fd.ic[4 * r + 3] = (float)(s * ic.translation[r]);
            }
        }
    }
    return ICG_OK;
}

// column factoring: every node of a grid column shares Phi (orthographic identity input camera,
// world-space grid)
// FieldOracle::has_texture (field.hpp:50): a texture rule (analytic) or texture MLP weights (PIFu)
bool field_has_texture(const icg_context* c, const FieldDev& fd) {
    return fd.kind == ICG_FIELD_PIFU ? c->has_tex : c->h_scene->tex_kind != ICG_TEXTURE_NONE;
}

bool fact_ok(const icg_context* c, const FieldDev& fd) {
    return fd.kind == ICG_FIELD_PIFU && (fd.precision == ICG_PREC_FP32 || fd.precision == ICG_PREC_BF16) &&
           !fd.icam && !fd.view &&
           c->geo_pair && c->geo_fact && c->use_fact;
}

// Column records of `cj`'s list window: the column GEMM (k_cols) or the pair kernel.
static int run_cols(icg_context* c, const FieldDev& fd, const EvalJob& cj, unsigned max_cols, int xi) {
    if (!(c->cg_ready && c->use_cg))
        return launch_pifu_pair_cols(fd, c->geo_tc, c->geo_fact_tmap[1][xi], cj, c->colrec.as<float>(), max_cols,
                                     xi == 0, c->stream);
    const size_t n1 = (size_t)cj.cells + 1, plane = n1 * n1;
    if (plane > c->cg_cap) {
        const size_t cap = (plane + 255) / 256 * 256;
        if (int r = c->cg_ah.ensure(cap * 512)) return r;
        if (int r = c->cg_al.ensure(cap * 512)) return r;
        if (int r = cg_make_tmap(c->cg_ah.p, cap, 256, 512, 64, 128, false, c->cg_mapA[0])) return r;
        if (int r = cg_make_tmap(c->cg_al.p, cap, 256, 512, 64, 128, false, c->cg_mapA[1])) return r;
        c->cg_cap = cap;
    }
    if (c->cg_rec != c->colrec.p || c->cg_rec_n != c->colrec.n) {
        const size_t rows = c->colrec.n / (kColRecord * sizeof(float));
        if (int r = cg_make_tmap(c->colrec.p, rows, kColRecord, kColRecord * 4, 32, 32, true, c->cg_mapR)) return r;
        c->cg_rec = c->colrec.p;
        c->cg_rec_n = c->colrec.n;
    }
    return launch_cols_gemm(fd, cj, c->geo_tc.w_last, c->cg_ah.as<__nv_bfloat16>(), c->cg_al.as<__nv_bfloat16>(),
                            c->colrec.as<float>(), c->cg_mapA[0], c->cg_mapA[1], c->cg_mapW[0], c->cg_mapW[1], c->cg_mapR,
                            max_cols, xi == 0, c->stream);
}

// Column-factored evaluation of a grid job (a level's node list, or all nodes of a dense grid):
// the orthographic projection gives every node of a column (i, j) the same Phi, so the Phi part
// of every layer is computed once per distinct column (COLS pass, k_mlp_pair.cu) and the per-node
// pass (FACT) only runs the hidden-input parts of layers 2-4.
int run_eval_fact(icg_context* c, const FieldDev& fd, const EvalJob& job, unsigned max_points) {
    const int xi = fd.precision == ICG_PREC_FP32 ? 0 : 1;
    const size_t n1 = (size_t)job.cells + 1, plane = n1 * n1;
    if (int r = c->colrec.ensure(plane * kColRecord * sizeof(float))) return r;
    if (int r = c->cmap.ensure(plane * sizeof(int))) return r;
    if (int r = c->collist.ensure(plane * sizeof(uint32_t))) return r;
    if (int r = c->colcnt.ensure(plane * sizeof(uint32_t))) return r;
    if (int r = c->sorted.ensure(nodes3(job.cells) * sizeof(uint32_t))) return r;
    if (int r = c->scan_bsum.ensure((plane + 8191) / 8192 * sizeof(unsigned))) return r;
    DevCounters* ctr = c->ctr.as<DevCounters>();
    int slot = prof_begin(c, 4);
    c->fact_used = true;
    EvalJob cj{};
    cj.cells = job.cells;
    const int* cm = nullptr;
    unsigned max_cols = (unsigned)plane;
    EvalJob pj = job;  // the per-node job, its list in column order (a tile spans few column records)
    pj.list = c->sorted.as<uint32_t>();
    if (job.list) {
        ICG_CUDA_TRY(cudaMemsetAsync(c->cmap.p, 0xFF, plane * sizeof(int), c->stream));
        ICG_CUDA_TRY(cudaMemsetAsync(&ctr->ncols, 0, sizeof(unsigned), c->stream));
        if (int r = launch_col_claim(job.list, job.count, job.cells, c->cmap.as<int>(), c->collist.as<uint32_t>(),
                                     ctr, max_points, c->stream))
            return r;
        if (int r = launch_sort_by_column(job.list, job.count, job.cells, c->cmap.as<int>(), c->colcnt.as<uint32_t>(),
                                          ctr, c->sorted.as<uint32_t>(), c->scan_bsum.as<unsigned>(), max_points, c->stream))
            return r;
        cj.list = c->collist.as<uint32_t>();
        cj.count = &ctr->ncols;
        cm = c->cmap.as<int>();
        if (max_points < max_cols) max_cols = max_points;
        c->launches += 4;
    } else {
        // dense grid (job.n_static = all nodes): every column, record = column index
        if (job.n_static != nodes3(job.cells)) return einval("factored field: dense job must cover the grid");
        cj.n_static = (unsigned)plane;
        if (int r = launch_dense_column_list(job.cells, c->sorted.as<uint32_t>(), c->stream)) return r;
        c->launches += 1;
    }
    if (int r = run_cols(c, fd, cj, max_cols, xi))
        return r;
    int r = c->use_fact2
                ? launch_pifu_fact2(fd, c->geo_tc, c->geo_fact2_tmap[xi], pj, c->colrec.as<float>(), cm, max_points,
                                    xi == 0, c->stream)
                : launch_pifu_pair_fact(fd, c->geo_tc, c->geo_fact_tmap[0][xi], pj, c->colrec.as<float>(), cm,
                                        max_points, xi == 0, c->stream);
    prof_end(c, slot);
    c->launches += 2;
    return r;
}

// A large conflict-loop batch (size class 1) through the column-factored kernels: the level's
// column records persist from its E0 pass, so only columns the batch adds are claimed and
// recorded (COLS over the record window [ncols_base, ncols)), then the batch is sorted by record
// and evaluated by k_fact2.  Every launch is sized by device counts; the claim and k_fact2 exit on
// device unless the batch is their class (job.min_count).
int run_chain_fact(icg_context* c, const FieldDev& fd, const EvalJob& job, unsigned max_points) {
    const int xi = fd.precision == ICG_PREC_FP32 ? 0 : 1;
    const size_t n1 = (size_t)job.cells + 1, plane = n1 * n1;
    DevCounters* ctr = c->ctr.as<DevCounters>();
    if (int r = c->scan_bsum.ensure((plane + 8191) / 8192 * sizeof(unsigned))) return r;
    if (int r = launch_col_claim(job.list, job.count, job.cells, c->cmap.as<int>(), c->collist.as<uint32_t>(), ctr,
                                 max_points, c->stream, job.min_count))
        return r;
    if (int r = launch_sort_by_column(job.list, job.count, job.cells, c->cmap.as<int>(), c->colcnt.as<uint32_t>(), ctr,
                                      c->sorted.as<uint32_t>(), c->scan_bsum.as<unsigned>(), max_points, c->stream, job.min_count))
        return r;
    EvalJob cj{};
    cj.cells = job.cells;
    cj.list = c->collist.as<uint32_t>();
    cj.count = &ctr->ncols;
    cj.base = &ctr->ncols_base;
    const unsigned max_cols = (unsigned)std::min<size_t>(plane, max_points);
    if (int r = run_cols(c, fd, cj, max_cols, xi))
        return r;
    EvalJob pj = job;
    pj.list = c->sorted.as<uint32_t>();
    int r = launch_pifu_fact2(fd, c->geo_tc, c->geo_fact2_tmap[xi], pj, c->colrec.as<float>(), c->cmap.as<int>(),
                              max_points, xi == 0, c->stream);
    c->launches += 6;
    return r;
}

// `dependent_chain`: the batch is one link of the serial conflict loop, usually
// small; it is routed on device between the tensor-core kernel and the
// layer-parallel latency path by its size.
int run_eval(icg_context* c, const FieldDev& fd, const EvalJob& job, unsigned max_points,
             bool dependent_chain = false) {
    if (!dependent_chain && job_is_grid_host(job) && fact_ok(c, fd)) return run_eval_fact(c, fd, job, max_points);
    int slot = prof_begin(c, 0);
    int r;
    if (fd.kind == ICG_FIELD_ANALYTIC) {
        r = launch_analytic_eval(fd, job, max_points, c->stream);
    } else if (fd.precision == ICG_PREC_FP32_SIMT) {
        r = launch_pifu_simt_eval(fd, c->geo_simt, job, max_points, c->stream);
    } else {
        r = launch_pifu_pair_eval(fd, c->geo_tc, c->geo_pair_tmap[fd.precision == ICG_PREC_FP32 ? 0 : 1], job,
                                  max_points, fd.precision == ICG_PREC_FP32, c->stream);
    }
    prof_end(c, slot);
    c->launches += 1;
    return r;
}

// The texture chain's weights: packed once both networks are set (icg_set_mlp).
static int tg_upload(icg_context* c) {
    c->tg_ready = false;
    if (!c->host_w_set[0] || !c->host_w_set[1]) return ICG_OK;
    const float* gw[5];
    const float* tw[5];
    for (int l = 0; l < 5; ++l) {
        gw[l] = c->host_w[0][l].data();
        tw[l] = c->host_w[1][l].data();
    }
    std::vector<__half> w(tg_weight_elems());
    if (int r = tg_pack_weights(gw, tw, w.data(), c->tg_off)) return r;
    if (int r = c->tg_w.ensure(w.size() * 2)) return r;
    ICG_CUDA_TRY(cudaMemcpy(c->tg_w.p, w.data(), w.size() * 2, cudaMemcpyHostToDevice));
    const int nout[7] = {1024, 512, 256, 1024, 512, 256, 128};
    const int kin[7] = {256, 1024 + 256, 512 + 256, 512, 1024 + 512, 512 + 512, 256 + 512};
    for (int l = 0; l < 7; ++l) {
        const unsigned box = nout[l] >= 256 ? 128u : (unsigned)nout[l] / 2;
        if (int r = tg_make_tmap(c->tg_w.as<__half>() + c->tg_off[l], (size_t)nout[l], (size_t)kin[l], box, c->tg_mapW[l]))
            return r;
    }
    std::vector<float> w5((size_t)3 * kTgW5Stride, 0.0f);
    for (int o = 0; o < 3; ++o)
        for (int k = 0; k < 128 + kTexSkip; ++k) w5[(size_t)o * kTgW5Stride + k] = tw[4][(size_t)o * (128 + kTexSkip) + k];
    if (int r = c->tg_w5.ensure(w5.size() * 4)) return r;
    ICG_CUDA_TRY(cudaMemcpy(c->tg_w5.p, w5.data(), w5.size() * 4, cudaMemcpyHostToDevice));
    c->tg_ready = true;
    return ICG_OK;
}

// per-point activations of up to `n` points (+ their TMA descriptors)
static int tg_ensure(icg_context* c, unsigned n) {
    if (n <= c->tg_cap) return ICG_OK;
    const size_t cap = ((size_t)n + 255) / 256 * 256;
    if (int r = c->tg_skip.ensure(cap * 512 * 2)) return r;
    if (int r = c->tg_h1.ensure(cap * 1024 * 2)) return r;
    if (int r = c->tg_h2.ensure(cap * 512 * 2)) return r;
    if (int r = c->tg_h3.ensure(cap * 256 * 2)) return r;
    if (int r = c->tg_z.ensure(cap * 4)) return r;
    if (int r = c->tg_sdot.ensure(cap * 12)) return r;
    if (int r = tg_make_tmap(c->tg_skip.p, cap, 512, 128, c->tg_mapS)) return r;
    if (int r = tg_make_tmap(c->tg_h1.p, cap, 1024, 128, c->tg_mapH[0])) return r;
    if (int r = tg_make_tmap(c->tg_h2.p, cap, 512, 128, c->tg_mapH[1])) return r;
    if (int r = tg_make_tmap(c->tg_h3.p, cap, 256, 128, c->tg_mapH[2])) return r;
    if (int r = tg_make_tmap(c->tg_h1.p, cap, 1024, 32, c->tg_mapO[0])) return r;
    if (int r = tg_make_tmap(c->tg_h2.p, cap, 512, 32, c->tg_mapO[1])) return r;
    if (int r = tg_make_tmap(c->tg_h3.p, cap, 256, 32, c->tg_mapO[2])) return r;
    if (int r = tg_make_tmap(c->tg_skip.p, cap, 512, 32, c->tg_mapO[3])) return r;
    c->tg_cap = (unsigned)cap;
    return ICG_OK;
}

// Texture field at `job`'s points as gather + 7 layer GEMMs (k_texgemm.cu).  Bias blocks per layer
// l of the tc epilogue layout: [b (out), w_z (out)] at sum_{i<l} 2 out_i; final biases after.
static int run_texture_chain(icg_context* c, const FieldDev& fd, const EvalJob& job, unsigned max_points) {
    if (int r = tg_ensure(c, max_points)) return r;
    __half* skip = c->tg_skip.as<__half>();
    float* z = c->tg_z.as<float>();
    float* sdot = c->tg_sdot.as<float>();
    const float* w5 = c->tg_w5.as<float>();
    const float* gb = c->geo_tc.bias;
    const float* tb = c->tex_tc.bias;
    c->tg_C = fd.C;
    {
        const int gs = prof_begin(c, 6);
        const int r = launch_tex_gather(fd, job, max_points, skip, z, sdot, w5, tb + 3840, c->stream);
        prof_end(c, gs);
        if (r) return r;
    }
    struct L {
        int w, hmap, omap, n_out, hid, s1;
        const float* bias;
        __half* out;
        int ldo, out_col, w5_off, fin;
    };
    const L ls[7] = {
        {0, 0, 0, 1024, 0, 4, gb + 0, c->tg_h1.as<__half>(), 1024, 0, -1, 0},
        {1, 0, 1, 512, 16, 4, gb + 2048, c->tg_h2.as<__half>(), 512, 0, -1, 0},
        {2, 1, 3, 256, 8, 4, gb + 3072, skip, 512, 256, 128 + 256, 0},  // h3 -> skip columns 256-511
        {3, 0, 0, 1024, 0, 8, tb + 0, c->tg_h1.as<__half>(), 1024, 0, -1, 0},
        {4, 0, 1, 512, 16, 8, tb + 2048, c->tg_h2.as<__half>(), 512, 0, -1, 0},
        {5, 1, 2, 256, 8, 8, tb + 3072, c->tg_h3.as<__half>(), 256, 0, -1, 0},
        {6, 2, 2, 128, 4, 8, tb + 3584, nullptr, 0, 0, 0, 1},
    };
    for (const L& l : ls) {
        TgLayer t{};
        t.count = job.count;
        t.n_static = job.n_static;
        t.n_out = l.n_out;
        t.hid_chunks = l.hid;
        t.skip_c0 = 0;
        t.skip_c1 = l.s1;
        t.bias = l.bias;
        t.z = z;
        t.slope = 0.02f;
        t.out = l.out;
        t.ldo = l.ldo;
        t.out_col = l.out_col;
        t.w5 = l.w5_off >= 0 ? w5 : nullptr;
        t.w5_off = l.w5_off;
        t.sdot = sdot;
        t.final_layer = l.fin;
        t.rgb = job.out;
        t.out_pixel = job.out_pixel;
        t.pdl = c->tg_pdl && &l != &ls[0];  // g1 follows the gather (a plain launch)
        if (int r = launch_tex_layer(c->tg_mapH[l.hmap], c->tg_mapS, c->tg_mapW[l.w], c->tg_mapO[l.omap], t, max_points,
                                     c->stream))
            return r;
    }
    c->launches += 7;  // + the gather (counted by the caller)
    return ICG_OK;
}

int run_texture(icg_context* c, const FieldDev& fd, const EvalJob& job, unsigned max_points) {
    int slot = prof_begin(c, 1);
    int r;
    if (fd.kind == ICG_FIELD_ANALYTIC)
        r = launch_analytic_texture(fd, job, max_points, c->stream);
    else if (fd.precision == ICG_PREC_FP32_SIMT)
        r = launch_pifu_simt_texture(fd, c->geo_simt, c->tex_simt, job, max_points, c->stream);
    else if (c->tg_ready && c->use_tg)
        r = run_texture_chain(c, fd, job, max_points);
    else
        // one fp16 copy of every weight and operand, one MMA per K step, at every precision:
        // colours within 5.2e-4 of fp64 (scripts/tex_precision.py; tolerance 1e-3)
        r = launch_pifu_pair_texture(fd, c->geo_tc, c->tex_tc, c->geo_pair_f16_tmap[1], c->tex_pair_tmap[1], job,
                                     max_points, false, c->stream);
    prof_end(c, slot);
    c->launches += 1;
    return r;
}

int issue_tail(icg_context* c, const FieldDev& fd, const LevelBufs& lb, int level, int fcells, int it, int max_iters,
               unsigned nf) {
    const unsigned cap_pts = 4096, cap_new = 4096;
    const size_t plane = ((size_t)fcells + 1) * ((size_t)fcells + 1);
    if (int r = c->tail_scratch.ensure(tail_scratch_bytes(cap_pts, cap_new, (unsigned)plane))) return r;
    TailParams tp{};
    tp.f = fd;
    tp.xext = lb.xext;
    tp.cells = fcells;
    tp.level = level;
    tp.it0 = it;
    tp.max_iters = max_iters;
    tp.cap = nf;
    tp.max_start = c->tail_max;
    tp.fv = lb.fv;
    tp.fs = lb.fs;
    tp.tentbin = lb.tentbin;
    tp.queued = c->queued.as<uint32_t>();
    for (int b = 0; b < 2; ++b) {
        tp.cf[b] = c->cf[b].as<uint32_t>();
        tp.nx[b] = c->nx[b].as<uint32_t>();
    }
    tp.ctr = c->ctr.as<DevCounters>();
    tp.colrec = c->colrec.as<float>();
    tp.cmap = c->cmap.as<int>();
    tp.collist = c->collist.as<uint32_t>();
    for (int l = 0; l < 4; ++l) tp.w[l] = c->geo_rows[l];
    tp.bias = c->geo_tc.bias;
    tp.wlast = c->geo_tc.w_last;
    tp.slope = 0.02f;
    return launch_tail(tp, c->tail_scratch.as<uint8_t>(), cap_pts, cap_new, (unsigned)plane, c->stream, c->tail_wide);
}

// Issues one whole extraction on the context stream (no host sync).
// keep_xext: the target level's x-line extents are kept in c->xext by the level pass and every
// evaluation epilogue (icg_frame's renderer then skips k_xline_extents; progressive variant only)
int issue_extract(icg_context* c, const FieldDev& fd, const icg_algo_config* cfg, bool keep_xext = false) {
    prof_discard(c);
    c->fact_used = false;
    DevCounters* ctr = c->ctr.as<DevCounters>();
    ICG_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(DevCounters), c->stream));
    const int L = cfg->target_level;
    const int RL = cfg->coarsest_cells << L;
    if (cfg->variant == ICG_VARIANT_BRUTE) {
        // extract_brute_force, localize.hpp:181-193
        EvalJob job{};
        job.cells = RL;
        job.n_static = (unsigned)nodes3(RL);
        job.values = c->vals[0].as<float>();
        job.states = c->sts[0].as<uint8_t>();
        job.evals = &ctr->evals[L];
        job.overflow = &ctr->overflow;
        if (int r = run_eval(c, fd, job, job.n_static)) return r;
        c->last_buf = 0;
        c->last_cells = RL;
        return ICG_OK;
    }
    // L0: evaluate_full (localize.hpp:322)
    int cells = cfg->coarsest_cells;
    int b = 0;
    {
        EvalJob job{};
        job.cells = cells;
        job.n_static = (unsigned)nodes3(cells);
        job.values = c->vals[b].as<float>();
        job.states = c->sts[b].as<uint8_t>();
        job.evals = &ctr->evals[0];
        job.overflow = &ctr->overflow;
        if (int r = run_eval(c, fd, job, job.n_static)) return r;
    }
    const bool octree = cfg->variant == ICG_VARIANT_OCTREE_BINARIZED || cfg->variant == ICG_VARIANT_OCTREE_THRESHOLD;
    for (int l = 1; l <= L; ++l) {
        const int fcells = 2 * cells;
        const size_t nf = nodes3(fcells);
        LevelBufs lb{};
        lb.cv = c->vals[b].as<float>();
        lb.cs = c->sts[b].as<uint8_t>();
        lb.fv = c->vals[b ^ 1].as<float>();
        lb.fs = c->sts[b ^ 1].as<uint8_t>();
        lb.cbin = c->cbin.as<uint32_t>();
        lb.mixed = c->mixed.as<uint32_t>();
        lb.tentbin = c->tentbin.as<uint32_t>();
        lb.sel = c->sel.as<uint32_t>();
        lb.queued = c->queued.as<uint32_t>();
        lb.block_counts = c->block_counts.as<uint32_t>();
        lb.list = c->list_e0.as<uint32_t>();
        lb.rc = cells;
        if (keep_xext && !octree && l == L) {
            if (int r = c->xext.ensure(((size_t)fcells + 1) * ((size_t)fcells + 1) * sizeof(int2))) return r;
            lb.xext = c->xext.as<int2>();
        }
        if (octree) {
            // Fig. 4 baselines: mark cells, build the fine grid, evaluate the nodes of marked cells
            const int mode = cfg->variant == ICG_VARIANT_OCTREE_BINARIZED ? 0 : 1;
            {
                int slot = prof_begin(c, 2);
                int r = launch_octree_level(lb, lb.queued, mode, cfg->threshold, ctr, l, c->stream);
                prof_end(c, slot);
                c->launches += mode == 0 ? 4 : 2;
                if (r) return r;
            }
            if (int r = c->set_scratch.ensure(bits_to_list_scratch_words(nf) * 4)) return r;
            if (int r = launch_bits_to_list(lb.sel, nf, c->set_scratch.as<uint32_t>(), lb.list, &ctr->list_count,
                                            c->stream))
                return r;
            c->launches += 3;
            EvalJob job{};
            job.list = lb.list;
            job.count = &ctr->list_count;
            job.cells = fcells;
            job.values = lb.fv;
            job.states = lb.fs;
            job.evals = &ctr->evals[l];
            job.overflow = &ctr->overflow;
            if (int r = run_eval(c, fd, job, (unsigned)nf)) return r;
            if (cfg->keep_level_sets) {
                const size_t ncell = (size_t)cells * cells * cells;
                if (int r = c->lvl_bits[0][l].ensure(words(nf) * 4 + 16)) return r;
                if (int r = c->lvl_bits[1][l].ensure(words(ncell) * 4 + 16)) return r;
                if (int r = launch_level_eval_bits(lb.fs, lb.cs, cells, c->lvl_bits[0][l].as<uint32_t>(), c->stream))
                    return r;
                ICG_CUDA_TRY(cudaMemcpyAsync(c->lvl_bits[1][l].p, c->mixed.p, words(ncell) * 4,
                                             cudaMemcpyDeviceToDevice, c->stream));
                c->launches += 1;
            }
            b ^= 1;
            cells = fcells;
            continue;
        }
        {
            int slot = prof_begin(c, l == cfg->target_level ? 8 : 2);
            int r = launch_level_classify(lb, ctr, l, c->stream);
            prof_end(c, slot);
            c->launches += 5;
            if (r) return r;
        }
        ICG_CUDA_TRY(cudaMemsetAsync(c->queued.p, 0, words(nf) * 4, c->stream));
        // evaluate E0 (localize.hpp:331-332) with the fused conflict test
        EvalJob job{};
        job.list = c->list_e0.as<uint32_t>();
        job.count = &ctr->list_count;
        job.cells = fcells;
        job.values = lb.fv;
        job.states = lb.fs;
        job.overflow = &ctr->overflow;
        job.xext = lb.xext;
        if (cfg->conflict_pass) {
            job.tentbin = lb.tentbin;
            job.conflicts = c->cf[0].as<uint32_t>();
            job.conflict_count = &ctr->cf_count[0];
            job.conflict_cap = (unsigned)nf;
        }
        if (int r = run_eval(c, fd, job, (unsigned)nf)) return r;
        if (cfg->conflict_pass) {
            int max_iters = cfg->max_conflict_iters > 0 ? cfg->max_conflict_iters : fcells;
            const int unroll = c->unroll[l];
            // size-class prediction: only the evaluators the previous frames needed at each
            // iteration are enqueued; a batch that meets none raises `mispredict` (checked on
            // device by the next expansion) and the frame is replayed with all of them
            const bool chain_pred = fact_ok(c, fd) && c->use_tail && c->geo_pair;
            const unsigned mid_max = 74u * 64u;
            // batches beyond one wave of 128-point pair tiles: column-factored (k_fact2, 256-point tiles)
            const bool x3c = fd.precision == ICG_PREC_FP32;
            const unsigned cfm = c->chain_fact_min ? c->chain_fact_min : (x3c ? 74u * 64u : 74u * 128u);
            const unsigned big_max = (c->chain_fact && c->use_fact2) ? cfm : 0u;
            int prev_mask = -1;
            for (int it = 0; it < unroll; ++it) {
                int p = it & 1;
                const int pm =
                    (chain_pred && c->pred_valid[l] && !c->pred_all[l] && it < kPredIters) ? c->pred[l][it] : 15;
                {
                    int slot = prof_begin(c, 7);
                    ChainClasses cc{c->tail_max, mid_max, l, chain_pred ? prev_mask : -1, big_max};
                    int r = launch_conflict_expand_cls(c->queued.as<uint32_t>(), lb.fs, fcells,
                                                       c->cf[p].as<uint32_t>(), ctr, it, max_iters,
                                                       c->nx[p].as<uint32_t>(), (unsigned)nf, cc, c->stream);
                    prev_mask = pm;
                    prof_end(c, slot);
                    c->launches += 1;
                    if (r) return r;
                }
                EvalJob cj{};
                cj.list = c->nx[p].as<uint32_t>();
                cj.count = &ctr->nx_count[p];
                cj.cells = fcells;
                cj.values = lb.fv;
                cj.states = lb.fs;
                cj.tentbin = lb.tentbin;
                cj.conflicts = c->cf[p ^ 1].as<uint32_t>();
                cj.conflict_count = &ctr->cf_count[p ^ 1];
                cj.conflict_cap = (unsigned)nf;
                cj.evals = &ctr->evals[l];
                cj.iters = &ctr->conflict_iters[l];
                cj.overflow = &ctr->overflow;
                cj.xext = lb.xext;
                if (chain_pred) {
                    // large batches: the CTA-pair kernel; the first small one starts the persistent tail,
                    // which finishes the level's chain (k_tail.cu)
                    // (mid-size batches: 64-point pair tiles, twice as many pairs busy per wave; the
                    // column-factored pass has a longer single-tile latency, so it is kept for bulk batches)
                    EvalJob huge = cj, big = cj, mid = cj;
                    huge.min_count = big_max + 1;
                    big.min_count = std::max(c->tail_max, mid_max) + 1;
                    big.max_count = big_max;
                    mid.min_count = c->tail_max + 1;
                    mid.max_count = mid_max;
                    int slot = prof_begin(c, 5);
                    const bool x3 = x3c;
                    const void* tm = c->geo_pair_tmap[x3 ? 0 : 1];
                    int r = ICG_OK;
                    if ((pm & 8) && big_max) r = run_chain_fact(c, fd, huge, (unsigned)nf);
                    if (!r && (pm & 1)) {
                        r = launch_pifu_pair_eval(fd, c->geo_tc, tm, big, (unsigned)nf, x3, c->stream);
                        c->launches += 1;
                    }
                    if (!r && (pm & 2) && c->tail_max < mid_max) {
                        r = launch_pifu_pair_eval_small(fd, c->geo_tc, tm, mid, mid_max, x3, c->stream);
                        c->launches += 1;
                    }
                    if (!r && (pm & 4)) {
                        r = issue_tail(c, fd, lb, l, fcells, it, max_iters, (unsigned)nf);
                        c->launches += 1;
                    }
                    prof_end(c, slot);
                    if (r) return r;
                    if (c->chain_trace) {  // dev aid: batch size of every iteration (synchronises)
                        DevCounters h;
                        cudaStreamSynchronize(c->stream);
                        cudaMemcpy(&h, ctr, sizeof(h), cudaMemcpyDeviceToHost);
                        fprintf(stderr, "[chain] level %d it %d batch %u tail_start %u\n", l, it, h.nx_count[p],
                                h.tail_start[l]);
                    }
                } else if (int r = run_eval(c, fd, cj, (unsigned)nf, true)) {
                    return r;
                }
            }
            {
                ChainClasses cc{c->tail_max, mid_max, l, chain_pred ? prev_mask : -1, big_max};
                if (int r = launch_unroll_check_cls(ctr, unroll & 1, l, cc, chain_pred ? unroll - 1 : -1, c->stream))
                    return r;
            }
            c->launches += 1;
        }
        if (cfg->keep_level_sets) {
            const size_t ncell = (size_t)cells * cells * cells;
            if (int r = c->lvl_bits[0][l].ensure(words(nf) * 4 + 16)) return r;
            if (int r = c->lvl_bits[1][l].ensure(words(ncell) * 4 + 16)) return r;
            if (int r = launch_level_eval_bits(lb.fs, lb.cs, cells, c->lvl_bits[0][l].as<uint32_t>(), c->stream))
                return r;
            ICG_CUDA_TRY(cudaMemcpyAsync(c->lvl_bits[1][l].p, c->mixed.p, words(ncell) * 4, cudaMemcpyDeviceToDevice,
                                         c->stream));
            c->launches += 1;
        }
        b ^= 1;
        cells = fcells;
    }
    c->last_buf = b;
    c->last_cells = cells;
    return ICG_OK;
}

// render_view's depth pass (render.hpp:89-215) on the context stream: view-space localization to
// level L-1 (issue_extract with the view-field wrap), then the level-L passes of k_depth.cu;
// `texture`: render_view (texture at covered pixels) else surface_depth_map.  Outputs in the
// context's render buffers, (R_L+1)^2 pixels.
int issue_depth_pass(icg_context* c, FieldDev fd, const icg_algo_config* cfg, const icg_camera* cam, const float* bg,
                     bool texture) {
    fd.view = 1;
    for (int k = 0; k < 9; ++k) fd.vr[k] = cam->rotation[k];
    for (int k = 0; k < 3; ++k) fd.vt[k] = cam->translation[k];
    fd.vs = cam->scale;
    icg_algo_config sub = *cfg;
    sub.target_level = cfg->target_level - 1;
    sub.keep_level_sets = 0;
    if (int r = issue_extract(c, fd, &sub)) return r;
    const int L = cfg->target_level, rc = c->last_cells, fcells = 2 * rc;
    const int b = c->last_buf;
    const size_t nf = nodes3(fcells), fn = (size_t)fcells + 1, npx = fn * fn;
    DevCounters* ctr = c->ctr.as<DevCounters>();
    LevelBufs lb{};
    lb.cv = c->vals[b].as<float>();
    lb.cs = c->sts[b].as<uint8_t>();
    lb.fv = c->vals[b ^ 1].as<float>();
    lb.fs = c->sts[b ^ 1].as<uint8_t>();
    lb.cbin = c->cbin.as<uint32_t>();
    lb.mixed = c->mixed.as<uint32_t>();
    lb.tentbin = c->tentbin.as<uint32_t>();
    lb.sel = c->sel.as<uint32_t>();
    lb.queued = c->queued.as<uint32_t>();
    lb.block_counts = c->block_counts.as<uint32_t>();
    lb.list = c->list_e0.as<uint32_t>();
    lb.rc = rc;
    {
        int slot = prof_begin(c, 2);
        int r = launch_level_carry(lb, ctr, L, c->stream);
        prof_end(c, slot);
        c->launches += 3;
        if (r) return r;
    }
    if (int r = c->set_scratch.ensure(bits_to_list_scratch_words(nf) * 4)) return r;
    DepthJob dj{};
    dj.cbin = lb.cbin;
    dj.rc = rc;
    dj.fv = lb.fv;
    dj.fs = lb.fs;
    dj.sel = lb.sel;
    if (int r = c->xext.ensure(npx * sizeof(int2))) return r;
    dj.colk = reinterpret_cast<int*>(c->xext.p);
    // evaluate the nodes of the sel bitset (ascending) into the level-L grid, counted at level L
    auto eval_sel = [&]() -> int {
        if (int r = launch_bits_to_list(lb.sel, nf, c->set_scratch.as<uint32_t>(), lb.list, &ctr->list_count,
                                        c->stream))
            return r;
        c->launches += 3;
        EvalJob job{};
        job.list = lb.list;
        job.count = &ctr->list_count;
        job.cells = fcells;
        job.values = lb.fv;
        job.states = lb.fs;
        job.evals = &ctr->evals[L];
        job.overflow = &ctr->overflow;
        return run_eval(c, fd, job, (unsigned)nf);
    };
    ICG_CUDA_TRY(cudaMemsetAsync(lb.sel, 0, (words(nf) + 1) * 4, c->stream));
    if (int r = launch_depth_shadow(dj, c->stream)) return r;
    if (int r = eval_sel()) return r;
    ICG_CUDA_TRY(cudaMemsetAsync(lb.sel, 0, (words(nf) + 1) * 4, c->stream));
    if (int r = launch_depth_bracket(dj, c->stream)) return r;
    if (int r = eval_sel()) return r;
    c->launches += 2;
    // per-pixel depth + surface points
    if (int r = c->depth.ensure(npx * 4)) return r;
    if (int r = c->rgb.ensure(npx * 12)) return r;
    if (int r = c->mask.ensure(npx)) return r;
    if (int r = c->surfk.ensure(npx * 4)) return r;
    if (int r = c->spts.ensure(npx * 24)) return r;
    if (int r = c->spx.ensure(npx * 4)) return r;
    ICG_CUDA_TRY(cudaMemsetAsync(&ctr->covered, 0, sizeof(DevCounters) - offsetof(DevCounters, covered), c->stream));
    for (int k = 0; k < 9; ++k) dj.vr[k] = cam->rotation[k];
    for (int k = 0; k < 3; ++k) {
        dj.vt[k] = cam->translation[k];
        dj.bg[k] = bg ? bg[k] : 0.0f;
    }
    dj.vs = cam->scale;
    dj.depth = c->depth.as<float>();
    dj.rgb = c->rgb.as<float>();
    dj.mask = c->mask.as<uint8_t>();
    dj.surface_k = c->surfk.as<int32_t>();
    dj.surface_pts = c->spts.as<double>();
    dj.surface_px = c->spx.as<uint32_t>();
    dj.ctr = ctr;
    {
        int slot = prof_begin(c, 3);
        int r = launch_depth_final(dj, c->stream);
        prof_end(c, slot);
        c->launches += 1;
        if (r) return r;
    }
    if (texture) {
        EvalJob tj{};
        tj.points = c->spts.as<double>();
        tj.count = &ctr->surface_count;
        tj.out = c->rgb.as<float>();
        tj.out_pixel = c->spx.as<uint32_t>();
        tj.out_clamp = 1.0f;
        FieldDev tf = fd;  // texture at world points: no view wrap
        tf.view = 0;
        if (int r = run_texture(c, tf, tj, (unsigned)npx)) return r;
    }
    c->last_buf = b ^ 1;
    c->last_cells = fcells;
    return ICG_OK;
}

int copy_out(icg_context* c, void* dst, const void* src, size_t bytes, int mem) {
    if (!dst) return ICG_OK;
    ICG_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, mem == ICG_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                 c->stream));
    return ICG_OK;
}

int finish_extract_outputs(icg_context* c, const icg_algo_config* cfg, icg_extraction* out) {
    if (!out) return ICG_OK;
    if (out->mem != ICG_MEM_HOST && out->mem != ICG_MEM_DEVICE) return einval("extraction: bad mem");
    size_t N = nodes3(c->last_cells);
    if (int r = copy_out(c, out->values, c->vals[c->last_buf].p, N * 4, out->mem)) return r;
    if (int r = copy_out(c, out->states, c->sts[c->last_buf].p, N, out->mem)) return r;
    if (out->binarized) {
        if (int r = c->binar.ensure(N)) return r;
        if (int r = launch_binarize(c->vals[c->last_buf].as<float>(), c->binar.as<uint8_t>(), N, c->stream)) return r;
        c->launches += 1;
        if (int r = copy_out(c, out->binarized, c->binar.p, N, out->mem)) return r;
    }
    (void)cfg;
    return ICG_OK;
}

void fill_extraction_scalars(icg_context* c, const icg_algo_config* cfg, icg_extraction* out, double secs) {
    if (!out) return;
    const DevCounters& h = *c->h_ctr;
    out->cells = c->last_cells;
    out->levels = cfg->target_level + 1;
    out->total_evals = 0;
    for (int l = 0; l < ICG_MAX_LEVELS; ++l) {
        out->evals_per_level[l] = l <= cfg->target_level ? h.evals[l] : 0;
        out->refined_cells_per_level[l] = l <= cfg->target_level ? h.refined[l] : 0;
        out->conflict_iters_per_level[l] = l <= cfg->target_level ? h.conflict_iters[l] : 0;
        out->total_evals += out->evals_per_level[l];
    }
    out->conflict_warning = h.warning ? 1 : 0;
    out->wall_seconds = secs;
}

int sync_counters(icg_context* c) {
    ICG_CUDA_TRY(cudaMemcpyAsync(c->h_ctr, c->ctr.p, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->stream));
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return ICG_OK;
}

// xext_ready: c->xext already holds the rendered grid's x-line extents (issue_extract keep_xext)
int issue_render(icg_context* c, const FieldDev& fd, const icg_camera* cam, int W, int H, const float* bg,
                 bool xext_ready = false) {
    size_t npx = (size_t)W * H;
    if (int r = c->depth.ensure(npx * 4)) return r;
    if (int r = c->rgb.ensure(npx * 12)) return r;
    if (int r = c->mask.ensure(npx)) return r;
    if (int r = c->surfk.ensure(npx * 4)) return r;
    if (int r = c->spts.ensure(npx * 24)) return r;
    if (int r = c->spx.ensure(npx * 4)) return r;
    DevCounters* ctr = c->ctr.as<DevCounters>();
    // clear render counters (covered .. surface_count)
    ICG_CUDA_TRY(cudaMemsetAsync(&ctr->covered, 0, sizeof(DevCounters) - offsetof(DevCounters, covered), c->stream));
    RenderJob rj{};
    rj.values = c->vals[c->last_buf].as<float>();
    rj.cells = c->last_cells;
    for (int i = 0; i < 9; ++i) rj.rot[i] = cam->rotation[i];
    for (int i = 0; i < 3; ++i) rj.trans[i] = cam->translation[i];
    rj.scale = cam->scale;
    rj.width = W;
    rj.height = H;
    for (int i = 0; i < 3; ++i) rj.bg[i] = bg ? bg[i] : 0.0f;
    rj.depth = c->depth.as<float>();
    rj.rgb = c->rgb.as<float>();
    rj.mask = c->mask.as<uint8_t>();
    rj.surface_k = c->surfk.as<int32_t>();
    rj.surface_pts = c->spts.as<double>();
    rj.surface_px = c->spx.as<uint32_t>();
    rj.ctr = ctr;
    if (int r = c->rtab.ensure(render_tab_doubles(W, H, rj.cells) * sizeof(double))) return r;
    rj.tab = c->rtab.as<double>();
    {
        int slot = prof_begin(c, 3);
        // rays along world x (the view direction R^T e_z has no y / z part): empty-space skipping
        if (c->use_xext && std::fabs(cam->rotation[7]) < 1e-9 && std::fabs(cam->rotation[8]) < 1e-9) {
            if (!xext_ready) {
                const size_t lines = ((size_t)rj.cells + 1) * ((size_t)rj.cells + 1);
                if (int r = c->xext.ensure(lines * sizeof(int2))) return r;
                if (int r = launch_xline_extents(rj.values, rj.cells, c->xext.as<int2>(), c->stream)) return r;
                c->launches += 1;
            }
            rj.xext = c->xext.as<int2>();
        }
        int r = launch_render_first_crossing(rj, c->stream);
        prof_end(c, slot);
        c->launches += 2;
        if (r) return r;
    }
    if (fd.kind == ICG_FIELD_PIFU && c->has_tex) {
        EvalJob tj{};
        tj.points = c->spts.as<double>();
        tj.count = &ctr->surface_count;
        tj.out = c->rgb.as<float>();
        tj.out_pixel = c->spx.as<uint32_t>();
        tj.out_clamp = 1.0f;
        if (int r = run_texture(c, fd, tj, (unsigned)npx)) return r;
    }
    return ICG_OK;
}

int finish_render_outputs(icg_context* c, int W, int H, icg_image* out) {
    if (!out) return ICG_OK;
    if (out->mem != ICG_MEM_HOST && out->mem != ICG_MEM_DEVICE) return einval("image: bad mem");
    size_t npx = (size_t)W * H;
    if (int r = copy_out(c, out->depth, c->depth.p, npx * 4, out->mem)) return r;
    if (int r = copy_out(c, out->rgb, c->rgb.p, npx * 12, out->mem)) return r;
    if (int r = copy_out(c, out->mask, c->mask.p, npx, out->mem)) return r;
    if (int r = copy_out(c, out->surface_k, c->surfk.p, npx * 4, out->mem)) return r;
    return ICG_OK;
}

void fill_image_scalars(icg_context* c, icg_image* out, double secs) {
    if (!out) return;
    const DevCounters& h = *c->h_ctr;
    out->covered_pixels = h.covered;
    out->degenerate_brackets = h.degenerate;
    out->grazing_pixels = h.grazing;
    out->texture_points = h.surface_count;
    out->wall_seconds = secs;
}

int check_render_args(icg_context* c, const icg_camera* cam, int W, int H) {
    if (!cam) return einval("render: null camera");
    if (W < 2 || H < 2 || (size_t)W * H > (size_t)1 << 26) return einval("render: image size out of range");
    if (!(cam->scale != 0.0)) return einval("render: camera scale must be nonzero");
    (void)c;
    return ICG_OK;
}

// fold one finished extraction / render into the profile totals
void prof_extract_done(icg_context* c, const icg_algo_config* cfg) {
    if (!c->prof_on) return;
    const DevCounters& h = *c->h_ctr;
    for (int l = 0; l <= cfg->target_level; ++l) c->prof.geo_points += h.evals[l];
    if (c->fact_used && cfg->variant == ICG_VARIANT_PROGRESSIVE) {
        c->prof.fact_points += h.evals[0];
        for (int l = 1; l <= cfg->target_level; ++l) {
            c->prof.fact_points += h.e0[l];
            c->prof.chain_points += h.evals[l] - h.e0[l];
        }
    }
    if (cfg->variant == ICG_VARIANT_PROGRESSIVE) {
        for (int l = 1; l <= cfg->target_level; ++l) {
            // level pass: fine value+state written, coarse read, index list
            const uint64_t b = 5 * nodes3(cfg->coarsest_cells << l) + 5 * nodes3(cfg->coarsest_cells << (l - 1)) +
                               4 * h.evals[l];
            c->prof.dense_bytes += b;
            if (l == cfg->target_level) c->prof.last_level_bytes += b;
        }
    }
}
void prof_render_done(icg_context* c, int W, int H) {
    if (!c->prof_on) return;
    c->prof.tex_points += c->h_ctr->surface_count;
    if (c->tg_ready && c->use_tg) {
        c->prof.gather_points += c->h_ctr->surface_count;
        c->prof.gather_bytes += 16ull * (uint64_t)c->tg_C * c->h_ctr->surface_count;
    }
    c->prof.render_bytes += 4 * nodes3(c->last_cells) + 17ull * (uint64_t)W * (uint64_t)H;
}

float elapsed(icg_context* c) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, c->e0, c->e1);
    return ms * 1e-3f;
}

// After a successful extraction, size each level's device loop to what this
// frame needed plus a margin; when a level ran out, deepen it and replay.
bool adapt_unroll(icg_context* c, const icg_algo_config* cfg) {
    const DevCounters& h = *c->h_ctr;
    bool replay = false;
    if (h.mispredict) {  // a conflict batch met no launched evaluator: all evaluators for that level
        for (int l = 1; l <= cfg->target_level; ++l)
            if (h.mispredict & (1u << l)) c->pred_all[l] = true;  // replay with every evaluator
        return true;
    }
    for (int l = 1; l <= cfg->target_level; ++l) {
        if (h.unroll_exhausted & (1u << l)) {
            c->unroll[l] *= 2;
            replay = true;
        }
    }
    if (!replay)
        for (int l = 1; l <= cfg->target_level; ++l) {
            // host-side iterations: up to the one where the persistent tail took over
            // (once started, the tail finishes the level: a margin of one iteration covers frames
            // whose chain hands over one iteration later)
            // grow-only: frames of a stream differ a little, and a stable depth keeps the frame's
            // CUDA graph valid (a shallower depth would only save a few early-exit launches)
            int need = h.tail_start[l] ? (int)h.tail_start[l] + 1
                                       : (int)h.conflict_iters[l] + std::max(2, (int)h.conflict_iters[l] / 4);
            c->unroll[l] = std::max(c->unroll_seen[l], need);
            c->unroll_seen[l] = c->unroll[l];
            // size classes: the first clean frame sets them, later ones only add (grow-only)
            for (int it = 0; it < kPredIters; ++it)
                c->pred[l][it] = c->pred_valid[l] ? (uint8_t)(c->pred[l][it] | h.cls[l][it]) : h.cls[l][it];
            c->pred_valid[l] = true;
            c->pred_all[l] = false;
        }
    return replay;
}

int do_extract(icg_context* c, const FieldDev& fd, const icg_algo_config* cfg) {
    for (int attempt = 0;; ++attempt) {
        if (int r = issue_extract(c, fd, cfg)) return r;
        if (int r = sync_counters(c)) return r;
        if (c->h_ctr->overflow) {
            set_error("extract: device work list overflow");
            return ICG_ECAPACITY;
        }
        if (!adapt_unroll(c, cfg)) return ICG_OK;
        if (attempt > 12) {
            set_error("extract: conflict loop did not converge");
            return ICG_ERUNTIME;
        }
    }
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int icg_abi_version(void) { return ICG_ABI_VERSION; }
const char* icg_last_error(void) { return g_err.c_str(); }

int icg_device_count(int* count) {
    if (!count) return einval("null count");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) n = 0;
    *count = n;
    return ICG_OK;
}

int icg_create(int device, icg_context** out) {
    if (!out) return einval("null output");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        set_error("no CUDA device");
        return ICG_ENODEV;
    }
    if (device < 0 || device >= n) return einval("device index out of range");
    ICG_CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    ICG_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        set_error("this build targets sm_100a (B200); device is sm_" + std::to_string(prop.major) +
                  std::to_string(prop.minor));
        return ICG_ENODEV;
    }
    auto* c = new icg_context();
    c->device = device;
    if (const char* e = getenv("ICG_NO_FACT")) c->use_fact = !(e[0] == '1');
    if (const char* e = getenv("ICG_NO_TAIL")) c->use_tail = !(e[0] == '1');
    if (const char* e = getenv("ICG_NO_GRAPH")) c->use_graph = !(e[0] == '1');
    if (getenv("ICG_TC_TRACE") || getenv("ICG_TAIL_TRACE")) c->use_graph = false;  // traces synchronise
    if (const char* e = getenv("ICG_FACT2")) c->use_fact2 = e[0] == '1';
    if (const char* e = getenv("ICG_TEX_PAIR")) c->use_tg = !(e[0] == '1');
    if (const char* e = getenv("ICG_TG_PDL")) c->tg_pdl = e[0] == '1';
    if (const char* e = getenv("ICG_COLS_PAIR")) c->use_cg = !(e[0] == '1');
    if (const char* e = getenv("ICG_CHAIN_FACT")) c->chain_fact = e[0] == '1';
    if (const char* e = getenv("ICG_CHAIN_FACT_MIN")) c->chain_fact_min = (unsigned)atoi(e);
    if (const char* e = getenv("ICG_NO_XEXT")) c->use_xext = !(e[0] == '1');
    if (getenv("ICG_CHAIN_TRACE")) {
        c->chain_trace = true;
        c->use_graph = false;
    }
    if (const char* e = getenv("ICG_TAIL_MAX")) c->tail_max = (unsigned)atoi(e);
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&c->e0) != cudaSuccess || cudaEventCreate(&c->e1) != cudaSuccess ||
        cudaMallocHost(&c->h_scene, sizeof(DevScene)) != cudaSuccess ||
        cudaMallocHost(&c->h_fscene, sizeof(FScene)) != cudaSuccess ||
        cudaMallocHost(&c->h_ctr, sizeof(DevCounters)) != cudaSuccess) {
        set_error("icg_create: CUDA resource allocation failed");
        delete c;
        return ICG_ERUNTIME;
    }
    if (int r = c->ctr.ensure(sizeof(DevCounters))) {
        delete c;
        return r;
    }
    *out = c;
    return ICG_OK;
}

int icg_destroy(icg_context* c) {
    if (!c) return ICG_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    DBuf* all[] = {&c->geo_bias, &c->geo_wlast, &c->tex_bias, &c->tex_wlast,
                   &c->scene, &c->fscene, &c->fmap_chw, &c->fmap_hwc, &c->vals[0], &c->vals[1], &c->sts[0], &c->sts[1],
                   &c->cbin, &c->mixed, &c->tentbin, &c->sel, &c->queued, &c->block_counts, &c->list_e0,
                   &c->cf[0], &c->cf[1], &c->nx[0], &c->nx[1], &c->ctr, &c->binar, &c->pts, &c->outv, &c->geo_pair_stream, &c->tex_pair_stream, &c->geo_pair_hi, &c->tex_pair_hi, &c->geo_pair_f16, &c->geo_pair_f16_hi,
                   &c->depth, &c->rgb, &c->mask, &c->surfk, &c->spts, &c->spx, &c->colrec, &c->cmap, &c->collist, &c->colcnt, &c->sorted, &c->tail_scratch,
                   &c->set_scratch, &c->set_list, &c->set_total, &c->set_bits, &c->mc_grid, &c->mc_blocks,
                   &c->mc_total, &c->mc_tri_keys, &c->mc_key_bits, &c->mc_keys, &c->mc_tri_ids, &c->mc_keep,
                   &c->mc_first, &c->mc_slot_bits, &c->mc_slots, &c->mc_tri_list, &c->mc_new_id, &c->mc_out_v,
                   &c->mc_out_t,
                   &c->geo_fact_stream[0][0], &c->geo_fact_stream[0][1], &c->geo_fact_stream[1][0],
                   &c->geo_fact_stream[1][1], &c->tg_w, &c->tg_w5, &c->tg_skip, &c->tg_h1, &c->tg_h2, &c->tg_h3,
                   &c->tg_z, &c->tg_sdot, &c->cg_ah, &c->cg_al, &c->cg_w};
    for (DBuf* b : all) b->release();
    for (auto& lv : c->lvl_bits)
        for (DBuf& b : lv) b.release();
    for (int l = 0; l < 5; ++l) {
        c->geo_wt[l].release();
        c->geo_wrow[l].release();
        c->geo_b[l].release();
        c->tex_wt[l].release();
        c->tex_b[l].release();
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    if (c->h_scene) cudaFreeHost(c->h_scene);
    if (c->h_fscene) cudaFreeHost(c->h_fscene);
    if (c->h_ctr) cudaFreeHost(c->h_ctr);
    if (c->e0) cudaEventDestroy(c->e0);
    if (c->e1) cudaEventDestroy(c->e1);
    for (auto& gs : c->gslot)
        if (gs.graph_exec) cudaGraphExecDestroy(gs.graph_exec);
    if (c->span_start) cudaEventDestroy(c->span_start);
    if (c->span_end) cudaEventDestroy(c->span_end);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return ICG_OK;
}

int icg_mlp_shape(int which, int32_t* out_dims, int32_t* in_dims, int32_t* skip_dim, size_t* n_weights,
                  size_t* n_biases) {
    if (which != ICG_MLP_GEOMETRY && which != ICG_MLP_TEXTURE) return einval("mlp: unknown network");
    const int* outs = which == ICG_MLP_GEOMETRY ? kGeoOut : kTexOut;
    int skip = which == ICG_MLP_GEOMETRY ? kGeoSkip : kTexSkip;
    size_t nw = 0, nb = 0;
    for (int l = 0; l < 5; ++l) {
        int in = (l ? outs[l - 1] : 0) + skip;
        if (out_dims) out_dims[l] = outs[l];
        if (in_dims) in_dims[l] = in;
        nw += (size_t)outs[l] * in;
        nb += (size_t)outs[l];
    }
    if (skip_dim) *skip_dim = skip;
    if (n_weights) *n_weights = nw;
    if (n_biases) *n_biases = nb;
    return ICG_OK;
}

int icg_set_mlp(icg_context* c, const icg_mlp_desc* d) {
    if (!c || !d) return einval("set_mlp: null argument");
    if (d->which != ICG_MLP_GEOMETRY && d->which != ICG_MLP_TEXTURE) return einval("set_mlp: unknown network");
    if (d->n_layers != ICG_MLP_LAYERS) return einval("set_mlp: the PIFu MLPs have 5 layers");
    int32_t outs[5], ins[5], skip;
    icg_mlp_shape(d->which, outs, ins, &skip, nullptr, nullptr);
    if (d->skip_dim != skip) return einval("set_mlp: skip dimension mismatch");
    for (int l = 0; l < 5; ++l) {
        if (d->out_dims[l] != outs[l]) return einval("set_mlp: layer width mismatch");
        if (!d->weights[l] || !d->biases[l]) return einval("set_mlp: null weights");
    }
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    bool geo = d->which == ICG_MLP_GEOMETRY;
    DBuf* wt = geo ? c->geo_wt : c->tex_wt;
    DBuf* bb = geo ? c->geo_b : c->tex_b;
    SimtMlp& sm = geo ? c->geo_simt : c->tex_simt;
    std::vector<float> t;
    for (int l = 0; l < 5; ++l) {
        int O = outs[l], K = ins[l];
        t.resize((size_t)O * K);
        for (int o = 0; o < O; ++o)
            for (int k = 0; k < K; ++k) t[(size_t)k * O + o] = d->weights[l][(size_t)o * K + k];
        if (int r = wt[l].ensure(t.size() * 4)) return r;
        if (int r = bb[l].ensure((size_t)O * 4)) return r;
        ICG_CUDA_TRY(cudaMemcpy(wt[l].p, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
        ICG_CUDA_TRY(cudaMemcpy(bb[l].p, d->biases[l], (size_t)O * 4, cudaMemcpyHostToDevice));
        if (geo) {
            if (int r = c->geo_wrow[l].ensure((size_t)O * K * 4)) return r;
            ICG_CUDA_TRY(cudaMemcpy(c->geo_wrow[l].p, d->weights[l], (size_t)O * K * 4, cudaMemcpyHostToDevice));
            c->geo_rows[l] = c->geo_wrow[l].as<float>();
        }
        sm.wt[l] = wt[l].as<float>();
        sm.b[l] = bb[l].as<float>();
        sm.out[l] = O;
        sm.in[l] = K;
    }
    sm.skip = skip;
    sm.slope = d->leaky_slope;
    // fp32 epilogue operands of the tensor-core kernels: biases + z-weight columns, final layer
    DBuf& bi = geo ? c->geo_bias : c->tex_bias;
    DBuf& wl = geo ? c->geo_wlast : c->tex_wlast;
    TcMlp& tc = geo ? c->geo_tc : c->tex_tc;
    tc.valid = 0;
    {
        std::vector<float> hb(tc_bias_floats(d->which)), hw(tc_wlast_floats(d->which));
        const float* ws[5];
        const float* bs[5];
        for (int l = 0; l < 5; ++l) {
            ws[l] = d->weights[l];
            bs[l] = d->biases[l];
        }
        if (int r = tc_pack_epilogue(d->which, ws, bs, hb.data(), hw.data())) return r;
        if (int r = bi.ensure(hb.size() * 4)) return r;
        if (int r = wl.ensure(hw.size() * 4)) return r;
        ICG_CUDA_TRY(cudaMemcpy(bi.p, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice));
        ICG_CUDA_TRY(cudaMemcpy(wl.p, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice));
        tc.bias = bi.as<float>();
        tc.w_last = wl.as<float>();
        int off = 0;
        for (int l = 0; l < 5; ++l) {
            tc.bias_off[l] = off;
            off += outs[l];
        }
        tc.valid = 1;
    }
    {
        // CTA-pair operand streams (k_mlp_pair.cu) + their TMA descriptors
        DBuf& px = geo ? c->geo_pair_stream : c->tex_pair_stream;
        DBuf& ph = geo ? c->geo_pair_hi : c->tex_pair_hi;
        const size_t bx = pair_stream_bytes(d->which, true), bh = pair_stream_bytes(d->which, false);
        std::vector<uint8_t> sx(bx), sh(bh);
        const float* ws[5];
        for (int l = 0; l < 5; ++l) ws[l] = d->weights[l];
        // (the texture stream carries fp16 skip items: the texture kernel's skip operand is fp16)
        if (int r = pair_pack(d->which, ws, sx.data(), sh.data(), !geo)) return r;
        if (int r = px.ensure(bx)) return r;
        if (int r = ph.ensure(bh)) return r;
        ICG_CUDA_TRY(cudaMemcpy(px.p, sx.data(), bx, cudaMemcpyHostToDevice));
        ICG_CUDA_TRY(cudaMemcpy(ph.p, sh.data(), bh, cudaMemcpyHostToDevice));
        unsigned char (*tm)[128] = geo ? c->geo_pair_tmap : c->tex_pair_tmap;
        if (int r = pair_make_tmap(px.p, bx, tm[0])) return r;
        if (int r = pair_make_tmap(ph.p, bh, tm[1])) return r;
        if (geo) {  // the geometry prefix of the texture kernel: same items, fp16 skip items
            if (int r = pair_pack(d->which, ws, sx.data(), sh.data(), true)) return r;
            if (int r = c->geo_pair_f16.ensure(bx)) return r;
            if (int r = c->geo_pair_f16_hi.ensure(bh)) return r;
            ICG_CUDA_TRY(cudaMemcpy(c->geo_pair_f16.p, sx.data(), bx, cudaMemcpyHostToDevice));
            ICG_CUDA_TRY(cudaMemcpy(c->geo_pair_f16_hi.p, sh.data(), bh, cudaMemcpyHostToDevice));
            if (int r = pair_make_tmap(c->geo_pair_f16.p, bx, c->geo_pair_f16_tmap[0])) return r;
            if (int r = pair_make_tmap(c->geo_pair_f16_hi.p, bh, c->geo_pair_f16_tmap[1])) return r;
        }
        (geo ? c->geo_pair : c->tex_pair) = true;
    }
    if (geo) {
        // column-factored streams: part 0 = hidden-input items of layers 2-4, part 1 = Phi items
        const float* ws[5];
        for (int l = 0; l < 5; ++l) ws[l] = d->weights[l];
        for (int part = 0; part < 2; ++part) {
            const size_t bx = pair_fact_stream_bytes(part, true), bh = pair_fact_stream_bytes(part, false);
            std::vector<uint8_t> sx(bx), sh(bh);
            if (int r = pair_pack_factored(ws, part, sx.data(), sh.data())) return r;
            if (int r = c->geo_fact_stream[part][0].ensure(bx)) return r;
            if (int r = c->geo_fact_stream[part][1].ensure(bh)) return r;
            ICG_CUDA_TRY(cudaMemcpy(c->geo_fact_stream[part][0].p, sx.data(), bx, cudaMemcpyHostToDevice));
            ICG_CUDA_TRY(cudaMemcpy(c->geo_fact_stream[part][1].p, sh.data(), bh, cudaMemcpyHostToDevice));
            if (int r = pair_make_tmap(c->geo_fact_stream[part][0].p, bx, c->geo_fact_tmap[part][0])) return r;
            if (int r = pair_make_tmap(c->geo_fact_stream[part][1].p, bh, c->geo_fact_tmap[part][1])) return r;
            if (part == 0) {
                if (int r = pair_make_tmap(c->geo_fact_stream[0][0].p, bx, c->geo_fact2_tmap[0], 128)) return r;
                if (int r = pair_make_tmap(c->geo_fact_stream[0][1].p, bh, c->geo_fact2_tmap[1], 128)) return r;
            }
        }
        c->geo_fact = true;
    }
    {
        const int w = geo ? 0 : 1;
        for (int l = 0; l < 5; ++l) c->host_w[w][l].assign(d->weights[l], d->weights[l] + (size_t)outs[l] * ins[l]);
        c->host_w_set[w] = true;
        if (int r = tg_upload(c)) return r;
    }
    if (geo) {  // the column GEMM's W_Phi (hi, lo)
        c->cg_ready = false;
        const float* ws[5];
        for (int l = 0; l < 5; ++l) ws[l] = d->weights[l];
        std::vector<__nv_bfloat16> wh((size_t)2048 * 256), wl((size_t)2048 * 256);
        if (int r = cg_pack_weights(ws, wh.data(), wl.data())) return r;
        if (int r = c->cg_w.ensure(wh.size() * 4)) return r;
        ICG_CUDA_TRY(cudaMemcpy(c->cg_w.p, wh.data(), wh.size() * 2, cudaMemcpyHostToDevice));
        __nv_bfloat16* lo = c->cg_w.as<__nv_bfloat16>() + wh.size();
        ICG_CUDA_TRY(cudaMemcpy(lo, wl.data(), wl.size() * 2, cudaMemcpyHostToDevice));
        if (int r = cg_make_tmap(c->cg_w.p, 2048, 256, 512, 64, 128, false, c->cg_mapW[0])) return r;
        if (int r = cg_make_tmap(lo, 2048, 256, 512, 64, 128, false, c->cg_mapW[1])) return r;
        c->cg_ready = true;
    }
    if (geo)
        c->has_geo = true;
    else
        c->has_tex = true;
    return ICG_OK;
}

int icg_extract(icg_context* c, const icg_field* field, const icg_algo_config* cfg, icg_extraction* out) {
    if (!c) return einval("extract: null context");
    if (int r = validate_algo(cfg)) return r;
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    FieldDev fd;
    if (int r = prepare_field(c, field, fd)) return r;
    if (int r = ensure_grid(c, cfg->coarsest_cells << cfg->target_level)) return r;
    InflightGuard inflight(c->device);
    c->tail_wide = inflight.alone;
    ICG_CUDA_TRY(cudaEventRecord(c->e0, c->stream));
    if (int r = do_extract(c, fd, cfg)) return r;
    ICG_CUDA_TRY(cudaEventRecord(c->e1, c->stream));
    if (int r = finish_extract_outputs(c, cfg, out)) return r;
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    fill_extraction_scalars(c, cfg, out, elapsed(c));
    c->kept_valid = cfg->keep_level_sets != 0;
    c->kept_cfg = *cfg;
    prof_extract_done(c, cfg);
    prof_collect(c);
    if (c->prof_on) {
        c->prof.frame_ms += elapsed(c) * 1e3;
        c->prof.frames += 1;
    }
    return ICG_OK;
}

int icg_level_set(icg_context* c, int level, int which, int mem, uint32_t* out, size_t cap, size_t* count) {
    if (!c || !count) return einval("level_set: null argument");
    *count = 0;
    if (which != ICG_SET_EVALUATED_NODES && which != ICG_SET_REFINED_CELLS) return einval("level_set: unknown set");
    if (mem != ICG_MEM_HOST && mem != ICG_MEM_DEVICE) return einval("level_set: mem must be ICG_MEM_HOST or ICG_MEM_DEVICE");
    if (!c->kept_valid)
        return einval("level_set: the last extraction on this context did not run with keep_level_sets");
    const icg_algo_config& k = c->kept_cfg;
    if (level < 0 || level > k.target_level) return einval("level_set: level out of range");
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    const int cells = k.coarsest_cells << level;
    const uint32_t* bits = nullptr;
    size_t nbits = 0;
    const bool brute = k.variant == ICG_VARIANT_BRUTE;
    if (which == ICG_SET_REFINED_CELLS) {
        if (level == 0 || brute) return ICG_OK;  // no refinement: empty
        nbits = (size_t)(cells / 2) * (cells / 2) * (cells / 2);
        bits = c->lvl_bits[1][level].as<uint32_t>();
    } else if (brute ? level == k.target_level : level == 0) {
        nbits = nodes3(cells);  // dense evaluation: every node
        if (int r = c->set_bits.ensure(words(nbits) * 4 + 16)) return r;
        if (int r = launch_all_bits(c->set_bits.as<uint32_t>(), nbits, c->stream)) return r;
        bits = c->set_bits.as<uint32_t>();
    } else if (brute) {
        return ICG_OK;  // brute force evaluates only the target level
    } else {
        nbits = nodes3(cells);
        bits = c->lvl_bits[0][level].as<uint32_t>();
    }
    if (int r = c->set_scratch.ensure(bits_to_list_scratch_words(nbits) * 4)) return r;
    if (int r = c->set_total.ensure(16)) return r;
    if (int r = launch_bits_to_list(bits, nbits, c->set_scratch.as<uint32_t>(), nullptr, c->set_total.as<unsigned>(),
                                    c->stream))
        return r;
    unsigned total = 0;
    ICG_CUDA_TRY(cudaMemcpyAsync(&total, c->set_total.p, 4, cudaMemcpyDeviceToHost, c->stream));
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    *count = total;
    if (!out || total == 0) return ICG_OK;
    if (cap < total) {
        set_error("level_set: capacity " + std::to_string(cap) + " < " + std::to_string(total) + " entries");
        return ICG_ECAPACITY;
    }
    uint32_t* dst = out;
    if (mem == ICG_MEM_HOST) {
        if (int r = c->set_list.ensure((size_t)total * 4)) return r;
        dst = c->set_list.as<uint32_t>();
    }
    if (int r = launch_bits_to_list(bits, nbits, c->set_scratch.as<uint32_t>(), dst, c->set_total.as<unsigned>(),
                                    c->stream))
        return r;
    if (mem == ICG_MEM_HOST)
        ICG_CUDA_TRY(cudaMemcpyAsync(out, dst, (size_t)total * 4, cudaMemcpyDeviceToHost, c->stream));
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return ICG_OK;
}

int icg_marching_cubes(icg_context* c, const float* values, int cells, int mem, double iso, icg_mesh* out) {
    if (!c || !out) return einval("marching_cubes: null argument");
    if (mem != ICG_MEM_HOST && mem != ICG_MEM_DEVICE) return einval("marching_cubes: bad mem");
    if (!values) {
        if (c->last_buf < 0) return einval("marching_cubes: no localized grid on this context");
        cells = c->last_cells;
    }
    if (cells < 1 || cells > 1023) return einval("marching_cubes: cells must lie in [1, 1023]");
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    if (int r = mc_init_tables()) return r;
    const size_t nn = nodes3(cells), ncell = (size_t)cells * cells * cells;
    const float* v = values ? values : c->vals[c->last_buf].as<float>();
    if (values && mem == ICG_MEM_HOST) {
        if (int r = c->mc_grid.ensure(nn * 4)) return r;
        ICG_CUDA_TRY(cudaMemcpyAsync(c->mc_grid.p, values, nn * 4, cudaMemcpyHostToDevice, c->stream));
        v = c->mc_grid.as<float>();
    }
    auto read_total = [&](unsigned& x) -> int {
        ICG_CUDA_TRY(cudaMemcpyAsync(&x, c->mc_total.p, 4, cudaMemcpyDeviceToHost, c->stream));
        ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
        return ICG_OK;
    };
    // triangles per block of 1024 cells -> offsets -> emit (weld keys in cell order)
    const unsigned nblocks = (unsigned)((ncell + 1023) / 1024);
    if (int r = c->mc_blocks.ensure((size_t)nblocks * 4 + 16)) return r;
    if (int r = c->mc_total.ensure(16)) return r;
    if (int r = launch_mc_count(v, cells, iso, c->mc_blocks.as<uint32_t>(), nblocks, c->stream)) return r;
    if (int r = launch_exclusive_scan(c->mc_blocks.as<uint32_t>(), nblocks, c->mc_total.as<unsigned>(), c->stream)) return r;
    unsigned ntri = 0;
    if (int r = read_total(ntri)) return r;
    const size_t nkeybits = 4 * nn;
    if (int r = c->mc_tri_keys.ensure((size_t)ntri * 12 + 16)) return r;
    if (int r = c->mc_key_bits.ensure(words(nkeybits) * 4 + 16)) return r;
    ICG_CUDA_TRY(cudaMemsetAsync(c->mc_key_bits.p, 0, words(nkeybits) * 4 + 16, c->stream));
    if (int r = launch_mc_emit(v, cells, iso, c->mc_blocks.as<uint32_t>(), nblocks, c->mc_tri_keys.as<uint32_t>(),
                               c->mc_key_bits.as<uint32_t>(), c->stream))
        return r;
    // the used weld keys, ascending (vertex ids before the first-use renumbering)
    if (int r = c->set_scratch.ensure(bits_to_list_scratch_words(std::max(nkeybits, (size_t)ntri * 3)) * 4)) return r;
    if (int r = launch_bits_to_list(c->mc_key_bits.as<uint32_t>(), nkeybits, c->set_scratch.as<uint32_t>(), nullptr,
                                    c->mc_total.as<unsigned>(), c->stream))
        return r;
    unsigned nkeys = 0;
    if (int r = read_total(nkeys)) return r;
    if (int r = c->mc_keys.ensure((size_t)nkeys * 4 + 16)) return r;
    if (int r = launch_bits_to_list(c->mc_key_bits.as<uint32_t>(), nkeybits, c->set_scratch.as<uint32_t>(),
                                    c->mc_keys.as<uint32_t>(), c->mc_total.as<unsigned>(), c->stream))
        return r;
    // degenerate filter + first use, surviving vertices in first-use order, surviving triangles
    if (int r = c->mc_tri_ids.ensure((size_t)ntri * 12 + 16)) return r;
    if (int r = c->mc_keep.ensure(words(ntri) * 4 + 16)) return r;
    if (int r = c->mc_first.ensure((size_t)nkeys * 4 + 16)) return r;
    if (int r = c->mc_slot_bits.ensure(words((size_t)ntri * 3) * 4 + 16)) return r;
    ICG_CUDA_TRY(cudaMemsetAsync(c->mc_keep.p, 0, words(ntri) * 4 + 16, c->stream));
    ICG_CUDA_TRY(cudaMemsetAsync(c->mc_first.p, 0xFF, (size_t)nkeys * 4 + 16, c->stream));
    ICG_CUDA_TRY(cudaMemsetAsync(c->mc_slot_bits.p, 0, words((size_t)ntri * 3) * 4 + 16, c->stream));
    if (int r = launch_mc_filter(c->mc_tri_keys.as<uint32_t>(), ntri, c->mc_keys.as<uint32_t>(), nkeys, v, cells, iso,
                                 c->mc_tri_ids.as<uint32_t>(), c->mc_keep.as<uint32_t>(), c->mc_first.as<uint32_t>(),
                                 c->stream))
        return r;
    if (int r = launch_mc_mark_first(c->mc_first.as<uint32_t>(), nkeys, c->mc_slot_bits.as<uint32_t>(), c->stream))
        return r;
    if (int r = c->mc_slots.ensure((size_t)nkeys * 4 + 16)) return r;
    if (int r = launch_bits_to_list(c->mc_slot_bits.as<uint32_t>(), (size_t)ntri * 3, c->set_scratch.as<uint32_t>(),
                                    c->mc_slots.as<uint32_t>(), c->mc_total.as<unsigned>(), c->stream))
        return r;
    unsigned nv = 0;
    if (int r = read_total(nv)) return r;
    if (int r = c->mc_tri_list.ensure((size_t)ntri * 4 + 16)) return r;
    if (int r = launch_bits_to_list(c->mc_keep.as<uint32_t>(), ntri, c->set_scratch.as<uint32_t>(),
                                    c->mc_tri_list.as<uint32_t>(), c->mc_total.as<unsigned>(), c->stream))
        return r;
    unsigned nt = 0;
    if (int r = read_total(nt)) return r;
    out->n_vertices = nv;
    out->n_triangles = nt;
    c->launches += 12;
    if ((nv && (!out->vertices || out->vertex_capacity < nv)) || (nt && (!out->triangles || out->triangle_capacity < nt))) {
        set_error("marching_cubes: output capacity too small (" + std::to_string(nv) + " vertices, " +
                  std::to_string(nt) + " triangles)");
        return ICG_ECAPACITY;
    }
    if (int r = c->mc_new_id.ensure((size_t)nkeys * 4 + 16)) return r;
    if (int r = c->mc_out_v.ensure((size_t)nv * 24 + 16)) return r;
    if (int r = c->mc_out_t.ensure((size_t)nt * 12 + 16)) return r;
    if (int r = launch_mc_vertices(c->mc_slots.as<uint32_t>(), nv, c->mc_tri_ids.as<uint32_t>(), c->mc_keys.as<uint32_t>(),
                                   v, cells, iso, c->mc_new_id.as<uint32_t>(), c->mc_out_v.as<double>(), c->stream))
        return r;
    if (int r = launch_mc_triangles(c->mc_tri_list.as<uint32_t>(), nt, c->mc_tri_ids.as<uint32_t>(),
                                    c->mc_new_id.as<uint32_t>(), c->mc_out_t.as<int32_t>(), c->stream))
        return r;
    if (nv) ICG_CUDA_TRY(cudaMemcpyAsync(out->vertices, c->mc_out_v.p, (size_t)nv * 24, cudaMemcpyDeviceToHost, c->stream));
    if (nt) ICG_CUDA_TRY(cudaMemcpyAsync(out->triangles, c->mc_out_t.p, (size_t)nt * 12, cudaMemcpyDeviceToHost, c->stream));
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return ICG_OK;
}

int icg_render_localized(icg_context* c, const icg_field* field, const icg_camera* cam, int W, int H,
                         const float* bg, icg_image* out) {
    if (!c) return einval("render: null context");
    if (c->last_buf < 0) return einval("render: no localized grid on this context (call icg_extract first)");
    if (int r = check_render_args(c, cam, W, H)) return r;
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    FieldDev fd;
    if (int r = prepare_field(c, field, fd)) return r;
    if (fd.kind == ICG_FIELD_PIFU && !c->has_tex) return einval("render: scene has no texture (icg_set_mlp TEXTURE)");
    prof_discard(c);
    ICG_CUDA_TRY(cudaEventRecord(c->e0, c->stream));
    if (int r = issue_render(c, fd, cam, W, H, bg)) return r;
    ICG_CUDA_TRY(cudaEventRecord(c->e1, c->stream));
    if (int r = finish_render_outputs(c, W, H, out)) return r;
    if (int r = sync_counters(c)) return r;
    fill_image_scalars(c, out, elapsed(c));
    prof_render_done(c, W, H);
    prof_collect(c);
    return ICG_OK;
}

static int view_render(icg_context* c, const icg_field* field, const icg_camera* cam, const icg_algo_config* cfg,
                       const float* bg, icg_image* out, bool texture) {
    if (!c) return einval("render: null context");
    if (int r = validate_algo(cfg)) return r;
    // depth_pass's checks, render.hpp:91-94 / 247
    if (cfg->variant != ICG_VARIANT_PROGRESSIVE) return einval("render: config variant must be progressive");
    if (cfg->target_level < 1) return einval("render: target level must be >= 1");
    if (!cam) return einval("render: null camera");
    if (!(cam->scale != 0.0)) return einval("render: camera scale must be nonzero");
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    FieldDev fd;
    if (int r = prepare_field(c, field, fd)) return r;
    if (texture && !field_has_texture(c, fd)) return einval("render_view: scene has no texture");
    const int RL = cfg->coarsest_cells << cfg->target_level;
    if (int r = ensure_grid(c, RL)) return r;
    InflightGuard inflight(c->device);
    c->tail_wide = inflight.alone;
    prof_discard(c);
    ICG_CUDA_TRY(cudaEventRecord(c->e0, c->stream));
    for (int attempt = 0;; ++attempt) {
        if (int r = issue_depth_pass(c, fd, cfg, cam, bg, texture)) return r;
        if (int r = sync_counters(c)) return r;
        if (c->h_ctr->overflow) {
            set_error("render: device work list overflow");
            return ICG_ECAPACITY;
        }
        icg_algo_config sub = *cfg;
        sub.target_level -= 1;
        if (!adapt_unroll(c, &sub)) break;  // the sub-extraction's conflict loop ran out: replay deeper
        if (attempt > 12) {
            set_error("render: conflict loop did not converge");
            return ICG_ERUNTIME;
        }
    }
    ICG_CUDA_TRY(cudaEventRecord(c->e1, c->stream));
    const int n = RL + 1;
    if (int r = finish_render_outputs(c, n, n, out)) return r;
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->kept_valid = false;
    if (out) {
        fill_image_scalars(c, out, elapsed(c));
        uint64_t calls = 0;
        for (int l = 0; l <= cfg->target_level; ++l) calls += c->h_ctr->evals[l];
        out->oracle_calls = calls;
    }
    prof_collect(c);
    return ICG_OK;
}

int icg_render_view(icg_context* c, const icg_field* field, const icg_camera* cam, const icg_algo_config* cfg,
                    const float* bg, icg_image* out) {
    return view_render(c, field, cam, cfg, bg, out, true);
}

int icg_surface_depth_map(icg_context* c, const icg_field* field, const icg_camera* cam, const icg_algo_config* cfg,
                          icg_image* out) {
    if (out) {
        icg_image o = *out;
        o.rgb = nullptr;  // no texture: depth / mask / surface_k only
        int r = view_render(c, field, cam, cfg, nullptr, &o, false);
        const float* keep_rgb = out->rgb;
        *out = o;
        out->rgb = const_cast<float*>(keep_rgb);
        return r;
    }
    return view_render(c, field, cam, cfg, nullptr, out, false);
}

int icg_frame(icg_context* c, const icg_field* field, const icg_algo_config* cfg, const icg_camera* cam, int W, int H,
              const float* bg, icg_extraction* ext, icg_image* img) {
    if (!c) return einval("frame: null context");
    if (int r = validate_algo(cfg)) return r;
    if (int r = check_render_args(c, cam, W, H)) return r;
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    FieldDev fd;
    if (int r = prepare_field(c, field, fd)) return r;
    if (fd.kind == ICG_FIELD_PIFU && !c->has_tex) return einval("frame: scene has no texture (icg_set_mlp TEXTURE)");
    if (int r = ensure_grid(c, cfg->coarsest_cells << cfg->target_level)) return r;
    InflightGuard inflight(c->device);
    c->tail_wide = inflight.alone;
    // the frame's device work: extraction, render + texture, output copies, counters back to the host
    // rays along grid x: the extraction keeps the final grid's x-line extents for the renderer
    const bool keep_xext = c->use_xext && cfg->variant == ICG_VARIANT_PROGRESSIVE && cfg->target_level >= 1 &&
                           std::fabs(cam->rotation[7]) < 1e-9 && std::fabs(cam->rotation[8]) < 1e-9;
    auto body = [&]() -> int {
        if (int r = issue_extract(c, fd, cfg, keep_xext)) return r;
        if (int r = issue_render(c, fd, cam, W, H, bg, keep_xext)) return r;
        if (int r = finish_render_outputs(c, W, H, img)) return r;
        ICG_CUDA_TRY(cudaMemcpyAsync(c->h_ctr, c->ctr.p, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->stream));
        return ICG_OK;
    };
    ICG_CUDA_TRY(cudaEventRecord(c->e0, c->stream));
    for (int attempt = 0;; ++attempt) {
        // Replayed as a CUDA graph once the same frame shape has run eagerly (allocations done):
        // one launch instead of ~150, no host work between dependent kernels.
        icg_context::FrameKey key{};
        key.cfg = *cfg;
        key.cam = *cam;
        key.W = W;
        key.H = H;
        key.kind = fd.kind;
        key.precision = fd.precision;
        key.alloc_gen = g_alloc_gen.load(std::memory_order_relaxed);
        key.fmap_c = fd.C;
        key.fmap_h = fd.H;
        key.fmap_w = fd.W;
        for (int i = 0; i < 3; ++i) key.bg[i] = bg ? bg[i] : 0.0f;
        if (img) {
            key.img_mem = img->mem;
            key.img_ptr[0] = img->depth;
            key.img_ptr[1] = img->rgb;
            key.img_ptr[2] = img->mask;
            key.img_ptr[3] = img->surface_k;
        }
        std::memcpy(key.unroll, c->unroll, sizeof(key.unroll));
        key.tail_wide = c->tail_wide ? 1 : 0;
        icg_context::GraphSlot& gs = c->gslot[key.tail_wide];
        std::memcpy(key.pred, c->pred, sizeof(key.pred));
        for (int l = 0; l < ICG_MAX_LEVELS; ++l) key.pred_valid[l] = (uint8_t)(c->pred_valid[l] | (c->pred_all[l] << 1));
        const bool graphs = c->use_graph && !c->prof_on;
        bool ran = false;
        if (getenv("ICG_GRAPH_DEBUG") && gs.warm_valid && !(gs.warm_key == key)) {
            const icg_context::FrameKey& w = gs.warm_key;
            fprintf(stderr, "[icg] frame key differs: cfg %d cam %d WH %d kind %d img %d bg %d unroll %d\n",
                    std::memcmp(&w.cfg, &key.cfg, sizeof(key.cfg)) != 0, std::memcmp(&w.cam, &key.cam, sizeof(key.cam)) != 0,
                    w.W != key.W || w.H != key.H, w.kind != key.kind || w.precision != key.precision,
                    std::memcmp(w.img_ptr, key.img_ptr, sizeof(key.img_ptr)) != 0 || w.img_mem != key.img_mem,
                    std::memcmp(w.bg, key.bg, sizeof(key.bg)) != 0, std::memcmp(w.unroll, key.unroll, sizeof(key.unroll)) != 0);
        }
        if (graphs && gs.graph_valid && gs.graph_key == key) {
            ICG_CUDA_TRY(cudaGraphLaunch(gs.graph_exec, c->stream));
            c->launches += gs.graph_launches;
            // the host-side bookkeeping body() would have done (issue_extract's final grid)
            c->last_cells = cfg->coarsest_cells << cfg->target_level;
            c->last_buf = cfg->variant == ICG_VARIANT_BRUTE ? 0 : (cfg->target_level & 1);
            c->fact_used = fact_ok(c, fd);
            ran = true;
        } else if (graphs && gs.warm_valid && gs.warm_key == key) {
            const uint64_t l0 = c->launches;
            cudaGraph_t g = nullptr;
            int r = ICG_OK;
            if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
                r = ICG_ERUNTIME;
            } else {
                r = body();
                cudaError_t e = cudaStreamEndCapture(c->stream, &g);
                if (e != cudaSuccess) r = r ? r : ICG_ERUNTIME;
            }
            cudaGetLastError();
            if (r == ICG_OK && g) {
                if (gs.graph_exec) cudaGraphExecDestroy(gs.graph_exec);
                gs.graph_exec = nullptr;
                if (cudaGraphInstantiate(&gs.graph_exec, g, 0) == cudaSuccess) {
                    gs.graph_key = key;
                    gs.graph_valid = true;
                    gs.graph_launches = c->launches - l0;
                    if (getenv("ICG_GRAPH_DEBUG")) fprintf(stderr, "[icg] frame graph captured: %llu launches\n",
                                                           (unsigned long long)gs.graph_launches);
                    ICG_CUDA_TRY(cudaGraphLaunch(gs.graph_exec, c->stream));
                    ran = true;
                } else {
                    gs.graph_exec = nullptr;
                }
            }
            if (g) cudaGraphDestroy(g);
            if (!ran) {  // capture not possible: stay eager on this context
                if (getenv("ICG_GRAPH_DEBUG"))
                    fprintf(stderr, "[icg] frame graph capture failed (%d: %s); staying eager\n", r, g_err.c_str());
                cudaGetLastError();
                c->use_graph = false;
                gs.graph_valid = false;
                c->launches = l0;
            }
        }
        if (!ran) {
            if (int r = body()) return r;
            gs.warm_key = key;
            gs.warm_valid = true;
        }
        ICG_CUDA_TRY(cudaEventRecord(c->e1, c->stream));
        ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (c->h_ctr->overflow) {
            set_error("frame: device work list overflow");
            return ICG_ECAPACITY;
        }
        if (!adapt_unroll(c, cfg)) break;
        if (attempt > 12) {
            set_error("frame: conflict loop did not converge");
            return ICG_ERUNTIME;
        }
        ICG_CUDA_TRY(cudaEventRecord(c->e0, c->stream));
    }
    double secs = elapsed(c);
    c->kept_valid = cfg->keep_level_sets != 0;
    c->kept_cfg = *cfg;
    prof_extract_done(c, cfg);
    prof_render_done(c, W, H);
    prof_collect(c);
    if (c->prof_on) {
        c->prof.frame_ms += secs * 1e3;
        c->prof.frames += 1;
    }
    if (ext) {
        if (int r = finish_extract_outputs(c, cfg, ext)) return r;
        ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
        fill_extraction_scalars(c, cfg, ext, secs);
    }
    fill_image_scalars(c, img, secs);
    return ICG_OK;
}

static int eval_points(icg_context* c, const icg_field* field, const double* points, size_t n, int mem, float* out,
                       bool texture) {
    if (!c || !field) return einval("batch: null argument");
    if (n == 0) return ICG_OK;  // empty list -> empty list, counter unchanged (SPEC field examples)
    if (!points || !out) return einval("batch: null buffer");
    if (mem != ICG_MEM_HOST && mem != ICG_MEM_DEVICE) return einval("batch: bad mem");
    if (n > (size_t)1 << 31) return einval("batch: too many points");
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    FieldDev fd;
    if (int r = prepare_field(c, field, fd)) return r;
    if (texture && !field_has_texture(c, fd)) return einval("FieldOracle: scene has no texture");
    const double* dpts = points;
    float* dout = out;
    size_t ob = n * 4 * (texture ? 3 : 1);
    if (mem == ICG_MEM_HOST) {
        if (int r = c->pts.ensure(n * 24)) return r;
        if (int r = c->outv.ensure(ob)) return r;
        ICG_CUDA_TRY(cudaMemcpyAsync(c->pts.p, points, n * 24, cudaMemcpyHostToDevice, c->stream));
        dpts = c->pts.as<double>();
        dout = c->outv.as<float>();
    }
    EvalJob job{};
    job.points = dpts;
    job.n_static = (unsigned)n;
    job.out = dout;
    prof_discard(c);
    int r = texture ? run_texture(c, fd, job, (unsigned)n) : run_eval(c, fd, job, (unsigned)n);
    if (r) return r;
    if (mem == ICG_MEM_HOST) ICG_CUDA_TRY(cudaMemcpyAsync(out, dout, ob, cudaMemcpyDeviceToHost, c->stream));
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->prof_on) {
        if (texture)
            c->prof.tex_points += n;
        else
            c->prof.geo_points += n;
        prof_collect(c);
    }
    return ICG_OK;
}

int icg_occupancy_batch(icg_context* c, const icg_field* f, const double* p, size_t n, int mem, float* out) {
    return eval_points(c, f, p, n, mem, out, false);
}

int icg_texture_batch(icg_context* c, const icg_field* f, const double* p, size_t n, int mem, float* out) {
    return eval_points(c, f, p, n, mem, out, true);
}

int icg_composite(const float* rgb, const uint8_t* mask, size_t n_image, const float* backdrop, size_t n_backdrop,
                  float* out) {
    if (n_image != n_backdrop) return einval("composite: dimension mismatch");
    if (n_image == 0) return ICG_OK;
    if (!rgb || !mask || !backdrop || !out) return einval("composite: null buffer");
    for (size_t i = 0; i < n_image; ++i) {
        const float* src = mask[i] ? rgb + 3 * i : backdrop + 3 * i;
        const float r = src[0], g = src[1], b = src[2];
        out[3 * i] = r;
        out[3 * i + 1] = g;
        out[3 * i + 2] = b;
    }
    return ICG_OK;
}

int icg_compare_iou(icg_context* c, const uint8_t* a, const uint8_t* b, size_t n, int mem, double* iou) {
    if (!iou) return einval("compare_iou: null output");
    if (n == 0) {
        *iou = 1.0;
        return ICG_OK;
    }
    if (!a || !b) return einval("compare_iou: null input");
    if (mem != ICG_MEM_HOST && mem != ICG_MEM_DEVICE) return einval("compare_iou: mem must be ICG_MEM_HOST or ICG_MEM_DEVICE");
    if (mem == ICG_MEM_DEVICE && !c) return einval("compare_iou: device arrays need a context");
    if (mem == ICG_MEM_HOST) {
        uint64_t inter = 0, uni = 0;
        for (size_t i = 0; i < n; ++i) {
            bool av = a[i] != 0, bv = b[i] != 0;
            inter += (av && bv);
            uni += (av || bv);
        }
        *iou = uni ? (double)inter / (double)uni : 1.0;
        return ICG_OK;
    }
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    if (int r = c->outv.ensure(16)) return r;
    ICG_CUDA_TRY(cudaMemsetAsync(c->outv.p, 0, 16, c->stream));
    if (int r = launch_iou(a, b, n, c->outv.as<unsigned long long>(), c->stream)) return r;
    unsigned long long iu[2];
    ICG_CUDA_TRY(cudaMemcpyAsync(iu, c->outv.p, 16, cudaMemcpyDeviceToHost, c->stream));
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    *iou = iu[1] ? (double)iu[0] / (double)iu[1] : 1.0;
    return ICG_OK;
}

int icg_span_begin(icg_context* const* ctxs, int n) {
    if (!ctxs || n < 1 || !ctxs[0]) return einval("span: no contexts");
    icg_context* c0 = ctxs[0];
    ICG_CUDA_TRY(cudaSetDevice(c0->device));
    if (!c0->span_start) ICG_CUDA_TRY(cudaEventCreate(&c0->span_start));
    ICG_CUDA_TRY(cudaEventRecord(c0->span_start, c0->stream));
    for (int i = 1; i < n; ++i) {
        if (!ctxs[i] || ctxs[i]->device != c0->device) return einval("span: contexts must share a device");
        ICG_CUDA_TRY(cudaStreamWaitEvent(ctxs[i]->stream, c0->span_start, 0));
    }
    return ICG_OK;
}

int icg_span_end(icg_context* const* ctxs, int n, float* ms) {
    if (!ctxs || n < 1 || !ctxs[0] || !ms) return einval("span: bad arguments");
    icg_context* c0 = ctxs[0];
    if (!c0->span_start) return einval("span: icg_span_begin was not called");
    ICG_CUDA_TRY(cudaSetDevice(c0->device));
    float best = 0.0f;
    for (int i = 0; i < n; ++i) {
        icg_context* c = ctxs[i];
        if (!c->span_end) ICG_CUDA_TRY(cudaEventCreate(&c->span_end));
        ICG_CUDA_TRY(cudaEventRecord(c->span_end, c->stream));
        ICG_CUDA_TRY(cudaEventSynchronize(c->span_end));
        float t = 0.0f;
        ICG_CUDA_TRY(cudaEventElapsedTime(&t, c0->span_start, c->span_end));
        if (t > best) best = t;
    }
    *ms = best;
    return ICG_OK;
}

int icg_profile_enable(icg_context* c, int on) {
    if (!c) return einval("null context");
    c->prof_on = on != 0;
    prof_discard(c);
    return ICG_OK;
}

int icg_profile_reset(icg_context* c) {
    if (!c) return einval("null context");
    c->prof = icg_profile{};
    c->launches = 0;
    prof_discard(c);
    return ICG_OK;
}

int icg_profile_get(icg_context* c, icg_profile* out) {
    if (!c || !out) return einval("null argument");
    *out = c->prof;
    out->kernel_launches = c->launches;
    return ICG_OK;
}

int icg_host_alloc(size_t bytes, void** p) {
    if (!p) return einval("null output");
    ICG_CUDA_TRY(cudaMallocHost(p, bytes ? bytes : 1));
    return ICG_OK;
}
int icg_host_free(void* p) {
    if (p) ICG_CUDA_TRY(cudaFreeHost(p));
    return ICG_OK;
}
int icg_device_alloc(icg_context* c, size_t bytes, void** p) {
    if (!c || !p) return einval("null argument");
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    ICG_CUDA_TRY(cudaMalloc(p, bytes ? bytes : 1));
    return ICG_OK;
}
int icg_device_free(icg_context* c, void* p) {
    if (!c) return einval("null context");
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    if (p) ICG_CUDA_TRY(cudaFree(p));
    return ICG_OK;
}
int icg_memcpy(icg_context* c, void* dst, const void* src, size_t bytes, int dst_mem, int src_mem) {
    if (!c) return einval("null context");
    if ((dst_mem != ICG_MEM_HOST && dst_mem != ICG_MEM_DEVICE) || (src_mem != ICG_MEM_HOST && src_mem != ICG_MEM_DEVICE))
        return einval("memcpy: mem must be ICG_MEM_HOST or ICG_MEM_DEVICE");
    if (bytes == 0) return ICG_OK;
    if (!dst || !src) return einval("memcpy: null pointer");
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    cudaMemcpyKind k = dst_mem == ICG_MEM_HOST
                           ? (src_mem == ICG_MEM_HOST ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost)
                           : (src_mem == ICG_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice);
    ICG_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, k, c->stream));
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return ICG_OK;
}

int icg_memset(icg_context* c, void* dst, int value, size_t bytes) {
    if (!c) return einval("null context");
    if (bytes == 0) return ICG_OK;
    if (!dst) return einval("memset: null pointer");
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    ICG_CUDA_TRY(cudaMemsetAsync(dst, value, bytes, c->stream));
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return ICG_OK;
}

// ---- seeded inputs: std::mt19937_64 + random.hpp:22-38 transforms ----------
static double u01(std::mt19937_64& g) { return (double)(g() >> 11) * 0x1.0p-53; }
static double urange(std::mt19937_64& g, double lo, double hi) { return lo + (hi - lo) * u01(g); }
static double normal(std::mt19937_64& g) {
    double a = u01(g);
    while (a <= 0.0) a = u01(g);
    double b = u01(g);
    return std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * 3.14159265358979323846 * b);
}

int icg_gen_capsules(uint64_t seed, int n, icg_primitive* out) {
    if (n < 0 || (n && !out)) return einval("gen_capsules: bad arguments");
    std::mt19937_64 g(seed);
    for (int c = 0; c < n; ++c) {
        std::memset(&out[c], 0, sizeof(icg_primitive));
        out[c].kind = ICG_PRIM_CAPSULE;
        for (int d = 0; d < 3; ++d) out[c].a[d] = urange(g, -0.5, 0.5);
        for (int d = 0; d < 3; ++d) out[c].b[d] = urange(g, -0.5, 0.5);
        out[c].radius = urange(g, 0.03, 0.08);
        out[c].inv_rotation[0] = out[c].inv_rotation[4] = out[c].inv_rotation[8] = 1.0;
    }
    return ICG_OK;
}

int icg_gen_normals(uint64_t seed, size_t n, float* out) {
    if (n && !out) return einval("gen_normals: null output");
    std::mt19937_64 g(seed);
    for (size_t i = 0; i < n; ++i) out[i] = (float)normal(g);
    return ICG_OK;
}

int icg_gen_feature_map_device(icg_context* c, uint64_t seed, int C, int H, int W, int mem, float* out) {
    if (!c || !out) return einval("gen_feature_map_device: null argument");
    if (C < 1 || H < 1 || W < 1) return einval("gen_feature_map_device: bad shape");
    if (mem != ICG_MEM_HOST && mem != ICG_MEM_DEVICE) return einval("gen_feature_map_device: bad mem");
    ICG_CUDA_TRY(cudaSetDevice(c->device));
    const size_t n = (size_t)C * H * W;
    float* dst = out;
    if (mem == ICG_MEM_HOST) {
        if (int r = c->outv.ensure(n * 4)) return r;
        dst = c->outv.as<float>();
    }
    if (int r = launch_feature_normals(seed, n, dst, c->stream)) return r;
    c->launches += 1;
    if (mem == ICG_MEM_HOST) ICG_CUDA_TRY(cudaMemcpyAsync(out, dst, n * 4, cudaMemcpyDeviceToHost, c->stream));
    ICG_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return ICG_OK;
}

int icg_gen_mlp(uint64_t seed, int which, float* w, float* b) {
    int32_t outs[5], ins[5];
    if (int r = icg_mlp_shape(which, outs, ins, nullptr, nullptr, nullptr)) return r;
    if (!w || !b) return einval("gen_mlp: null output");
    const double slope = 0.02, gain = std::sqrt(2.0 / (1.0 + slope * slope));
    std::mt19937_64 g(seed);
    size_t wo = 0, bo = 0;
    for (int l = 0; l < 5; ++l) {
        double bound = gain * std::sqrt(3.0 / (double)ins[l]);
        for (size_t i = 0; i < (size_t)outs[l] * ins[l]; ++i) w[wo + i] = (float)urange(g, -bound, bound);
        double bb = 1.0 / std::sqrt((double)ins[l]);
        for (int o = 0; o < outs[l]; ++o) b[bo + o] = (float)urange(g, -bb, bb);
        wo += (size_t)outs[l] * ins[l];
        bo += (size_t)outs[l];
    }
    return ICG_OK;
}

int icg_camera_from_angles(double yaw_deg, double pitch_deg, double dist, double scale, icg_camera* out) {
    if (!out) return einval("camera: null output");
    const double kPi = 3.14159265358979323846;
    double yaw = std::fmod(yaw_deg, 360.0), pitch = std::fmod(pitch_deg, 360.0);
    double rx = pitch * kPi / 180.0, ry = yaw * kPi / 180.0;  // deg_to_rad, geom.hpp:11
    double cx = std::cos(rx), sx = std::sin(rx), cy = std::cos(ry), sy = std::sin(ry);
    double A[9] = {1, 0, 0, 0, cx, -sx, 0, sx, cx};
    double B[9] = {cy, 0, sy, 0, 1, 0, -sy, 0, cy};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int k = 0; k < 3; ++k) s += A[3 * i + k] * B[3 * k + j];
            out->rotation[3 * i + j] = s;
        }
    out->translation[0] = 0.0;
    out->translation[1] = 0.0;
    out->translation[2] = -dist;
    out->scale = scale;
    return ICG_OK;
}

}  // extern "C"

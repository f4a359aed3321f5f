// k_mlp_pair.cu — the PIFu geometry and texture fields on CTA PAIRS
// (tcgen05 cta_group::2).
//
// A fused "weights x activations^T" dataflow: every MMA is M=256 x N x K=16
// executed by the two SMs of a TPC: each CTA of the cluster holds 128 of the
// 256 weight rows (A) and N/2 of the N points (B) in its shared memory; its
// TMEM holds its 128 output rows for all N points.  Per SM this halves the
// shared-memory operand bytes per FLOP and doubles the tensor work per
// pipeline stage relative to a single-CTA 128xN MMA (a round-1 single-CTA
// kernel measured ~25% tensor-pipe activity, bound by per-stage overheads and
// SMEM operand traffic; it was removed in round 2).
//   geometry : N = 128 (64 points per CTA), 257->1024->512->256->128->1
//   texture  : N = 64 (32 points per CTA; the 513-wide skip input is twice as
//              large): the geometry prefix (layers 1-3) writes its layer-3
//              activations h3 straight into the skip operand, then the texture
//              body 513->1024->512->256->128->3 runs over [Phi, h3, z]
//              (render.hpp:262-277 evaluates f_T at the surface points).
//
//   weights  : both CTAs' producers TMA (2-SM form) their 16 KB half-tile
//              into their own ring; transaction bytes land on the leader's
//              barrier; the leader's MMA commit frees both rings (multicast).
//   epilogue : CTA r's TMEM lane q = output feature r*128+q of the 256-row
//              block; its warps convert (bias, z-term, leaky-ReLU, bf16 hi/lo)
//              and write the next layer's B operand straight into the shared
//              memory of the CTA that owns each point (DSMEM for the peer's).
//   layer 1  : 4 chunks of 256 features streamed through TMEM into layer 2.
//   final    : layer 4 is padded to 256 rows (peer half zero); CTA 0 reduces
//              the 128 -> 1 (3) outputs for all points on CUDA cores.  The
//              skip-input part of the final layer is a fp32 dot computed where
//              the data is produced (Phi during the gather, h3 once it is in
//              the skip operand); the peer's arrive over DSMEM.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "eval_common.cuh"
#include "tc_ptx.cuh"

namespace icg {

namespace pair {

constexpr uint32_t kHalf = 16384;   // one 128 x 64 bf16 tile
constexpr uint32_t kStage = 32768;  // one TMA box: (hi, lo) of one item (bf16x3) or hi of two items (bf16)
constexpr int kEpiWarpsMax = 16;
constexpr int kMaxNP = 128;
constexpr int kMaxStages = 6;

// Kernel modes.
//   GEO  : geometry field, full network per point (257-wide skip operand gathered per point)
//   TEX  : texture field at surface points (geometry prefix + texture body)
//   COLS : column pass of the column-factored geometry field: for a list of grid COLUMNS (i,j)
//          computes the Phi-part of every layer's pre-activation, S = W_Phi . Phi(x_i, y_j), and
//          the Phi-part of the output dot, into a fp32 record per column (kSRow floats)
//   FACT : column-factored geometry field: under the orthographic projection every node of a
//          column shares Phi, so layer 1 is act(S1[col] + w1z z + b1) (no MMA) and layers 2-4
//          only multiply the hidden part: W_h . h + S_l[col]
enum { kModeGeo = 0, kModeTex = 1, kModeCols = 2, kModeFact = 3, kModeGeo64 = 4 };
constexpr int kSRow = 1936;    // floats per column record: [1024 | 512 | 256 | 128 | final Phi dot | pad]
constexpr int kSFinal = 1920;  // offset of the final layer's Phi dot
__host__ __device__ constexpr int kSOffL(int l) { return l == 0 ? 0 : l == 1 ? 1024 : l == 2 ? 1536 : 1792; }

template <int MODE>
struct Cfg {
    static constexpr bool TEX = MODE == kModeTex;
    static constexpr int NPC = MODE == kModeGeo64 ? 32 : 64;  // points per CTA
    static constexpr int NP = 2 * NPC;               // points per pair tile = MMA N
    // [Phi] or [Phi, h3] in 64-wide K-chunks (none for FACT: Phi enters through the column records)
    static constexpr int kSkipChunks = TEX ? 8 : (MODE == kModeFact ? 0 : 4);
    static constexpr int kHBufs = MODE == kModeFact ? 2 : (MODE == kModeCols ? 0 : 1);  // h operand buffers
    // 32 KB stages (per-copy TMA cost is size-independent)
    static constexpr int kStages = (MODE == kModeCols || MODE == kModeGeo64) ? 4 : (MODE == kModeTex ? 3 : 2);
    // TEX: the skip operand [Phi, h3] is ONE fp16 copy (its weights fp16 hi + lo): 10 more mantissa
    // bits than a bf16 copy keep colours within 1e-3 (max 1.9e-4 simulated) and free the shared
    // memory of a lo copy, so the texture tile is 128 points like the geometry one
    static constexpr bool kF16Skip = TEX;
    static constexpr int kSkipCopies = kF16Skip ? 1 : 2;
    // TEX: the hidden activations too are one fp16 copy (all weights fp16 hi / lo): 2 MMAs per
    // K step instead of 3, half the h-operand bytes; colours within 2.5e-4 of the oracle (simulated)
    static constexpr bool kF16H = TEX;
    static constexpr uint32_t kChunk = NPC * 128;  // NPC point rows x 64 bf16 (SW128)
    static constexpr uint32_t kSkipHalf = kSkipChunks * kChunk;
    static constexpr uint32_t kHHalf = 4 * kChunk;  // one 256-feature block
    static constexpr uint32_t kOffSkip = 0;
    static constexpr uint32_t kOffH = kOffSkip + kSkipCopies * kSkipHalf;
    static constexpr uint32_t kOffRing = kOffH + kHBufs * (kF16H ? 1 : 2) * kHHalf;
    static constexpr uint32_t kOffMisc = kOffRing + kStages * kStage;
    static constexpr uint32_t kMisc = 24576;
    static constexpr uint32_t kTotal = kOffMisc + kMisc + 1024;
    static constexpr int kOut = TEX ? 3 : 1;
    // epilogue warps: 8 = 4 TMEM lane quarters x 2 point halves; FACT (no transposes, fewer
    // registers) uses 16 = 4 quarters x 4 point quarters to hide the per-block latency chain
    static constexpr int kEpiWarps = 8;
    static constexpr int kEpiThreads = 32 * kEpiWarps;
    // FACT: two auxiliary warps gather the next tiles (positions, column records, sdf bias) so the
    // epilogue warps only convert and emit h blocks (their work bounds the FACT tile time)
    static constexpr int kAuxWarps = MODE == kModeFact ? 2 : 0;
    static constexpr int kThreads = 64 + kEpiThreads + 32 * kAuxWarps;
    static constexpr int kHF = (NPC / 32) / (kEpiWarps / 8);  // 32-point chunks per epilogue thread
    // one CTA per SM: the register file split over the CTA's warps, allocated in groups of 4
    // warps, per thread a multiple of 8
    static constexpr int kWarpsAlloc = ((kThreads / 32) + 3) / 4 * 4;
    static constexpr int kMaxReg = (65536 / (kWarpsAlloc * 32)) / 8 * 8;
    static constexpr int kSkipDim = TEX ? kTexSkip : kGeoSkip;
    static_assert(kStages <= kMaxStages, "stages");
};

// weight-item schedule of one MLP body: (layer, 256-row block, K column offset).
// ks = skip K-chunks (4 geometry, 8 texture); the geometry prefix of the texture
// network is the same schedule without layer 4, i.e. the first items of the
// geometry stream.
template <class Emit>
__host__ __device__ void schedule(int ks, bool with_l4, Emit&& emit) {
    auto L1 = [&](int c) {
        for (int j = 0; j < ks; ++j) emit(0, c, j * 64);
    };
    L1(0);
    L1(1);
    for (int m = 0; m < 2; ++m)
        for (int j = 0; j < ks; ++j) emit(1, m, 1024 + j * 64);
    for (int c = 0; c < 4; ++c) {
        for (int jj = 0; jj < 4; ++jj)  // jj-major: h halves (K chunks 0-1 / 2-3) are released in turn
            for (int m = 0; m < 2; ++m) emit(1, m, c * 256 + jj * 64);
        if (c + 2 < 4) L1(c + 2);
    }
    for (int j = 0; j < ks; ++j) emit(2, 0, 512 + j * 64);
    for (int c = 0; c < 2; ++c)
        for (int jj = 0; jj < 4; ++jj) emit(2, 0, c * 256 + jj * 64);
    if (with_l4) {
        for (int j = 0; j < ks; ++j) emit(3, 0, 256 + j * 64);
        for (int jj = 0; jj < 4; ++jj) emit(3, 0, jj * 64);
    }
}
__host__ __device__ constexpr int items(int ks, bool with_l4) {
    return 4 * ks + 2 * ks + 32 + ks + 8 + (with_l4 ? ks + 4 : 0);
}
constexpr int kGeoItems = items(4, true);      // 76
constexpr int kPrefixItems = items(4, false);  // 68
constexpr int kTexItems = items(8, true);      // 108

// FACT stream: only the hidden-input items of layers 2-4, in the order the MMA issuer consumes
// them (h1 chunk c: K chunks jj, row blocks m; then h2 blocks for layer 3; then h3 for layer 4)
template <class Emit>
__host__ __device__ void schedule_fact(Emit&& emit) {
    for (int c = 0; c < 4; ++c)
        for (int jj = 0; jj < 4; ++jj)
            for (int m = 0; m < 2; ++m) emit(1, m, c * 256 + jj * 64);
    for (int c = 0; c < 2; ++c)
        for (int jj = 0; jj < 4; ++jj) emit(2, 0, c * 256 + jj * 64);
    for (int jj = 0; jj < 4; ++jj) emit(3, 0, jj * 64);
}
constexpr int kFactItems = 44;
// COLS stream: the Phi items (K = skip columns 0..255) of every 256-row block of layers 1-4
template <class Emit>
__host__ __device__ void schedule_cols(Emit&& emit) {
    const int prev[4] = {0, 1024, 512, 256};
    const int blocks[4] = {4, 2, 1, 1};
    for (int l = 0; l < 4; ++l)
        for (int m = 0; m < blocks[l]; ++m)
            for (int j = 0; j < 4; ++j) emit(l, m, prev[l] + j * 64);
}
constexpr int kColsItems = 32;
constexpr int kColsBlocks = 8;

struct Misc {
    uint64_t full[kMaxStages], empty[kMaxStages];
    uint64_t f_ready, h_ready[2][2], h_free[2][2], l1done[2], d2done, d3done, d4done, sd_ready[2], skip_free, d4_free;
    uint64_t accb[4], acc_free[4];  // COLS: accumulator ring
    uint64_t g_ready[2], fin_done[2];  // FACT: tile gathered (aux -> epilogue), final layer done (-> aux)
    uint32_t tmem_base;
    int slot[2][kMaxNP];  // FACT: column record of each point of the tile (by tile parity)
    // FACT: per 32-point chunk of a (column-sorted) tile: first / last record, mask of the points
    // on the last record, and whether those two records are all the chunk uses
    int cfirst[2][kMaxNP / 32], clast[2][kMaxNP / 32];
    uint32_t cmask[2][kMaxNP / 32], cok[2][kMaxNP / 32];
    float z[2][kMaxNP];       // by tile parity (the next tile is gathered before this one's final layer)
    float pos[2][kMaxNP][3];
    float red[4][3][kMaxNP];      // final layer: per-lane-quarter partial sums over features
    float skipdot[2][3][kMaxNP];  // final layer: skip-input dots (leader, all points), by tile parity
    float sdl[3][kMaxNP / 2];     // texture: this CTA's Phi-part skip dots until h3 is known
    float cterm[3][kMaxNP];       // b5 + w5z*z (- sdf_scale*sdf for geometry); FACT: [tile parity][point]
    // the bias scene as capsules (a, b - a, |b - a|^2, r), when every primitive is a capsule
    float caps[ICG_MAX_PRIMS][8];
    int ncaps;  // -1: not all capsules (use the general fp32 scene path)
};
static_assert(sizeof(Misc) + 16 <= Cfg<kModeGeo>::kMisc, "misc smem too small");

struct Params {
    FieldDev f;
    EvalJob job;
    const float* bias_g;  // geometry per-layer [b, wz] blocks (same layout as the single-CTA stream)
    const float* bias_t;  // texture per-layer [b, wz] blocks
    const float* wlast;   // final layer of the evaluated network, [out][128 + skip]
    int items_a, items_b;  // items used from stream A / B
    int total_a, total_b;  // items in stream A / B (per-rank segment length)
    float slope;
    int x3;
    unsigned long long* trace;
    float* s_out;        // COLS: column records, kSRow floats per list entry
    const float* s_in;   // FACT: column records
    const int* cmap;     // FACT: column (i + n j) -> record index (nullptr: the column index itself)
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t k) {
    return row * 128u + ((((k >> 3) ^ row) & 7u) << 4) + (k & 7u) * 2u;
}

__device__ __forceinline__ float warp_transpose_reduce(float* v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        const bool upper = lane & w;
#pragma unroll
        for (int i = 0; i < w; ++i) {
            float send = upper ? v[i] : v[i + w];
            float keep = upper ? v[i + w] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
        }
    }
    return v[0];
}

// 8x8 transpose inside each 8-lane group: lane i of a group holds one feature (8g + i) for 32
// points; afterwards it holds all 8 features of the group, as bf16 hi (and lo) 16-byte rows, for
// points 8u + i (u = 0..3).  Three butterfly rounds swap point-index bits with lane bits.
template <bool LO, bool F16 = false>
__device__ __forceinline__ void transpose8_bf16(const float* v, uint4* hi, uint4* lo) {
    const int lane = threadIdx.x & 31;
    const bool i0 = lane & 1, i1 = lane & 2, i2 = lane & 4;
    // round 0 (fp32): keep points q with q0 == i0; pack the two features as bf16x2 (lower feature first)
    uint32_t wh[16], wl[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        const float keep = i0 ? v[2 * m + 1] : v[2 * m];
        const float send = i0 ? v[2 * m] : v[2 * m + 1];
        const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
        const float a = i0 ? recv : keep, b = i0 ? keep : recv;
        if (F16) {
            __half2 f2 = __floats2half2_rn(a, b);
            wh[m] = *reinterpret_cast<uint32_t*>(&f2);
        } else {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
            wh[m] = *reinterpret_cast<uint32_t*>(&h2);
        }
        if (LO && !F16) {
            __nv_bfloat162 l2 =
                __floats2bfloat162_rn(a - __uint_as_float(wh[m] << 16), b - __uint_as_float(wh[m] & 0xFFFF0000u));
            wl[m] = *reinterpret_cast<uint32_t*>(&l2);
        }
    }
    // round 1: words m (point 2m + i0); keep m with m0 == i1 -> 2 words (features 0-3 of the half-group)
    uint32_t xh[8][2], xl[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t kh = i1 ? wh[2 * j + 1] : wh[2 * j], sh = i1 ? wh[2 * j] : wh[2 * j + 1];
        const uint32_t rh = __shfl_xor_sync(0xffffffffu, sh, 2);
        xh[j][0] = i1 ? rh : kh;
        xh[j][1] = i1 ? kh : rh;
        if (LO) {
            const uint32_t kl = i1 ? wl[2 * j + 1] : wl[2 * j], sl = i1 ? wl[2 * j] : wl[2 * j + 1];
            const uint32_t rl = __shfl_xor_sync(0xffffffffu, sl, 2);
            xl[j][0] = i1 ? rl : kl;
            xl[j][1] = i1 ? kl : rl;
        }
    }
    // round 2: words j (point 4j + 2 i1 + i0); keep j with j0 == i2 -> 4 words = 8 features
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        uint32_t k0 = i2 ? xh[2 * u + 1][0] : xh[2 * u][0], k1 = i2 ? xh[2 * u + 1][1] : xh[2 * u][1];
        uint32_t s0 = i2 ? xh[2 * u][0] : xh[2 * u + 1][0], s1 = i2 ? xh[2 * u][1] : xh[2 * u + 1][1];
        uint32_t r0 = __shfl_xor_sync(0xffffffffu, s0, 4), r1 = __shfl_xor_sync(0xffffffffu, s1, 4);
        hi[u] = i2 ? make_uint4(r0, r1, k0, k1) : make_uint4(k0, k1, r0, r1);
        if (LO) {
            k0 = i2 ? xl[2 * u + 1][0] : xl[2 * u][0];
            k1 = i2 ? xl[2 * u + 1][1] : xl[2 * u][1];
            s0 = i2 ? xl[2 * u][0] : xl[2 * u + 1][0];
            s1 = i2 ? xl[2 * u][1] : xl[2 * u + 1][1];
            r0 = __shfl_xor_sync(0xffffffffu, s0, 4);
            r1 = __shfl_xor_sync(0xffffffffu, s1, 4);
            lo[u] = i2 ? make_uint4(r0, r1, k0, k1) : make_uint4(k0, k1, r0, r1);
        }
    }
}

template <int N>
__device__ __forceinline__ void epi_bar_n() { asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory"); }

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(Cfg<MODE>::kMaxReg)
    k_mlp_pair(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB, Params P) {
    using C = Cfg<MODE>;
    constexpr int kEpiWarps = C::kEpiWarps, kEpiThreads = C::kEpiThreads, kHF = C::kHF;
    auto epi_bar = [] { epi_bar_n<C::kEpiThreads>(); };
    constexpr bool TEX = MODE == kModeTex, COLS = MODE == kModeCols, FACT = MODE == kModeFact;
    // h operands (and TEX's h3 skip chunks) MN-major: one 128-byte row per feature, written
    // without register transposes (b_major = MN in the instruction descriptor)
    constexpr bool kMnH = FACT || TEX;
    constexpr int NPC = C::NPC, NP = C::NP, NOUT = C::kOut, kStages = C::kStages;
    constexpr uint32_t kChunk = C::kChunk, kSkipHalf = C::kSkipHalf, kHHalf = C::kHHalf;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* skip = smem + C::kOffSkip;
    uint8_t* hbuf = smem + C::kOffH;
    uint8_t* ring = smem + C::kOffRing;
    Misc& ms = *reinterpret_cast<Misc*>(smem + C::kOffMisc);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_rank();
    const bool leader = rank == 0;
    const EvalJob& job = P.job;
    const unsigned pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    // COLS: the job may be a window [*base, *count) of the column list (records of new columns only)
    const unsigned jbase = (COLS && job.base) ? *job.base : 0u;
    const unsigned n = job_count(job) - jbase;
    float* const s_out = COLS ? P.s_out + (size_t)jbase * kSRow : nullptr;  // record of entry gi: row jbase + gi
    if (n < job.min_count || (job.max_count && n > job.max_count)) return;  // not this kernel's size class
    if (pair_id * NP >= n) {        // both CTAs of the pair take the same decision
        job_account(job);
        return;
    }
    const unsigned ntiles = (n + NP - 1) / NP;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&ms.full[s], 1);
            ptx::mbar_init(&ms.empty[s], 1);
        }
        ptx::mbar_init(&ms.f_ready, 2 * kEpiWarps);  // one arrival per epilogue warp (after __syncwarp)
        // h buffer halves: K chunks 0-1 (features 0-127) are written by CTA 0, chunks 2-3 by CTA 1
        for (int b = 0; b < 2; ++b)
            for (int h = 0; h < 2; ++h) {
                ptx::mbar_init(&ms.h_ready[b][h], kEpiWarps);
                ptx::mbar_init(&ms.h_free[b][h], 1);
            }
        for (int a = 0; a < 4; ++a) {
            ptx::mbar_init(&ms.accb[a], 1);
            ptx::mbar_init(&ms.acc_free[a], 2 * kEpiThreads);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&ms.g_ready[b], C::kAuxWarps > 0 ? C::kAuxWarps : 1);
            ptx::mbar_init(&ms.fin_done[b], kEpiWarps);
        }
        ptx::mbar_init(&ms.l1done[0], 1);
        ptx::mbar_init(&ms.l1done[1], 1);
        ptx::mbar_init(&ms.d2done, 1);
        ptx::mbar_init(&ms.d3done, 1);
        ptx::mbar_init(&ms.d4done, 1);
        ptx::mbar_init(&ms.sd_ready[0], NPC);
        ptx::mbar_init(&ms.sd_ready[1], NPC);
        ptx::mbar_init(&ms.skip_free, 1);
        ptx::mbar_init(&ms.d4_free, kEpiThreads);
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmapA);
        if (TEX) ptx::prefetch_tmap(&tmapB);
    }
    // (loaded before the start-up cluster barrier, which publishes it to every warp)
    if constexpr (MODE == kModeFact) {
        // the capsule figure of the -sdf_scale * sdf bias in shared memory (read by every tile)
        if (threadIdx.x >= 64 && threadIdx.x < 64 + kEpiThreads) {
            const int i = threadIdx.x - 64;
            const int np = __ldg(&P.f.fscene->n_prims);
            if (i < np) {
                const FPrim* pr = &P.f.fscene->prims[i];
                const float a0 = __ldg(&pr->a[0]), a1 = __ldg(&pr->a[1]), a2 = __ldg(&pr->a[2]);
                const float b0 = __ldg(&pr->b[0]) - a0, b1 = __ldg(&pr->b[1]) - a1, b2 = __ldg(&pr->b[2]) - a2;
                ms.caps[i][0] = a0;
                ms.caps[i][1] = a1;
                ms.caps[i][2] = a2;
                ms.caps[i][3] = b0;
                ms.caps[i][4] = b1;
                ms.caps[i][5] = b2;
                ms.caps[i][6] = b0 * b0 + b1 * b1 + b2 * b2;
                ms.caps[i][7] = __ldg(&pr->radius);
            }
            if (i == 0) {
                bool all = np <= ICG_MAX_PRIMS;
                for (int k = 0; k < np && all; ++k)
                    all = __ldg(&P.f.fscene->prims[k].kind) == ICG_PRIM_CAPSULE && !__ldg(&P.f.fscene->prims[k].rotated);
                ms.ncaps = all ? np : -1;
            }
        }
    }
    if (warp == 1) ptx::tmem_alloc2<512>(&ms.tmem_base);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = ms.tmem_base;
    job_account(job);


    // leader-CTA addresses of the barriers that receive cross-CTA traffic
    const uint32_t full0 = ptx::mapa(ptx::smem_u32(&ms.full[0]), 0);
    const uint32_t f_ready0 = ptx::mapa(ptx::smem_u32(&ms.f_ready), 0);
    // this CTA's half of h buffer b: h_ready0 + 16 * b
    const uint32_t h_ready0 = ptx::mapa(ptx::smem_u32(&ms.h_ready[0][rank]), 0);
    const uint32_t acc_free0 = ptx::mapa(ptx::smem_u32(&ms.acc_free[0]), 0);
    const uint32_t sd_ready0 = ptx::mapa(ptx::smem_u32(&ms.sd_ready[0]), 0);
    const uint16_t both = 0x3;

    if (warp == 0) {
        // ===================== weight producer (both CTAs) =====================
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const int per_stage = P.x3 ? 1 : 2;  // items per 32 KB box
            const uint32_t ring0 = ptx::smem_u32(ring);
            if constexpr (FACT) {
                // the MMA's consumption order, software-pipelined across tiles (see the issuer):
                // A(0) B(0) C(0) | A(1) D(0) B(1) C(1) | ... | D(last), where A/B = layer-2 items of
                // h1 chunks 0-1 / 2-3, C = layer 3, D = layer 4 (item ranges of the FACT stream)
                auto load_range = [&](int i0, int i1) {
                    for (int i = i0; i < i1; i += per_stage) {
                        ptx::mbar_wait(&ms.empty[s], ph ^ 1);
                        if (leader) ptx::mbar_arrive_expect_tx(&ms.full[s], 2 * kStage);
                        const int row0 = ((int)rank * P.total_a + i) * (P.x3 ? 256 : 128);
                        ptx::tma_load_2d_2sm(ring0 + s * kStage, &tmapA, full0 + s * 8, 0, row0);
                        if (++s == kStages) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                };
                for (unsigned t = pair_id; t < ntiles; t += npairs) {
                    load_range(0, 16);                   // A(t)
                    if (t != pair_id) load_range(40, 44);  // D(t-1)
                    load_range(16, 32);                  // B(t)
                    load_range(32, 40);                  // C(t)
                }
                load_range(40, 44);  // D(last)
            } else
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                for (int seg = 0; seg < (TEX ? 2 : 1); ++seg) {
                    const CUtensorMap* tm = seg ? &tmapB : &tmapA;
                    const int cnt = seg ? P.items_b : P.items_a;
                    const int total = seg ? P.total_b : P.total_a;
                    for (int i = 0; i < cnt; i += per_stage) {
                        ptx::mbar_wait(&ms.empty[s], ph ^ 1);
                        if (leader) ptx::mbar_arrive_expect_tx(&ms.full[s], 2 * kStage);
                        // stream layout [rank][item][hi, lo] (x3) or [rank][item][hi] (bf16), 128-row tiles
                        const int row0 = ((int)rank * total + i) * (P.x3 ? 256 : 128);
                        ptx::tma_load_2d_2sm(ring0 + s * kStage, tm, full0 + s * 8, 0, row0);
                        if (++s == kStages) {
                            s = 0;
                            ph ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader only) =====================
        if (leader && lane == 0) {
            const uint32_t idesc = ptx::idesc_bf16_f32(256, NP);
            int s = 0;
            uint32_t ph = 0, fph = 0, hph[2] = {0, 0};
            const uint32_t skip_hi = ptx::smem_u32(skip), skip_lo = skip_hi + kSkipHalf;
            const uint32_t h_hi = ptx::smem_u32(hbuf), h_lo = h_hi + kHHalf;
            const uint32_t ring0 = ptx::smem_u32(ring);
            const bool tr = P.trace && blockIdx.x == 0;
            unsigned long long w_full = 0, w_h = 0, w_f = 0, t_begin = gtime();
            auto next_stage = [&]() {
                if (++s == kStages) {
                    s = 0;
                    ph ^= 1;
                }
            };
            auto wait_full = [&]() {
                const unsigned long long t0 = tr ? gtime() : 0;
                ptx::mbar_wait(&ms.full[s], ph);
                if (tr) w_full += gtime() - t0;
                ptx::tc_fence_after();
            };
            int sub = 0;  // bf16: which of the two items of the current box
            // B operand (point activations): K-major (gathered skip operand) or MN-major (h
            // blocks written one feature per thread, FACT); A (weights) is always K-major
            const uint32_t idesc_mn = idesc | (1u << 16);
            const uint32_t idesc_f16 = idesc & ~((7u << 7) | (7u << 10));  // A, B fp16 (fp32 accumulate)
            // f16: a skip item of the TEX kernel: fp16 weights (hi, lo) x the single fp16 operand
            auto item = [&](uint32_t dcol, uint32_t b_hi, uint32_t b_lo, bool acc, bool mn = false, bool f16 = false) {
                const uint64_t bd_hi = mn ? ptx::sdesc_sw128_mn(b_hi) : ptx::sdesc_sw128(b_hi);
                const uint64_t bd_lo = mn ? ptx::sdesc_sw128_mn(b_lo) : ptx::sdesc_sw128(b_lo);
                const uint32_t id = (f16 ? idesc_f16 : idesc) | (mn ? (1u << 16) : 0u);
                if (P.x3) {
                    wait_full();
                    const uint64_t ad_hi = ptx::sdesc_sw128(ring0 + s * kStage);
                    const uint64_t ad_lo = ptx::sdesc_sw128(ring0 + s * kStage + kHalf);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t koff = (uint64_t)(kk * 2);
                        const uint64_t kb = mn ? (uint64_t)(kk * 128) : koff;  // 16 k = 16 rows of 128 B (MN)
                        ptx::mma_bf16_pair(tmem + dcol, ad_hi + koff, bd_hi + kb, id, (acc || kk > 0) ? 1u : 0u);
                        if (!f16) ptx::mma_bf16_pair(tmem + dcol, ad_hi + koff, bd_lo + kb, id, 1u);
                        ptx::mma_bf16_pair(tmem + dcol, ad_lo + koff, bd_hi + kb, id, 1u);
                    }
                    ptx::mma_commit_pair(&ms.empty[s], both);
                    next_stage();
                } else {
                    if (sub == 0) wait_full();
                    const uint64_t ad = ptx::sdesc_sw128(ring0 + s * kStage + sub * kHalf);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t koff = (uint64_t)(kk * 2);
                        const uint64_t kb = mn ? (uint64_t)(kk * 128) : koff;
                        ptx::mma_bf16_pair(tmem + dcol, ad + koff, bd_hi + kb, id, (acc || kk > 0) ? 1u : 0u);
                    }
                    if (sub == 1) {
                        ptx::mma_commit_pair(&ms.empty[s], both);
                        next_stage();
                    }
                    sub ^= 1;
                }
            };
            uint32_t hph_bits = 0;  // parity of h_ready[buf][half] at bit 2 buf + half (no local array)
            int nev = 0;  // trace: event log of block 0 (times at [64..320), codes at [320..576))
            auto ev = [&](int code) {
                if (tr && nev < 256) {
                    P.trace[64 + nev] = gtime();
                    P.trace[320 + nev] = (unsigned long long)code;
                    ++nev;
                }
            };
            auto wait_h = [&](int buf, int half) {
                ev(100 + 10 * buf + half);
                const unsigned long long t0 = tr ? gtime() : 0;
                const uint32_t bit = (uint32_t)(2 * buf + half);
                ptx::mbar_wait(&ms.h_ready[buf][half], (hph_bits >> bit) & 1u);
                if (tr) w_h += gtime() - t0;
                hph_bits ^= 1u << bit;
                ptx::tc_fence_after();
                ev(200 + 10 * buf + half);
            };
            (void)hph;
            // consume one h block (4 K chunks) of buffer `buf` for `nm` 256-row blocks, half by half;
            // `first`: the block starts the accumulation (FACT: no skip items precede it)
            auto h_block = [&](int nm, uint32_t dcol0, int buf = 0, bool first = false) {
                const uint32_t bh = h_hi + (uint32_t)buf * 2 * kHHalf, bl = bh + kHHalf;
                for (int half = 0; half < 2; ++half) {
                    wait_h(buf, half);
                    for (int jj = 2 * half; jj < 2 * half + 2; ++jj)
                        for (int m = 0; m < nm; ++m)
                            item(dcol0 + m * NP, bh + jj * kChunk, bl + jj * kChunk, !(first && jj == 0), kMnH,
                                 C::kF16H);
                    ptx::mma_commit_pair(&ms.h_free[buf][half], both);
                }
            };
            auto skipk = [&](int j) { return skip_hi + j * kChunk; };
            auto skipmn = [&](int j) { return TEX && j >= 4; };  // TEX: [Phi K-major | h3 MN-major]
            auto skipl = [&](int j) { return skip_lo + j * kChunk; };
            // TMEM columns: D2[m] = m*NP, BUF[b] = 2NP + b*NP, D3 = BUF[0], D4 = D2[0]
            uint32_t d4fph = 0;
            uint32_t cblk = 0, hblk = 0;  // COLS accumulator blocks / FACT h blocks issued so far
            auto body = [&](int ks, bool with_l4, bool wait_d4) {
                auto L1 = [&](int c) {
                    for (int j = 0; j < ks; ++j) item(2 * NP + (c & 1) * NP, skipk(j), skipl(j), j > 0, skipmn(j), C::kF16Skip);
                    ptx::mma_commit_pair(&ms.l1done[c & 1], both);
                };
                L1(0);
                L1(1);
                if (wait_d4) {  // D2[0] doubles as the previous tile's D4: its final layer must have read it
                    ptx::mbar_wait(&ms.d4_free, d4fph);
                    d4fph ^= 1;
                    ptx::tc_fence_after();
                }
                for (int m = 0; m < 2; ++m)
                    for (int j = 0; j < ks; ++j) item(m * NP, skipk(j), skipl(j), j > 0, skipmn(j), C::kF16Skip);
                for (int c = 0; c < 4; ++c) {
                    h_block(2, 0);
                    if (c + 2 < 4) L1(c + 2);
                }
                ptx::mma_commit_pair(&ms.d2done, both);
                for (int j = 0; j < ks; ++j) item(2 * NP, skipk(j), skipl(j), j > 0, skipmn(j), C::kF16Skip);
                for (int c = 0; c < 2; ++c) h_block(1, 2 * NP);
                ptx::mma_commit_pair(&ms.d3done, both);
                if (with_l4) {
                    for (int j = 0; j < ks; ++j) item(0, skipk(j), skipl(j), j > 0, skipmn(j), C::kF16Skip);
                    ptx::mma_commit_pair(&ms.skip_free, both);  // last reader of the skip operand
                    h_block(1, 0);
                    ptx::mma_commit_pair(&ms.d4done, both);
                } else {
                    // prefix: h3 is in the skip operands of both CTAs
                    for (int half = 0; half < 2; ++half) {
                        wait_h(0, half);
                        ptx::mma_commit_pair(&ms.h_free[0][half], both);
                    }
                }
            };
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                if constexpr (!FACT) {  // FACT: operands arrive through the h buffers only
                    const unsigned long long t0 = tr ? gtime() : 0;
                    ptx::mbar_wait(&ms.f_ready, fph);
                    if (tr) w_f += gtime() - t0;
                }
                fph ^= 1;
                ptx::tc_fence_after();
                const bool later = t != pair_id;
                if constexpr (TEX) {
                    body(4, false, later);
                    body(8, true, false);
                } else if constexpr (COLS) {
                    // 8 blocks of 256 rows, each K = 256 (the Phi channels), through a ring of 4 accumulators
                    for (int b = 0; b < kColsBlocks; ++b) {
                        const int a = (int)(cblk & 3u);
                        ptx::mbar_wait(&ms.acc_free[a], ((cblk >> 2) & 1u) ^ 1u);
                        ptx::tc_fence_after();
                        for (int j = 0; j < 4; ++j) item((uint32_t)a * NP, skipk(j), skipl(j), j > 0);
                        ptx::mma_commit_pair(&ms.accb[a], both);
                        ++cblk;
                    }
                    ptx::mma_commit_pair(&ms.skip_free, both);
                } else if constexpr (FACT) {
                    // TMEM: D2[m] = m*NP, D3 = 2NP, D4 = 3NP; h blocks alternate between two buffers.
                    // Software-pipelined across tiles: the previous tile's layer 4 runs after this
                    // tile's first two layer-2 chunks, so the tensor cores have work while the
                    // epilogue emits the previous tile's layer-3 output (h3).
                    for (int c = 0; c < 2; ++c) h_block(2, 0, (int)(hblk++ & 1u), c == 0);  // A(t)
                    if (later) {                                                               // D(t-1)
                        h_block(1, 3 * NP, (int)(hblk++ & 1u), true);
                        ptx::mma_commit_pair(&ms.d4done, both);
                        ev(304);
                    }
                    for (int c = 2; c < 4; ++c) h_block(2, 0, (int)(hblk++ & 1u), false);  // B(t)
                    ptx::mma_commit_pair(&ms.d2done, both);
                    ev(302);
                    for (int c = 0; c < 2; ++c) h_block(1, 2 * NP, (int)(hblk++ & 1u), c == 0);  // C(t)
                    ptx::mma_commit_pair(&ms.d3done, both);
                    ev(303);
                    if (t + npairs >= ntiles) {  // D(last)
                        h_block(1, 3 * NP, (int)(hblk++ & 1u), true);
                        ptx::mma_commit_pair(&ms.d4done, both);
                        ev(304);
                    }
                } else {
                    body(4, true, later);
                }
            }
            if (tr) {
                P.trace[0] = gtime() - t_begin;
                P.trace[1] = w_full;
                P.trace[2] = w_h;
                P.trace[3] = w_f;
            }
        }
    } else if (C::kAuxWarps > 0 && warp >= 2 + kEpiWarps) {
        // ===================== FACT auxiliary warps: gather tiles ahead =====================
        const int at = (int)threadIdx.x - (64 + kEpiThreads);
        constexpr int kAT = 32 * C::kAuxWarps;
        const int aw = at >> 5;
        auto aux_bar = [] { asm volatile("bar.sync 2, %0;" ::"n"(32 * C::kAuxWarps) : "memory"); };
        const float* b5 = P.bias_g + 2 * (1024 + 512 + 256 + 128);
        constexpr int wls = 128 + kGeoSkip;
        uint32_t fph_bits = 0;
        unsigned tl = 0;
        for (unsigned t = pair_id; t < ntiles; t += npairs, ++tl) {
            const int gb = (int)(tl & 1u);
            if (tl >= 2) {  // the epilogue's final layer of tile tl-2 is done with these buffers
                ptx::mbar_wait(&ms.fin_done[gb], (fph_bits >> gb) & 1u);
                fph_bits ^= 1u << gb;
            }
            // positions, column records
            for (int p = at; p < NP; p += kAT) {
                const unsigned idx = t * NP + (unsigned)p;
                double pd[3] = {0.0, 0.0, 0.0};
                int sl = 0;
                if (idx < n) {
                    job_point_d(job, idx, pd);
                    const uint32_t n1 = (uint32_t)job.cells + 1u, col = job_node(job, idx) % (n1 * n1);
                    sl = P.cmap ? __ldg(&P.cmap[col]) : (int)col;
                }
                ms.slot[gb][p] = sl;
                for (int d = 0; d < 3; ++d) ms.pos[gb][p][d] = (float)pd[d];
                ms.z[gb][p] = (float)pd[2];
            }
            aux_bar();
            // per 32-point chunk: first / last record and which points use the last one
            for (int c = aw; c < NP / 32; c += C::kAuxWarps) {
                const int sv = ms.slot[gb][32 * c + lane];
                const int first = __shfl_sync(0xffffffffu, sv, 0), last = __shfl_sync(0xffffffffu, sv, 31);
                const uint32_t m = __ballot_sync(0xffffffffu, sv == last);
                const uint32_t ok = __all_sync(0xffffffffu, sv == first || sv == last);
                if (lane == 0) {
                    ms.cfirst[gb][c] = first;
                    ms.clast[gb][c] = last;
                    ms.cmask[gb][c] = m;
                    ms.cok[gb][c] = ok;
                }
            }
            if (leader) {  // the final layer's Phi dot and constant term (-sdf_scale sdf + b5 + w5z z)
                for (int p = at; p < NP; p += kAT) {
                    ms.skipdot[gb][0][p] = __ldg(&P.s_in[(size_t)ms.slot[gb][p] * kSRow + kSFinal]);
                    const float* P3 = ms.pos[gb][p];
                    float d = 3.0e38f;
                    const int nc = ms.ncaps;
                    if (nc >= 0) {
                        for (int i = 0; i < nc; ++i) {
                            const float* c = ms.caps[i];
                            const float pa0 = P3[0] - c[0], pa1 = P3[1] - c[1], pa2 = P3[2] - c[2];
                            float hh = 0.0f;
                            if (c[6] > 0.0f) hh = fminf(fmaxf((pa0 * c[3] + pa1 * c[4] + pa2 * c[5]) / c[6], 0.0f), 1.0f);
                            const float v0 = pa0 - hh * c[3], v1 = pa1 - hh * c[4], v2 = pa2 - hh * c[5];
                            d = fminf(d, sqrtf(v0 * v0 + v1 * v1 + v2 * v2) - c[7]);
                        }
                        if (nc == 0) d = 0.0f;
                    } else {
                        d = scene_sdf_f(P.f.fscene, P3);
                    }
                    ms.cterm[gb][p] = __ldg(&b5[0]) + __ldg(&P.wlast[wls - 1]) * ms.z[gb][p] -
                                      __ldg(&P.f.fscene->sdf_scale) * d;
                }
            }
            aux_bar();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&ms.g_ready[gb]);
        }
    } else {
        // ===================== gather + epilogue (8 warps, both CTAs) =====================
        const int et = threadIdx.x - 64;
        const int ew = et >> 5;
        const int quarter = warp & 3;
        const int colq = (warp - 2) >> 2;
        const int colh = colq / (kEpiWarps / 8);  // point half this warp converts = destination CTA
        const int hf0 = (colq % (kEpiWarps / 8)) * kHF;  // its first 32-point chunk inside that half
        const int row = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(colh * NPC);
        uint32_t l1ph[2] = {0, 0}, d2ph = 0, d3ph = 0, d4ph = 0, hfph = 1, sdph_bits = 0, sfph = 0;
        unsigned tile_iter = 0;
        const float* zc = ms.z[0];  // z of the tile being converted
        const int* slc = ms.slot[0];  // FACT: column records of the tile being converted
        int ms_tile_parity = 0;       // FACT: parity of that tile (chunk record info)
        uint32_t hfph_bits = 3u;      // h_free parity per h buffer (bit buf)
        uint32_t hbe = 0;             // FACT: h blocks emitted so far (buffer = hbe & 1)
        const FieldDev& f = P.f;
        const bool odd = lane & 1;
        // this thread's feature inside a 256-row block, and its K position in the next layer's operand
        const uint32_t feat = rank * 128u + (uint32_t)row;
        const uint32_t kc_off = (feat >> 6) * kChunk;
        const uint32_t c16 = (feat & 63u) >> 3;  // 16-byte chunk of this lane group's 8 features
        // h buffer of the owning CTA: warps converting this CTA's own points store locally (plain
        // st.shared, CTA-scope proxy fence), the others through DSMEM (cluster-scope fence)
        const bool local_dst = (uint32_t)colh == rank;
        const uint32_t hdst = local_dst ? ptx::smem_u32(hbuf) : ptx::mapa(ptx::smem_u32(hbuf), (uint32_t)colh);
        const uint32_t sdst = local_dst ? ptx::smem_u32(skip) + 4 * kChunk
                                        : ptx::mapa(ptx::smem_u32(skip) + 4 * kChunk, (uint32_t)colh);  // texture: h3 -> skip
        auto st_h = [local_dst](uint32_t a, uint4 v) {
            if (local_dst)
                ptx::st_shared_v4(a, v);
            else
                ptx::st_cluster_v4(a, v);
        };

        const bool etr = P.trace && blockIdx.x == 0 && et == 0;
        int nee = 0;  // trace: epilogue event log (times at [576..832), codes at [832..1088))
        auto eev = [&](int code) {
            if (etr && nee < 256) {
                P.trace[576 + nee] = gtime();
                P.trace[832 + nee] = (unsigned long long)code;
                ++nee;
            }
        };
        unsigned long long e_acc = 0, e_hf = 0, e_emit = 0, e_t0 = 0, e_begin = gtime();
        unsigned long long e_cyc[3] = {0, 0, 0};
        // TMEM columns [col, col + NPC) of this thread's lane -> next layer's operand in the owning CTA
        // soff >= 0 (FACT): add the column-record term S[slot(p)][soff + o]; from_tmem == false
        // (FACT layer 1): there is no accumulator, the pre-activation is the column term alone
        // FACT: a block's global operands (bias, z weight, the two column-record terms of each
        // 32-point chunk), loaded one block ahead so their latency overlaps the previous block
        struct Pre {
            float bo, wz, sA[kHF], sB[kHF];
        };
        auto fact_pre = [&](const float* bias_blk, int out_dim, int feat0, int soff, int cp) {
            Pre q;
            const int o = feat0 + (int)feat;
            q.bo = __ldg(&bias_blk[o]);
            q.wz = __ldg(&bias_blk[out_dim + o]);
#pragma unroll
            for (int hi = 0; hi < kHF; ++hi) {
                const int c = colh * (NPC / 32) + hf0 + hi;
                q.sA[hi] = __ldg(P.s_in + soff + o + (size_t)ms.cfirst[cp][c] * kSRow);
                q.sB[hi] = __ldg(P.s_in + soff + o + (size_t)ms.clast[cp][c] * kSRow);
            }
            return q;
        };
        auto emit_block = [&](uint32_t col, const float* bias_blk, int out_dim, int feat0, uint32_t dst,
                              uint32_t lo_off, bool write_lo, int soff = -1, bool from_tmem = true,
                              const Pre* pre = nullptr, bool f16 = false) {
            const int o = feat0 + (int)feat;
            const float bo = FACT ? pre->bo : __ldg(&bias_blk[o]);
            const float wz = FACT ? pre->wz : __ldg(&bias_blk[out_dim + o]);
            float sA[kHF], sB[kHF];
            uint32_t smask[kHF], sok[kHF];
            if constexpr (FACT) {
                const int cp = ms_tile_parity;
#pragma unroll
                for (int hi = 0; hi < kHF; ++hi) {
                    const int c = colh * (NPC / 32) + hf0 + hi;
                    sok[hi] = ms.cok[cp][c];
                    smask[hi] = ms.cmask[cp][c];
                    sA[hi] = pre->sA[hi];
                    sB[hi] = pre->sB[hi];
                }
            }
            unsigned long long c0 = etr ? clock64() : 0;
#pragma unroll
            for (int hi = 0; hi < kHF; ++hi) {
                const int hf = hf0 + hi;
                uint32_t r[32];
                if constexpr (FACT) {
                    const float* sbase = P.s_in + soff + o;
                    const int* sl = slc + colh * NPC + hf * 32;
                    if (from_tmem) ptx::tmem_ld32(lane_base + col + hf * 32, r);
                    // points are sorted by column record: a 32-point chunk uses one or two records
                    if (sok[hi]) {
                        if (from_tmem) ptx::tmem_ld_wait();
                        const uint32_t m = smask[hi];
#pragma unroll
                        for (int q = 0; q < 32; ++q) {
                            const float sq = (m >> q) & 1u ? sB[hi] : sA[hi];
                            r[q] = __float_as_uint((from_tmem ? __uint_as_float(r[q]) : 0.0f) + sq);
                        }
                    } else {  // three or more records in the chunk (rare): one load per point
                        if (from_tmem) ptx::tmem_ld_wait();
#pragma unroll
                        for (int q = 0; q < 32; ++q)
                            r[q] = __float_as_uint((from_tmem ? __uint_as_float(r[q]) : 0.0f) +
                                                   __ldg(sbase + (size_t)sl[q] * kSRow));
                    }
                } else {
                    ptx::tmem_ld32(lane_base + col + hf * 32, r);
                    ptx::tmem_ld_wait();
                }
                if (etr) {
                    const unsigned long long c1 = clock64();
                    e_cyc[0] += c1 - c0;
                    c0 = c1;
                }
                float v[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const float x = __uint_as_float(r[q]) + fmaf(wz, zc[colh * NPC + hf * 32 + q], bo);
                    v[q] = x < 0.0f ? x * P.slope : x;
                }
                if constexpr (kMnH) {
                    // MN-major operand: this thread's feature is one 128-byte row (64 points) of its
                    // K-chunk; points hf*32 + 8u .. +7 are the 16-byte chunk hf*4 + u (swizzled by row)
                    const uint32_t fr = feat & 63u;
                    const uint32_t rbase = (feat >> 6) * kChunk + fr * 128u;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        uint4 hv, lv;
                        uint32_t* hp = reinterpret_cast<uint32_t*>(&hv);
                        uint32_t* lp = reinterpret_cast<uint32_t*>(&lv);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float a = v[8 * u + 2 * i], b = v[8 * u + 2 * i + 1];
                            if (f16) {
                                __half2 f2 = __floats2half2_rn(a, b);
                                hp[i] = *reinterpret_cast<uint32_t*>(&f2);
                                lp[i] = 0u;
                            } else {
                                hp[i] = pack_bf16(a, b);
                                lp[i] = pack_bf16(a - __uint_as_float(hp[i] << 16), b - __uint_as_float(hp[i] & 0xFFFF0000u));
                            }
                        }
                        const uint32_t off = rbase + ((((uint32_t)(hf * 4 + u)) ^ (fr & 7u)) << 4);
                        st_h(dst + off, hv);
                        if (write_lo) st_h(dst + lo_off + off, lv);
                    }
                    continue;
                }
                // rows (points) 8u + (lane & 7) of this hf block, 16-byte chunk of this lane group's 8 features
                uint4 hv[4], lv[4];
                if (f16)
                    transpose8_bf16<false, true>(v, hv, lv);
                else if (write_lo)
                    transpose8_bf16<true>(v, hv, lv);
                else
                    transpose8_bf16<false>(v, hv, lv);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t pl = (uint32_t)(hf * 32 + 8 * u + (lane & 7));
                    const uint32_t off = kc_off + pl * 128u + (((c16 ^ pl) & 7u) << 4);
                    st_h(dst + off, hv[u]);
                    if (write_lo) st_h(dst + lo_off + off, lv[u]);
                }
                if (etr) {
                    const unsigned long long c1 = clock64();
                    e_cyc[1] += c1 - c0;
                    c0 = c1;
                }
            }
        };
        auto h_begin = [&](int buf = 0) {
            const unsigned long long t0 = etr ? gtime() : 0;
            ptx::mbar_wait(&ms.h_free[buf][rank], (hfph_bits >> buf) & 1u);
            hfph_bits ^= 1u << buf;
            (void)hfph;
            if (etr) {
                e_t0 = gtime();
                e_hf += e_t0 - t0;
            }
        };
        auto h_end = [&](int buf = 0) {
            const unsigned long long c0 = etr ? clock64() : 0;
            // every lane makes its own stores visible to the async proxy; after the warp
            // barrier one lane arrives for the warp (256 remote arrivals per block would serialise)
            if (local_dst)
                ptx::fence_proxy_async_smem();
            else
                ptx::fence_proxy_async_cluster();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                // own shared memory only: CTA-scope release (no MEMBAR.ALL.GPU); DSMEM stores to the
                // peer keep the cluster-scope release
                if (local_dst)
                    ptx::mbar_arrive_remote(h_ready0 + 16u * (uint32_t)buf);
                else
                    ptx::mbar_arrive_cluster(h_ready0 + 16u * (uint32_t)buf);
            }
            if (etr) {
                e_cyc[2] += clock64() - c0;
                e_emit += gtime() - e_t0;
            }
        };
        auto wait_acc = [&](uint64_t* bar, uint32_t& par) {
            eev(400);
            const unsigned long long t0 = etr ? gtime() : 0;
            ptx::mbar_wait(bar, par);
            eev(401);
            par ^= 1;
            ptx::tc_fence_after();
            if (etr) e_acc += gtime() - t0;
        };
        // epilogue of one MLP body (layers 1-3); `after_l1c0` runs once layer-1 chunk 0 is done
        auto body_epi = [&](const float* bias, bool prefix, auto&& after_l1c0) {
            const float* b1 = bias;
            const float* b2 = b1 + 2 * 1024;
            const float* b3 = b2 + 2 * 512;
            for (int c = 0; c < 4; ++c) {
                wait_acc(&ms.l1done[c & 1], l1ph[c & 1]);
                if (c == 0) after_l1c0();
                h_begin();
                emit_block(2 * NP + (c & 1) * NP, b1, 1024, c * 256, hdst, kHHalf, P.x3 && !C::kF16H, -1, true, nullptr,
                           C::kF16H);
                h_end();
            }
            wait_acc(&ms.d2done, d2ph);
            for (int m = 0; m < 2; ++m) {
                h_begin();
                emit_block(m * NP, b2, 512, m * 256, hdst, kHHalf, P.x3 && !C::kF16H, -1, true, nullptr, C::kF16H);
                h_end();
            }
            wait_acc(&ms.d3done, d3ph);
            h_begin();
            if (prefix)  // h3 -> skip K-chunks 4..7 (TEX: the single fp16 skip copy)
                emit_block(2 * NP, b3, 256, 0, sdst, kSkipHalf, !C::kF16Skip, -1, true, nullptr, C::kF16Skip);
            else
                emit_block(2 * NP, b3, 256, 0, hdst, kHHalf, P.x3 && !C::kF16H, -1, true, nullptr, C::kF16H);
            h_end();
        };

        const float* bias = TEX ? P.bias_t : P.bias_g;
        const float* b4 = bias + 2 * (1024 + 512 + 256);
        const float* b5 = b4 + 2 * 128;
        constexpr int wl_stride = 128 + C::kSkipDim;

        // positions + Phi gather of pair tile tg into the skip operand (parity gb buffers)
        auto gather_tile = [&](unsigned tg, int gb) {
            // ---- positions of all points of the pair tile (every CTA needs z for its epilogue) ----
            if (et < NP) {
                const unsigned idx = tg * NP + et;
                double pd[3] = {0.0, 0.0, 0.0};
                if constexpr (COLS) {
                    // list entry = a column i + n j of the level grid; its node at k = 0 gives (x, y)
                    if (idx < n) node_pos_d(job_node(job, jbase + idx), job.cells, pd);
                } else {
                    // world point (view-space fields: view_to_world of the node, render.hpp:98-99)
                    if (idx < n) field_point_d(f, job, idx, pd);
                }
                if constexpr (FACT) {
                    int sl = 0;
                    if (idx < n) {
                        const uint32_t n1 = (uint32_t)job.cells + 1u, col = job_node(job, idx) % (n1 * n1);
                        sl = P.cmap ? __ldg(&P.cmap[col]) : (int)col;
                    }
                    ms.slot[gb][et] = sl;
                }
                for (int d = 0; d < 3; ++d) ms.pos[gb][et][d] = (float)pd[d];
                float q[3];
                input_coords(f, ms.pos[gb][et], q);
                ms.z[gb][et] = q[2];  // depth feature of the input camera
            }
            epi_bar();
            if constexpr (FACT) {
                // no Phi operand: the final layer's Phi dot is part of the column record
                if (leader && et < NP) ms.skipdot[gb][0][et] = __ldg(&P.s_in[(size_t)ms.slot[gb][et] * kSRow + kSFinal]);
                if (et < NP) {  // one warp per 32-point chunk
                    const int c = et >> 5, sv = ms.slot[gb][et];
                    const int first = __shfl_sync(0xffffffffu, sv, 0), last = __shfl_sync(0xffffffffu, sv, 31);
                    const uint32_t m = __ballot_sync(0xffffffffu, sv == last);
                    const uint32_t ok = __all_sync(0xffffffffu, sv == first || sv == last);
                    if (lane == 0) {
                        ms.cfirst[gb][c] = first;
                        ms.clast[gb][c] = last;
                        ms.cmask[gb][c] = m;
                        ms.cok[gb][c] = ok;
                    }
                }
                epi_bar();
            } else
            // ---- gather Phi for this CTA's points into its skip operand ----
            // warp per point (2 in flight); lane = 8 consecutive channels = one 16-byte
            // SW128 chunk of the bf16 operand; the same pass computes the final
            // layer's Phi-part skip dot in fp32.
            {
                const int c0 = 8 * lane;
                const uint32_t chunk = (uint32_t)(c0 >> 6) * kChunk;
                const uint32_t c16 = (uint32_t)((c0 & 63) >> 3);
                const size_t rowW = (size_t)f.W * f.C;
                float w5s[NOUT][8];
#pragma unroll
                for (int c = 0; c < NOUT; ++c)
#pragma unroll
                    for (int i = 0; i < 8; ++i) w5s[c][i] = __ldg(&P.wlast[c * wl_stride + 128 + c0 + i]);
                constexpr int kPerWarp = NPC / kEpiWarps;
                for (int it = 0; it < kPerWarp / 2; ++it) {
                    float4 tv[2][8];
                    float wts[2][4];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int p = (int)rank * NPC + ew * kPerWarp + it * 2 + j;
                        float q[3];
                        input_coords(f, ms.pos[gb][p], q);  // Phi at the input camera's (x, y)
                        float u = (q[0] + 1.0f) * 0.5f * (float)(f.W - 1);
                        float v = (1.0f - q[1]) * 0.5f * (float)(f.H - 1);
                        u = fminf(fmaxf(u, 0.0f), (float)(f.W - 1));
                        v = fminf(fmaxf(v, 0.0f), (float)(f.H - 1));
                        const int x0 = min((int)floorf(u), f.W - 2), y0 = min((int)floorf(v), f.H - 2);
                        const float ax = u - (float)x0, ay = v - (float)y0;
                        wts[j][0] = (1.0f - ax) * (1.0f - ay);
                        wts[j][1] = ax * (1.0f - ay);
                        wts[j][2] = (1.0f - ax) * ay;
                        wts[j][3] = ax * ay;
                        const float* m00 = f.fmap_hwc + ((size_t)y0 * f.W + x0) * (size_t)f.C + c0;
                        const float* taps[4] = {m00, m00 + f.C, m00 + rowW, m00 + rowW + f.C};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            tv[j][2 * q] = __ldg(reinterpret_cast<const float4*>(taps[q]));
                            tv[j][2 * q + 1] = __ldg(reinterpret_cast<const float4*>(taps[q] + 4));
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int pl = ew * kPerWarp + it * 2 + j;
                        float val[8];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const float4 a0 = tv[j][h], a1 = tv[j][2 + h], a2 = tv[j][4 + h], a3 = tv[j][6 + h];
                            val[4 * h + 0] = wts[j][0] * a0.x + wts[j][1] * a1.x + wts[j][2] * a2.x + wts[j][3] * a3.x;
                            val[4 * h + 1] = wts[j][0] * a0.y + wts[j][1] * a1.y + wts[j][2] * a2.y + wts[j][3] * a3.y;
                            val[4 * h + 2] = wts[j][0] * a0.z + wts[j][1] * a1.z + wts[j][2] * a2.z + wts[j][3] * a3.z;
                            val[4 * h + 3] = wts[j][0] * a0.w + wts[j][1] * a1.w + wts[j][2] * a2.w + wts[j][3] * a3.w;
                        }
                        uint4 hv, lv;
                        uint32_t* hp = reinterpret_cast<uint32_t*>(&hv);
                        uint32_t* lp = reinterpret_cast<uint32_t*>(&lv);
                        float dot[NOUT];
#pragma unroll
                        for (int c = 0; c < NOUT; ++c) dot[c] = 0.0f;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float a = val[2 * i], b = val[2 * i + 1];
                            if constexpr (C::kF16Skip) {
                                __half2 f2 = __floats2half2_rn(a, b);
                                hp[i] = *reinterpret_cast<uint32_t*>(&f2);
                                lp[i] = 0u;
                            } else {
                                hp[i] = pack_bf16(a, b);
                                lp[i] = pack_bf16(a - __uint_as_float(hp[i] << 16), b - __uint_as_float(hp[i] & 0xFFFF0000u));
                            }
#pragma unroll
                            for (int c = 0; c < NOUT; ++c) {
                                dot[c] = fmaf(w5s[c][2 * i], a, dot[c]);
                                dot[c] = fmaf(w5s[c][2 * i + 1], b, dot[c]);
                            }
                        }
                        const uint32_t off = chunk + (uint32_t)pl * 128u + (((c16 ^ (uint32_t)pl) & 7u) << 4);
                        *reinterpret_cast<uint4*>(skip + off) = hv;
                        if constexpr (!C::kF16Skip) *reinterpret_cast<uint4*>(skip + kSkipHalf + off) = lv;
#pragma unroll
                        for (int c = 0; c < NOUT; ++c)
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) dot[c] += __shfl_xor_sync(0xffffffffu, dot[c], o);
                        if (lane == 0) {
                            if constexpr (COLS) {
                                const unsigned gi = tg * NP + rank * NPC + (unsigned)pl;
                                if (gi < n) s_out[(size_t)gi * kSRow + kSFinal] = dot[0];
                            } else if (TEX) {
#pragma unroll
                                for (int c = 0; c < NOUT; ++c) ms.sdl[c][pl] = dot[c];
                            } else {
                                const int p = (int)rank * NPC + pl;
                                if (leader) {
                                    ms.skipdot[gb][0][p] = dot[0];
                                } else {
                                    ptx::st_cluster_f32(ptx::mapa(ptx::smem_u32(&ms.skipdot[gb][0][p]), 0), dot[0]);
                                    ptx::mbar_arrive_cluster(sd_ready0 + 8 * gb);
                                }
                            }
                        }
                    }
                }
            }
            ptx::fence_proxy_async_smem();  // the skip operand is this CTA's own shared memory
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(f_ready0);
        };

        // ---- final layer (CTA 0 holds layer-4 rows 0..127 for all points) ----
        auto final_layer = [&](unsigned t, int tp) {
            const unsigned base = t * NP;
            if (leader) {
                const float bo = __ldg(&b4[row]), wz = __ldg(&b4[128 + row]);
                float w5[NOUT];
#pragma unroll
                for (int c = 0; c < NOUT; ++c) w5[c] = __ldg(&P.wlast[c * wl_stride + row]);
#pragma unroll
                for (int hi = 0; hi < kHF; ++hi) {
                const int hf = hf0 + hi;
                    uint32_t r[32];
                    float s4a = 0.0f, s4b = 0.0f;
                    uint32_t s4m = 0, s4ok = 1;
                    if (FACT) {
                        const int c = colh * (NPC / 32) + hf;
                        s4ok = ms.cok[tp][c];
                        s4m = ms.cmask[tp][c];
                        s4a = __ldg(&P.s_in[(size_t)ms.cfirst[tp][c] * kSRow + kSOffL(3) + row]);
                        s4b = __ldg(&P.s_in[(size_t)ms.clast[tp][c] * kSRow + kSOffL(3) + row]);
                    }
                    ptx::tmem_ld32(lane_base + (FACT ? 3 * NP : 0) + hf * 32, r);
                    ptx::tmem_ld_wait();
                    float hx[32];
#pragma unroll
                    if (FACT && !s4ok) {  // three or more records in the chunk (rare)
#pragma unroll 4
                        for (int q = 0; q < 32; ++q)
                            r[q] = __float_as_uint(__uint_as_float(r[q]) +
                                                   __ldg(&P.s_in[(size_t)slc[colh * NPC + hf * 32 + q] * kSRow + kSOffL(3) + row]));
                    }
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const float acc4 =
                            FACT && s4ok ? __uint_as_float(r[q]) + ((s4m >> q) & 1u ? s4b : s4a) : __uint_as_float(r[q]);
                        const float x = acc4 + fmaf(wz, zc[colh * NPC + hf * 32 + q], bo);
                        hx[q] = x < 0.0f ? x * P.slope : x;
                    }
                    if constexpr (NOUT == 1) {  // in place: fewer live registers
#pragma unroll
                        for (int q = 0; q < 32; ++q) hx[q] *= w5[0];
                        ms.red[quarter][0][colh * NPC + hf * 32 + lane] = warp_transpose_reduce(hx);
                    } else {
#pragma unroll
                        for (int c = 0; c < NOUT; ++c) {
                            float v[32];
#pragma unroll
                            for (int q = 0; q < 32; ++q) v[q] = w5[c] * hx[q];
                            ms.red[quarter][c][colh * NPC + hf * 32 + lane] = warp_transpose_reduce(v);
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            epi_bar();
            if (leader) {
                if (!FACT) {  // FACT: the leader read every point's Phi dot from the column records
                    ptx::mbar_wait_cluster(&ms.sd_ready[tp], (sdph_bits >> tp) & 1u);
                    sdph_bits ^= 1u << tp;
                }
                for (int e = et; e < NP * NOUT; e += kEpiThreads) {  // (texture: 384 outputs, 256 threads)
                    const int p = e % NP, c = e / NP;
                    const unsigned idx = base + p;
                    const float s = ms.red[0][c][p] + ms.red[1][c][p] + ms.red[2][c][p] + ms.red[3][c][p] +
                                    ms.skipdot[tp][c][p] + ms.cterm[FACT ? tp : c][p];
                    if (idx < n) {
                        float v = 1.0f / (1.0f + expf(-s));
                        if (TEX) {
                            if (job.out_pixel) {
                                v = fminf(fmaxf(v, 0.0f), 1.0f);  // clamp01, render.hpp:276
                                job.out[(size_t)job.out_pixel[idx] * 3 + c] = v;
                            } else {
                                job.out[(size_t)idx * 3 + c] = v;
                            }
                        } else if (job_is_grid(job)) {
                            grid_epilogue(job, job_node(job, idx), v);
                        } else {
                            job.out[idx] = v;
                        }
                    }
                }
                if (!FACT) ptx::mbar_arrive(&ms.d4_free);  // D4 and this tile's skip dots consumed
            }
            epi_bar();
        };

        if constexpr (COLS) {
            // ---- column pass: drain each 256-row block of S = W_Phi . Phi into the column records ----
            uint32_t cb = 0;
            gather_tile(pair_id, 0);
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                const int tp = (int)(tile_iter & 1u);
                for (int b = 0; b < kColsBlocks; ++b) {
                    const int a = (int)(cb & 3u);
                    ptx::mbar_wait(&ms.accb[a], (cb >> 2) & 1u);
                    ptx::tc_fence_after();
                    // block b: layer-1 blocks 0-3, layer-2 blocks 0-1, layer 3, layer 4 (128 rows)
                    const int roff = b < 4 ? b * 256 : (b < 6 ? 1024 + (b - 4) * 256 : (b == 6 ? 1536 : 1792));
                    const bool valid = b < 7 || feat < 128u;
#pragma unroll
                    for (int hi = 0; hi < kHF; ++hi) {
                const int hf = hf0 + hi;
                        uint32_t r[32];
                        ptx::tmem_ld32(lane_base + (uint32_t)a * NP + hf * 32, r);
                        ptx::tmem_ld_wait();
                        if (valid) {
#pragma unroll
                            for (int q = 0; q < 32; ++q) {
                                const unsigned gi = t * NP + (unsigned)(colh * NPC + hf * 32 + q);
                                if (gi < n) s_out[(size_t)gi * kSRow + roff + feat] = __uint_as_float(r[q]);
                            }
                        }
                    }
                    ptx::tc_fence_before();
                    ptx::mbar_arrive_remote(acc_free0 + 8u * (uint32_t)a);
                    ++cb;
                }
                if (t + npairs < ntiles) {
                    ptx::mbar_wait(&ms.skip_free, sfph);
                    sfph ^= 1;
                    gather_tile(t + npairs, tp ^ 1);
                }
                ++tile_iter;
            }
        } else if constexpr (FACT) {
            const float* b1 = P.bias_g;
            const float* b2 = b1 + 2 * 1024;
            const float* b3 = b2 + 2 * 512;
            auto emit_h = [&](uint32_t col, const float* bb, int od, int f0, int soff, bool tm, const Pre& pre) {
                const int buf = (int)(hbe++ & 1u);
                eev(500 + buf);
                h_begin(buf);
                eev(510 + buf);
                emit_block(col, bb, od, f0, hdst + (uint32_t)buf * 2u * kHHalf, kHHalf, P.x3, soff, tm, &pre);
                eev(520 + buf);
                h_end(buf);
                eev(530 + buf);
            };
            auto step_pre = [&](int kk, int cp) {
                const int l = kk < 4 ? 0 : (kk < 6 ? 1 : 2);
                const int blk = kk < 4 ? kk : (kk < 6 ? kk - 4 : 0);
                return fact_pre(l == 0 ? b1 : (l == 1 ? b2 : b3), 1024 >> l, blk * 256, kSOffL(l), cp);
            };
            // -sdf_scale * sdf(P) + b5 + w5z z of the tile's points (parity gb): two threads per point
            // split the capsules (same per-capsule arithmetic as scene_sdf_f)
            auto fact_cterm = [&](int gb) {
                const int p = et >> 1, h = et & 1;
                const float* P3 = ms.pos[gb][p];
                float d = 3.0e38f;
                const int nc = ms.ncaps;
                if (nc >= 0) {
                    for (int i = h; i < nc; i += 2) {
                        const float* c = ms.caps[i];
                        const float pa0 = P3[0] - c[0], pa1 = P3[1] - c[1], pa2 = P3[2] - c[2];
                        float hh = 0.0f;
                        if (c[6] > 0.0f) hh = fminf(fmaxf((pa0 * c[3] + pa1 * c[4] + pa2 * c[5]) / c[6], 0.0f), 1.0f);
                        const float v0 = pa0 - hh * c[3], v1 = pa1 - hh * c[4], v2 = pa2 - hh * c[5];
                        d = fminf(d, sqrtf(v0 * v0 + v1 * v1 + v2 * v2) - c[7]);
                    }
                    d = fminf(d, __shfl_xor_sync(0xffffffffu, d, 1));
                    if (nc == 0) d = 0.0f;
                } else if (h == 0) {
                    d = scene_sdf_f(f.fscene, P3);
                }
                if (h == 0 && p < NP)
                    ms.cterm[gb][p] = __ldg(&b5[0]) + __ldg(&P.wlast[wl_stride - 1]) * ms.z[gb][p] -
                                      __ldg(&f.fscene->sdf_scale) * d;
            };
            // Per tile t the epilogue emits layer-1 chunks 2-3 of t; then, while the tensor cores
            // finish layer 2 of t, the final layer of t-1 and the gather of t+1; then h2 of t, the
            // layer-1 chunks 0-1 of t+1 and h3 of t -- the order the issuer consumes them in
            // (A(t+1) before D(t), so the tensor cores work while h3 is converted).
            // One emit site: the epilogue is large and inlining it per step costs registers.
            const float* b_of[3] = {b1, b2, b3};
            (void)b_of;
            auto run_steps = [&](int k0, int k1, int cp) {
                Pre cur = step_pre(k0, cp);
#pragma unroll 1
                for (int k = k0; k < k1; ++k) {
                    Pre nxt = cur;
                    if (k + 1 < k1) nxt = step_pre(k + 1, cp);  // in flight during this block
                    if (k == 4) wait_acc(&ms.d2done, d2ph);
                    if (k == 6) wait_acc(&ms.d3done, d3ph);
                    const int l = k < 4 ? 0 : (k < 6 ? 1 : 2);
                    const int blk = k < 4 ? k : (k < 6 ? k - 4 : 0);
                    emit_h(l == 0 ? 0u : (uint32_t)(l == 1 ? blk : 2) * NP, l == 0 ? b1 : (l == 1 ? b2 : b3),
                           1024 >> l, blk * 256, kSOffL(l), l > 0, cur);
                    cur = nxt;
                }
            };
            auto set_tile = [&](int gb) {
                zc = ms.z[gb];
                slc = ms.slot[gb];
                ms_tile_parity = gb;
            };
            // tiles are gathered ahead by the auxiliary warps (g_ready per parity buffer)
            uint32_t gph_bits = 0;
            auto wait_g = [&](int gb) {
                ptx::mbar_wait(&ms.g_ready[gb], (gph_bits >> gb) & 1u);
                gph_bits ^= 1u << gb;
            };
            (void)fact_cterm;
            wait_g(0);
            set_tile(0);
            run_steps(0, 2, 0);
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                const int tp = (int)(tile_iter & 1u);
                const bool has_next = t + npairs < ntiles;
                set_tile(tp);
                run_steps(2, 4, tp);
                if (t != pair_id) {  // the previous tile's final layer (its D4 is long done)
                    set_tile(tp ^ 1);
                    wait_acc(&ms.d4done, d4ph);
                    eev(600);
                    final_layer(t - npairs, tp ^ 1);
                    eev(601);
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&ms.fin_done[tp ^ 1]);  // its buffers may be refilled
                }
                set_tile(tp);
                run_steps(4, 6, tp);  // h2 of t
                if (has_next) {       // the next tile's first layer-1 chunks, before h3 of t: the MMA
                    wait_g(tp ^ 1);    // runs layer 2 of t+1 while h3 is converted (issuer order)
                    set_tile(tp ^ 1);
                    run_steps(0, 2, tp ^ 1);
                }
                set_tile(tp);
                run_steps(6, 7, tp);  // h3 of t
                ++tile_iter;
            }
            {  // the last tile's final layer
                const int tp = (int)((tile_iter - 1u) & 1u);
                set_tile(tp);
                wait_acc(&ms.d4done, d4ph);
                final_layer(pair_id + (tile_iter - 1u) * npairs, tp);
            }
        } else {
        gather_tile(pair_id, 0);
        for (unsigned t = pair_id; t < ntiles; t += npairs) {
            const unsigned base = t * NP;
            const int tp = (int)(tile_iter & 1u);
            zc = ms.z[tp];
            // constant part of the final logits, b5 + w5z*z (- sdf_scale*sdf(P) for geometry), off the
            // MMA critical path: the tensor cores are busy with layer 1 now
            if (leader && et < NP) {
                float extra = 0.0f;
                if (!TEX) extra = -__ldg(&f.fscene->sdf_scale) * scene_sdf_f(f.fscene, ms.pos[tp][et]);
                for (int c = 0; c < NOUT; ++c)
                    ms.cterm[c][et] = __ldg(&b5[c]) + __ldg(&P.wlast[c * wl_stride + wl_stride - 1]) * ms.z[tp][et] + extra;
            }

            if (TEX) {
                body_epi(P.bias_g, true, [] {});
                // texture body: when its layer-1 chunk 0 is done, h3 (skip chunks 4..7) has been
                // consumed by the tensor cores, i.e. it is complete in both CTAs -> add the h3
                // part of the final skip dot for this CTA's points (fp32 from hi + lo)
                body_epi(P.bias_t, false, [&] {
                    epi_bar();  // ms.sdl from the gather warps
                    // NPC points x kSl slices of 256 / kSl features (h3 = skip K 256..511, fp16)
                    constexpr int kSl = kEpiThreads / NPC, kSF = 256 / kSl;
                    const int pl = et / kSl, part = et % kSl;
                    float acc[NOUT];
#pragma unroll
                    for (int c = 0; c < NOUT; ++c) acc[c] = 0.0f;
                    for (int j = part * kSF; j < part * kSF + kSF; j += 2) {
                        const int k = 256 + j;
                        float x0, x1;
                        if constexpr (kMnH) {
                            // MN-major h3 chunk: feature row fr, point pl at 16-byte chunk pl / 8 (swizzled)
                            const uint32_t fr = (uint32_t)(k & 63), cb = (uint32_t)(k >> 6) * kChunk + ((uint32_t)pl & 7u) * 2u;
                            const uint32_t o0 = cb + fr * 128u + (((((uint32_t)pl >> 3) ^ fr) & 7u) << 4);
                            const uint32_t o1 = cb + (fr + 1u) * 128u + (((((uint32_t)pl >> 3) ^ (fr + 1u)) & 7u) << 4);
                            x0 = __half2float(*reinterpret_cast<const __half*>(skip + o0));
                            x1 = __half2float(*reinterpret_cast<const __half*>(skip + o1));
                        } else {
                        const uint32_t off = (uint32_t)(k >> 6) * kChunk + sw128((uint32_t)pl, (uint32_t)(k & 63));
                        const uint32_t hv = *reinterpret_cast<const uint32_t*>(skip + off);
                        if constexpr (C::kF16Skip) {
                            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&hv));
                            x0 = f.x;
                            x1 = f.y;
                        } else {
                            const uint32_t lv = *reinterpret_cast<const uint32_t*>(skip + kSkipHalf + off);
                            x0 = __uint_as_float(hv << 16) + __uint_as_float(lv << 16);
                            x1 = __uint_as_float(hv & 0xFFFF0000u) + __uint_as_float(lv & 0xFFFF0000u);
                        }
                        }
#pragma unroll
                        for (int c = 0; c < NOUT; ++c) {
                            acc[c] = fmaf(__ldg(&P.wlast[c * wl_stride + 128 + k]), x0, acc[c]);
                            acc[c] = fmaf(__ldg(&P.wlast[c * wl_stride + 128 + k + 1]), x1, acc[c]);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < NOUT; ++c)
#pragma unroll
                        for (int o = 1; o < kSl; o <<= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
                    if (part == 0) {
                        const int p = (int)rank * NPC + pl;
#pragma unroll
                        for (int c = 0; c < NOUT; ++c) {
                            const float v = acc[c] + ms.sdl[c][pl];
                            if (leader)
                                ms.skipdot[tp][c][p] = v;
                            else
                                ptx::st_cluster_f32(ptx::mapa(ptx::smem_u32(&ms.skipdot[tp][c][p]), 0), v);
                        }
                        if (!leader) ptx::mbar_arrive_cluster(sd_ready0 + 8 * tp);
                    }
                });
            } else {
                body_epi(P.bias_g, false, [] {});
            }
            // the next tile's gather overlaps this tile's last MMAs and final layer
            if (t + npairs < ntiles) {
                ptx::mbar_wait(&ms.skip_free, sfph);
                sfph ^= 1;
                gather_tile(t + npairs, tp ^ 1);
            }
            wait_acc(&ms.d4done, d4ph);
            final_layer(t, tp);
            ++tile_iter;
        }
        }  // GEO / TEX
        if (etr) {
            P.trace[4] = gtime() - e_begin;
            P.trace[5] = e_acc;
            P.trace[6] = e_hf;
            P.trace[7] = e_emit;
            P.trace[8] = e_cyc[0];
            P.trace[9] = e_cyc[1];
            P.trace[10] = e_cyc[2];
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc2<512>(tmem);
    }
}

}  // namespace pair

// ===========================================================================
// Host side: pair weight streams + tensor maps + launch
// ===========================================================================
static inline uint16_t f2bf_p(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    uint32_t r = ((u >> 16) & 1u) + 0x7FFFu;
    return (uint16_t)((u + r) >> 16);
}
static inline float bf2f_p(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// x3 stream: [rank][item][hi, lo] 16 KB tiles; hi stream (bf16 mode): [rank][item][hi]
size_t pair_stream_bytes(int which, bool x3) {
    return (size_t)(which == ICG_MLP_GEOMETRY ? pair::kGeoItems : pair::kTexItems) * (x3 ? 4 : 2) * pair::kHalf;
}

// item i, rank r (rows r*128.. of the 256-row block), part (hi/lo): 16 KB SW128 tile
// sched: 0 = full network (pair::schedule), 1 = FACT items, 2 = COLS items (geometry only)
// f16skip: items over the skip input (K columns >= the hidden width) as fp16 hi / lo (the TEX
// kernel's single fp16 skip operand); everything else bf16 hi / lo
static int pair_pack_sched(int which, int sched, const float* const* w, uint8_t* stream_x3, uint8_t* stream_hi,
                           bool f16skip = false, bool f16all = false) {
    const bool geo = which == ICG_MLP_GEOMETRY;
    const int* outs = geo ? kGeoOut : kTexOut;
    const int skip = geo ? kGeoSkip : kTexSkip;
    const int nitems = sched == 1 ? pair::kFactItems
                                  : sched == 2 ? pair::kColsItems : (geo ? pair::kGeoItems : pair::kTexItems);
    int ins[5];
    for (int l = 0; l < 5; ++l) ins[l] = (l ? outs[l - 1] : 0) + skip;
    int item = 0;
    auto emit = [&](int l, int m, int col0) {
        const bool f16 = f16all || (f16skip && col0 >= (l ? outs[l - 1] : 0));
        for (int h = 0; h < 2; ++h) {
            uint8_t* hi = stream_x3 + ((size_t)(h * nitems + item) * 2 + 0) * pair::kHalf;
            uint8_t* lo = stream_x3 + ((size_t)(h * nitems + item) * 2 + 1) * pair::kHalf;
            uint8_t* h2 = stream_hi + (size_t)(h * nitems + item) * pair::kHalf;
            for (int r = 0; r < 128; ++r) {
                const int o = m * 256 + h * 128 + r;
                for (int k = 0; k < 64; ++k) {
                    float v = o < outs[l] ? w[l][(size_t)o * ins[l] + col0 + k] : 0.0f;
                    uint16_t a, b;
                    if (f16) {
                        const __half ha = __float2half_rn(v);
                        const __half hb = __float2half_rn(v - __half2float(ha));
                        std::memcpy(&a, &ha, 2);
                        std::memcpy(&b, &hb, 2);
                    } else {
                        a = f2bf_p(v);
                        b = f2bf_p(v - bf2f_p(a));
                    }
                    size_t off = (size_t)r * 128 + (size_t)(((k >> 3) ^ (r & 7)) << 4) + (size_t)(k & 7) * 2;
                    std::memcpy(hi + off, &a, 2);
                    std::memcpy(lo + off, &b, 2);
                    std::memcpy(h2 + off, &a, 2);
                }
            }
        }
        ++item;
    };
    if (sched == 1)
        pair::schedule_fact(emit);
    else if (sched == 2)
        pair::schedule_cols(emit);
    else
        pair::schedule(geo ? 4 : 8, true, emit);
    return item == nitems ? ICG_OK : ICG_ERUNTIME;
}

int pair_pack(int which, const float* const* w, uint8_t* stream_x3, uint8_t* stream_hi, bool f16skip) {
    // f16skip: the texture kernel's streams -- every item fp16 hi / lo (its operands are fp16)
    return pair_pack_sched(which, 0, w, stream_x3, stream_hi, f16skip, f16skip);
}

size_t pair_fact_stream_bytes(int part, bool x3) {
    return (size_t)(part == 0 ? pair::kFactItems : pair::kColsItems) * (x3 ? 4 : 2) * pair::kHalf;
}

int pair_pack_factored(const float* const* w, int part, uint8_t* stream_x3, uint8_t* stream_hi) {
    return pair_pack_sched(ICG_MLP_GEOMETRY, part == 0 ? 1 : 2, w, stream_x3, stream_hi);
}

int pair_make_tmap(const void* dev_stream, size_t bytes, void* tmap_out /* 128-byte CUtensorMap */, unsigned box_rows) {
    // the pre-swizzled stream as bytes: rows of 128 B, one stage = box_rows rows
    return make_tmap_2d(dev_stream, CU_TENSOR_MAP_DATA_TYPE_UINT8, bytes / 128, 128, 128, 128, box_rows,
                        CU_TENSOR_MAP_SWIZZLE_NONE, tmap_out);
}

template <int MODE>
static int launch_pair(pair::Params p, const void* tmapA, const void* tmapB, unsigned max_points, cudaStream_t s) {
    using C = pair::Cfg<MODE>;
    constexpr bool TEX = MODE == pair::kModeTex;
    static PerDeviceOnce once;
    if (int r = once.run([] {
            ICG_CUDA_TRY(cudaFuncSetAttribute(pair::k_mlp_pair<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)C::kTotal));
            return ICG_OK;
        }))
        return r;
    // dev trace buffer (ICG_TC_TRACE=1), created once (thread-safe static initialisation)
    static unsigned long long* const trace = [] {
        const char* e = getenv("ICG_TC_TRACE");
        unsigned long long* t = nullptr;
        if (e && e[0] == '1' && cudaMallocManaged(&t, 2048 * sizeof(unsigned long long)) != cudaSuccess) t = nullptr;
        return t;
    }();
    p.trace = trace;
    if (p.trace) cudaMemsetAsync(p.trace, 0, 2048 * 8, s);
    unsigned pairs = (max_points + C::NP - 1) / C::NP;
    if (pairs > 74) pairs = 74;
    if (pairs == 0) pairs = 1;
    CUtensorMap ta, tb;
    std::memcpy(&ta, tmapA, sizeof(CUtensorMap));
    std::memcpy(&tb, tmapB ? tmapB : tmapA, sizeof(CUtensorMap));
    pair::k_mlp_pair<MODE><<<2 * pairs, C::kThreads, C::kTotal, s>>>(ta, tb, p);
    if (const cudaError_t e = cudaGetLastError()) {
        set_error("k_mlp_pair<" + std::to_string(MODE) + ">: " + cudaGetErrorString(e));
        return ICG_ERUNTIME;
    }
    if (p.trace) {
        cudaStreamSynchronize(s);
        const unsigned long long* t = p.trace;
        fprintf(stderr,
                "[pair-trace %s] mma: total %.1f us, wait data %.1f, wait h %.1f, wait f %.1f | epi: total %.1f, wait acc "
                "%.1f, wait hfree %.1f, emit %.1f\n",
                TEX ? "tex" : (MODE == pair::kModeGeo ? "geo" : (MODE == pair::kModeCols ? "cols" : (MODE == pair::kModeGeo64 ? "geo64" : "fact"))), t[0] * 1e-3, t[1] * 1e-3, t[2] * 1e-3, t[3] * 1e-3, t[4] * 1e-3, t[5] * 1e-3,
                t[6] * 1e-3, t[7] * 1e-3);
        fprintf(stderr, "    epi cycles: tmem-ld %llu, convert+store %llu, fence+arrive %llu\n", t[8], t[9], t[10]);
        if (getenv("ICG_TC_EVENTS") && (t[64] || t[576])) {
            // merged event log of block 0: MMA (m) and epilogue thread 0 (e), us from the first event
            unsigned long long t0 = ~0ull;
            for (int i = 0; i < 256; ++i) {
                if (t[64 + i] && t[64 + i] < t0) t0 = t[64 + i];
                if (t[576 + i] && t[576 + i] < t0) t0 = t[576 + i];
            }
            int a = 0, b = 0;
            while ((a < 256 && t[64 + a]) || (b < 256 && t[576 + b])) {
                const bool ta = a < 256 && t[64 + a], tb = b < 256 && t[576 + b];
                if (ta && (!tb || t[64 + a] <= t[576 + b])) {
                    fprintf(stderr, "  m %8.2f %llu\n", (t[64 + a] - t0) * 1e-3, t[320 + a]);
                    ++a;
                } else {
                    fprintf(stderr, "  e %8.2f %llu\n", (t[576 + b] - t0) * 1e-3, t[832 + b]);
                    ++b;
                }
            }
        }
    }
    return ICG_OK;
}

int launch_pifu_pair_eval(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& job,
                          unsigned max_points, bool x3, cudaStream_t s) {
    pair::Params p{};
    p.f = f;
    p.job = job;
    p.bias_g = geo.bias;
    p.wlast = geo.w_last;
    p.items_a = pair::kGeoItems;
    p.total_a = pair::kGeoItems;
    p.slope = 0.02f;
    p.x3 = x3 ? 1 : 0;
    return launch_pair<pair::kModeGeo>(p, tmap, nullptr, max_points, s);
}

int launch_pifu_pair_eval_small(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& job,
                                unsigned max_points, bool x3, cudaStream_t s) {
    pair::Params p{};
    p.f = f;
    p.job = job;
    p.bias_g = geo.bias;
    p.wlast = geo.w_last;
    p.items_a = pair::kGeoItems;
    p.total_a = pair::kGeoItems;
    p.slope = 0.02f;
    p.x3 = x3 ? 1 : 0;
    return launch_pair<pair::kModeGeo64>(p, tmap, nullptr, max_points, s);
}

int launch_pifu_pair_cols(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& cols, float* records,
                          unsigned max_cols, bool x3, cudaStream_t s) {
    pair::Params p{};
    p.f = f;
    p.job = cols;
    p.bias_g = geo.bias;
    p.wlast = geo.w_last;
    p.items_a = pair::kColsItems;
    p.total_a = pair::kColsItems;
    p.slope = 0.02f;
    p.x3 = x3 ? 1 : 0;
    p.s_out = records;
    return launch_pair<pair::kModeCols>(p, tmap, nullptr, max_cols, s);
}

int launch_pifu_pair_fact(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& job,
                          const float* records, const int* cmap, unsigned max_points, bool x3, cudaStream_t s) {
    pair::Params p{};
    p.f = f;
    p.job = job;
    p.bias_g = geo.bias;
    p.wlast = geo.w_last;
    p.items_a = pair::kFactItems;
    p.total_a = pair::kFactItems;
    p.slope = 0.02f;
    p.x3 = x3 ? 1 : 0;
    p.s_in = records;
    p.cmap = cmap;
    return launch_pair<pair::kModeFact>(p, tmap, nullptr, max_points, s);
}

int launch_pifu_pair_texture(const FieldDev& f, const TcMlp& geo, const TcMlp& tex, const void* tmap_geo,
                             const void* tmap_tex, const EvalJob& job, unsigned max_points, bool x3,
                             cudaStream_t s) {
    pair::Params p{};
    p.f = f;
    p.job = job;
    p.bias_g = geo.bias;
    p.bias_t = tex.bias;
    p.wlast = tex.w_last;
    p.items_a = pair::kPrefixItems;  // the geometry prefix = the first items of the geometry stream
    p.items_b = pair::kTexItems;
    p.total_a = pair::kGeoItems;
    p.total_b = pair::kTexItems;
    p.slope = 0.02f;
    p.x3 = x3 ? 1 : 0;
    return launch_pair<pair::kModeTex>(p, tmap_geo, tmap_tex, max_points, s);
}

}  // namespace icg

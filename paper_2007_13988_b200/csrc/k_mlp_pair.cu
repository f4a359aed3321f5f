// k_mlp_pair.cu — the PIFu geometry and texture fields on CTA PAIRS
// (tcgen05 cta_group::2).
//
// Same fused "weights x activations^T" dataflow as k_mlp_tc.cu, but every MMA
// is M=256 x N x K=16 executed by the two SMs of a TPC: each CTA of the
// cluster holds 128 of the 256 weight rows (A) and N/2 of the N points (B) in
// its shared memory; its TMEM holds its 128 output rows for all N points.  Per
// SM this halves the shared-memory operand bytes per FLOP and doubles the
// tensor work per pipeline stage relative to the single-CTA 128xN MMA (the
// single-CTA kernel measured ~25% tensor-pipe activity, bound by per-stage
// overheads and SMEM operand traffic).
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
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kEpiThreads;
constexpr int kMaxNP = 128;
constexpr int kMaxStages = 6;

template <bool TEX>
struct Cfg {
    static constexpr int NPC = TEX ? 32 : 64;        // points per CTA
    static constexpr int NP = 2 * NPC;               // points per pair tile = MMA N
    static constexpr int kSkipChunks = TEX ? 8 : 4;  // [Phi] or [Phi, h3] in 64-wide K-chunks
    static constexpr int kStages = TEX ? 3 : 2;  // 32 KB stages (per-copy TMA cost is size-independent)
    static constexpr uint32_t kChunk = NPC * 128;  // NPC point rows x 64 bf16 (SW128)
    static constexpr uint32_t kSkipHalf = kSkipChunks * kChunk;
    static constexpr uint32_t kHHalf = 4 * kChunk;  // one 256-feature block
    static constexpr uint32_t kOffSkip = 0;
    static constexpr uint32_t kOffH = kOffSkip + 2 * kSkipHalf;
    static constexpr uint32_t kOffRing = kOffH + 2 * kHHalf;
    static constexpr uint32_t kOffMisc = kOffRing + kStages * kStage;
    static constexpr uint32_t kMisc = 20480;
    static constexpr uint32_t kTotal = kOffMisc + kMisc + 1024;
    static constexpr int kOut = TEX ? 3 : 1;
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

struct Misc {
    uint64_t full[kMaxStages], empty[kMaxStages];
    uint64_t f_ready, h_ready[2], h_free[2], l1done[2], d2done, d3done, d4done, sd_ready[2], skip_free, d4_free;
    uint32_t tmem_base;
    float z[2][kMaxNP];       // by tile parity (the next tile is gathered before this one's final layer)
    float pos[2][kMaxNP][3];
    float red[4][3][kMaxNP];      // final layer: per-lane-quarter partial sums over features
    float skipdot[2][3][kMaxNP];  // final layer: skip-input dots (leader, all points), by tile parity
    float sdl[3][kMaxNP / 2];     // texture: this CTA's Phi-part skip dots until h3 is known
    float cterm[3][kMaxNP];       // b5 + w5z*z (- sdf_scale*sdf for geometry)
};
static_assert(sizeof(Misc) + 16 <= Cfg<false>::kMisc, "misc smem too small");

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
template <bool LO>
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
        __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
        wh[m] = *reinterpret_cast<uint32_t*>(&h2);
        if (LO) {
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

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); }

template <bool TEX>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_mlp_pair(const __grid_constant__ CUtensorMap tmapA, const __grid_constant__ CUtensorMap tmapB, Params P) {
    using C = Cfg<TEX>;
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
    const unsigned n = job_count(job);
    if (n < job.min_count) return;  // small batch: latency path
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
        ptx::mbar_init(&ms.f_ready, 2 * kEpiThreads);
        // h buffer halves: K chunks 0-1 (features 0-127) are written by CTA 0, chunks 2-3 by CTA 1
        ptx::mbar_init(&ms.h_ready[0], kEpiThreads);
        ptx::mbar_init(&ms.h_ready[1], kEpiThreads);
        ptx::mbar_init(&ms.h_free[0], 1);
        ptx::mbar_init(&ms.h_free[1], 1);
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
    if (warp == 1) ptx::tmem_alloc2<512>(&ms.tmem_base);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = ms.tmem_base;
    job_account(job);

    // leader-CTA addresses of the barriers that receive cross-CTA traffic
    const uint32_t full0 = ptx::mapa(ptx::smem_u32(&ms.full[0]), 0);
    const uint32_t f_ready0 = ptx::mapa(ptx::smem_u32(&ms.f_ready), 0);
    const uint32_t h_ready0 = ptx::mapa(ptx::smem_u32(&ms.h_ready[rank]), 0);  // this CTA's half
    const uint32_t sd_ready0 = ptx::mapa(ptx::smem_u32(&ms.sd_ready[0]), 0);
    const uint16_t both = 0x3;

    if (warp == 0) {
        // ===================== weight producer (both CTAs) =====================
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const int per_stage = P.x3 ? 1 : 2;  // items per 32 KB box
            const uint32_t ring0 = ptx::smem_u32(ring);
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
            auto item = [&](uint32_t dcol, uint32_t b_hi, uint32_t b_lo, bool acc) {
                const uint64_t bd_hi = ptx::sdesc_sw128(b_hi), bd_lo = ptx::sdesc_sw128(b_lo);
                if (P.x3) {
                    wait_full();
                    const uint64_t ad_hi = ptx::sdesc_sw128(ring0 + s * kStage);
                    const uint64_t ad_lo = ptx::sdesc_sw128(ring0 + s * kStage + kHalf);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t koff = (uint64_t)(kk * 2);
                        ptx::mma_bf16_pair(tmem + dcol, ad_hi + koff, bd_hi + koff, idesc, (acc || kk > 0) ? 1u : 0u);
                        ptx::mma_bf16_pair(tmem + dcol, ad_hi + koff, bd_lo + koff, idesc, 1u);
                        ptx::mma_bf16_pair(tmem + dcol, ad_lo + koff, bd_hi + koff, idesc, 1u);
                    }
                    ptx::mma_commit_pair(&ms.empty[s], both);
                    next_stage();
                } else {
                    if (sub == 0) wait_full();
                    const uint64_t ad = ptx::sdesc_sw128(ring0 + s * kStage + sub * kHalf);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t koff = (uint64_t)(kk * 2);
                        ptx::mma_bf16_pair(tmem + dcol, ad + koff, bd_hi + koff, idesc, (acc || kk > 0) ? 1u : 0u);
                    }
                    if (sub == 1) {
                        ptx::mma_commit_pair(&ms.empty[s], both);
                        next_stage();
                    }
                    sub ^= 1;
                }
            };
            auto wait_h = [&](int half) {
                const unsigned long long t0 = tr ? gtime() : 0;
                ptx::mbar_wait_cluster(&ms.h_ready[half], hph[half]);
                if (tr) w_h += gtime() - t0;
                hph[half] ^= 1;
                ptx::tc_fence_after();
            };
            // consume one h block (4 K chunks) for `nm` 256-row blocks, half by half
            auto h_block = [&](int nm, uint32_t dcol0) {
                for (int half = 0; half < 2; ++half) {
                    wait_h(half);
                    for (int jj = 2 * half; jj < 2 * half + 2; ++jj)
                        for (int m = 0; m < nm; ++m)
                            item(dcol0 + m * NP, h_hi + jj * kChunk, h_lo + jj * kChunk, true);
                    ptx::mma_commit_pair(&ms.h_free[half], both);
                }
            };
            auto skipk = [&](int j) { return skip_hi + j * kChunk; };
            auto skipl = [&](int j) { return skip_lo + j * kChunk; };
            // TMEM columns: D2[m] = m*NP, BUF[b] = 2NP + b*NP, D3 = BUF[0], D4 = D2[0]
            uint32_t d4fph = 0;
            auto body = [&](int ks, bool with_l4, bool wait_d4) {
                auto L1 = [&](int c) {
                    for (int j = 0; j < ks; ++j) item(2 * NP + (c & 1) * NP, skipk(j), skipl(j), j > 0);
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
                    for (int j = 0; j < ks; ++j) item(m * NP, skipk(j), skipl(j), j > 0);
                for (int c = 0; c < 4; ++c) {
                    h_block(2, 0);
                    if (c + 2 < 4) L1(c + 2);
                }
                ptx::mma_commit_pair(&ms.d2done, both);
                for (int j = 0; j < ks; ++j) item(2 * NP, skipk(j), skipl(j), j > 0);
                for (int c = 0; c < 2; ++c) h_block(1, 2 * NP);
                ptx::mma_commit_pair(&ms.d3done, both);
                if (with_l4) {
                    for (int j = 0; j < ks; ++j) item(0, skipk(j), skipl(j), j > 0);
                    ptx::mma_commit_pair(&ms.skip_free, both);  // last reader of the skip operand
                    h_block(1, 0);
                    ptx::mma_commit_pair(&ms.d4done, both);
                } else {
                    // prefix: h3 is in the skip operands of both CTAs
                    for (int half = 0; half < 2; ++half) {
                        wait_h(half);
                        ptx::mma_commit_pair(&ms.h_free[half], both);
                    }
                }
            };
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                {
                    const unsigned long long t0 = tr ? gtime() : 0;
                    ptx::mbar_wait_cluster(&ms.f_ready, fph);
                    if (tr) w_f += gtime() - t0;
                }
                fph ^= 1;
                ptx::tc_fence_after();
                const bool later = t != pair_id;
                if (TEX) {
                    body(4, false, later);
                    body(8, true, false);
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
    } else {
        // ===================== gather + epilogue (8 warps, both CTAs) =====================
        const int et = threadIdx.x - 64;
        const int ew = et >> 5;
        const int quarter = warp & 3;
        const int colh = (warp - 2) >> 2;  // point half this warp converts = destination CTA
        const int row = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(colh * NPC);
        uint32_t l1ph[2] = {0, 0}, d2ph = 0, d3ph = 0, d4ph = 0, hfph = 1, sdph[2] = {0, 0}, sfph = 0;
        unsigned tile_iter = 0;
        const float* zc = ms.z[0];  // z of the tile being converted
        const FieldDev& f = P.f;
        const bool odd = lane & 1;
        // this thread's feature inside a 256-row block, and its K position in the next layer's operand
        const uint32_t feat = rank * 128u + (uint32_t)row;
        const uint32_t kc_off = (feat >> 6) * kChunk;
        const uint32_t c16 = (feat & 63u) >> 3;  // 16-byte chunk of this lane group's 8 features
        const uint32_t hdst = ptx::mapa(ptx::smem_u32(hbuf), (uint32_t)colh);  // h buffer of the owning CTA
        const uint32_t sdst = ptx::mapa(ptx::smem_u32(skip) + 4 * kChunk, (uint32_t)colh);  // texture: h3 -> skip

        const bool etr = P.trace && blockIdx.x == 0 && et == 0;
        unsigned long long e_acc = 0, e_hf = 0, e_emit = 0, e_t0 = 0, e_begin = gtime();
        unsigned long long e_cyc[3] = {0, 0, 0};
        // TMEM columns [col, col + NPC) of this thread's lane -> next layer's operand in the owning CTA
        auto emit_block = [&](uint32_t col, const float* bias_blk, int out_dim, int feat0, uint32_t dst,
                              uint32_t lo_off, bool write_lo) {
            const int o = feat0 + (int)feat;
            const float bo = __ldg(&bias_blk[o]);
            const float wz = __ldg(&bias_blk[out_dim + o]);
            unsigned long long c0 = etr ? clock64() : 0;
#pragma unroll
            for (int hf = 0; hf < NPC / 32; ++hf) {
                uint32_t r[32];
                ptx::tmem_ld32(lane_base + col + hf * 32, r);
                ptx::tmem_ld_wait();
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
                // rows (points) 8u + (lane & 7) of this hf block, 16-byte chunk of this lane group's 8 features
                uint4 hv[4], lv[4];
                if (write_lo)
                    transpose8_bf16<true>(v, hv, lv);
                else
                    transpose8_bf16<false>(v, hv, lv);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t pl = (uint32_t)(hf * 32 + 8 * u + (lane & 7));
                    const uint32_t off = kc_off + pl * 128u + (((c16 ^ pl) & 7u) << 4);
                    ptx::st_cluster_v4(dst + off, hv[u]);
                    if (write_lo) ptx::st_cluster_v4(dst + lo_off + off, lv[u]);
                }
                if (etr) {
                    const unsigned long long c1 = clock64();
                    e_cyc[1] += c1 - c0;
                    c0 = c1;
                }
            }
        };
        auto h_begin = [&]() {
            const unsigned long long t0 = etr ? gtime() : 0;
            ptx::mbar_wait(&ms.h_free[rank], hfph);
            hfph ^= 1;
            if (etr) {
                e_t0 = gtime();
                e_hf += e_t0 - t0;
            }
        };
        auto h_end = [&]() {
            const unsigned long long c0 = etr ? clock64() : 0;
            ptx::fence_proxy_async_cluster();
            ptx::tc_fence_before();
            ptx::mbar_arrive_cluster(h_ready0);
            if (etr) {
                e_cyc[2] += clock64() - c0;
                e_emit += gtime() - e_t0;
            }
        };
        auto wait_acc = [&](uint64_t* bar, uint32_t& par) {
            const unsigned long long t0 = etr ? gtime() : 0;
            ptx::mbar_wait(bar, par);
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
                emit_block(2 * NP + (c & 1) * NP, b1, 1024, c * 256, hdst, kHHalf, P.x3);
                h_end();
            }
            wait_acc(&ms.d2done, d2ph);
            for (int m = 0; m < 2; ++m) {
                h_begin();
                emit_block(m * NP, b2, 512, m * 256, hdst, kHHalf, P.x3);
                h_end();
            }
            wait_acc(&ms.d3done, d3ph);
            h_begin();
            if (prefix)  // h3 -> skip K-chunks 4..7 (lo always: the final skip dot reads hi + lo)
                emit_block(2 * NP, b3, 256, 0, sdst, kSkipHalf, true);
            else
                emit_block(2 * NP, b3, 256, 0, hdst, kHHalf, P.x3);
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
                if (idx < n) job_point_d(job, idx, pd);
                for (int d = 0; d < 3; ++d) ms.pos[gb][et][d] = (float)pd[d];
                ms.z[gb][et] = (float)pd[2];
            }
            epi_bar();
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
                        float u = (ms.pos[gb][p][0] + 1.0f) * 0.5f * (float)(f.W - 1);
                        float v = (1.0f - ms.pos[gb][p][1]) * 0.5f * (float)(f.H - 1);
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
                            hp[i] = pack_bf16(a, b);
                            lp[i] = pack_bf16(a - __uint_as_float(hp[i] << 16), b - __uint_as_float(hp[i] & 0xFFFF0000u));
#pragma unroll
                            for (int c = 0; c < NOUT; ++c) {
                                dot[c] = fmaf(w5s[c][2 * i], a, dot[c]);
                                dot[c] = fmaf(w5s[c][2 * i + 1], b, dot[c]);
                            }
                        }
                        const uint32_t off = chunk + (uint32_t)pl * 128u + (((c16 ^ (uint32_t)pl) & 7u) << 4);
                        *reinterpret_cast<uint4*>(skip + off) = hv;
                        *reinterpret_cast<uint4*>(skip + kSkipHalf + off) = lv;
#pragma unroll
                        for (int c = 0; c < NOUT; ++c)
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) dot[c] += __shfl_xor_sync(0xffffffffu, dot[c], o);
                        if (lane == 0) {
                            if (TEX) {
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
            ptx::fence_proxy_async_cluster();
            ptx::mbar_arrive_cluster(f_ready0);
        };

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
                    const int pl = et >> 3, part = et & 7;  // NPC = 32 points x 8 slices of 32 features
                    float acc[NOUT];
#pragma unroll
                    for (int c = 0; c < NOUT; ++c) acc[c] = 0.0f;
                    for (int j = part * 32; j < part * 32 + 32; j += 2) {
                        const int k = 256 + j;
                        const uint32_t off = (uint32_t)(k >> 6) * kChunk + sw128((uint32_t)pl, (uint32_t)(k & 63));
                        const uint32_t hv = *reinterpret_cast<const uint32_t*>(skip + off);
                        const uint32_t lv = *reinterpret_cast<const uint32_t*>(skip + kSkipHalf + off);
                        const float x0 = __uint_as_float(hv << 16) + __uint_as_float(lv << 16);
                        const float x1 = __uint_as_float(hv & 0xFFFF0000u) + __uint_as_float(lv & 0xFFFF0000u);
#pragma unroll
                        for (int c = 0; c < NOUT; ++c) {
                            acc[c] = fmaf(__ldg(&P.wlast[c * wl_stride + 128 + k]), x0, acc[c]);
                            acc[c] = fmaf(__ldg(&P.wlast[c * wl_stride + 128 + k + 1]), x1, acc[c]);
                        }
                    }
#pragma unroll
                    for (int c = 0; c < NOUT; ++c)
#pragma unroll
                        for (int o = 1; o < 8; o <<= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
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
            // ---- final layer (CTA 0 holds layer-4 rows 0..127 for all points) ----
            if (leader) {
                const float bo = __ldg(&b4[row]), wz = __ldg(&b4[128 + row]);
                float w5[NOUT];
#pragma unroll
                for (int c = 0; c < NOUT; ++c) w5[c] = __ldg(&P.wlast[c * wl_stride + row]);
#pragma unroll
                for (int hf = 0; hf < NPC / 32; ++hf) {
                    uint32_t r[32];
                    ptx::tmem_ld32(lane_base + hf * 32, r);
                    ptx::tmem_ld_wait();
                    float hx[32];
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const float x = __uint_as_float(r[q]) + fmaf(wz, zc[colh * NPC + hf * 32 + q], bo);
                        hx[q] = x < 0.0f ? x * P.slope : x;
                    }
#pragma unroll
                    for (int c = 0; c < NOUT; ++c) {
                        float v[32];
#pragma unroll
                        for (int q = 0; q < 32; ++q) v[q] = w5[c] * hx[q];
                        ms.red[quarter][c][colh * NPC + hf * 32 + lane] = warp_transpose_reduce(v);
                    }
                }
            }
            ptx::tc_fence_before();
            epi_bar();
            if (leader) {
                ptx::mbar_wait_cluster(&ms.sd_ready[tp], sdph[tp]);
                sdph[tp] ^= 1;
                if (et < NP * NOUT) {
                    const int p = et % NP, c = et / NP;
                    const unsigned idx = base + p;
                    const float s = ms.red[0][c][p] + ms.red[1][c][p] + ms.red[2][c][p] + ms.red[3][c][p] +
                                    ms.skipdot[tp][c][p] + ms.cterm[c][p];
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
                ptx::mbar_arrive(&ms.d4_free);  // D4 and this tile's skip dots consumed
            }
            epi_bar();
            ++tile_iter;
        }
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
int pair_pack(int which, const float* const* w, uint8_t* stream_x3, uint8_t* stream_hi) {
    const bool geo = which == ICG_MLP_GEOMETRY;
    const int* outs = geo ? kGeoOut : kTexOut;
    const int skip = geo ? kGeoSkip : kTexSkip;
    const int nitems = geo ? pair::kGeoItems : pair::kTexItems;
    int ins[5];
    for (int l = 0; l < 5; ++l) ins[l] = (l ? outs[l - 1] : 0) + skip;
    int item = 0;
    auto emit = [&](int l, int m, int col0) {
        for (int h = 0; h < 2; ++h) {
            uint8_t* hi = stream_x3 + ((size_t)(h * nitems + item) * 2 + 0) * pair::kHalf;
            uint8_t* lo = stream_x3 + ((size_t)(h * nitems + item) * 2 + 1) * pair::kHalf;
            uint8_t* h2 = stream_hi + (size_t)(h * nitems + item) * pair::kHalf;
            for (int r = 0; r < 128; ++r) {
                const int o = m * 256 + h * 128 + r;
                for (int k = 0; k < 64; ++k) {
                    float v = o < outs[l] ? w[l][(size_t)o * ins[l] + col0 + k] : 0.0f;
                    uint16_t a = f2bf_p(v);
                    uint16_t b = f2bf_p(v - bf2f_p(a));
                    size_t off = (size_t)r * 128 + (size_t)(((k >> 3) ^ (r & 7)) << 4) + (size_t)(k & 7) * 2;
                    std::memcpy(hi + off, &a, 2);
                    std::memcpy(lo + off, &b, 2);
                    std::memcpy(h2 + off, &a, 2);
                }
            }
        }
        ++item;
    };
    pair::schedule(geo ? 4 : 8, true, emit);
    return item == nitems ? ICG_OK : ICG_ERUNTIME;
}

int pair_make_tmap(const void* dev_stream, size_t bytes, void* tmap_out /* 128-byte CUtensorMap */) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        ICG_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) {
            set_error("cuTensorMapEncodeTiled not available");
            return ICG_ERUNTIME;
        }
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t dims[2] = {128, (cuuint64_t)(bytes / 128)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, 256};  // one 32 KB stage
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(reinterpret_cast<CUtensorMap*>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                        const_cast<void*>(dev_stream), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
        return ICG_ERUNTIME;
    }
    return ICG_OK;
}

template <bool TEX>
static int launch_pair(pair::Params p, const void* tmapA, const void* tmapB, unsigned max_points, cudaStream_t s) {
    using C = pair::Cfg<TEX>;
    static bool attr = false;
    if (!attr) {
        ICG_CUDA_TRY(cudaFuncSetAttribute(pair::k_mlp_pair<TEX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)C::kTotal));
        attr = true;
    }
    static unsigned long long* trace = nullptr;
    static int tron = -1;
    if (tron < 0) {
        const char* e = getenv("ICG_TC_TRACE");
        tron = e && e[0] == '1';
        if (tron) cudaMallocManaged(&trace, 64 * sizeof(unsigned long long));
    }
    p.trace = tron ? trace : nullptr;
    if (p.trace) cudaMemsetAsync(p.trace, 0, 64 * 8, s);
    unsigned pairs = (max_points + C::NP - 1) / C::NP;
    if (pairs > 74) pairs = 74;
    if (pairs == 0) pairs = 1;
    CUtensorMap ta, tb;
    std::memcpy(&ta, tmapA, sizeof(CUtensorMap));
    std::memcpy(&tb, tmapB ? tmapB : tmapA, sizeof(CUtensorMap));
    pair::k_mlp_pair<TEX><<<2 * pairs, pair::kThreads, C::kTotal, s>>>(ta, tb, p);
    ICG_CUDA_TRY(cudaGetLastError());
    if (p.trace) {
        cudaStreamSynchronize(s);
        const unsigned long long* t = p.trace;
        fprintf(stderr,
                "[pair-trace %s] mma: total %.1f us, wait data %.1f, wait h %.1f, wait f %.1f | epi: total %.1f, wait acc "
                "%.1f, wait hfree %.1f, emit %.1f\n",
                TEX ? "tex" : "geo", t[0] * 1e-3, t[1] * 1e-3, t[2] * 1e-3, t[3] * 1e-3, t[4] * 1e-3, t[5] * 1e-3,
                t[6] * 1e-3, t[7] * 1e-3);
        fprintf(stderr, "    epi cycles: tmem-ld %llu, convert+store %llu, fence+arrive %llu\n", t[8], t[9], t[10]);
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
    return launch_pair<false>(p, tmap, nullptr, max_points, s);
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
    return launch_pair<true>(p, tmap_geo, tmap_tex, max_points, s);
}

}  // namespace icg

// k_mlp_tc.cu — the PIFu field as ONE fused tcgen05/TMEM kernel per point
// batch (ICG_PREC_FP32: bf16x3 split products; ICG_PREC_BF16: bf16 operands;
// fp32 accumulation in TMEM for both).
//
// Work unit: a tile of NP points (64 for geometry, 32 for texture), one CTA
// per SM, persistent over tiles.  Per tile:
//   gather   Phi(P_xy): bilinear over the H x W x C map (each tap of a point is a
//            coalesced 1 KB row), split into bf16 hi/lo, written straight into
//            the MMA B-operand layout in shared memory (K-major, 128B swizzle);
//   MLP      "weights x activations^T": A = 128-row weight tiles streamed from
//            L2 by the bulk-copy (TMA) engine through a 3-stage mbarrier ring,
//            B = the point tile, D = fp32 accumulators in TMEM (lane = output
//            feature, column = point).  Layer 1 (1024 wide) is never
//            materialised: each 128-feature chunk goes TMEM -> epilogue ->
//            shared memory and is immediately consumed as a K-chunk of layer 2
//            while the next chunk is on the tensor cores.  The skip input is
//            re-used from shared memory by every layer (skip concat without
//            copies); its z column (rank 1) and the biases are applied in the
//            epilogue.
//   final    the 1- / 3-wide output layer on CUDA cores (warp transpose-reduce),
//            + bias - sdf_scale*sdf(P), sigmoid, then the grid epilogue of
//            evaluate_nodes (localize.hpp:86-88) with the fused conflict test.
// Warp roles: 0 = weight producer (1 thread), 1 = MMA issuer (1 thread, also
// owns TMEM), 2..5 = gather + epilogue (128 threads, TMEM lanes 0..127).
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <vector>

#include "eval_common.cuh"
#include "tc_ptx.cuh"

namespace icg {

namespace tc {

constexpr uint32_t kTileHalf = 16384;       // one 128 x 64 bf16 tile
constexpr uint32_t kTileBytes = 2 * kTileHalf;  // hi + lo in the packed stream

// ---------------------------------------------------------------------------
// The weight-tile schedule.  The packer (host) and the MMA issuer (device)
// walk the same sequence; `Emit` gets (layer, m_block, k_col0).
// ---------------------------------------------------------------------------
template <class Emit>
__host__ __device__ void body_schedule(int ks, bool with_l4, Emit&& emit) {
    auto L1 = [&](int c) {
        for (int j = 0; j < ks; ++j) emit(0, c, j * 64);
    };
    L1(0);
    L1(1);
    for (int m = 0; m < 4; ++m)
        for (int j = 0; j < ks; ++j) emit(1, m, 1024 + j * 64);
    for (int c = 0; c < 8; ++c) {
        for (int m = 0; m < 4; ++m)
            for (int jj = 0; jj < 2; ++jj) emit(1, m, c * 128 + jj * 64);
        if (c + 2 < 8) L1(c + 2);
    }
    for (int m = 0; m < 2; ++m)
        for (int j = 0; j < ks; ++j) emit(2, m, 512 + j * 64);
    for (int c = 0; c < 4; ++c)
        for (int m = 0; m < 2; ++m)
            for (int jj = 0; jj < 2; ++jj) emit(2, m, c * 128 + jj * 64);
    if (with_l4) {
        for (int j = 0; j < ks; ++j) emit(3, 0, 256 + j * 64);
        for (int c = 0; c < 2; ++c)
            for (int jj = 0; jj < 2; ++jj) emit(3, 0, c * 128 + jj * 64);
    }
}

__host__ __device__ constexpr int body_tiles(int ks, bool with_l4) {
    return 8 * ks + 4 * ks + 8 * 4 * 2 + 2 * ks + 4 * 2 * 2 + (with_l4 ? ks + 4 : 0);
}

// geometry: skip = [Phi] (4 chunks of 64; z handled in the epilogue)
// texture : skip = [Phi, h3] (8 chunks); preceded by the geometry prefix (L1-L3)
constexpr int kGeoTiles = body_tiles(4, true);    // 144
constexpr int kGeoPrefixTiles = body_tiles(4, false);
constexpr int kTexBodyTiles = body_tiles(8, true);

}  // namespace tc

// ===========================================================================
// Host: pack weights into the consumption-ordered bf16 hi/lo tile stream.
// ===========================================================================
static inline uint16_t f2bf(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    uint32_t r = ((u >> 16) & 1u) + 0x7FFFu;  // round to nearest even
    return (uint16_t)((u + r) >> 16);
}
static inline float bf2f(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

size_t tc_stream_bytes(int which) {
    return (size_t)(which == ICG_MLP_GEOMETRY ? tc::kGeoTiles : tc::kTexBodyTiles) * tc::kTileBytes;
}
size_t tc_bias_floats(int which) { return which == ICG_MLP_GEOMETRY ? (1024 + 512 + 256 + 128 + 1) * 2 + 2 : (1024 + 512 + 256 + 128 + 3) * 2 + 2; }
size_t tc_wlast_floats(int which) { return which == ICG_MLP_GEOMETRY ? 1 * (128 + 257) : 3 * (128 + 513); }

// bias block layout per layer l (l < 4): [b_l (out), wz_l (out)] where wz is
// the weight column of the skip's z input; then final-layer biases.
int tc_pack_mlp(int which, const float* const* w, const float* const* b, uint8_t* stream, float* bias,
                float* wlast) {
    const bool geo = which == ICG_MLP_GEOMETRY;
    const int* outs = geo ? kGeoOut : kTexOut;
    const int skip = geo ? kGeoSkip : kTexSkip;
    int ins[5];
    for (int l = 0; l < 5; ++l) ins[l] = (l ? outs[l - 1] : 0) + skip;
    size_t tile = 0;
    auto emit = [&](int l, int m, int col0) {
        uint8_t* hi = stream + tile * tc::kTileBytes;
        uint8_t* lo = hi + tc::kTileHalf;
        for (int r = 0; r < 128; ++r)
            for (int k = 0; k < 64; ++k) {
                float v = w[l][(size_t)(m * 128 + r) * ins[l] + col0 + k];
                uint16_t h = f2bf(v);
                uint16_t q = f2bf(v - bf2f(h));
                size_t off = (size_t)r * 128 + (size_t)(((k >> 3) ^ (r & 7)) << 4) + (size_t)(k & 7) * 2;
                std::memcpy(hi + off, &h, 2);
                std::memcpy(lo + off, &q, 2);
            }
        ++tile;
    };
    tc::body_schedule(geo ? 4 : 8, true, emit);
    size_t off = 0;
    for (int l = 0; l < 4; ++l) {
        for (int o = 0; o < outs[l]; ++o) bias[off + o] = b[l][o];
        for (int o = 0; o < outs[l]; ++o) bias[off + outs[l] + o] = w[l][(size_t)o * ins[l] + ins[l] - 1];
        off += 2 * (size_t)outs[l];
    }
    for (int o = 0; o < outs[4]; ++o) bias[off + o] = b[4][o];
    for (int o = 0; o < outs[4]; ++o)
        for (int k = 0; k < ins[4]; ++k) wlast[(size_t)o * ins[4] + k] = w[4][(size_t)o * ins[4] + k];
    return ICG_OK;
}

// ===========================================================================
// Device kernel
// ===========================================================================
namespace tc {

constexpr int kStages = 4;          // weight ring: 4 x 16 KB (one bf16 128x64 tile each)
constexpr int kEpiWarps = 8;        // gather + epilogue: two warps per TMEM lane quarter
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreadsV2 = 64 + kEpiThreads;

template <int NP>
struct Smem {
    // skip operand: KS chunks of [NP rows x 64 bf16] (K-major, SW128), hi block
    // then lo block (geometry 4 chunks, texture 8).  h operand: two buffers of
    // 2 chunks (hi, lo) so the epilogue of chunk c+1 overlaps the MMAs of c.
    static constexpr uint32_t kChunk = NP * 128;
    static constexpr int kSkipChunks = NP == 64 ? 4 : 8;
    static constexpr uint32_t kSkipHalf = kSkipChunks * kChunk;
    static constexpr uint32_t kHHalf = 2 * kChunk;
    static constexpr uint32_t kHBuf = 2 * kHHalf;
    static constexpr uint32_t kOffSkip = 0;
    static constexpr uint32_t kOffH = kOffSkip + 2 * kSkipHalf;
    static constexpr uint32_t kOffRing = kOffH + 2 * kHBuf;
    static constexpr uint32_t kOffMisc = kOffRing + kStages * kTileHalf;
    static constexpr uint32_t kMisc = 16384;
    static constexpr uint32_t kTotal = kOffMisc + kMisc + 1024;  // + alignment slack
};

struct Misc {
    uint64_t full[kStages], empty[kStages];
    uint64_t f_ready, h_ready[2], h_free[2], l1done[2], d2done, d3done, d4done;
    uint32_t tmem_base;
    float z[64];
    float pos[64][3];
    double posd[64][3];
    float red[4][3][64];      // final layer: per-quarter partial sums over features
    float skipdot[8][3][64];  // final layer: skip-input partial dots
};
static_assert(sizeof(Misc) + 16 <= Smem<64>::kMisc, "misc smem area too small");

struct Params {
    FieldDev f;
    EvalJob job;
    const uint8_t* stream_a;   // geometry stream (or geometry prefix for texture)
    int tiles_a;
    const uint8_t* stream_b;   // texture stream (texture kernel only)
    int tiles_b;
    const float* bias_g;       // geometry bias/wz blocks
    const float* bias_t;       // texture bias/wz blocks
    const float* wlast;        // final layer of the network being evaluated
    float slope;
    int x3;                    // bf16x3 split products
    unsigned long long* trace; // optional per-role wait accounting (CTA 0), see ICG_TC_TRACE
    int exp;                   // debug experiments: 1 = skip MMAs, 2 = skip weight loads
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

// byte offset of element (row, k) inside a K-major SW128 operand chunk
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t k) {
    return row * 128u + ((((k >> 3) ^ row) & 7u) << 4) + (k & 7u) * 2u;
}

// transpose-reduce: lane l returns sum over lanes of v[l] (v has 32 entries)
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

template <int NC>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t* r) {
    if constexpr (NC == 32)
        ptx::tmem_ld32(taddr, r);
    else
        ptx::tmem_ld16(taddr, r);
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); }

template <int NP>
__global__ void __launch_bounds__(kThreadsV2, 1) k_mlp_tc(Params P) {
    using S = Smem<NP>;
    constexpr int NC = NP / 2;  // point columns per epilogue warp
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* skip = smem + S::kOffSkip;
    uint8_t* hbase = smem + S::kOffH;
    uint8_t* ring = smem + S::kOffRing;
    Misc& ms = *reinterpret_cast<Misc*>(smem + S::kOffMisc);
    __shared__ DevScene scene;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool texture = P.tiles_b > 0;
    const EvalJob& job = P.job;
    {
        // empty work list (e.g. a converged conflict iteration): leave before any setup
        const unsigned n0 = job_count(job);
        if (n0 < job.min_count) return;  // small batch: the latency path (k_small.cu) evaluates it
        if (blockIdx.x * NP >= n0) {
            job_account(job);
            return;
        }
    }

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&ms.full[s], 1);
            ptx::mbar_init(&ms.empty[s], 1);
        }
        ptx::mbar_init(&ms.f_ready, kEpiThreads);
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&ms.h_ready[b], kEpiThreads);
            ptx::mbar_init(&ms.h_free[b], 1);
            ptx::mbar_init(&ms.l1done[b], 1);
        }
        ptx::mbar_init(&ms.d2done, 1);
        ptx::mbar_init(&ms.d3done, 1);
        ptx::mbar_init(&ms.d4done, 1);
        ptx::fence_mbar_init();
    }
    if (!texture)
        for (int i = threadIdx.x; i < (int)(sizeof(DevScene) / 8); i += blockDim.x)
            reinterpret_cast<double*>(&scene)[i] = reinterpret_cast<const double*>(P.f.scene)[i];
    if (warp == 1) ptx::tmem_alloc<512>(&ms.tmem_base);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = ms.tmem_base;
    job_account(job);

    const unsigned n = job_count(job);
    const unsigned ntiles = (n + NP - 1) / NP;

    if (warp == 0) {
        // ===================== weight producer (bulk copies, 16 KB stages) =====================
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const int halves = P.x3 ? 2 : 1;
            for (unsigned t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int seg = 0; seg < 2; ++seg) {
                    const uint8_t* src = seg ? P.stream_b : P.stream_a;
                    const int cnt = seg ? P.tiles_b : P.tiles_a;
                    for (int i = 0; i < cnt; ++i)
                        for (int h = 0; h < halves; ++h) {
                            ptx::mbar_wait(&ms.empty[s], ph ^ 1);
                            if (P.exp & 2) {
                                ptx::mbar_arrive(&ms.full[s]);
                            } else {
                                ptx::mbar_arrive_expect_tx(&ms.full[s], kTileHalf);
                                ptx::bulk_g2s(ring + s * kTileHalf, src + (size_t)i * kTileBytes + h * kTileHalf,
                                              kTileHalf, &ms.full[s]);
                            }
                            if (++s == kStages) {
                                s = 0;
                                ph ^= 1;
                            }
                        }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            const uint32_t idesc = ptx::idesc_bf16_f32(128, NP);
            int s = 0;
            uint32_t ph = 0, fph = 0, hr_ph[2] = {0, 0};
            int eh = 0;  // h-event counter
            const uint32_t skip_hi = ptx::smem_u32(skip), skip_lo = skip_hi + S::kSkipHalf;
            const uint32_t h0 = ptx::smem_u32(hbase);
            const uint32_t ring0 = ptx::smem_u32(ring);
            unsigned long long w_full = 0, w_h = 0, w_f = 0, t_begin = gtime();
            const bool tr = P.trace && blockIdx.x == 0;
            auto twait = [&](uint64_t* bar, uint32_t par, unsigned long long& acc) {
                if (tr) {
                    unsigned long long t0 = gtime();
                    ptx::mbar_wait(bar, par);
                    acc += gtime() - t0;
                } else {
                    ptx::mbar_wait(bar, par);
                }
            };
            auto next_stage = [&]() {
                if (++s == kStages) {
                    s = 0;
                    ph ^= 1;
                }
            };
            // TMEM columns: D2[m] = m*NP, BUF[b] = 4NP + b*NP (D3[m] reuses BUF), D4 = 6NP
            auto item = [&](uint32_t dcol, uint32_t b_hi, uint32_t b_lo, bool acc) {
                const uint64_t bd_hi = ptx::sdesc_sw128(b_hi), bd_lo = ptx::sdesc_sw128(b_lo);
                twait(&ms.full[s], ph, w_full);
                ptx::tc_fence_after();
                const uint64_t ad_hi = ptx::sdesc_sw128(ring0 + s * kTileHalf);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    if (P.exp & 1) break;
                    const uint64_t koff = (uint64_t)(kk * 2);  // +32 bytes per K=16 step
                    ptx::mma_bf16(tmem + dcol, ad_hi + koff, bd_hi + koff, idesc, (acc || kk > 0) ? 1u : 0u);
                    if (P.x3) ptx::mma_bf16(tmem + dcol, ad_hi + koff, bd_lo + koff, idesc, 1u);
                }
                ptx::mma_commit(&ms.empty[s]);
                next_stage();
                if (P.x3) {
                    twait(&ms.full[s], ph, w_full);
                    ptx::tc_fence_after();
                    const uint64_t ad_lo = ptx::sdesc_sw128(ring0 + s * kTileHalf);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        if (P.exp & 1) break;
                        const uint64_t koff = (uint64_t)(kk * 2);
                        ptx::mma_bf16(tmem + dcol, ad_lo + koff, bd_hi + koff, idesc, 1u);
                    }
                    ptx::mma_commit(&ms.empty[s]);
                    next_stage();
                }
            };
            auto wait_h = [&]() -> int {
                const int b = eh & 1;
                twait(&ms.h_ready[b], hr_ph[b], w_h);
                hr_ph[b] ^= 1;
                ptx::tc_fence_after();
                return b;
            };
            auto done_h = [&](int b) {
                ptx::mma_commit(&ms.h_free[b]);
                ++eh;
            };
            // one MLP body: layers 1-3 (+4); skip chunks [0, ks)
            auto body = [&](int ks, bool with_l4) {
                auto L1 = [&](int c) {
                    for (int j = 0; j < ks; ++j)
                        item(4 * NP + (c & 1) * NP, skip_hi + j * S::kChunk, skip_lo + j * S::kChunk, j > 0);
                    ptx::mma_commit(&ms.l1done[c & 1]);
                };
                L1(0);
                L1(1);
                for (int m = 0; m < 4; ++m)
                    for (int j = 0; j < ks; ++j)
                        item(m * NP, skip_hi + j * S::kChunk, skip_lo + j * S::kChunk, j > 0);
                for (int c = 0; c < 8; ++c) {
                    const int b = wait_h();
                    const uint32_t hh = h0 + b * S::kHBuf, hl = hh + S::kHHalf;
                    for (int m = 0; m < 4; ++m)
                        for (int jj = 0; jj < 2; ++jj) item(m * NP, hh + jj * S::kChunk, hl + jj * S::kChunk, true);
                    done_h(b);
                    if (c + 2 < 8) L1(c + 2);
                }
                ptx::mma_commit(&ms.d2done);
                for (int m = 0; m < 2; ++m)
                    for (int j = 0; j < ks; ++j)
                        item(4 * NP + m * NP, skip_hi + j * S::kChunk, skip_lo + j * S::kChunk, j > 0);
                for (int c = 0; c < 4; ++c) {
                    const int b = wait_h();
                    const uint32_t hh = h0 + b * S::kHBuf, hl = hh + S::kHHalf;
                    for (int m = 0; m < 2; ++m)
                        for (int jj = 0; jj < 2; ++jj)
                            item(4 * NP + m * NP, hh + jj * S::kChunk, hl + jj * S::kChunk, true);
                    done_h(b);
                }
                ptx::mma_commit(&ms.d3done);
                if (with_l4) {
                    for (int j = 0; j < ks; ++j)
                        item(6 * NP, skip_hi + j * S::kChunk, skip_lo + j * S::kChunk, j > 0);
                    for (int c = 0; c < 2; ++c) {
                        const int b = wait_h();
                        const uint32_t hh = h0 + b * S::kHBuf, hl = hh + S::kHHalf;
                        for (int jj = 0; jj < 2; ++jj) item(6 * NP, hh + jj * S::kChunk, hl + jj * S::kChunk, true);
                        done_h(b);
                    }
                    ptx::mma_commit(&ms.d4done);
                } else {
                    // prefix mode: h3 goes into skip chunks 4..7 (two events, nothing to consume)
                    for (int c = 0; c < 2; ++c) done_h(wait_h());
                }
            };
            for (unsigned t = blockIdx.x; t < ntiles; t += gridDim.x) {
                twait(&ms.f_ready, fph, w_f);
                fph ^= 1;
                ptx::tc_fence_after();
                if (texture) {
                    body(4, false);
                    body(8, true);
                } else {
                    body(4, true);
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
        // ===================== gather + epilogue (8 warps) =====================
        const int et = threadIdx.x - 64;              // 0..255
        const int quarter = warp & 3;                 // TMEM lane quarter of this warp
        const int colh = (warp - 2) >> 2;             // which half of the point columns
        const int col0 = colh * NC;
        const int row = quarter * 32 + lane;          // TMEM lane = output feature within the block
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)col0;
        uint32_t l1ph[2] = {0, 0}, d2ph = 0, d3ph = 0, d4ph = 0, hf_ph[2] = {1, 1};
        int ee = 0;  // h-event counter (matches the MMA issuer's)
        const bool tr = P.trace && blockIdx.x == 0 && threadIdx.x == 64;
        unsigned long long e_acc = 0, e_hfree = 0, e_gather = 0, e_emit = 0, e_final = 0, e_begin = gtime();
        auto ewait = [&](uint64_t* bar, uint32_t par, unsigned long long& acc) {
            if (tr) {
                unsigned long long t0 = gtime();
                ptx::mbar_wait(bar, par);
                acc += gtime() - t0;
            } else {
                ptx::mbar_wait(bar, par);
            }
        };
        const FieldDev& f = P.f;
        const bool odd = lane & 1;
        const uint32_t kk = (uint32_t)(row & 63) & ~1u;
        const uint32_t rchunk = (uint32_t)(row >> 6) * S::kChunk;

        // one 128-feature activation chunk: this thread = feature `row`, points
        // [col0, col0+NC) from TMEM column `col`, into operand region `dst`.
        auto emit_chunk = [&](uint32_t col, const float* bias_blk, int out_dim, int feat0, uint8_t* dst,
                              uint32_t lo_off, bool write_lo) {
            const int o = feat0 + row;
            const float bo = __ldg(&bias_blk[o]);
            const float wz = __ldg(&bias_blk[out_dim + o]);
            uint32_t r[NC];
            tmem_ld<NC>(lane_base + col, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q = 0; q < NC; q += 2) {
                const int p = col0 + q;
                float v0 = __uint_as_float(r[q]) + fmaf(wz, ms.z[p], bo);
                float v1 = __uint_as_float(r[q + 1]) + fmaf(wz, ms.z[p + 1], bo);
                v0 = v0 < 0.0f ? v0 * P.slope : v0;
                v1 = v1 < 0.0f ? v1 * P.slope : v1;
                // even lane writes (p, feats kk,kk+1); odd lane writes (p+1, feats kk,kk+1)
                const float send = odd ? v0 : v1;
                const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                const float a = odd ? recv : v0;
                const float b = odd ? v1 : recv;
                const uint32_t off = rchunk + sw128((uint32_t)(p + (odd ? 1 : 0)), kk);
                const uint32_t hv = pack_bf16(a, b);
                *reinterpret_cast<uint32_t*>(dst + off) = hv;
                if (write_lo) {
                    const float ah = __uint_as_float(hv << 16), bh = __uint_as_float(hv & 0xFFFF0000u);
                    *reinterpret_cast<uint32_t*>(dst + lo_off + off) = pack_bf16(a - ah, b - bh);
                }
            }
        };

        auto h_begin = [&]() -> int {
            const int b = ee & 1;
            ewait(&ms.h_free[b], hf_ph[b], e_hfree);
            hf_ph[b] ^= 1;
            return b;
        };
        auto h_end = [&](int b) {
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&ms.h_ready[b]);
            ++ee;
        };

        // epilogue of one body; returns after D3 (prefix) or before D4
        auto body_epi = [&](const float* bias, bool prefix) {
            const float* b1 = bias;
            const float* b2 = b1 + 2 * 1024;
            const float* b3 = b2 + 2 * 512;
            for (int c = 0; c < 8; ++c) {
                ewait(&ms.l1done[c & 1], l1ph[c & 1], e_acc);
                l1ph[c & 1] ^= 1;
                ptx::tc_fence_after();
                const int b = h_begin();
                uint8_t* hb = hbase + b * S::kHBuf;
                emit_chunk(4 * NP + (c & 1) * NP, b1, 1024, c * 128, hb, S::kHHalf, P.x3);
                h_end(b);
            }
            ewait(&ms.d2done, d2ph, e_acc);
            d2ph ^= 1;
            ptx::tc_fence_after();
            for (int m = 0; m < 4; ++m) {
                const int b = h_begin();
                emit_chunk(m * NP, b2, 512, m * 128, hbase + b * S::kHBuf, S::kHHalf, P.x3);
                h_end(b);
            }
            ewait(&ms.d3done, d3ph, e_acc);
            d3ph ^= 1;
            ptx::tc_fence_after();
            for (int m = 0; m < 2; ++m) {
                const int b = h_begin();
                if (prefix)  // h3 -> skip chunks 4 + 2m, 5 + 2m
                    emit_chunk(4 * NP + m * NP, b3, 256, m * 128, skip + (4 + 2 * m) * S::kChunk, S::kSkipHalf, true);
                else
                    emit_chunk(4 * NP + m * NP, b3, 256, m * 128, hbase + b * S::kHBuf, S::kHHalf, P.x3);
                h_end(b);
            }
        };

        for (unsigned t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const unsigned base = t * NP;
            // ---- positions ----
            if (et < NP) {
                const unsigned idx = base + et;
                double pd[3] = {0.0, 0.0, 0.0};
                if (idx < n) job_point_d(job, idx, pd);
                for (int d = 0; d < 3; ++d) {
                    ms.posd[et][d] = pd[d];
                    ms.pos[et][d] = (float)pd[d];
                }
                ms.z[et] = (float)pd[2];
            }
            epi_bar();
            // ---- gather Phi into the skip operand (hi/lo): 2 channels x NP/2 points per thread ----
            unsigned long long tg0 = tr ? gtime() : 0;
            {
                const int c0 = 2 * (et & 127);
                const int p0 = (et >> 7) * (NP / 2);
                const uint32_t chunk = (uint32_t)(c0 >> 6) * S::kChunk;
                const uint32_t ck = (uint32_t)(c0 & 63);
                const size_t rowW = (size_t)f.W * f.C;
#pragma unroll 4
                for (int p = p0; p < p0 + NP / 2; ++p) {
                    float u = (ms.pos[p][0] + 1.0f) * 0.5f * (float)(f.W - 1);
                    float v = (1.0f - ms.pos[p][1]) * 0.5f * (float)(f.H - 1);
                    u = fminf(fmaxf(u, 0.0f), (float)(f.W - 1));
                    v = fminf(fmaxf(v, 0.0f), (float)(f.H - 1));
                    const int x0 = min((int)floorf(u), f.W - 2), y0 = min((int)floorf(v), f.H - 2);
                    const float ax = u - (float)x0, ay = v - (float)y0;
                    const float* m00 = f.fmap_hwc + ((size_t)y0 * f.W + x0) * (size_t)f.C + c0;
                    const float2 t00 = __ldg(reinterpret_cast<const float2*>(m00));
                    const float2 t10 = __ldg(reinterpret_cast<const float2*>(m00 + f.C));
                    const float2 t01 = __ldg(reinterpret_cast<const float2*>(m00 + rowW));
                    const float2 t11 = __ldg(reinterpret_cast<const float2*>(m00 + rowW + f.C));
                    const float w00 = (1.0f - ax) * (1.0f - ay), w10 = ax * (1.0f - ay), w01 = (1.0f - ax) * ay,
                                w11 = ax * ay;
                    const float a = w00 * t00.x + w10 * t10.x + w01 * t01.x + w11 * t11.x;
                    const float b = w00 * t00.y + w10 * t10.y + w01 * t01.y + w11 * t11.y;
                    const uint32_t off = chunk + sw128((uint32_t)p, ck);
                    const uint32_t hv = pack_bf16(a, b);
                    *reinterpret_cast<uint32_t*>(skip + off) = hv;
                    const float ah = __uint_as_float(hv << 16), bh = __uint_as_float(hv & 0xFFFF0000u);
                    *reinterpret_cast<uint32_t*>(skip + S::kSkipHalf + off) = pack_bf16(a - ah, b - bh);
                }
            }
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(&ms.f_ready);
            if (tr) e_gather += gtime() - tg0;

            if (texture) body_epi(P.bias_g, true);
            const float* bias = texture ? P.bias_t : P.bias_g;
            body_epi(bias, false);

            // ---- layer 4 -> h4 (fp32, registers) -> final layer on CUDA cores ----
            const int nout = texture ? 3 : 1;
            const int K4 = 128;
            const int skipdim = texture ? kTexSkip : kGeoSkip;
            const float* b4 = bias + 2 * (1024 + 512 + 256);
            const float* b5 = b4 + 2 * 128;
            ewait(&ms.d4done, d4ph, e_acc);
            unsigned long long tf0 = tr ? gtime() : 0;
            d4ph ^= 1;
            ptx::tc_fence_after();
            {
                const float bo = __ldg(&b4[row]), wz = __ldg(&b4[128 + row]);
                uint32_t r[NC];
                tmem_ld<NC>(lane_base + 6 * NP, r);
                ptx::tmem_ld_wait();
                float h[NC];
#pragma unroll
                for (int q = 0; q < NC; ++q) {
                    float v = __uint_as_float(r[q]) + fmaf(wz, ms.z[col0 + q], bo);
                    h[q] = v < 0.0f ? v * P.slope : v;
                }
                for (int c = 0; c < nout; ++c) {
                    const float w5 = __ldg(&P.wlast[(size_t)c * (K4 + skipdim) + row]);
                    float v[32];
#pragma unroll
                    for (int q = 0; q < 32; ++q) v[q] = q < NC ? w5 * h[q] : 0.0f;
                    const float sum = warp_transpose_reduce(v);  // lane l: point col0 + l
                    if (lane < NC) ms.red[quarter][c][col0 + lane] = sum;
                }
            }
            ptx::tc_fence_before();
            // skip part of the final layer: sum_j w5s[j] * skip[p][j] (the z term is added below)
            {
                constexpr int split = kEpiThreads / NP;  // threads per point
                const int p = et / split, part = et % split;
                const int nch = (texture ? 512 : 256) / split;
                for (int c = 0; c < nout; ++c) {
                    const float* ws = P.wlast + (size_t)c * (K4 + skipdim) + K4;
                    float acc = 0.0f;
                    for (int j = part * nch; j < (part + 1) * nch; j += 2) {
                        const uint32_t off = (uint32_t)(j >> 6) * S::kChunk + sw128((uint32_t)p, (uint32_t)(j & 63));
                        const uint32_t hv = *reinterpret_cast<const uint32_t*>(skip + off);
                        const uint32_t lv = *reinterpret_cast<const uint32_t*>(skip + S::kSkipHalf + off);
                        const float x0 = __uint_as_float(hv << 16) + __uint_as_float(lv << 16);
                        const float x1 = __uint_as_float(hv & 0xFFFF0000u) + __uint_as_float(lv & 0xFFFF0000u);
                        acc = fmaf(__ldg(&ws[j]), x0, acc);
                        acc = fmaf(__ldg(&ws[j + 1]), x1, acc);
                    }
                    ms.skipdot[part][c][p] = acc;
                }
            }
            epi_bar();
            if (et < NP * nout) {
                constexpr int split = kEpiThreads / NP;
                const int p = et % NP, c = et / NP;
                const unsigned idx = base + p;
                float s = ms.red[0][c][p] + ms.red[1][c][p] + ms.red[2][c][p] + ms.red[3][c][p];
                for (int q = 0; q < split; ++q) s += ms.skipdot[q][c][p];
                const float* ws = P.wlast + (size_t)c * (K4 + skipdim) + K4;
                s += __ldg(&ws[skipdim - 1]) * ms.z[p] + __ldg(&b5[c]);
                if (idx < n) {
                    if (texture) {
                        float v = 1.0f / (1.0f + expf(-s));
                        if (job.out_pixel) {
                            v = fminf(fmaxf(v, 0.0f), 1.0f);  // clamp01, render.hpp:276
                            job.out[(size_t)job.out_pixel[idx] * 3 + c] = v;
                        } else {
                            job.out[(size_t)idx * 3 + c] = v;
                        }
                    } else {
                        const double sdf = scene_sdf(scene, ms.posd[p]);
                        const float logit = s + (float)(-scene.sdf_scale * sdf);
                        const float v = 1.0f / (1.0f + expf(-logit));
                        if (job_is_grid(job))
                            grid_epilogue(job, job_node(job, idx), v);
                        else
                            job.out[idx] = v;
                    }
                }
            }
            epi_bar();
            if (tr) e_final += gtime() - tf0;
        }
        if (tr) {
            P.trace[4] = gtime() - e_begin;
            P.trace[5] = e_acc;
            P.trace[6] = e_hfree;
            P.trace[7] = e_gather;
            P.trace[8] = e_final;
            P.trace[9] = ntiles;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

}  // namespace tc

static unsigned long long* trace_buffer() {
    static unsigned long long* buf = nullptr;
    static int enabled = -1;
    if (enabled < 0) {
        const char* e = getenv("ICG_TC_TRACE");
        enabled = e && e[0] == '1';
        if (enabled) cudaMallocManaged(&buf, 64 * sizeof(unsigned long long));
    }
    return enabled ? buf : nullptr;
}

template <int NP>
static int launch_tc(tc::Params p, unsigned max_points, cudaStream_t s) {
    p.trace = trace_buffer();
    {
        const char* e = getenv("ICG_TC_EXP");
        p.exp = e ? atoi(e) : 0;
    }
    if (p.trace) cudaMemsetAsync(p.trace, 0, 64 * sizeof(unsigned long long), s);
    static bool attr = false;
    const uint32_t smem = tc::Smem<NP>::kTotal;
    if (!attr) {
        ICG_CUDA_TRY(cudaFuncSetAttribute(tc::k_mlp_tc<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    unsigned blocks = (max_points + NP - 1) / NP;
    if (blocks > 148) blocks = 148;
    if (blocks == 0) blocks = 1;
    tc::k_mlp_tc<NP><<<blocks, tc::kThreadsV2, smem, s>>>(p);
    ICG_CUDA_TRY(cudaGetLastError());
    if (p.trace) {
        cudaStreamSynchronize(s);
        const unsigned long long* t = p.trace;
        fprintf(stderr,
                "[tc-trace NP=%d] mma: total %.1f us, wait data %.1f, wait h %.1f, wait f %.1f | epi: total %.1f us, "
                "wait acc %.1f, wait hfree %.1f, gather %.1f, final %.1f | tiles(cta0) %llu\n",
                NP, t[0] * 1e-3, t[1] * 1e-3, t[2] * 1e-3, t[3] * 1e-3, t[4] * 1e-3, t[5] * 1e-3, t[6] * 1e-3,
                t[7] * 1e-3, t[8] * 1e-3, t[9]);
    }
    return ICG_OK;
}

int launch_pifu_tc_eval(const FieldDev& f, const TcMlp& geo, const EvalJob& job, unsigned int max_points, bool x3,
                        cudaStream_t s) {
    tc::Params p{};
    p.f = f;
    p.job = job;
    p.stream_a = geo.stream;
    p.tiles_a = tc::kGeoTiles;
    p.stream_b = nullptr;
    p.tiles_b = 0;
    p.bias_g = geo.bias;
    p.bias_t = nullptr;
    p.wlast = geo.w_last;
    p.slope = 0.02f;
    p.x3 = x3 ? 1 : 0;
    return launch_tc<64>(p, max_points, s);
}

int launch_pifu_tc_texture(const FieldDev& f, const TcMlp& geo, const TcMlp& tex, const EvalJob& job,
                           unsigned int max_points, bool x3, cudaStream_t s) {
    tc::Params p{};
    p.f = f;
    p.job = job;
    p.stream_a = geo.stream;  // the geometry prefix is the first kGeoPrefixTiles tiles of the geometry stream
    p.tiles_a = tc::kGeoPrefixTiles;
    p.stream_b = tex.stream;
    p.tiles_b = tc::kTexBodyTiles;
    p.bias_g = geo.bias;
    p.bias_t = tex.bias;
    p.wlast = tex.w_last;
    p.slope = 0.02f;
    p.x3 = x3 ? 1 : 0;
    return launch_tc<32>(p, max_points, s);
}

}  // namespace icg

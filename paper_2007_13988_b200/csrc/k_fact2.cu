// k_fact2.cu — column-factored geometry field, bulk batches, with the operands swapped:
// A = the point tile's activations, B = the weight tiles.
//
// Same arithmetic as k_mlp_pair<FACT> (localize.hpp:76-90 evaluation of
// a node list): layer 1 = act(S1[col] + w1z z + b1) from the column record, layers 2-4 =
// act(W_h . h + S_l[col] + w_lz z + b_l) with W_h on the tensor cores (bf16x3), output =
// sigmoid(w5 . h4 + S5[col] + b5 + w5z z - sdf_scale sdf).  What changes is the MMA shape:
//
//   tcgen05.mma.cta_group::2, M = 256 POINTS (128 per CTA), N = 256 output features,
//   A = activations, K-major, each CTA's own 128 points in its own shared memory,
//   B = weight tile, K-major, 128 of the 256 feature rows per CTA (the FACT stream as is),
//   D = TMEM, lane = point, column = feature.
//
// Consequences (the reasons for the swap):
//   * an epilogue thread owns one point (its TMEM lane) and reads that point's features, so the
//     next layer's operand is written by the CTA that owns the point: no DSMEM exchange, no
//     register transposes, and the final 128 -> 1 layer is an in-thread dot product;
//   * N = 256 instead of 128: per MMA the shared-memory port reads 4 KB of A + 4 KB of B per CTA
//     for 2x the MACs (scripts/mma_bench.cu: pair M256 N128 87 clk, N256 152 clk per MMA).
//
// TMEM (512 columns x 128 lanes per CTA): layer 2's D2 fills it (512 features); D3 reuses
// columns 0-255 once h2 chunks 0-3 are read, D4 (N = 256, upper half zero weights) columns
// 256-511.  The next tile's layer 2 starts when the final layer has read D4.
//
// Activation chunks (64 K x 128 points, bf16 hi + lo = 32 KB) stream through a ring of 4 slots:
// 16 h1 chunks (from the records), 8 h2 chunks (from D2), 4 h3 chunks (from D3) per tile.
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "eval_common.cuh"
#include "tc_ptx.cuh"

namespace icg {

namespace fact2 {

constexpr uint32_t kHalf = 16384;                   // 128 x 64 bf16 tile
constexpr uint32_t kStage = 16384;                  // a weight stage: 128 rows x 64 K (hi or lo of an item)
constexpr int kStagesMax = 5;
// bf16x3 (X3): chunks of 128 points x 64 K as hi then lo (32 KB), a 4-slot ring (128 KB);
// bf16: hi only (16 KB), 4 slots (64 KB: the tensor cores drain a bf16 chunk faster than the
// epilogue fills one, so a deeper ring would idle) -- the freed shared memory goes to L1, which
// holds the record rows and biases the epilogue streams (its loads are latency-bound)
// kG: chunks published per proxy fence (each fence stalls its warp until the stores land; the
// bf16 tensor work per chunk is short, so bf16 publishes 4 at a time into a deeper ring)
// kWS: weight-ring stages (5 x 16 KB).  The epilogue's bias and z-weight rows sit in shared memory
// (broadcast loads instead of global ones): bf16 all of layers 1-4 (15 KB, the activation ring
// one slot shorter), bf16x3 those of layers 2-4 (7 KB: the drains; layer 1 is paced by the MMA)
template <bool X3>
struct Prec {
    static constexpr int kWS = 5;
    static constexpr bool kBiasL1 = !X3;  // layer-1 rows in shared memory too
    static constexpr uint32_t kAChunk = X3 ? 32768u : 16384u;
    static constexpr int kA = X3 ? 4 : 7;
    static constexpr uint32_t kARing = kA * kAChunk;
    // layer 3 reuses D2 columns 0-255: it starts once h2 chunks 0-3 are all in the ring
    static_assert(kA >= 4 && kA <= 8, "activation ring: 4..8 slots");
    static constexpr int kStagesPerItem = X3 ? 2 : 1;
    static constexpr int kG = X3 ? 2 : 4;
};
constexpr int kAMax = 8;
#ifndef FACT2_CQ
#define FACT2_CQ 4
#endif
constexpr int kCQ = FACT2_CQ;                       // column groups per TMEM lane quarter
constexpr int kFW = 64 / kCQ;                       // features per thread of a 64-feature chunk
constexpr int kEpiWarps = 4 * kCQ;                  // 4 TMEM lane quarters x kCQ column groups
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kEpiThreads;
constexpr int NPC = 128;                            // points per CTA
constexpr int NP = 256;                             // points per pair tile
constexpr int kSRow = 1936;
constexpr int kSFinal = 1920;
constexpr int kItems = 44;                          // FACT stream: L2 (kc, m) 32, L3 8, L4 4
constexpr uint32_t kOffRing = 0;
constexpr uint32_t kMisc = 11264;
constexpr int kBiasFloats = 2 * (1024 + 512 + 256 + 128);  // [b, w_z] of layers 1-4
constexpr int kBiasL1Floats = 2 * 1024;
template <bool X3>
struct Layout {
    static constexpr int kSBias = Prec<X3>::kBiasL1 ? kBiasFloats : kBiasFloats - kBiasL1Floats;
    static constexpr uint32_t kOffA = kOffRing + Prec<X3>::kWS * kStage;
    static constexpr uint32_t kOffBias = kOffA + Prec<X3>::kARing;
    static constexpr uint32_t kOffMisc = kOffBias + kSBias * 4;
    static constexpr uint32_t kTotal = kOffMisc + kMisc + 1024;
    static_assert(kTotal <= 232448, "shared memory");
};

struct Misc {
    uint64_t full[kStagesMax], empty[kStagesMax];
    uint64_t a_ready[kAMax], a_free[kAMax];
    uint64_t d2a, d2done, d3done, d4done, tm_free;  // d2a: D2 columns 0-255 final
    uint32_t tmem_base;
    int ncaps;
    float caps[16][8];
    float dmin[2][kCQ][NPC];  // capsule distance, split over the column groups (tile parity)
    float ppos[2][NPC][3];  // the tile's point positions (tile parity)
    int pslot[2][NPC];
    float red[kCQ][NPC];
};
static_assert(sizeof(Misc) <= kMisc, "misc");

struct Params {
    FieldDev f;
    EvalJob job;
    const float* bias;   // [b, wz] per layer (tc layout), then b5
    const float* wlast;  // [128 + 257]: w5 hidden part, Phi part, z
    const float* s_in;   // column records
    const int* cmap;     // column -> record
    float slope;
    unsigned long long* trace;  // optional wait accounting of CTA 0 (ICG_TC_TRACE=1)
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

// FACT stream item consumed at MMA position p.  The stream holds layer 2 as (kc, m) pairs, kc =
// h1 chunk, m = feature half; the issuer takes the last R chunks' m = 0 items first (R = the
// activation ring depth: those chunks are resident together), so D2 columns 0-255 are final R
// items before the end of layer 2 and h2 chunks 0-3 drain while the m = 1 items run
template <int R>  // R = chunks reordered (the activation ring depth, <= 16)
__device__ __forceinline__ int mma_item(int p) {
    if (p >= 32 - 2 * R && p < 32) {
        const int q = p - (32 - 2 * R);
        return 2 * (16 - R + q % R) + q / R;
    }
    return p;
}

template <bool X3>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_fact2(const __grid_constant__ CUtensorMap tmapW, Params P) {
    constexpr uint32_t kAChunk = Prec<X3>::kAChunk;
    constexpr int kA = Prec<X3>::kA;
    constexpr int kStages = Prec<X3>::kWS;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1 KB-aligned base kept as smem_raw + offset (shared-space loads for the bias rows)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* ring = smem + kOffRing;
    uint8_t* abuf = smem + Layout<X3>::kOffA;
    float* sbias = reinterpret_cast<float*>(smem + Layout<X3>::kOffBias);
    {
        const float* src = P.bias + (Prec<X3>::kBiasL1 ? 0 : kBiasL1Floats);
        for (int i = threadIdx.x; i < Layout<X3>::kSBias; i += kThreads) sbias[i] = __ldg(&src[i]);
    }
    Misc& ms = *reinterpret_cast<Misc*>(smem + Layout<X3>::kOffMisc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_rank();
    const bool leader = rank == 0;
    const EvalJob& job = P.job;
    const unsigned pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const unsigned n = job_count(job);
    if (n < job.min_count || (job.max_count && n > job.max_count)) return;
    if (pair_id * NP >= n) {
        job_account(job);
        return;
    }
    const unsigned ntiles = (n + NP - 1) / NP;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&ms.full[s], 1);
            ptx::mbar_init(&ms.empty[s], 1);
        }
        for (int a = 0; a < kA; ++a) {
            ptx::mbar_init(&ms.a_ready[a], 2 * kEpiWarps);  // every epilogue warp of both CTAs
            ptx::mbar_init(&ms.a_free[a], 1);
        }
        ptx::mbar_init(&ms.d2a, 1);
        ptx::mbar_init(&ms.d2done, 1);
        ptx::mbar_init(&ms.d3done, 1);
        ptx::mbar_init(&ms.d4done, 1);
        ptx::mbar_init(&ms.tm_free, 2 * kEpiWarps);
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmapW);
    if (threadIdx.x >= 64 && threadIdx.x < 64 + 32) {  // capsule figure of the sdf bias
        const int i = threadIdx.x - 64;
        const int np = __ldg(&P.f.fscene->n_prims);
        if (i < np && i < 16) {
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
            bool all = np <= 16;
            for (int k = 0; k < np && all; ++k)
                all = __ldg(&P.f.fscene->prims[k].kind) == ICG_PRIM_CAPSULE && !__ldg(&P.f.fscene->prims[k].rotated);
            ms.ncaps = all ? np : -1;
        }
    }
    if (warp == 1) ptx::tmem_alloc2<512>(&ms.tmem_base);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = ms.tmem_base;
    job_account(job);

    const uint32_t full0 = ptx::mapa(ptx::smem_u32(&ms.full[0]), 0);
    const uint32_t a_ready0 = ptx::mapa(ptx::smem_u32(&ms.a_ready[0]), 0);
    const uint32_t tm_free0 = ptx::mapa(ptx::smem_u32(&ms.tm_free), 0);
    const uint16_t both = 0x3;

    if (warp == 0) {
        // ===================== weight producer (both CTAs) =====================
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const uint32_t ring0 = ptx::smem_u32(ring);
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                // stream [rank][item][hi, lo] (X3) or [rank][item] (bf16), 128-row stages
                for (int i = 0; i < Prec<X3>::kStagesPerItem * kItems; ++i) {
                    ptx::mbar_wait(&ms.empty[s], ph ^ 1);
                    if (leader) ptx::mbar_arrive_expect_tx(&ms.full[s], 2 * kStage);
                    constexpr int kSPI = Prec<X3>::kStagesPerItem;
                    const int row0 = (((int)rank * kItems + mma_item<Prec<X3>::kA>(i / kSPI)) * kSPI + i % kSPI) * 128;
                    ptx::tma_load_2d_2sm(ring0 + s * kStage, &tmapW, full0 + s * 8, 0, row0);
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader only) =====================
        if (leader && lane == 0) {
            const uint32_t idesc = ptx::idesc_bf16_f32(256, 256);
            const uint32_t ring0 = ptx::smem_u32(ring), a0 = ptx::smem_u32(abuf);
            int s = 0;
            uint32_t ph = 0;
            uint32_t ac = 0;  // activation chunks consumed
            uint32_t tfph = 0;
            const bool tr = P.trace && blockIdx.x == 0;
            unsigned long long w_chunk = 0, w_full = 0, w_tm = 0, t_begin = gtime();
            unsigned long long w_ph[4] = {0, 0, 0, 0};  // chunk waits by phase: h1 first / h1 rest / h2 / h3
            unsigned long long w_wph[4] = {0, 0, 0, 0};  // weight waits by the same phases
            int wph = 0;
            auto wait_chunk = [&](uint32_t c) {
                const unsigned long long t0 = tr ? gtime() : 0;
                ptx::mbar_wait(&ms.a_ready[c % kA], (c / kA) & 1u);
                if (tr) {
                    w_chunk += gtime() - t0;
                    w_ph[wph] += gtime() - t0;
                }
                ptx::tc_fence_after();
            };
            // one weight item (4 K steps) against activation chunk c into D columns dcol
            auto next_stage = [&]() {
                ptx::mma_commit_pair(&ms.empty[s], both);
                if (++s == kStages) {
                    s = 0;
                    ph ^= 1;
                }
            };
            auto wait_stage = [&]() {
                const unsigned long long t0 = tr ? gtime() : 0;
                ptx::mbar_wait(&ms.full[s], ph);
                if (tr) {
                    w_full += gtime() - t0;
                    w_wph[wph] += gtime() - t0;
                }
                ptx::tc_fence_after();
            };
            // one weight item (4 K steps) against activation chunk c into D columns dcol: the weights'
            // hi stage (x act hi, x act lo), then their lo stage (x act hi)
            auto item = [&](uint32_t c, uint32_t dcol, bool first) {
                const uint32_t ab = a0 + (c % kA) * kAChunk;
                const uint64_t ah = ptx::sdesc_sw128(ab), al = ptx::sdesc_sw128(ab + kHalf);
                wait_stage();
                const uint64_t bh = ptx::sdesc_sw128(ring0 + s * kStage);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t ko = (uint64_t)(kk * 2);
                    ptx::mma_bf16_pair(tmem + dcol, ah + ko, bh + ko, idesc, (first && kk == 0) ? 0u : 1u);
                    if constexpr (X3) ptx::mma_bf16_pair(tmem + dcol, al + ko, bh + ko, idesc, 1u);
                }
                next_stage();
                if constexpr (!X3) return;
                wait_stage();
                const uint64_t bl = ptx::sdesc_sw128(ring0 + s * kStage);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t ko = (uint64_t)(kk * 2);
                    ptx::mma_bf16_pair(tmem + dcol, ah + ko, bl + ko, idesc, 1u);
                }
                next_stage();
            };
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                // layer 2: 16 h1 chunks x 2 feature halves into D2 (columns 0-511).  Columns 0-255
                // (the previous tile's D3) are free once its h3 chunks were emitted, so the first
                // item goes ahead; columns 256-511 (its D4) wait for the output layer to read them.
                constexpr int kR = kA;  // chunks whose feature halves are issued apart (mma_item)
                for (int kc = 0; kc < 16 - kR; ++kc) {
                    wph = kc == 0 ? 0 : 1;
                    wait_chunk(ac);
                    item(ac, 0, kc == 0);
                    if (kc == 0 && t != pair_id) {
                        const unsigned long long t0 = tr ? gtime() : 0;
                        ptx::mbar_wait(&ms.tm_free, tfph);
                        if (tr) w_tm += gtime() - t0;
                        tfph ^= 1;
                        ptx::tc_fence_after();
                    }
                    item(ac, 256, kc == 0);
                    ptx::mma_commit_pair(&ms.a_free[ac % kA], both);
                    ++ac;
                }
                // the last kR chunks (resident together): their m = 0 items, then their m = 1 items
                // (mma_item), each chunk's slot freed after its second item
                for (int q = 0; q < kR; ++q) {
                    wait_chunk(ac + q);
                    item(ac + q, 0, false);
                }
                ptx::mma_commit_pair(&ms.d2a, both);  // D2 columns 0-255 final: h2 chunks 0-3 may be drained
                for (int q = 0; q < kR; ++q) {
                    item(ac + q, 256, false);
                    ptx::mma_commit_pair(&ms.a_free[(ac + q) % kA], both);
                }
                ac += kR;
                ptx::mma_commit_pair(&ms.d2done, both);
                // layer 3 into D3 = columns 0-255: its first MMA needs h2 chunks 0-3 (D2 columns
                // 0-255) read, i.e. all four of them emitted
                wph = 2;
                for (uint32_t c = ac; c < ac + 4; ++c) wait_chunk(c);
                for (int kc = 0; kc < 8; ++kc) {
                    if (kc >= 4) wait_chunk(ac);
                    item(ac, 0, kc == 0);
                    ptx::mma_commit_pair(&ms.a_free[ac % kA], both);
                    ++ac;
                }
                ptx::mma_commit_pair(&ms.d3done, both);
                // layer 4 into D4 = columns 256-511 (D2's upper half was read as h2 chunks 4-7)
                wph = 3;
                for (int kc = 0; kc < 4; ++kc) {
                    wait_chunk(ac);
                    item(ac, 256, kc == 0);
                    ptx::mma_commit_pair(&ms.a_free[ac % kA], both);
                    ++ac;
                }
                ptx::mma_commit_pair(&ms.d4done, both);
            }
            if (tr) {
                P.trace[0] = gtime() - t_begin;
                P.trace[1] = w_chunk;
                P.trace[2] = w_full;
                P.trace[3] = w_tm;
                for (int q = 0; q < 4; ++q) P.trace[10 + q] = w_ph[q];
                for (int q = 0; q < 4; ++q) P.trace[20 + q] = w_wph[q];
            }
        }
    } else {
        // ===================== epilogue: thread = (point row, column group) =====================
        const int et = threadIdx.x - 64;
        const int quarter = warp & 3;
        const int cq = (warp - 2) >> 2;  // column group
        const int row = quarter * 32 + lane;  // this CTA's point = TMEM lane
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t arow = ptx::smem_u32(abuf) + (uint32_t)row * 128u;
        const uint32_t sw = (uint32_t)row & 7u;
        auto epi_bar = [] { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); };
        const float* b1 = Prec<X3>::kBiasL1 ? sbias : P.bias;  // [b, w_z] per layer (shared memory, see Prec)
        const float* b2 = Prec<X3>::kBiasL1 ? sbias + kBiasL1Floats : sbias;
        const float* b3 = b2 + 2 * 512;
        const float* b4 = b3 + 2 * 256;
        const float* b5 = P.bias + kBiasFloats;
        const float w5z = __ldg(&P.wlast[128 + kGeoSkip - 1]);
        uint32_t ac = 0, d2aph = 0, d2ph = 0, d3ph = 0, d4ph = 0;
        const bool etr = P.trace && blockIdx.x == 0 && et == 0;
        unsigned long long e_free = 0, e_d = 0, e_prep = 0, e_h1 = 0, e_fin = 0, e_dr = 0, e_begin = gtime();
        // kFW activations of this thread (features cq kFW .. of the chunk) -> chunk slot, hi and lo
        auto store_chunk = [&](const float* v, uint32_t a) {
            const uint32_t base = arow + (a % kA) * kAChunk;
#pragma unroll
            for (int j = 0; j < kFW / 8; ++j) {
                uint4 hv, lv;
                uint32_t* hp = reinterpret_cast<uint32_t*>(&hv);
                uint32_t* lp = reinterpret_cast<uint32_t*>(&lv);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float a = v[8 * j + 2 * i], b = v[8 * j + 2 * i + 1];
                    hp[i] = pack_bf16(a, b);
                    if constexpr (X3)
                        lp[i] = pack_bf16(a - __uint_as_float(hp[i] << 16), b - __uint_as_float(hp[i] & 0xFFFF0000u));
                }
                const uint32_t off = ((((uint32_t)(cq * (kFW / 8) + j)) ^ sw) << 4);
                ptx::st_shared_v4(base + off, hv);
                if constexpr (X3) ptx::st_shared_v4(base + kHalf + off, lv);
            }
        };
        auto begin_chunk = [&](uint32_t a) {
            const unsigned long long t0 = etr ? gtime() : 0;
            ptx::mbar_wait(&ms.a_free[a % kA], ((a / kA) & 1u) ^ 1u);
            if (etr) e_free += gtime() - t0;
        };
        // publish chunks ac .. ac+cnt-1: ONE proxy fence for all of this thread's stores (the fence
        // waits for them to land, so it is paid per batch, not per chunk)
        auto publish = [&](uint32_t first, int cnt) {
            ptx::fence_proxy_async_smem();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0)
                for (int i = 0; i < cnt; ++i) ptx::mbar_arrive_remote(a_ready0 + 8u * ((first + i) % kA));
        };
        auto end_chunks = [&](int cnt) {
            publish(ac, cnt);
            ac += cnt;
        };
        auto wait_d = [&](uint64_t* bar, uint32_t& par) {
            const unsigned long long t0 = etr ? gtime() : 0;
            ptx::mbar_wait(bar, par);
            if (etr) e_d += gtime() - t0;
            par ^= 1;
            ptx::tc_fence_after();
        };
        // kFW consecutive floats at p (16-byte aligned) into v as float4 loads
        auto loads = [](const float* p, float* v) {  // shared memory (bias rows)
#pragma unroll
            for (int q = 0; q < kFW / 4; ++q) {
                const float4 x = reinterpret_cast<const float4*>(p)[q];
                v[4 * q + 0] = x.x;
                v[4 * q + 1] = x.y;
                v[4 * q + 2] = x.z;
                v[4 * q + 3] = x.w;
            }
        };
        auto loadw = [](const float* p, float* v) {
#pragma unroll
            for (int q = 0; q < kFW / 4; ++q) {
                const float4 x = __ldg(reinterpret_cast<const float4*>(p) + q);
                v[4 * q + 0] = x.x;
                v[4 * q + 1] = x.y;
                v[4 * q + 2] = x.z;
                v[4 * q + 3] = x.w;
            }
        };
        // per-thread state of a tile's point (both column halves compute it; the capsule distance
        // is split between them and combined by the final layer)
        struct Pt {
            const float* rec;
            float z;
            unsigned idx;
            bool valid;
        };
        // the node index and record slot of this thread's point of tile tg, loaded ahead of prep()
        struct Pre {
            uint32_t node;
            int slot;
        };
        auto preload = [&](unsigned tg) {
            Pre r{0u, 0};
            const unsigned idx = tg * NP + rank * NPC + (unsigned)row;
            if (cq == 0 && idx < n) {
                r.node = job_node(job, idx);
                const uint32_t n1 = (uint32_t)job.cells + 1u, col = r.node % (n1 * n1);
                r.slot = P.cmap ? __ldg(&P.cmap[col]) : (int)col;
            }
            return r;
        };
        auto prep = [&](unsigned tg, int pb, const Pre& pr) {
            Pt q;
            q.idx = tg * NP + rank * NPC + (unsigned)row;
            q.valid = q.idx < n;
            if (cq == 0) {  // position (node -> NDC: dyadic, so fp32 equals the reference's fp64) and slot
                float pf[3] = {0.0f, 0.0f, 0.0f};
                if (q.valid) node_pos_f(pr.node, job.cells, pf);
                ms.ppos[pb][row][0] = pf[0];
                ms.ppos[pb][row][1] = pf[1];
                ms.ppos[pb][row][2] = pf[2];
                ms.pslot[pb][row] = pr.slot;
            }
            epi_bar();
            const float p3[3] = {ms.ppos[pb][row][0], ms.ppos[pb][row][1], ms.ppos[pb][row][2]};
            const int sl = ms.pslot[pb][row];
            // the tile's column records into L2 (one bulk prefetch per distinct column; the list is
            // sorted by column): the records of a large level do not stay in L2 after the column
            // pass, and the epilogue's loads would wait on DRAM one chunk at a time
            if (cq == 0 && q.valid && (row == 0 || ms.pslot[pb][row - 1] != sl))
                ptx::prefetch_l2_bulk(P.s_in + (size_t)sl * kSRow, kSRow * 4);
            float d = 3.0e38f;
            const int nc = ms.ncaps;
            if (nc >= 0) {
                for (int i = cq; i < nc; i += kCQ) {
                    const float* c = ms.caps[i];
                    const float pa0 = p3[0] - c[0], pa1 = p3[1] - c[1], pa2 = p3[2] - c[2];
                    float hh = 0.0f;
                    if (c[6] > 0.0f) hh = fminf(fmaxf((pa0 * c[3] + pa1 * c[4] + pa2 * c[5]) / c[6], 0.0f), 1.0f);
                    const float v0 = pa0 - hh * c[3], v1 = pa1 - hh * c[4], v2 = pa2 - hh * c[5];
                    d = fminf(d, sqrtf(v0 * v0 + v1 * v1 + v2 * v2) - c[7]);
                }
                if (nc == 0) d = 0.0f;
            } else if (cq == 0) {
                d = scene_sdf_f(P.f.fscene, p3);
            }
            ms.dmin[pb][cq][row] = d;
            q.z = p3[2];
            q.rec = P.s_in + (size_t)sl * kSRow;
            return q;
        };
        // layer 1 (no MMA): chunks [c0, c1) of act(S1 + w1z z + b1)
        // layer 1 in pairs of chunks [c0, c1) (c1 - c0 even)
        constexpr int kG = Prec<X3>::kG;
        // layer-1 chunk c of point q (act(S1 + w1z z + b1)) into ring slot a
        auto h1_chunk = [&](const Pt& q, int c, uint32_t a) {
            const int f0 = c * 64 + cq * kFW;
            float v[kFW], bb[kFW], wz[kFW];
            loadw(q.rec + f0, v);
            loads(b1 + f0, bb);
            loads(b1 + 1024 + f0, wz);
#pragma unroll
            for (int i = 0; i < kFW; ++i) {
                const float x = v[i] + fmaf(wz[i], q.z, bb[i]);
                v[i] = fmaxf(x, x * P.slope);  // leaky-ReLU (0 < slope < 1)
            }
            begin_chunk(a);
            store_chunk(v, a);
        };
        // layer 1, chunks [c0, c1) in ring order, published kG at a time
        auto emit_h1 = [&](const Pt& q, int c0, int c1) {  // (c1 - c0 even)
            int pend = 0;
#pragma unroll 1
            for (int c = c0; c < c1; c += 2) {
                // two chunks per step, unrolled: both chunks' record loads in flight together
#pragma unroll
                for (int u = 0; u < 2; ++u) h1_chunk(q, c + u, ac + pend + u);
                pend += 2;
                if (pend == kG) {
                    end_chunks(pend);
                    pend = 0;
                }
            }
            if (pend) end_chunks(pend);
        };
        // bf16: the next tile's first layer-1 chunks, written `off` ring slots ahead of ac while the
        // epilogue would otherwise wait for layer 3 (their slots' previous chunks, h2 5-6, are layer-3
        // operands: freed without the epilogue); published out of ring order, ac not advanced
        auto emit_h1_ahead = [&](const Pt& q, int c0, int c1, uint32_t off) {
#pragma unroll 1
            for (int c = c0; c < c1; ++c) h1_chunk(q, c, ac + off + (uint32_t)(c - c0));
            publish(ac + off, c1 - c0);
        };
        // hidden layers 2, 3: drain D (columns col0 + feature) into the next layer's chunks
        // two chunks per step: both TMEM loads and both record loads in flight before either is used
        // (the drain is latency-bound: one chunk at a time left the tensor pipe waiting ~1 us per chunk)
        // g: chunks published per proxy fence (kG; 2 for h3, whose chunks layer 4 takes one by one)
        auto drain = [&](const Pt& q, int cbeg, int cend, uint32_t col0, const float* bl, int od, int soff, int g) {
            static_assert(kFW == 16, "drain: 16 features per thread and chunk");
            int pend = 0;  // chunks stored since the last publish (chunk index = ac + pend)
            auto one = [&](const uint32_t* r, float* v, int f) {
                float bb[kFW], wz[kFW];
                loads(bl + f, bb);
                loads(bl + od + f, wz);
#pragma unroll
                for (int i = 0; i < kFW; ++i) {
                    const float x = (__uint_as_float(r[i]) + v[i]) + fmaf(wz[i], q.z, bb[i]);
                    v[i] = fmaxf(x, x * P.slope);
                }
                begin_chunk(ac + pend);
                store_chunk(v, ac + pend);
                if (++pend == g) {
                    end_chunks(pend);
                    pend = 0;
                }
            };
#pragma unroll 1
            for (int c = cbeg; c < cend; c += 2) {
                const int f0 = c * 64 + cq * kFW, f1 = f0 + 64;
                uint32_t r0[kFW], r1[kFW];
                ptx::tmem_ld16(lane_base + col0 + (uint32_t)f0, r0);
                ptx::tmem_ld16(lane_base + col0 + (uint32_t)f1, r1);
                float v0[kFW], v1[kFW];
                loadw(q.rec + soff + f0, v0);
                loadw(q.rec + soff + f1, v1);
                ptx::tmem_ld_wait();
                one(r0, v0, f0);
                one(r1, v1, f1);
            }
            if (pend) end_chunks(pend);
        };
        // layer 4 + output: this thread's 64 of the 128 layer-4 features, dot with w5
        auto final_layer = [&](const Pt& q, int pb) {
            float part = 0.0f;
            constexpr int kFin = 128 / kCQ;  // layer-4 features of this thread
#pragma unroll 1
            for (int c = 0; c < kFin / kFW; ++c) {
                const int f0 = cq * kFin + c * kFW;
                uint32_t r[kFW];
                if constexpr (kFW == 32)
                    ptx::tmem_ld32(lane_base + 256u + (uint32_t)f0, r);
                else
                    ptx::tmem_ld16(lane_base + 256u + (uint32_t)f0, r);
                float v[kFW], bb[kFW], wz[kFW];
                loadw(q.rec + 1792 + f0, v);
                loads(b4 + f0, bb);
                loads(b4 + 128 + f0, wz);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < kFW; ++i) {
                    const float x = (__uint_as_float(r[i]) + v[i]) + fmaf(wz[i], q.z, bb[i]);
                    const float h = fmaxf(x, x * P.slope);
                    part = fmaf(__ldg(&P.wlast[f0 + i]), h, part);
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(tm_free0);  // D3 / D4 are free for the next tile
            ms.red[cq][row] = part;
            epi_bar();
            if (cq == 0 && q.valid) {
                float d = ms.dmin[pb][0][row], sum = part;
#pragma unroll
                for (int g = 1; g < kCQ; ++g) {
                    d = fminf(d, ms.dmin[pb][g][row]);
                    sum += ms.red[g][row];
                }
                const float cterm = __ldg(&b5[0]) + w5z * q.z - __ldg(&P.f.fscene->sdf_scale) * d;
                const float s = sum + __ldg(q.rec + kSFinal) + cterm;
                const float v = 1.0f / (1.0f + expf(-s));
                if (job_is_grid(job))
                    grid_epilogue(job, job_node(job, q.idx), v);
                else
                    job.out[q.idx] = v;
            }
            epi_bar();
        };
        // Per tile t: h1(t) 4-15, prep(t+1), h2(t), h3(t), h1(t+1) 0-3, final(t): the next tile's first
        // layer-1 chunks are ready when its layer 2 may start (after final(t) has read D4).
        int pb = 0;
        unsigned long long tq = etr ? gtime() : 0;
        Pt cur = prep(pair_id, 0, preload(pair_id));
        if (etr) e_prep += gtime() - tq;
        emit_h1(cur, 0, 4);
        for (unsigned t = pair_id; t < ntiles; t += npairs) {
            const bool has_next = t + npairs < ntiles;
            const Pre pre_next = has_next ? preload(t + npairs) : Pre{0u, 0};  // in flight during h1
            tq = etr ? gtime() : 0;
            emit_h1(cur, 4, 16);
            if (etr) e_h1 += gtime() - tq;
            Pt nxt = cur;
            tq = etr ? gtime() : 0;
            if (has_next) nxt = prep(t + npairs, pb ^ 1, pre_next);
            if (etr) e_prep += gtime() - tq;
            wait_d(&ms.d2a, d2aph);
            tq = etr ? gtime() : 0;
            drain(cur, 0, 4, 0, b2, 512, 1024, kG);
            if (etr) e_dr += gtime() - tq;
            wait_d(&ms.d2done, d2ph);
            drain(cur, 4, 8, 0, b2, 512, 1024, kG);
            // bf16 (7-slot ring): next tile's h1 chunks 0-1 go to the slots after the 4 h3 chunks
            constexpr int kAhead = X3 ? 0 : 2;
            static_assert(X3 || kA >= 4 + kAhead + 1, "ring: h3 chunks + the early h1 chunks + one");
            if (kAhead && has_next) emit_h1_ahead(nxt, 0, kAhead, 4);
            wait_d(&ms.d3done, d3ph);
            drain(cur, 0, 4, 0, b3, 256, 1536, 1);  // layer 4 takes h3 chunk by chunk
            tq = etr ? gtime() : 0;
            if (has_next) {
                ac += kAhead;  // (already written and published)
                emit_h1(nxt, kAhead, 4);
            }
            if (etr) e_h1 += gtime() - tq;
            wait_d(&ms.d4done, d4ph);
            tq = etr ? gtime() : 0;
            final_layer(cur, pb);
            if (etr) e_fin += gtime() - tq;
            cur = nxt;
            pb ^= 1;
        }
        if (etr) {
            P.trace[4] = gtime() - e_begin;
            P.trace[5] = e_free;
            P.trace[6] = e_d;
            P.trace[7] = e_prep;
            P.trace[8] = e_h1;
            P.trace[9] = e_fin;
            P.trace[14] = e_dr;
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc2<512>(tmem);
    }
}

}  // namespace fact2

int launch_pifu_fact2(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& job, const float* records,
                      const int* cmap, unsigned max_points, bool x3, cudaStream_t s) {
    static PerDeviceOnce once;
    if (int r = once.run([] {
            ICG_CUDA_TRY(cudaFuncSetAttribute(fact2::k_fact2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)fact2::Layout<true>::kTotal));
            ICG_CUDA_TRY(cudaFuncSetAttribute(fact2::k_fact2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)fact2::Layout<false>::kTotal));
            return ICG_OK;
        }))
        return r;
    fact2::Params p{};
    p.f = f;
    p.job = job;
    p.bias = geo.bias;
    p.wlast = geo.w_last;
    p.s_in = records;
    p.cmap = cmap;
    p.slope = 0.02f;
    unsigned pairs = (max_points + fact2::NP - 1) / fact2::NP;
    if (pairs > 74) pairs = 74;
    if (pairs == 0) pairs = 1;
    CUtensorMap tm;
    std::memcpy(&tm, tmap, sizeof(CUtensorMap));
    // dev trace buffer (ICG_TC_TRACE=1), created once (thread-safe static initialisation)
    static unsigned long long* const trace = [] {
        const char* e = getenv("ICG_TC_TRACE");
        unsigned long long* t = nullptr;
        if (e && e[0] == '1' && cudaMallocManaged(&t, 64 * sizeof(unsigned long long)) != cudaSuccess) t = nullptr;
        return t;
    }();
    p.trace = trace;
    if (p.trace) cudaMemsetAsync(p.trace, 0, 64 * 8, s);
    if (x3)
        fact2::k_fact2<true><<<2 * pairs, fact2::kThreads, fact2::Layout<true>::kTotal, s>>>(tm, p);
    else
        fact2::k_fact2<false><<<2 * pairs, fact2::kThreads, fact2::Layout<false>::kTotal, s>>>(tm, p);
    if (const cudaError_t e = cudaGetLastError()) {
        set_error(std::string("k_fact2: ") + cudaGetErrorString(e));
        return ICG_ERUNTIME;
    }
    if (p.trace) {
        cudaStreamSynchronize(s);
        const unsigned long long* t = p.trace;
        fprintf(stderr,
                "[fact2-trace] mma: total %.1f us, wait chunk %.1f, wait weights %.1f, wait tmem %.1f | epi: total %.1f, "
                "wait slot %.1f, wait acc %.1f, prep %.1f, h1 %.1f, final %.1f\n",
                t[0] * 1e-3, t[1] * 1e-3, t[2] * 1e-3, t[3] * 1e-3, t[4] * 1e-3, t[5] * 1e-3, t[6] * 1e-3, t[7] * 1e-3,
                t[8] * 1e-3, t[9] * 1e-3);
        fprintf(stderr, "[fact2-trace] weight waits by phase: L2 first %.1f, L2 rest %.1f, L3 %.1f, L4 %.1f us\n",
                t[20] * 1e-3, t[21] * 1e-3, t[22] * 1e-3, t[23] * 1e-3);
        fprintf(stderr, "[fact2-trace] chunk waits by phase: h1 first %.1f, h1 rest %.1f, h2 %.1f, h3 %.1f us; drain h2 0-3 %.1f\n",
                t[10] * 1e-3, t[11] * 1e-3, t[12] * 1e-3, t[13] * 1e-3, t[14] * 1e-3);
    }
    return ICG_OK;
}

}  // namespace icg

// k_mlp_pair.cu — the PIFu geometry field on CTA PAIRS (tcgen05 cta_group::2).
//
// Same fused "weights x activations^T" dataflow as k_mlp_tc.cu, but every MMA
// is M=256 x N=128 x K=16 executed by two SMs of a TPC: each CTA of the
// cluster holds 128 of the 256 weight rows (A) and 64 of the 128 points (B)
// in its shared memory; its TMEM holds its 128 output rows for all 128
// points.  Per SM this halves the shared-memory operand bytes per FLOP and
// doubles the tensor work per pipeline stage relative to the single-CTA
// 128x64 MMA (the single-CTA kernel measured ~25% tensor-pipe activity,
// bound by per-stage overheads and SMEM operand traffic).
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
//              the 128 -> 1 output for all 128 points on CUDA cores, the peer
//              contributes its points' skip-input dot products over DSMEM.
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

constexpr uint32_t kHalf = 16384;                 // one 128 x 64 bf16 tile
constexpr int kStages = 4;
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kEpiThreads;
constexpr int NP = 128;                           // points per pair tile (64 per CTA)
constexpr uint32_t kChunk = 64 * 128;             // 64 point rows x 64 bf16 (SW128)
constexpr uint32_t kSkipHalf = 4 * kChunk;        // Phi: 4 K-chunks
constexpr uint32_t kHHalf = 4 * kChunk;           // one 256-feature block: 4 K-chunks
constexpr uint32_t kOffSkip = 0;
constexpr uint32_t kOffH = kOffSkip + 2 * kSkipHalf;   // 64 KB
constexpr uint32_t kOffRing = kOffH + 2 * kHHalf;      // 128 KB
constexpr uint32_t kOffMisc = kOffRing + kStages * kHalf;  // 192 KB
constexpr uint32_t kMisc = 16384;
constexpr uint32_t kTotal = kOffMisc + kMisc + 1024;

// weight-item schedule (pairs): (layer, 256-row block, K column offset)
template <class Emit>
__host__ __device__ void schedule(Emit&& emit) {
    auto L1 = [&](int c) {
        for (int j = 0; j < 4; ++j) emit(0, c, j * 64);
    };
    L1(0);
    L1(1);
    for (int m = 0; m < 2; ++m)
        for (int j = 0; j < 4; ++j) emit(1, m, 1024 + j * 64);
    for (int c = 0; c < 4; ++c) {
        for (int m = 0; m < 2; ++m)
            for (int jj = 0; jj < 4; ++jj) emit(1, m, c * 256 + jj * 64);
        if (c + 2 < 4) L1(c + 2);
    }
    for (int j = 0; j < 4; ++j) emit(2, 0, 512 + j * 64);
    for (int c = 0; c < 2; ++c)
        for (int jj = 0; jj < 4; ++jj) emit(2, 0, c * 256 + jj * 64);
    for (int j = 0; j < 4; ++j) emit(3, 0, 256 + j * 64);
    for (int jj = 0; jj < 4; ++jj) emit(3, 0, jj * 64);
}
constexpr int kItems = 16 + 8 + 32 + 4 + 8 + 4 + 4;  // 76

struct Misc {
    uint64_t full[kStages], empty[kStages];
    uint64_t f_ready, h_ready, h_free, l1done[2], d2done, d3done, d4done, sd_ready[2];
    uint32_t tmem_base;
    float z[NP];
    float pos[NP][3];
    double posd[NP][3];
    float red[4][NP];
    float skipdot[2][NP];  // final-layer skip-input dot per point, double-buffered by tile parity
    float cterm[NP];       // b5 + w5z * z - sdf_scale * sdf(P), per point (leader)
};
static_assert(sizeof(Misc) + 16 <= kMisc, "misc smem too small");

struct Params {
    FieldDev f;
    EvalJob job;
    const float* bias;   // per layer [b, wz] blocks (same layout as the single-CTA stream)
    const float* wlast;  // final layer [1][128 + 257]
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

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_mlp_pair(const __grid_constant__ CUtensorMap tmap, Params P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* skip = smem + kOffSkip;
    uint8_t* hbuf = smem + kOffH;
    uint8_t* ring = smem + kOffRing;
    Misc& ms = *reinterpret_cast<Misc*>(smem + kOffMisc);
    __shared__ DevScene scene;

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
        ptx::mbar_init(&ms.h_ready, 2 * kEpiThreads);
        ptx::mbar_init(&ms.h_free, 1);
        ptx::mbar_init(&ms.l1done[0], 1);
        ptx::mbar_init(&ms.l1done[1], 1);
        ptx::mbar_init(&ms.d2done, 1);
        ptx::mbar_init(&ms.d3done, 1);
        ptx::mbar_init(&ms.d4done, 1);
        ptx::mbar_init(&ms.sd_ready[0], 64);
        ptx::mbar_init(&ms.sd_ready[1], 64);
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmap);
    for (int i = threadIdx.x; i < (int)(sizeof(DevScene) / 8); i += blockDim.x)
        reinterpret_cast<double*>(&scene)[i] = reinterpret_cast<const double*>(P.f.scene)[i];
    if (warp == 1) ptx::tmem_alloc2<512>(&ms.tmem_base);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = ms.tmem_base;
    job_account(job);

    // leader-CTA addresses of the barriers that receive cross-CTA traffic
    const uint32_t full0 = ptx::mapa(ptx::smem_u32(&ms.full[0]), 0);
    const uint32_t f_ready0 = ptx::mapa(ptx::smem_u32(&ms.f_ready), 0);
    const uint32_t h_ready0 = ptx::mapa(ptx::smem_u32(&ms.h_ready), 0);
    const uint32_t sd_ready0 = ptx::mapa(ptx::smem_u32(&ms.sd_ready[0]), 0);
    const uint16_t both = 0x3;

    if (warp == 0) {
        // ===================== weight producer (both CTAs) =====================
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const int parts = P.x3 ? 2 : 1;
            const uint32_t ring0 = ptx::smem_u32(ring);
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                for (int i = 0; i < kItems; ++i)
                    for (int part = 0; part < parts; ++part) {
                        ptx::mbar_wait(&ms.empty[s], ph ^ 1);
                        if (leader) ptx::mbar_arrive_expect_tx(&ms.full[s], 2 * kHalf);
                        const int row0 = ((i * 2 + (int)rank) * 2 + part) * 128;
                        ptx::tma_load_2d_2sm(ring0 + s * kHalf, &tmap, full0 + s * 8, 0, row0);
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
            const uint32_t idesc = ptx::idesc_bf16_f32(256, NP);
            int s = 0;
            uint32_t ph = 0, fph = 0, hph = 0;
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
            auto item = [&](uint32_t dcol, uint32_t b_hi, uint32_t b_lo, bool acc) {
                const uint64_t bd_hi = ptx::sdesc_sw128(b_hi), bd_lo = ptx::sdesc_sw128(b_lo);
                {
                    unsigned long long t0 = tr ? gtime() : 0;
                    ptx::mbar_wait(&ms.full[s], ph);
                    if (tr) w_full += gtime() - t0;
                }
                ptx::tc_fence_after();
                const uint64_t ad_hi = ptx::sdesc_sw128(ring0 + s * kHalf);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t koff = (uint64_t)(kk * 2);
                    ptx::mma_bf16_pair(tmem + dcol, ad_hi + koff, bd_hi + koff, idesc, (acc || kk > 0) ? 1u : 0u);
                    if (P.x3) ptx::mma_bf16_pair(tmem + dcol, ad_hi + koff, bd_lo + koff, idesc, 1u);
                }
                ptx::mma_commit_pair(&ms.empty[s], both);
                next_stage();
                if (P.x3) {
                    {
                        unsigned long long t0 = tr ? gtime() : 0;
                        ptx::mbar_wait(&ms.full[s], ph);
                        if (tr) w_full += gtime() - t0;
                    }
                    ptx::tc_fence_after();
                    const uint64_t ad_lo = ptx::sdesc_sw128(ring0 + s * kHalf);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t koff = (uint64_t)(kk * 2);
                        ptx::mma_bf16_pair(tmem + dcol, ad_lo + koff, bd_hi + koff, idesc, 1u);
                    }
                    ptx::mma_commit_pair(&ms.empty[s], both);
                    next_stage();
                }
            };
            auto wait_h = [&]() {
                unsigned long long t0 = tr ? gtime() : 0;
                ptx::mbar_wait_cluster(&ms.h_ready, hph);
                if (tr) w_h += gtime() - t0;
                hph ^= 1;
                ptx::tc_fence_after();
            };
            auto skipk = [&](int j) { return skip_hi + j * kChunk; };
            auto skipl = [&](int j) { return skip_lo + j * kChunk; };
            // TMEM columns: D2[m] = m*128, BUF[b] = 256 + b*128, D3 = BUF[0], D4 = D2[0]
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                {
                    unsigned long long t0 = tr ? gtime() : 0;
                    ptx::mbar_wait_cluster(&ms.f_ready, fph);
                    if (tr) w_f += gtime() - t0;
                }
                fph ^= 1;
                ptx::tc_fence_after();
                auto L1 = [&](int c) {
                    for (int j = 0; j < 4; ++j) item(256 + (c & 1) * 128, skipk(j), skipl(j), j > 0);
                    ptx::mma_commit_pair(&ms.l1done[c & 1], both);
                };
                L1(0);
                L1(1);
                for (int m = 0; m < 2; ++m)
                    for (int j = 0; j < 4; ++j) item(m * 128, skipk(j), skipl(j), j > 0);
                for (int c = 0; c < 4; ++c) {
                    wait_h();
                    for (int m = 0; m < 2; ++m)
                        for (int jj = 0; jj < 4; ++jj) item(m * 128, h_hi + jj * kChunk, h_lo + jj * kChunk, true);
                    ptx::mma_commit_pair(&ms.h_free, both);
                    if (c + 2 < 4) L1(c + 2);
                }
                ptx::mma_commit_pair(&ms.d2done, both);
                for (int j = 0; j < 4; ++j) item(256, skipk(j), skipl(j), j > 0);
                for (int c = 0; c < 2; ++c) {
                    wait_h();
                    for (int jj = 0; jj < 4; ++jj) item(256, h_hi + jj * kChunk, h_lo + jj * kChunk, true);
                    ptx::mma_commit_pair(&ms.h_free, both);
                }
                ptx::mma_commit_pair(&ms.d3done, both);
                for (int j = 0; j < 4; ++j) item(0, skipk(j), skipl(j), j > 0);
                wait_h();
                for (int jj = 0; jj < 4; ++jj) item(0, h_hi + jj * kChunk, h_lo + jj * kChunk, true);
                ptx::mma_commit_pair(&ms.h_free, both);
                ptx::mma_commit_pair(&ms.d4done, both);
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
        const int quarter = warp & 3;
        const int colh = (warp - 2) >> 2;  // point half this warp converts = destination CTA
        const int row = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(colh * 64);
        uint32_t l1ph[2] = {0, 0}, d2ph = 0, d3ph = 0, d4ph = 0, hfph = 1, sdph[2] = {0, 0};
        unsigned tile_iter = 0;
        const FieldDev& f = P.f;
        const bool odd = lane & 1;
        // this thread's feature inside a 256-row block, and its K position in the next layer's operand
        const uint32_t feat = rank * 128u + (uint32_t)row;
        const uint32_t kc_off = (feat >> 6) * kChunk;
        const uint32_t kk = (feat & 63u) & ~1u;
        const uint32_t hdst = ptx::mapa(ptx::smem_u32(hbuf), (uint32_t)colh);  // h buffer of the owning CTA
        const bool tr = P.trace && blockIdx.x == 0 && et == 0;
        unsigned long long e_acc = 0, e_hf = 0, e_g = 0, e_fin = 0, e_emit = 0, e_begin = gtime();
        auto ew = [&](uint64_t* bar, uint32_t par) {
            unsigned long long t0 = tr ? gtime() : 0;
            ptx::mbar_wait(bar, par);
            if (tr) e_acc += gtime() - t0;
        };

        auto emit_block = [&](uint32_t col, const float* bias_blk, int out_dim, int feat0) {
            const int o = feat0 + (int)feat;
            const float bo = __ldg(&bias_blk[o]);
            const float wz = __ldg(&bias_blk[out_dim + o]);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                uint32_t r[32];
                ptx::tmem_ld32(lane_base + col + hf * 32, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int q = 0; q < 32; q += 2) {
                    const int pl = hf * 32 + q;          // point within the destination CTA (0..63)
                    const int p = colh * 64 + pl;        // point within the pair tile
                    float v0 = __uint_as_float(r[q]) + fmaf(wz, ms.z[p], bo);
                    float v1 = __uint_as_float(r[q + 1]) + fmaf(wz, ms.z[p + 1], bo);
                    v0 = v0 < 0.0f ? v0 * P.slope : v0;
                    v1 = v1 < 0.0f ? v1 * P.slope : v1;
                    const float send = odd ? v0 : v1;
                    const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                    const float a = odd ? recv : v0;
                    const float b = odd ? v1 : recv;
                    const uint32_t off = kc_off + sw128((uint32_t)(pl + (odd ? 1 : 0)), kk);
                    const uint32_t hv = pack_bf16(a, b);
                    ptx::st_cluster_u32(hdst + off, hv);
                    if (P.x3) {
                        const float ah = __uint_as_float(hv << 16), bh = __uint_as_float(hv & 0xFFFF0000u);
                        ptx::st_cluster_u32(hdst + kHHalf + off, pack_bf16(a - ah, b - bh));
                    }
                }
            }
        };
        auto h_begin = [&]() {
            unsigned long long t0 = tr ? gtime() : 0;
            ptx::mbar_wait(&ms.h_free, hfph);
            if (tr) e_hf += gtime() - t0;
            hfph ^= 1;
        };
        auto h_end = [&]() {
            ptx::fence_proxy_async_cluster();
            ptx::tc_fence_before();
            ptx::mbar_arrive_cluster(h_ready0);
        };

        const float* b1 = P.bias;
        const float* b2 = b1 + 2 * 1024;
        const float* b3 = b2 + 2 * 512;
        const float* b4 = b3 + 2 * 256;
        const float* b5 = b4 + 2 * 128;

        for (unsigned t = pair_id; t < ntiles; t += npairs) {
            const unsigned base = t * NP;
            // ---- positions of all 128 points (every CTA needs z for its epilogue) ----
            const int tp = (int)(tile_iter & 1u);
            if (et < NP) {
                const unsigned idx = base + et;
                double pd[3] = {0.0, 0.0, 0.0};
                if (idx < n) job_point_d(job, idx, pd);
                for (int d = 0; d < 3; ++d) {
                    ms.posd[et][d] = pd[d];
                    ms.pos[et][d] = (float)pd[d];
                }
                ms.z[et] = (float)pd[2];
                if (leader)  // constant part of the final logit: b5 + w5z*z - sdf_scale*sdf(P) (fp64 SDF)
                    ms.cterm[et] = __ldg(&b5[0]) + __ldg(&P.wlast[128 + kGeoSkip - 1]) * (float)pd[2] +
                                   (float)(-scene.sdf_scale * scene_sdf(scene, pd));
            }
            epi_bar();
            // ---- gather Phi for this CTA's 64 points into its skip operand ----
            // warp per point (8 points per warp, 2 in flight); lane = 8 consecutive
            // channels = one 16-byte SW128 chunk of the bf16 operand; the same pass
            // computes the final layer's skip-input dot product in fp32.
            unsigned long long tg = tr ? gtime() : 0;
            {
                const int ew = et >> 5;
                const int c0 = 8 * lane;
                const uint32_t chunk = (uint32_t)(c0 >> 6) * kChunk;
                const uint32_t c16 = (uint32_t)((c0 & 63) >> 3);
                const size_t rowW = (size_t)f.W * f.C;
                float w5s[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) w5s[i] = __ldg(&P.wlast[128 + c0 + i]);
                for (int it = 0; it < 4; ++it) {
                    float4 t[2][8];
                    float wts[2][4];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int p = (int)rank * 64 + ew * 8 + it * 2 + j;
                        float u = (ms.pos[p][0] + 1.0f) * 0.5f * (float)(f.W - 1);
                        float v = (1.0f - ms.pos[p][1]) * 0.5f * (float)(f.H - 1);
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
                            t[j][2 * q] = __ldg(reinterpret_cast<const float4*>(taps[q]));
                            t[j][2 * q + 1] = __ldg(reinterpret_cast<const float4*>(taps[q] + 4));
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int pl = ew * 8 + it * 2 + j;
                        float val[8];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const float4 a0 = t[j][h], a1 = t[j][2 + h], a2 = t[j][4 + h], a3 = t[j][6 + h];
                            val[4 * h + 0] = wts[j][0] * a0.x + wts[j][1] * a1.x + wts[j][2] * a2.x + wts[j][3] * a3.x;
                            val[4 * h + 1] = wts[j][0] * a0.y + wts[j][1] * a1.y + wts[j][2] * a2.y + wts[j][3] * a3.y;
                            val[4 * h + 2] = wts[j][0] * a0.z + wts[j][1] * a1.z + wts[j][2] * a2.z + wts[j][3] * a3.z;
                            val[4 * h + 3] = wts[j][0] * a0.w + wts[j][1] * a1.w + wts[j][2] * a2.w + wts[j][3] * a3.w;
                        }
                        uint4 hv, lv;
                        uint32_t* hp = reinterpret_cast<uint32_t*>(&hv);
                        uint32_t* lp = reinterpret_cast<uint32_t*>(&lv);
                        float dot = 0.0f;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float a = val[2 * i], b = val[2 * i + 1];
                            hp[i] = pack_bf16(a, b);
                            lp[i] = pack_bf16(a - __uint_as_float(hp[i] << 16), b - __uint_as_float(hp[i] & 0xFFFF0000u));
                            dot = fmaf(w5s[2 * i], a, dot);
                            dot = fmaf(w5s[2 * i + 1], b, dot);
                        }
                        const uint32_t off = chunk + (uint32_t)pl * 128u + (((c16 ^ (uint32_t)pl) & 7u) << 4);
                        *reinterpret_cast<uint4*>(skip + off) = hv;
                        *reinterpret_cast<uint4*>(skip + kSkipHalf + off) = lv;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
                        if (lane == 0) {
                            const int p = (int)rank * 64 + pl;
                            if (leader) {
                                ms.skipdot[tp][p] = dot;
                            } else {
                                ptx::st_cluster_f32(ptx::mapa(ptx::smem_u32(&ms.skipdot[tp][p]), 0), dot);
                                ptx::mbar_arrive_cluster(sd_ready0 + 8 * tp);
                            }
                        }
                    }
                }
            }
            ptx::fence_proxy_async_cluster();
            ptx::mbar_arrive_cluster(f_ready0);
            if (tr) e_g += gtime() - tg;

            // ---- layer 1 chunks (256 features each) -> h buffers of both CTAs ----
            for (int c = 0; c < 4; ++c) {
                ew(&ms.l1done[c & 1], l1ph[c & 1]);
                l1ph[c & 1] ^= 1;
                ptx::tc_fence_after();
                h_begin();
                emit_block(256 + (c & 1) * 128, b1, 1024, c * 256);
                h_end();
            }
            ew(&ms.d2done, d2ph);
            d2ph ^= 1;
            ptx::tc_fence_after();
            for (int m = 0; m < 2; ++m) {
                h_begin();
                emit_block(m * 128, b2, 512, m * 256);
                h_end();
            }
            ew(&ms.d3done, d3ph);
            d3ph ^= 1;
            ptx::tc_fence_after();
            h_begin();
            emit_block(256, b3, 256, 0);
            h_end();
            ew(&ms.d4done, d4ph);
            d4ph ^= 1;
            ptx::tc_fence_after();
            unsigned long long tf = tr ? gtime() : 0;
            // ---- final layer (CTA 0 holds layer-4 rows 0..127 for all 128 points) ----
            if (leader) {
                const float bo = __ldg(&b4[row]), wz = __ldg(&b4[128 + row]);
                const float w5 = __ldg(&P.wlast[row]);
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t r[32];
                    ptx::tmem_ld32(lane_base + 0 + hf * 32, r);
                    ptx::tmem_ld_wait();
                    float v[32];
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        float x = __uint_as_float(r[q]) + fmaf(wz, ms.z[colh * 64 + hf * 32 + q], bo);
                        x = x < 0.0f ? x * P.slope : x;
                        v[q] = w5 * x;
                    }
                    const float sum = warp_transpose_reduce(v);
                    ms.red[quarter][colh * 64 + hf * 32 + lane] = sum;
                }
            }
            ptx::tc_fence_before();
            epi_bar();
            if (leader) {
                ptx::mbar_wait_cluster(&ms.sd_ready[tp], sdph[tp]);
                sdph[tp] ^= 1;
                if (et < NP) {
                    const int p = et;
                    const unsigned idx = base + p;
                    const float s = ms.red[0][p] + ms.red[1][p] + ms.red[2][p] + ms.red[3][p] + ms.skipdot[tp][p] +
                                    ms.cterm[p];
                    if (idx < n) {
                        const float vv = 1.0f / (1.0f + expf(-s));
                        if (job_is_grid(job))
                            grid_epilogue(job, job_node(job, idx), vv);
                        else
                            job.out[idx] = vv;
                    }
                }
            }
            epi_bar();
            if (tr) e_fin += gtime() - tf;
            ++tile_iter;
        }
        if (tr) {
            P.trace[4] = gtime() - e_begin;
            P.trace[5] = e_acc;
            P.trace[6] = e_hf;
            P.trace[7] = e_g;
            P.trace[8] = e_fin;
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
// Host side: pair weight stream + tensor map + launch
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

size_t pair_stream_bytes() { return (size_t)pair::kItems * 4 * pair::kHalf; }

// item i, half h (rows h*128.. of the 256-row block), part (hi/lo): 16 KB SW128 tile
int pair_pack_geometry(const float* const* w, uint8_t* stream) {
    const int* outs = kGeoOut;
    int ins[5];
    for (int l = 0; l < 5; ++l) ins[l] = (l ? outs[l - 1] : 0) + kGeoSkip;
    int item = 0;
    auto emit = [&](int l, int m, int col0) {
        for (int h = 0; h < 2; ++h) {
            uint8_t* hi = stream + ((size_t)(item * 2 + h) * 2 + 0) * pair::kHalf;
            uint8_t* lo = stream + ((size_t)(item * 2 + h) * 2 + 1) * pair::kHalf;
            for (int r = 0; r < 128; ++r) {
                const int o = m * 256 + h * 128 + r;
                for (int k = 0; k < 64; ++k) {
                    float v = o < outs[l] ? w[l][(size_t)o * ins[l] + col0 + k] : 0.0f;
                    uint16_t a = f2bf_p(v);
                    uint16_t b = f2bf_p(v - bf2f_p(a));
                    size_t off = (size_t)r * 128 + (size_t)(((k >> 3) ^ (r & 7)) << 4) + (size_t)(k & 7) * 2;
                    std::memcpy(hi + off, &a, 2);
                    std::memcpy(lo + off, &b, 2);
                }
            }
        }
        ++item;
    };
    pair::schedule(emit);
    return item == pair::kItems ? ICG_OK : ICG_ERUNTIME;
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
    cuuint32_t box[2] = {128, 128};
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

int launch_pifu_pair_eval(const FieldDev& f, const TcMlp& geo, const void* tmap, const EvalJob& job,
                          unsigned max_points, bool x3, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        ICG_CUDA_TRY(cudaFuncSetAttribute(pair::k_mlp_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)pair::kTotal));
        attr = true;
    }
    pair::Params p{};
    p.f = f;
    p.job = job;
    p.bias = geo.bias;
    p.wlast = geo.w_last;
    p.slope = 0.02f;
    p.x3 = x3 ? 1 : 0;
    unsigned pairs = (max_points + pair::NP - 1) / pair::NP;
    if (pairs > 74) pairs = 74;
    if (pairs == 0) pairs = 1;
    static unsigned long long* trace = nullptr;
    static int tron = -1;
    if (tron < 0) {
        const char* e = getenv("ICG_TC_TRACE");
        tron = e && e[0] == '1';
        if (tron) cudaMallocManaged(&trace, 64 * sizeof(unsigned long long));
    }
    p.trace = tron ? trace : nullptr;
    if (p.trace) cudaMemsetAsync(p.trace, 0, 64 * 8, s);
    CUtensorMap tm;
    std::memcpy(&tm, tmap, sizeof(CUtensorMap));
    pair::k_mlp_pair<<<2 * pairs, pair::kThreads, pair::kTotal, s>>>(tm, p);
    ICG_CUDA_TRY(cudaGetLastError());
    if (p.trace) {
        cudaStreamSynchronize(s);
        const unsigned long long* t = p.trace;
        fprintf(stderr,
                "[pair-trace] mma: total %.1f us, wait data %.1f, wait h %.1f, wait f %.1f | epi: total %.1f, wait acc "
                "%.1f, wait hfree %.1f, gather %.1f, final %.1f\n",
                t[0] * 1e-3, t[1] * 1e-3, t[2] * 1e-3, t[3] * 1e-3, t[4] * 1e-3, t[5] * 1e-3, t[6] * 1e-3, t[7] * 1e-3,
                t[8] * 1e-3);
    }
    return ICG_OK;
}

}  // namespace icg

// k_lp.cu — latency path of the PIFu geometry field: LAYER-parallel tensor-core
// evaluation of small and medium batches over the whole GPU.
//
// The conflict loop (localize.hpp:338-353) is a chain of dependent batches of
// ~10-25000 nodes.  The CTA-pair kernel (k_mlp_pair.cu) parallelises over
// POINTS: a batch of n points occupies ceil(n/128) pairs, each streaming all
// ~5 MB of weight tiles through one TPC, so a small batch costs a full tile
// latency (~100 us) on a mostly idle GPU.  Here every layer is spread over
// all SMs instead: work units are (128-row output block, K-range, 128-point
// block); a unit loads its weight tiles and activation tiles with the TMA
// engine (1-D bulk copies of pre-swizzled 32 KB hi|lo tiles), runs the
// bf16x3 (or bf16) tcgen05 MMAs into TMEM and either
//   * K-split: stores fp32 partial sums, reduced after a grid barrier in a
//     fixed order by a reduce phase that applies bias + z-term + leaky ReLU
//     and writes the next layer's bf16 hi/lo activation tiles, or
//   * full K: applies the activation in its own epilogue (staged in shared
//     memory, stored as whole tiles); for the last hidden layer the epilogue
//     also computes the 128 -> 1 output layer and the grid epilogue.
// One cooperative persistent kernel, grid barriers between phases.  Exits at
// once when the batch is empty or larger than `max_count` (the pair kernel
// takes those: both are enqueued, no host round trip).
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "eval_common.cuh"
#include "tc_ptx.cuh"

namespace cg = cooperative_groups;

namespace icg {

namespace lp {

constexpr int kThreads = 256;
constexpr int NB = 128;                 // points per point block (MMA N)
constexpr uint32_t kTile = 32768;       // one 128 x 64 bf16 hi tile + its lo tile
constexpr uint32_t kTileHalf = 16384;
constexpr int kStages = 3;
constexpr uint32_t kOffStage = 0;                            // stage s: W tile, X tile (64 KB)
constexpr uint32_t kOffOut = 0;                              // activation staging (2 tiles) reuses stages 0..1
constexpr uint32_t kOffMisc = kStages * 2 * kTile;           // 192 KB
constexpr uint32_t kSmem = kOffMisc + 4096 + 1024;
constexpr int kActKC = 16;                                   // activation tiles per point block (max K-chunks)
constexpr int kLayers = 4;                                   // hidden layers on tensor cores

__host__ __device__ constexpr int layer_out(int l) { return l == 0 ? 1024 : l == 1 ? 512 : l == 2 ? 256 : 128; }
__host__ __device__ constexpr int layer_prev(int l) { return l == 0 ? 0 : layer_out(l - 1); }
__host__ __device__ constexpr int layer_kc(int l) { return (layer_prev(l) + kC) / 64; }   // 4, 20, 12, 8
__host__ __device__ constexpr int layer_rb(int l) { return layer_out(l) / 128; }          // 8, 4, 2, 1
__host__ __device__ constexpr int layer_tile0(int l) {
    return l == 0 ? 0 : layer_tile0(l - 1) + layer_rb(l - 1) * layer_kc(l - 1);
}
__host__ __device__ constexpr int layer_bias0(int l) { return l == 0 ? 0 : layer_bias0(l - 1) + 2 * layer_out(l - 1); }
constexpr int kTiles = layer_tile0(kLayers);  // 144

struct Params {
    FieldDev f;
    EvalJob job;
    const uint8_t* wst;   // weight tiles [layer][rb][kc] (hi | lo, SW128)
    const float* bias;    // per layer [b, wz] (tc layout), then b5
    const float* wlast;   // final layer [128 + 257]
    uint8_t* act_skip;    // Phi tiles [pb][4]
    uint8_t* act[2];      // hidden activations [pb][kActKC], ping-pong by layer parity
    float* part;          // K-split partial sums [split][O][n_pad]
    float* zf;            // z per point
    float* cterm;         // b5 + w5z*z - sdf_scale*sdf + Phi-part of the output dot
    unsigned max_count;
    int max_split[kLayers];
    int target_units;
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
__device__ __forceinline__ uint32_t lo_of(uint32_t hv, float a, float b) {
    return pack_bf16(a - __uint_as_float(hv << 16), b - __uint_as_float(hv & 0xFFFF0000u));
}
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t k) {
    return row * 128u + ((((k >> 3) ^ row) & 7u) << 4) + (k & 7u) * 2u;
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

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

// number of K-splits of layer l for npb point blocks
__device__ __forceinline__ int choose_split(const Params& P, int l, unsigned npb) {
    const int kc = layer_kc(l);
    const unsigned base = (unsigned)layer_rb(l) * npb;
    int s = (int)((P.target_units + base - 1) / base);
    s = max(1, min(s, min(kc, P.max_split[l])));
    const int g = (kc + s - 1) / s;
    return (kc + g - 1) / g;
}

struct Misc {
    uint64_t full[kStages], empty[kStages], accb;
    uint32_t tmem_base;
    float red[4][NB];
};

__global__ void __launch_bounds__(kThreads, 1) k_lp(Params P) {
    const EvalJob& job = P.job;
    const unsigned n = job_count(job);
    if (n == 0 || n > P.max_count) return;  // grid-uniform decision
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Misc& ms = *reinterpret_cast<Misc*>(smem + kOffMisc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned npb = (n + NB - 1) / NB, n_pad = npb * NB;
    const FieldDev& f = P.f;
    const bool tr = P.trace && blockIdx.x == 0 && threadIdx.x == 0;
    int ti = 1;
    if (tr) P.trace[0] = gtime();
    if (P.trace && threadIdx.x == 0) atomicMax(&P.trace[31], gtime());  // last CTA start
    // grid barrier; trace: [ti] = barrier exit (block 0), [16 + ti] = last arrival over blocks
    auto gsync = [&]() {
        if (P.trace && threadIdx.x == 0) atomicMax(&P.trace[16 + ti], gtime());
        grid.sync();
        if (tr) P.trace[ti] = gtime();
        ++ti;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&ms.full[s], 1);
            ptx::mbar_init(&ms.empty[s], 1);
        }
        ptx::mbar_init(&ms.accb, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc<128>(&ms.tmem_base);
    job_account(job);
    // pull the weight tiles into L2 while the gather runs (one tile per CTA)
    if (threadIdx.x == 0)
        for (unsigned t = blockIdx.x; t < (unsigned)kTiles; t += gridDim.x)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.wst + (size_t)t * kTile), "r"(kTile)
                         : "memory");

    // ---- phase 0: gather Phi (bf16 hi/lo tiles), z, constant part of the output logit ----
    {
        const float* wl = P.wlast;
        const float* b5 = P.bias + layer_bias0(kLayers);
        const int c0 = 8 * lane;
        float w5s[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w5s[i] = __ldg(&wl[128 + c0 + i]);
        const float w5z = __ldg(&wl[128 + kGeoSkip - 1]);
        const size_t rowW = (size_t)f.W * f.C;
        const unsigned gw = (blockIdx.x * kThreads + threadIdx.x) >> 5, nw = (gridDim.x * kThreads) >> 5;
        for (unsigned p = gw; p < n_pad; p += nw) {
            const unsigned pb = p / NB, r = p % NB;
            uint8_t* tile = P.act_skip + ((size_t)pb * 4 + (lane >> 3)) * kTile;
            const uint32_t off = r * 128u + ((((uint32_t)lane & 7u) ^ r) & 7u) * 16u;
            if (p >= n) {  // padded point: zeros
                *reinterpret_cast<uint4*>(tile + off) = make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4*>(tile + kTileHalf + off) = make_uint4(0, 0, 0, 0);
                if (lane == 0) P.zf[p] = 0.0f;
                continue;
            }
            double pd[3];
            job_point_d(job, p, pd);
            float u = ((float)pd[0] + 1.0f) * 0.5f * (float)(f.W - 1);
            float v = (1.0f - (float)pd[1]) * 0.5f * (float)(f.H - 1);
            u = fminf(fmaxf(u, 0.0f), (float)(f.W - 1));
            v = fminf(fmaxf(v, 0.0f), (float)(f.H - 1));
            const int x0 = min((int)floorf(u), f.W - 2), y0 = min((int)floorf(v), f.H - 2);
            const float ax = u - (float)x0, ay = v - (float)y0;
            const float w00 = (1.0f - ax) * (1.0f - ay), w10 = ax * (1.0f - ay), w01 = (1.0f - ax) * ay,
                        w11 = ax * ay;
            const float* m00 = f.fmap_hwc + ((size_t)y0 * f.W + x0) * (size_t)f.C + c0;
            const float* taps[4] = {m00, m00 + f.C, m00 + rowW, m00 + rowW + f.C};
            float4 t[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                t[2 * q] = __ldg(reinterpret_cast<const float4*>(taps[q]));
                t[2 * q + 1] = __ldg(reinterpret_cast<const float4*>(taps[q] + 4));
            }
            float val[8];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                val[4 * h + 0] = w00 * t[h].x + w10 * t[2 + h].x + w01 * t[4 + h].x + w11 * t[6 + h].x;
                val[4 * h + 1] = w00 * t[h].y + w10 * t[2 + h].y + w01 * t[4 + h].y + w11 * t[6 + h].y;
                val[4 * h + 2] = w00 * t[h].z + w10 * t[2 + h].z + w01 * t[4 + h].z + w11 * t[6 + h].z;
                val[4 * h + 3] = w00 * t[h].w + w10 * t[2 + h].w + w01 * t[4 + h].w + w11 * t[6 + h].w;
            }
            uint4 hv, lv;
            uint32_t* hp = reinterpret_cast<uint32_t*>(&hv);
            uint32_t* lp = reinterpret_cast<uint32_t*>(&lv);
            float dot = 0.0f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                hp[i] = pack_bf16(val[2 * i], val[2 * i + 1]);
                lp[i] = lo_of(hp[i], val[2 * i], val[2 * i + 1]);
                dot = fmaf(w5s[2 * i], val[2 * i], dot);
                dot = fmaf(w5s[2 * i + 1], val[2 * i + 1], dot);
            }
            *reinterpret_cast<uint4*>(tile + off) = hv;
            *reinterpret_cast<uint4*>(tile + kTileHalf + off) = lv;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            const double sdf = scene_sdf_warp(*f.scene, pd);
            if (lane == 0) {
                P.zf[p] = (float)pd[2];
                P.cterm[p] = dot + __ldg(&b5[0]) + w5z * (float)pd[2] + (float)(-f.scene->sdf_scale * sdf);
            }
        }
    }
    fence_proxy_async_global();
    ptx::tc_fence_before();
    gsync();
    ptx::tc_fence_after();
    const uint32_t tmem = ms.tmem_base;
    const uint32_t idesc = ptx::idesc_bf16_f32(128, NB);
    uint32_t g_issue = 0, g_mma = 0, g_acc = 0;
    const int quarter = warp & 3, colh = warp >> 2;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(colh * 64);
    uint8_t* stage0 = smem + kOffStage;
    uint8_t* outst = smem + kOffOut;

    for (int l = 0; l < kLayers; ++l) {
        const int O = layer_out(l), KC = layer_kc(l), KCh = layer_prev(l) / 64, RB = layer_rb(l);
        const int nsplit = l == kLayers - 1 ? 1 : choose_split(P, l, npb);
        const int G = (KC + nsplit - 1) / nsplit;
        const unsigned units = (unsigned)RB * nsplit * npb;
        const uint8_t* act_in = P.act[(l + 1) & 1];  // layer l reads act[(l+1)&1] (l >= 1), writes act[l&1]
        uint8_t* act_out = P.act[l & 1];
        const float* bl = P.bias + layer_bias0(l);
        // ---- MMA phase ----
        for (unsigned u = blockIdx.x; u < units; u += gridDim.x) {
            const unsigned pb = u % npb;
            const int rb = (int)((u / npb) % (unsigned)RB);
            const int sp = (int)(u / (npb * (unsigned)RB));
            const int k0 = sp * G, k1 = min(KC, k0 + G), nk = k1 - k0;
            if (threadIdx.x == 0) {
                const uint8_t* wbase = P.wst + ((size_t)layer_tile0(l) + (size_t)rb * KC) * kTile;
                int issued = 0, done = 0;
                while (done < nk) {
                    while (issued < nk && issued - done < kStages) {
                        const int s = (int)(g_issue % kStages);
                        if (g_issue >= (uint32_t)kStages) ptx::mbar_wait(&ms.empty[s], ((g_issue / kStages) - 1) & 1);
                        const int kc = k0 + issued;
                        const uint8_t* xsrc = kc < KCh ? act_in + ((size_t)pb * kActKC + kc) * kTile
                                                       : P.act_skip + ((size_t)pb * 4 + (kc - KCh)) * kTile;
                        uint8_t* st = stage0 + (size_t)s * 2 * kTile;
                        ptx::mbar_arrive_expect_tx(&ms.full[s], 2 * kTile);
                        ptx::bulk_g2s(st, wbase + (size_t)kc * kTile, kTile, &ms.full[s]);
                        ptx::bulk_g2s(st + kTile, xsrc, kTile, &ms.full[s]);
                        ++issued;
                        ++g_issue;
                    }
                    const int s = (int)(g_mma % kStages);
                    ptx::mbar_wait(&ms.full[s], (g_mma / kStages) & 1);
                    if (tr && done == 0 && u == blockIdx.x) P.trace[32 + l * 6 + 0] = gtime();
                    ptx::tc_fence_after();
                    const uint32_t a = ptx::smem_u32(stage0 + (size_t)s * 2 * kTile), b = a + kTile;
                    const uint64_t ah = ptx::sdesc_sw128(a), al = ptx::sdesc_sw128(a + kTileHalf);
                    const uint64_t bh = ptx::sdesc_sw128(b), bl_ = ptx::sdesc_sw128(b + kTileHalf);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t ko = (uint64_t)(kk * 2);
                        ptx::mma_bf16(tmem, ah + ko, bh + ko, idesc, (done > 0 || kk > 0) ? 1u : 0u);
                        if (P.x3) {
                            ptx::mma_bf16(tmem, ah + ko, bl_ + ko, idesc, 1u);
                            ptx::mma_bf16(tmem, al + ko, bh + ko, idesc, 1u);
                        }
                    }
                    ptx::mma_commit(&ms.empty[s]);
                    ++done;
                    ++g_mma;
                }
                ptx::mma_commit(&ms.accb);
            }
            __syncwarp();
            if (tr && u == blockIdx.x) P.trace[32 + l * 6 + 1] = gtime();
            ptx::mbar_wait(&ms.accb, g_acc & 1);
            if (tr && u == blockIdx.x) P.trace[32 + l * 6 + 2] = gtime();
            ++g_acc;
            ptx::tc_fence_after();
            // ---- epilogue: thread = output row (lane quarter), 64 points (column half) ----
            const int o = rb * 128 + quarter * 32 + lane;
            const bool fin = l == kLayers - 1;
            const float bo = nsplit > 1 ? 0.0f : __ldg(&bl[o]), wz = nsplit > 1 ? 0.0f : __ldg(&bl[O + o]);
            const float w5 = fin ? __ldg(&P.wlast[o]) : 0.0f;
            const bool odd = lane & 1;
            const uint32_t kt = (uint32_t)((quarter * 32 + lane) >> 6);  // local K tile (0/1) of the output
            const uint32_t kk = (uint32_t)((quarter * 32 + lane) & 63) & ~1u;
#pragma unroll 1
            for (int hf = 0; hf < 2; ++hf) {
                uint32_t r[32];
                ptx::tmem_ld32(lane_base + hf * 32, r);
                ptx::tmem_ld_wait();
                if (tr && u == blockIdx.x && hf == 0) P.trace[32 + l * 6 + 5] = gtime();
                const unsigned p0 = pb * NB + colh * 64 + hf * 32;
                if (nsplit > 1) {
                    float* dst = P.part + ((size_t)sp * O + o) * n_pad + p0;
#pragma unroll
                    for (int q = 0; q < 32; q += 4)
                        *reinterpret_cast<float4*>(dst + q) =
                            make_float4(__uint_as_float(r[q]), __uint_as_float(r[q + 1]), __uint_as_float(r[q + 2]),
                                        __uint_as_float(r[q + 3]));
                    continue;
                }
                float h[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const float x = __uint_as_float(r[q]) + fmaf(wz, P.zf[p0 + q], bo);
                    h[q] = x < 0.0f ? x * P.slope : x;
                }
                if (fin) {
                    // output layer 128 -> 1: per-warp transpose-reduce over its 32 rows
#pragma unroll
                    for (int q = 0; q < 32; ++q) h[q] *= w5;
                    ms.red[quarter][colh * 64 + hf * 32 + lane] = warp_transpose_reduce(h);
                } else {
                    // activation tiles of this row block, staged in shared memory (SW128, hi | lo)
#pragma unroll
                    for (int q = 0; q < 32; q += 2) {
                        const float send = odd ? h[q] : h[q + 1];
                        const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                        const float a = odd ? recv : h[q];
                        const float b = odd ? h[q + 1] : recv;
                        const uint32_t row = (uint32_t)(colh * 64 + hf * 32 + q + (odd ? 1 : 0));
                        const uint32_t off = kt * kTile + sw128(row, kk);
                        const uint32_t hv = pack_bf16(a, b);
                        *reinterpret_cast<uint32_t*>(outst + off) = hv;
                        *reinterpret_cast<uint32_t*>(outst + kTileHalf + off) = lo_of(hv, a, b);
                    }
                }
            }
            ptx::tc_fence_before();
            if (tr && u == blockIdx.x) P.trace[24 + l] = gtime();
            if (nsplit == 1) {
                __syncthreads();
                if (fin) {
                    if (threadIdx.x < NB) {
                        const unsigned p = pb * NB + threadIdx.x;
                        if (p < n) {
                            const float s = ms.red[0][threadIdx.x] + ms.red[1][threadIdx.x] + ms.red[2][threadIdx.x] +
                                            ms.red[3][threadIdx.x] + P.cterm[p];
                            const float vv = 1.0f / (1.0f + expf(-s));
                            if (job_is_grid(job))
                                grid_epilogue(job, job_node(job, p), vv);
                            else
                                job.out[p] = vv;
                        }
                    }
                } else {
                    uint8_t* dst = act_out + ((size_t)pb * kActKC + rb * 2) * kTile;  // 2 contiguous tiles
                    for (int i = threadIdx.x; i < (int)(2 * kTile / 16); i += kThreads)
                        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(outst)[i];
                    ptx::fence_proxy_async_smem();  // the stages are refilled by the TMA engine next
                }
            }
            __syncthreads();
            ptx::tc_fence_after();
            if (tr && u == blockIdx.x) P.trace[32 + l * 6 + 3] = gtime();
        }
        fence_proxy_async_global();
        if (tr) P.trace[32 + l * 6 + 4] = gtime();
        ptx::tc_fence_before();
        gsync();
        ptx::tc_fence_after();
        // ---- reduce phase (K-split layers): fixed-order sum of the partials ----
        if (nsplit > 1) {
            const unsigned items = (unsigned)(O / 2) * n_pad;
            for (unsigned it = blockIdx.x * kThreads + threadIdx.x; it < items; it += gridDim.x * kThreads) {
                const unsigned p = it % n_pad;
                const int o = (int)(it / n_pad) * 2;
                float s0 = 0.0f, s1 = 0.0f;
                for (int sp = 0; sp < nsplit; ++sp) {
                    const float* src = P.part + ((size_t)sp * O + o) * n_pad + p;
                    s0 += src[0];
                    s1 += src[n_pad];
                }
                const float z = P.zf[p];
                float a = s0 + fmaf(__ldg(&bl[O + o]), z, __ldg(&bl[o]));
                float b = s1 + fmaf(__ldg(&bl[O + o + 1]), z, __ldg(&bl[o + 1]));
                a = a < 0.0f ? a * P.slope : a;
                b = b < 0.0f ? b * P.slope : b;
                const unsigned pb = p / NB, row = p % NB;
                uint8_t* tile = act_out + ((size_t)pb * kActKC + (o >> 6)) * kTile;
                const uint32_t off = sw128(row, (uint32_t)(o & 63));
                const uint32_t hv = pack_bf16(a, b);
                *reinterpret_cast<uint32_t*>(tile + off) = hv;
                *reinterpret_cast<uint32_t*>(tile + kTileHalf + off) = lo_of(hv, a, b);
            }
            fence_proxy_async_global();
            gsync();
        }
    }
    if (tr) P.trace[15] = n;
    if (P.trace && threadIdx.x == 0) atomicMax(&P.trace[30], gtime());  // last CTA end
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<128>(ms.tmem_base);
    }
}

}  // namespace lp

// ===========================================================================
// Host side
// ===========================================================================
static inline uint16_t f2bf_l(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    uint32_t r = ((u >> 16) & 1u) + 0x7FFFu;
    return (uint16_t)((u + r) >> 16);
}
static inline float bf2f_l(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

size_t lp_stream_bytes() { return (size_t)lp::kTiles * lp::kTile; }

// tile (l, rb, kc): rows = outputs rb*128.., K = input columns kc*64.. ([prev, Phi]), hi then lo, SW128
int lp_pack_geometry(const float* const* w, uint8_t* stream) {
    for (int l = 0; l < lp::kLayers; ++l) {
        const int ins = lp::layer_prev(l) + kGeoSkip;
        for (int rb = 0; rb < lp::layer_rb(l); ++rb)
            for (int kc = 0; kc < lp::layer_kc(l); ++kc) {
                uint8_t* hi = stream + ((size_t)lp::layer_tile0(l) + (size_t)rb * lp::layer_kc(l) + kc) * lp::kTile;
                uint8_t* lo = hi + lp::kTileHalf;
                for (int r = 0; r < 128; ++r)
                    for (int k = 0; k < 64; ++k) {
                        const float v = w[l][(size_t)(rb * 128 + r) * ins + kc * 64 + k];
                        const uint16_t a = f2bf_l(v), b = f2bf_l(v - bf2f_l(a));
                        const size_t off = (size_t)r * 128 + (size_t)(((k >> 3) ^ (r & 7)) << 4) + (size_t)(k & 7) * 2;
                        std::memcpy(hi + off, &a, 2);
                        std::memcpy(lo + off, &b, 2);
                    }
            }
    }
    return ICG_OK;
}

static int lp_env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

// scratch layout for max_count points: act_skip | act[0] | act[1] | part | zf | cterm
size_t lp_scratch_bytes(unsigned max_count) {
    const size_t npb = (max_count + lp::NB - 1) / lp::NB, n_pad = npb * lp::NB;
    size_t part = 0;
    for (unsigned b = 1; b <= npb; ++b)
        for (int l = 0; l < lp::kLayers - 1; ++l) {
            const size_t s = lp::layer_kc(l);  // upper bound on the split count
            const size_t bytes = s * lp::layer_out(l) * (size_t)b * lp::NB * 4;
            if (bytes > part) part = bytes;
        }
    return npb * 4 * lp::kTile + 2 * npb * lp::kActKC * lp::kTile + part + 2 * n_pad * 4 + 4096;
}

int launch_lp_eval(const FieldDev& f, const TcMlp& geo, const uint8_t* lp_stream, const EvalJob& job, uint8_t* scratch,
                   unsigned max_count, bool x3, cudaStream_t s) {
    static int grid = 0;
    static bool attr = false;
    if (!attr) {
        ICG_CUDA_TRY(cudaFuncSetAttribute(lp::k_lp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lp::kSmem));
        attr = true;
    }
    if (grid == 0) {
        int per_sm = 0, sms = 0, dev = 0;
        ICG_CUDA_TRY(cudaGetDevice(&dev));
        ICG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        ICG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lp::k_lp, lp::kThreads, lp::kSmem));
        if (per_sm < 1) {
            set_error("k_lp: does not fit on an SM");
            return ICG_ERUNTIME;
        }
        grid = sms;
    }
    lp::Params p{};
    p.f = f;
    p.job = job;
    p.wst = lp_stream;
    p.bias = geo.bias;
    p.wlast = geo.w_last;
    const size_t npb = (max_count + lp::NB - 1) / lp::NB, n_pad = npb * lp::NB;
    uint8_t* q = scratch;
    p.act_skip = q;
    q += npb * 4 * lp::kTile;
    p.act[0] = q;
    q += npb * lp::kActKC * lp::kTile;
    p.act[1] = q;
    q += npb * lp::kActKC * lp::kTile;
    p.zf = reinterpret_cast<float*>(q);
    q += n_pad * 4;
    p.cterm = reinterpret_cast<float*>(q);
    q += n_pad * 4;
    q = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(q) + 255) & ~uintptr_t(255));
    p.part = reinterpret_cast<float*>(q);
    p.max_count = max_count;
    p.max_split[0] = lp_env_int("ICG_LP_S1", 1);
    p.max_split[1] = lp_env_int("ICG_LP_S2", 10);
    p.max_split[2] = lp_env_int("ICG_LP_S3", 6);
    p.max_split[3] = 1;
    p.target_units = lp_env_int("ICG_LP_UNITS", 148);
    p.slope = 0.02f;
    p.x3 = x3 ? 1 : 0;
    static unsigned long long* trace = nullptr;
    static int tron = -1;
    if (tron < 0) {
        tron = lp_env_int("ICG_TC_TRACE", 0) == 1;
        if (tron) cudaMalloc(&trace, 64 * sizeof(unsigned long long));
    }
    p.trace = tron ? trace : nullptr;
    if (p.trace) cudaMemsetAsync(p.trace, 0, 64 * 8, s);
    void* args[] = {&p};
    ICG_CUDA_TRY(cudaLaunchCooperativeKernel((void*)lp::k_lp, grid, lp::kThreads, args, lp::kSmem, s));
    if (p.trace) {
        unsigned long long t[64];
        cudaMemcpyAsync(t, p.trace, sizeof(t), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (t[0]) {
            fprintf(stderr, "[lp-trace] n=%llu start-skew %.1f | work/sync:", t[15], (t[31] - t[0]) * 1e-3);
            for (int i = 1; i < 15 && t[i]; ++i)
                fprintf(stderr, " %.1f/%.1f", (t[16 + i] - t[i - 1]) * 1e-3, (t[i] - t[16 + i]) * 1e-3);
            int last = 1;
            while (last < 15 && t[last]) ++last;
            fprintf(stderr, " final %.1f | total %.1f us\n", (t[30] - t[last - 1]) * 1e-3, (t[30] - t[0]) * 1e-3);
            // block 0, first unit of each layer: data / issued / acc / epilogue / fence (from phase start)
            for (int l = 0; l < 4; ++l) {
                const unsigned long long* d = t + 32 + l * 6;
                if (!d[0]) continue;
                unsigned long long b = 0;
                for (int i = 1; i < 15 && t[i]; ++i)
                    if (t[i] <= d[0]) b = t[i];
                fprintf(stderr, "    L%d: data %.2f mma-issued %.2f acc %.2f tld %.2f own-epi %.2f epi %.2f fence %.2f\n", l + 1,
                        (d[0] - b) * 1e-3, (d[1] - b) * 1e-3, (d[2] - b) * 1e-3, (d[5] - b) * 1e-3, (t[24 + l] - b) * 1e-3,
                        (d[3] - b) * 1e-3, d[4] ? (d[4] - b) * 1e-3 : 0.0);
            }
        }
    }
    return ICG_OK;
}

}  // namespace icg

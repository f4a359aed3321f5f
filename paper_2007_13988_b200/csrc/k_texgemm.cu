// k_texgemm.cu — the texture field at the surface points (render.hpp:262-277 evaluates f_T at
// each covered pixel's first crossing) as a chain of per-layer GEMMs over all surface points.
//
// Why a chain: the fused pair kernel (k_mlp_pair<TEX>) keeps a point tile's activations in shared
// memory and streams the weights through it, so every weight byte serves only 128 points and the
// weight stream (TMA write + MMA read of ~47 B/clk/SM) keeps shared memory at its port limit with
// the tensor pipe ~30 % busy.  Here each layer is one GEMM, D[points x features] = A[points x K] .
// W[features x K]^T, over the whole batch: A (fp16 activations, row-major in HBM/L2) and W (fp16,
// row-major) both arrive by TMA in 128-byte-swizzled 64-wide K chunks, and one CTA-pair MMA is
// M = 256 points x N = 256 features x K = 16 (tcgen05.mma.cta_group::2), i.e. every operand byte
// in shared memory serves 256 MACs.
//
//   gather   : per point Phi (bilinear, fp32) -> fp16 skip row [Phi | h3], z, and the fp32 output-
//              layer terms of Phi and z (+ b5) into sdot;
//   geometry : g1 [Phi] -> 1024, g2 [h1 | Phi] -> 512, g3 [h2 | Phi] -> 256 = h3, written into the
//              skip rows (columns 256-511), its output-layer dot added to sdot (fp32);
//   texture  : t1 [Phi | h3] -> 1024, t2 [h1 | Phi | h3] -> 512, t3 -> 256, t4 -> 128, and the
//              output layer fused into t4's epilogue in fp32: rgb = sigmoid(w5 . h4 + sdot).
// Every hidden pre-activation is acc + b + w_z z in fp32 (the z input column stays fp32, as in the
// pair kernel), leaky-ReLU, then one fp16 rounding for the next layer's operand -- the same
// rounding points as k_mlp_pair<TEX> (colours within ~5e-4 of the fp64 oracle; tolerance 1e-3).
//
// Kernel structure (persistent, one CTA pair per TPC, 320 threads): warp 0 = TMA producer (both
// CTAs: its 128 A rows and its half of the 256 W rows per stage, 5 stages of 32 KB), warp 1 = MMA
// issuer (leader CTA), warps 2-9 = epilogue (TMEM lane quarter = warp % 4, column half =
// (warp - 2) / 4).  Two TMEM accumulators (2 x 256 columns): a tile's epilogue overlaps the next
// tile's main loop.  Tiles run M-major (consecutive tiles share their A rows in L2).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "eval_common.cuh"
#include "tc_ptx.cuh"

namespace icg {

namespace tg {

#ifndef TG_STAGES
#define TG_STAGES 5
#endif
constexpr int kStages = TG_STAGES;
constexpr uint32_t kATile = 16384;  // 128 rows x 64 fp16
constexpr uint32_t kBTile = 16384;  // up to 128 weight rows x 64 fp16
constexpr uint32_t kStage = kATile + kBTile;
#ifndef TG_EPI_WARPS
#define TG_EPI_WARPS 8
#endif
constexpr int kEpiWarps = TG_EPI_WARPS;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kMaxChunks = 32;
constexpr int kMaxOut = 1024;
// stages | Misc | the layer's epilogue constants (b, w_z, and the output-layer rows of its features)
constexpr uint32_t kMisc = 8192;
constexpr uint32_t kConsts = (2 * kMaxOut + 3 * 256) * 4;  // 11 KB, keeps 1 KB alignment
constexpr uint32_t kStaging = 4096;                           // per epilogue warp: 32 rows x 128 B
constexpr uint32_t kSmem = kStages * kStage + kMisc + kConsts + kEpiWarps * kStaging + 1024;
constexpr int kW5S = kTgW5Stride;  // padded row stride of the fp32 output-layer weights

struct Misc {
    uint64_t full[kStages], empty[kStages];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
    float red[kEpiWarps / 4][128][3];
};
static_assert(sizeof(Misc) <= kMisc, "misc");

struct Params {
    const unsigned* count;  // points (device counter) or nullptr -> n_static
    unsigned n_static;
    int bn;                 // N per tile: 256 or 128
    int n_out;              // output features (multiple of bn)
    int nchunks;            // K chunks of 64
    uint8_t amap[kMaxChunks];   // chunk j: A tensor map (0 = hidden, 1 = skip)
    uint16_t acol[kMaxChunks];  // chunk j: A column (elements)
    const float* bias;      // [b (n_out), w_z (n_out)]
    const float* z;         // per point depth feature
    float slope;
    __half* out;            // fp16 activations out (nullptr: fused output layer)
    int ldo, out_col;
    // fused output-layer terms
    const float* w5;        // final layer fp32 [3][kW5S]: [h4 (128) | Phi | h3 | z | pad]
    int w5_off;             // column of this layer's features in a w5 row (g3: 128 + 256; t4: 0)
    float* sdot;            // per point [3] fp32 output-layer partial sums
    int final_layer;        // t4: rgb = sigmoid(w5 . h4 + sdot)
    float* rgb;
    const uint32_t* out_pixel;
};

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
    __half2 v = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_layer(const __grid_constant__ CUtensorMap mapH, const __grid_constant__ CUtensorMap mapS,
            const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapO,
            const __grid_constant__ Params P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1 KB-aligned base, kept as smem_raw + offset so the compiler sees shared-space accesses
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    Misc& ms = *reinterpret_cast<Misc*>(smem + kStages * kStage);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_rank();
    const bool leader = rank == 0;
    const unsigned pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const unsigned n = P.count ? *P.count : P.n_static;
    const unsigned mt = (n + 255) / 256, nt = (unsigned)(P.n_out / P.bn), ntiles = mt * nt;
    if (pair_id >= ntiles) return;  // both CTAs of a pair agree

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&ms.full[s], 1);
            ptx::mbar_init(&ms.empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&ms.acc_full[a], 1);
            ptx::mbar_init(&ms.acc_empty[a], 2 * kEpiWarps);
        }
        ptx::fence_mbar_init();
    }
    // epilogue constants into shared memory (every epilogue thread reads all of them: broadcast)
    float* cb = reinterpret_cast<float*>(smem + kStages * kStage + kMisc);  // [b | w_z] of the layer
    float* cw5 = cb + 2 * kMaxOut;                                         // [3][256] output-layer terms
    for (int i = threadIdx.x; i < 2 * P.n_out; i += kThreads) cb[i] = __ldg(&P.bias[i]);
    if (P.w5)
        for (int i = threadIdx.x; i < 3 * P.n_out && i < 3 * 256; i += kThreads)
            cw5[i] = __ldg(&P.w5[(i / P.n_out) * kW5S + P.w5_off + i % P.n_out]);
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&mapH);
        ptx::prefetch_tmap(&mapS);
        ptx::prefetch_tmap(&mapW);
        ptx::prefetch_tmap(&mapO);
    }
    if (warp == 1) ptx::tmem_alloc2<512>(&ms.tmem_base);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    // programmatic dependent launch: everything above overlaps the previous layer's tail; its
    // outputs (this layer's A operand, z, sdot) are read only after it has completed
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t tmem = ms.tmem_base;
    const uint32_t full0 = ptx::mapa(ptx::smem_u32(&ms.full[0]), 0);
    const uint32_t acc_empty0 = ptx::mapa(ptx::smem_u32(&ms.acc_empty[0]), 0);
    const uint16_t both = 0x3;
    const int bn = P.bn, nch = P.nchunks;
    const uint32_t btile = (uint32_t)bn / 2 * 128;  // this CTA's weight rows x 128 B

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const uint32_t base = ptx::smem_u32(smem);
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                const int row0 = (int)((t / nt) * 256 + rank * 128);
                const int wrow0 = (int)((t % nt) * (unsigned)bn + rank * (unsigned)bn / 2);
                for (int j = 0; j < nch; ++j) {
                    ptx::mbar_wait(&ms.empty[s], ph ^ 1);
                    if (leader) ptx::mbar_arrive_expect_tx(&ms.full[s], 2 * (kATile + btile));
                    const uint32_t st = base + (uint32_t)s * kStage;
                    ptx::tma_load_2d_2sm(st, P.amap[j] ? (const void*)&mapS : (const void*)&mapH, full0 + s * 8,
                                         (int)P.acol[j], row0);
                    ptx::tma_load_2d_2sm(st + kATile, &mapW, full0 + s * 8, j * 64, wrow0);
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
            // kind::f16 with fp16 A and B (format 0), fp32 D, M = 256, N = bn
            const uint32_t idesc = ptx::idesc_bf16_f32(256, (uint32_t)bn) & ~((7u << 7) | (7u << 10));
            const uint32_t base = ptx::smem_u32(smem);
            int s = 0;
            uint32_t ph = 0, k = 0;
            for (unsigned t = pair_id; t < ntiles; t += npairs, ++k) {
                const uint32_t a = k & 1u;
                if (k >= 2) {
                    ptx::mbar_wait(&ms.acc_empty[a], ((k >> 1) - 1) & 1u);
                    ptx::tc_fence_after();
                }
                const uint32_t d = tmem + a * 256u;
                for (int j = 0; j < nch; ++j) {
                    ptx::mbar_wait(&ms.full[s], ph);
                    ptx::tc_fence_after();
                    const uint32_t st = base + (uint32_t)s * kStage;
                    const uint64_t ad = ptx::sdesc_sw128(st), bd = ptx::sdesc_sw128(st + kATile);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        ptx::mma_bf16_pair(d, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), idesc,
                                           (j > 0 || kk > 0) ? 1u : 0u);
                    ptx::mma_commit_pair(&ms.empty[s], both);
                    if (++s == kStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                ptx::mma_commit_pair(&ms.acc_full[a], both);
            }
        }
    } else {
        // ===================== epilogue: thread = (point row, column half) =====================
        const int quarter = warp & 3, half = (warp - 2) >> 2;  // half: column slice (kEpiWarps / 4 of them)
        const int row = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const int cols = bn / (kEpiWarps / 4);  // this thread's features of the tile
        // output staging of this warp: 32 rows (its TMEM lanes) x 64 features, 128-byte swizzled,
        // written to HBM by one TMA store per 64 features (full 128-byte lines)
        uint8_t* stg = smem + kStages * kStage + kMisc + kConsts + (uint32_t)(warp - 2) * kStaging;
        const uint32_t stg_s = ptx::smem_u32(stg);
        bool stg_busy = false;
        uint32_t k = 0;
        for (unsigned t = pair_id; t < ntiles; t += npairs, ++k) {
            const uint32_t a = k & 1u;
            const unsigned idx = (t / nt) * 256 + rank * 128 + (unsigned)row;
            const int f_tile = (int)(t % nt) * bn;
            const bool valid = idx < n;
            const float z = valid ? __ldg(&P.z[idx]) : 0.0f;
            ptx::mbar_wait(&ms.acc_full[a], (k >> 1) & 1u);
            ptx::tc_fence_after();
            float part[3] = {0.0f, 0.0f, 0.0f};
            const bool dot = P.w5 != nullptr;
            for (int g = 0; g < cols; g += 32) {
                const int fl = half * cols + g;  // feature within the tile
                const int f = f_tile + fl;       // feature within the layer
                uint32_t r[32];
                ptx::tmem_ld32(lane_base + a * 256u + (uint32_t)fl, r);
                float v[32];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const float4 b = reinterpret_cast<const float4*>(cb + f)[q];
                    const float4 w = reinterpret_cast<const float4*>(cb + P.n_out + f)[q];
                    v[4 * q + 0] = fmaf(w.x, z, b.x);
                    v[4 * q + 1] = fmaf(w.y, z, b.y);
                    v[4 * q + 2] = fmaf(w.z, z, b.z);
                    v[4 * q + 3] = fmaf(w.w, z, b.w);
                }
                ptx::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float x = __uint_as_float(r[i]) + v[i];
                    v[i] = fmaxf(x, x * P.slope);  // leaky-ReLU (0 < slope < 1)
                }
                if (dot) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float* wr = cw5 + c * P.n_out + f;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 w = reinterpret_cast<const float4*>(wr)[q];
                            part[c] = fmaf(w.x, v[4 * q], part[c]);
                            part[c] = fmaf(w.y, v[4 * q + 1], part[c]);
                            part[c] = fmaf(w.z, v[4 * q + 2], part[c]);
                            part[c] = fmaf(w.w, v[4 * q + 3], part[c]);
                        }
                    }
                }
                if (P.out) {
                    if ((g & 63) == 0 && stg_busy) {  // the previous store has read the staging rows
                        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        __syncwarp();
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t c16 = (uint32_t)(((g & 63) >> 3) + q);
                        ptx::st_shared_v4(stg_s + (uint32_t)lane * 128u + ((c16 ^ ((uint32_t)lane & 7u)) << 4),
                                          make_uint4(pack_h2(v[8 * q], v[8 * q + 1]), pack_h2(v[8 * q + 2], v[8 * q + 3]),
                                                     pack_h2(v[8 * q + 4], v[8 * q + 5]),
                                                     pack_h2(v[8 * q + 6], v[8 * q + 7])));
                    }
                    if ((g & 63) == 32) {
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            const int x = P.out_col + f - 32, y = (int)(idx - (unsigned)lane);
                            asm volatile(
                                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n\t"
                                "cp.async.bulk.commit_group;" ::"l"(&mapO),
                                "r"(x), "r"(y), "r"(stg_s)
                                : "memory");
                        }
                        stg_busy = true;
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(acc_empty0 + 8u * a);  // the accumulator is free
            if (dot) {
                // the output layer's terms of this layer: both column halves of the point, in order
#pragma unroll
                for (int c = 0; c < 3; ++c) ms.red[half][row][c] = part[c];
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
                if (half == 0 && valid) {
                    float s3[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        float acc = ms.red[0][row][c];
                        for (int h = 1; h < kEpiWarps / 4; ++h) acc += ms.red[h][row][c];
                        s3[c] = acc + P.sdot[3 * (size_t)idx + c];
                    }
                    if (P.final_layer) {
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            float o = 1.0f / (1.0f + expf(-s3[c]));
                            if (P.out_pixel) {
                                o = fminf(fmaxf(o, 0.0f), 1.0f);  // clamp01, render.hpp:276
                                P.rgb[(size_t)P.out_pixel[idx] * 3 + c] = o;
                            } else {
                                P.rgb[(size_t)idx * 3 + c] = o;
                            }
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < 3; ++c) P.sdot[3 * (size_t)idx + c] = s3[c];
                    }
                }
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
            }
        }
    }
    if (warp >= 2 && lane == 0 && P.out) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc2<512>(tmem);
    }
}

// Bilinear taps of one point: input coordinates -> the four tap rows of the H x W x C map and weights.
__device__ __forceinline__ void tap_rows(const FieldDev& f, const float* q, const float*& m00, float* w) {
    float u = (q[0] + 1.0f) * 0.5f * (float)(f.W - 1);
    float v = (1.0f - q[1]) * 0.5f * (float)(f.H - 1);
    u = fminf(fmaxf(u, 0.0f), (float)(f.W - 1));
    v = fminf(fmaxf(v, 0.0f), (float)(f.H - 1));
    const int x0 = min((int)floorf(u), f.W - 2), y0 = min((int)floorf(v), f.H - 2);
    const float ax = u - (float)x0, ay = v - (float)y0;
    w[0] = (1.0f - ax) * (1.0f - ay);
    w[1] = ax * (1.0f - ay);
    w[2] = (1.0f - ax) * ay;
    w[3] = ax * ay;
    m00 = f.fmap_hwc + ((size_t)y0 * f.W + x0) * (size_t)f.C;
}

// lane L's 8 channels {4L..4L+3, 128+4L..128+4L+3}: every 16-byte load of a warp is one contiguous
// 512-byte run of a tap row; both points' 16 loads are issued before either is used
__device__ __forceinline__ void tap_loads(const FieldDev& f, const float* m00, int c0, float4* tv) {
    const size_t rowW = (size_t)f.W * f.C;
    const float* taps[4] = {m00, m00 + f.C, m00 + rowW, m00 + rowW + f.C};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        tv[2 * t] = __ldg(reinterpret_cast<const float4*>(taps[t] + c0));
        tv[2 * t + 1] = __ldg(reinterpret_cast<const float4*>(taps[t] + c0 + 128));
    }
}

__device__ __forceinline__ void tap_blend(const float4* tv, const float* w, float* val) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const float4 a0 = tv[h], a1 = tv[2 + h], a2 = tv[4 + h], a3 = tv[6 + h];
        val[4 * h + 0] = w[0] * a0.x + w[1] * a1.x + w[2] * a2.x + w[3] * a3.x;
        val[4 * h + 1] = w[0] * a0.y + w[1] * a1.y + w[2] * a2.y + w[3] * a3.y;
        val[4 * h + 2] = w[0] * a0.z + w[1] * a1.z + w[2] * a2.z + w[3] * a3.z;
        val[4 * h + 3] = w[0] * a0.w + w[1] * a1.w + w[2] * a2.w + w[3] * a3.w;
    }
}

// Per point (one warp, two points per step): world point -> input coordinates, Phi bilinear in
// fp32 (lane = 8 channels), fp16 into the skip row [Phi | h3], z, and the output layer's Phi and z
// terms + b5 (fp32).
__global__ void __launch_bounds__(256) k_gather(FieldDev f, EvalJob job, __half* skip, float* zbuf, float* sdot,
                                                const float* w5, const float* b5) {
    const unsigned n = job_count(job);
    if (blockIdx.x == 0 && threadIdx.x == 0) job_account(job);
    const int lane = threadIdx.x & 31;
    const unsigned warp_g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    const int c0 = 4 * lane;
    float w5s[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int i = 0; i < 8; ++i) w5s[c][i] = __ldg(&w5[c * kW5S + 128 + c0 + (i & 3) + (i >> 2) * 128]);
    for (unsigned i0 = warp_g; i0 < n; i0 += 2 * nwarps) {
        unsigned idx[2] = {i0, i0 + nwarps};
        float q[2][3], w[2][4];
        float4 tv[2][8];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            if (idx[p] >= n) continue;
            double pd[3];
            field_point_d(f, job, idx[p], pd);
            const float pw[3] = {(float)pd[0], (float)pd[1], (float)pd[2]};
            input_coords(f, pw, q[p]);
            const float* m00;
            tap_rows(f, q[p], m00, w[p]);
            tap_loads(f, m00, c0, tv[p]);
        }
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            if (idx[p] >= n) continue;
            float val[8];
            tap_blend(tv[p], w[p], val);
            __half* row = skip + (size_t)idx[p] * 512;
            *reinterpret_cast<uint2*>(row + c0) = make_uint2(pack_h2(val[0], val[1]), pack_h2(val[2], val[3]));
            *reinterpret_cast<uint2*>(row + 128 + c0) = make_uint2(pack_h2(val[4], val[5]), pack_h2(val[6], val[7]));
            float dot[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                dot[c] = 0.0f;
#pragma unroll
                for (int i = 0; i < 8; ++i) dot[c] = fmaf(w5s[c][i], val[i], dot[c]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) dot[c] += __shfl_xor_sync(0xffffffffu, dot[c], o);
            }
            if (lane == 0) {
                zbuf[idx[p]] = q[p][2];
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    sdot[3 * (size_t)idx[p] + c] =
                        dot[c] + fmaf(__ldg(&w5[c * kW5S + 128 + kTexSkip - 1]), q[p][2], __ldg(&b5[c]));
            }
        }
    }
}

}  // namespace tg

// 2D tiled tensor map (one encoder for every TMA descriptor of the library): element type `dtype`
// (CUtensorMapDataType), row pitch row_bytes, boxes of box_cols x box_rows, swizzle (CUtensorMapSwizzle)
int make_tmap_2d(const void* base, int dtype, size_t rows, size_t cols, size_t row_bytes, unsigned box_cols,
                 unsigned box_rows, int swizzle, void* out) {
    static std::once_flag once;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess && fn &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!encode) {
        set_error("cuTensorMapEncodeTiled not available");
        return ICG_ERUNTIME;
    }
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(reinterpret_cast<CUtensorMap*>(out), (CUtensorMapDataType)dtype, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)swizzle,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
        return ICG_ERUNTIME;
    }
    return ICG_OK;
}

// fp16 row-major [rows][cols] tensor map, boxes of 64 columns x box_rows rows, 128-byte swizzle
int tg_make_tmap(const void* base, size_t rows, size_t cols, unsigned box_rows, void* out) {
    return make_tmap_2d(base, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rows, cols, cols * 2, 64, box_rows,
                        CU_TENSOR_MAP_SWIZZLE_128B, out);
}

// fp16 weights of the texture chain, row-major [n_out][K] with K ordered like the layer's A chunks:
// [hidden | Phi (| h3)], the z column left out (it enters the epilogue in fp32).  Layer order
// g1 g2 g3 t1 t2 t3 t4; returns the element offsets of each layer in `off`.
size_t tg_weight_elems() {
    const int gk[3] = {256, 1024 + 256, 512 + 256}, go[3] = {1024, 512, 256};
    const int tk[4] = {512, 1024 + 512, 512 + 512, 256 + 512}, to[4] = {1024, 512, 256, 128};
    size_t e = 0;
    for (int l = 0; l < 3; ++l) e += (size_t)gk[l] * go[l];
    for (int l = 0; l < 4; ++l) e += (size_t)tk[l] * to[l];
    return e;
}

int tg_pack_weights(const float* const* gw, const float* const* tw, __half* dst, size_t* off) {
    size_t e = 0;
    int li = 0;
    for (int net = 0; net < 2; ++net) {
        const float* const* w = net ? tw : gw;
        const int skip = net ? kTexSkip : kGeoSkip;
        const int* outs = net ? kTexOut : kGeoOut;
        for (int l = 0; l < (net ? 4 : 3); ++l) {
            const int prev = l ? outs[l - 1] : 0, in = prev + skip, K = in - 1, O = outs[l];
            off[li++] = e;
            for (int o = 0; o < O; ++o)
                for (int k = 0; k < K; ++k) dst[e + (size_t)o * K + k] = __float2half_rn(w[l][(size_t)o * in + k]);
            e += (size_t)O * K;
        }
    }
    return e == tg_weight_elems() ? ICG_OK : ICG_ERUNTIME;
}

int launch_tex_gather(const FieldDev& f, const EvalJob& job, unsigned max_points, __half* skip, float* z, float* sdot,
                      const float* w5, const float* b5, cudaStream_t s) {
    unsigned blocks = (max_points + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks == 0) blocks = 1;
    tg::k_gather<<<blocks, 256, 0, s>>>(f, job, skip, z, sdot, w5, b5);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// one layer: A chunks = `hid` chunks of the hidden map, then skip chunks [s0, s1) of the skip map
int launch_tex_layer(const void* mapH, const void* mapS, const void* mapW, const void* mapO, const TgLayer& L,
                     unsigned max_points, cudaStream_t s) {
    static PerDeviceOnce once;
    if (int r = once.run([] {
            ICG_CUDA_TRY(cudaFuncSetAttribute(tg::k_layer, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tg::kSmem));
            return ICG_OK;
        }))
        return r;
    tg::Params p{};
    p.count = L.count;
    p.n_static = L.n_static;
    p.bn = L.n_out >= 256 ? 256 : L.n_out;
    p.n_out = L.n_out;
    int j = 0;
    for (int c = 0; c < L.hid_chunks; ++c, ++j) {
        p.amap[j] = 0;
        p.acol[j] = (uint16_t)(64 * c);
    }
    for (int c = L.skip_c0; c < L.skip_c1; ++c, ++j) {
        p.amap[j] = 1;
        p.acol[j] = (uint16_t)(64 * c);
    }
    if (j > tg::kMaxChunks) {
        set_error("texture layer: too many K chunks");
        return ICG_ERUNTIME;
    }
    p.nchunks = j;
    p.bias = L.bias;
    p.z = L.z;
    p.slope = L.slope;
    p.out = L.out;
    p.ldo = L.ldo;
    p.out_col = L.out_col;
    p.w5 = L.w5;
    p.w5_off = L.w5_off;
    p.sdot = L.sdot;
    p.final_layer = L.final_layer;
    p.rgb = L.rgb;
    p.out_pixel = L.out_pixel;
    const unsigned tiles = (max_points + 255) / 256 * (unsigned)(L.n_out / p.bn);
    unsigned pairs = tiles < 74 ? tiles : 74;
    if (pairs == 0) pairs = 1;
    CUtensorMap h, sk, w, o;
    std::memcpy(&h, mapH, sizeof(CUtensorMap));
    std::memcpy(&sk, mapS, sizeof(CUtensorMap));
    std::memcpy(&w, mapW, sizeof(CUtensorMap));
    std::memcpy(&o, mapO, sizeof(CUtensorMap));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(tg::kThreads);
    cfg.dynamicSmemBytes = tg::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = L.pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ICG_CUDA_TRY(cudaLaunchKernelEx(&cfg, tg::k_layer, h, sk, w, o, p));
    if (const cudaError_t e = cudaGetLastError()) {
        set_error(std::string("k_layer (texture GEMM): ") + cudaGetErrorString(e));
        return ICG_ERUNTIME;
    }
    return ICG_OK;
}


// ============================================================================================
// Column pass of the column-factored geometry field as one GEMM (replaces k_mlp_pair<COLS>):
// records[slot] = W_Phi . Phi(column) for the Phi columns of layers 1-4 (1920 outputs), with
// M = 256 columns x N = 256 outputs per CTA-pair tile, K = the 256 Phi channels, bf16x3 (A and
// B as bf16 hi + lo, three MMAs per K step: fp32-accurate) or bf16.  The output layer's Phi dot
// (record column 1920) is an fp32 dot in the gather.  Records are written by TMA bulk stores of
// 32 x 32 fp32 boxes from per-warp swizzled staging.
// ============================================================================================
namespace cg {

constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kTile = 16384;  // 128 rows x 64 bf16
constexpr int kNOut = 1920;        // record columns computed by the GEMM (layers 1-4)
constexpr int kNTiles = 8;         // 2048 weight rows (the last 128 zero)
constexpr uint32_t kStaging = 4096;  // per epilogue warp: 32 rows x 32 fp32
template <bool X3>
struct Cfg {
    static constexpr int kStages = X3 ? 3 : 5;
    static constexpr uint32_t kStage = (X3 ? 4 : 2) * kTile;  // A hi (lo), B hi (lo)
    static constexpr uint32_t kSmem = kStages * kStage + 1024 + kEpiWarps * kStaging + 1024;
};

struct Misc {
    uint64_t full[5], empty[5];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};

struct Params {
    const unsigned* count;  // list entries [*base, *count) (count null: n_static)
    const unsigned* base;
    unsigned n_static;
};

template <bool X3>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_cols(const __grid_constant__ CUtensorMap mapAh, const __grid_constant__ CUtensorMap mapAl,
           const __grid_constant__ CUtensorMap mapWh, const __grid_constant__ CUtensorMap mapWl,
           const __grid_constant__ CUtensorMap mapR, const __grid_constant__ Params P) {
    using C = Cfg<X3>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    Misc& ms = *reinterpret_cast<Misc*>(smem + C::kStages * C::kStage);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_rank();
    const bool leader = rank == 0;
    const unsigned pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const unsigned base = P.base ? *P.base : 0u;
    const unsigned cnt = P.count ? *P.count : P.n_static;
    const unsigned n = cnt > base ? cnt - base : 0u;
    const unsigned mt = (n + 255) / 256, ntiles = mt * kNTiles;
    if (pair_id >= ntiles) return;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&ms.full[s], 1);
            ptx::mbar_init(&ms.empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&ms.acc_full[a], 1);
            ptx::mbar_init(&ms.acc_empty[a], 2 * kEpiWarps);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&mapAh);
        ptx::prefetch_tmap(&mapWh);
        ptx::prefetch_tmap(&mapR);
        if (X3) {
            ptx::prefetch_tmap(&mapAl);
            ptx::prefetch_tmap(&mapWl);
        }
    }
    if (warp == 1) ptx::tmem_alloc2<512>(&ms.tmem_base);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = ms.tmem_base;
    const uint32_t full0 = ptx::mapa(ptx::smem_u32(&ms.full[0]), 0);
    const uint32_t acc_empty0 = ptx::mapa(ptx::smem_u32(&ms.acc_empty[0]), 0);
    const uint16_t both = 0x3;

    if (warp == 0) {
        // ===================== TMA producer (both CTAs) =====================
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            const uint32_t sbase = ptx::smem_u32(smem);
            for (unsigned t = pair_id; t < ntiles; t += npairs) {
                const int row0 = (int)((t / kNTiles) * 256 + rank * 128);
                const int wrow0 = (int)((t % kNTiles) * 256 + rank * 128);
                for (int j = 0; j < 4; ++j) {
                    ptx::mbar_wait(&ms.empty[s], ph ^ 1);
                    if (leader) ptx::mbar_arrive_expect_tx(&ms.full[s], 2 * C::kStage);
                    const uint32_t st = sbase + (uint32_t)s * C::kStage;
                    ptx::tma_load_2d_2sm(st, &mapAh, full0 + s * 8, j * 64, row0);
                    ptx::tma_load_2d_2sm(st + kTile, &mapWh, full0 + s * 8, j * 64, wrow0);
                    if (X3) {
                        ptx::tma_load_2d_2sm(st + 2 * kTile, &mapAl, full0 + s * 8, j * 64, row0);
                        ptx::tma_load_2d_2sm(st + 3 * kTile, &mapWl, full0 + s * 8, j * 64, wrow0);
                    }
                    if (++s == C::kStages) {
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
            const uint32_t sbase = ptx::smem_u32(smem);
            int s = 0;
            uint32_t ph = 0, k = 0;
            for (unsigned t = pair_id; t < ntiles; t += npairs, ++k) {
                const uint32_t a = k & 1u;
                if (k >= 2) {
                    ptx::mbar_wait(&ms.acc_empty[a], ((k >> 1) - 1) & 1u);
                    ptx::tc_fence_after();
                }
                const uint32_t d = tmem + a * 256u;
                for (int j = 0; j < 4; ++j) {
                    ptx::mbar_wait(&ms.full[s], ph);
                    ptx::tc_fence_after();
                    const uint32_t st = sbase + (uint32_t)s * C::kStage;
                    const uint64_t ah = ptx::sdesc_sw128(st), bh = ptx::sdesc_sw128(st + kTile);
                    const uint64_t al = ptx::sdesc_sw128(st + 2 * kTile), bl = ptx::sdesc_sw128(st + 3 * kTile);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t ko = (uint64_t)(kk * 2);
                        ptx::mma_bf16_pair(d, ah + ko, bh + ko, idesc, (j > 0 || kk > 0) ? 1u : 0u);
                        if (X3) {
                            ptx::mma_bf16_pair(d, al + ko, bh + ko, idesc, 1u);
                            ptx::mma_bf16_pair(d, ah + ko, bl + ko, idesc, 1u);
                        }
                    }
                    ptx::mma_commit_pair(&ms.empty[s], both);
                    if (++s == C::kStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                ptx::mma_commit_pair(&ms.acc_full[a], both);
            }
        }
    } else {
        // ===================== epilogue: raw fp32 records through TMA stores =====================
        const int quarter = warp & 3, half = (warp - 2) >> 2;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        uint8_t* stg = smem + C::kStages * C::kStage + 1024 + (uint32_t)(warp - 2) * kStaging;
        const uint32_t stg_s = ptx::smem_u32(stg);
        bool busy = false;
        uint32_t k = 0;
        for (unsigned t = pair_id; t < ntiles; t += npairs, ++k) {
            const uint32_t a = k & 1u;
            const int y = (int)(base + (t / kNTiles) * 256 + rank * 128 + (unsigned)quarter * 32);
            const int f_tile = (int)(t % kNTiles) * 256;
            ptx::mbar_wait(&ms.acc_full[a], (k >> 1) & 1u);
            ptx::tc_fence_after();
            for (int g = 0; g < 128; g += 32) {
                const int fl = half * 128 + g, f = f_tile + fl;
                uint32_t r[32];
                ptx::tmem_ld32(lane_base + a * 256u + (uint32_t)fl, r);
                if (busy) {  // the previous box has been read out of the staging rows
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                }
                ptx::tmem_ld_wait();
                if (f < kNOut) {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        ptx::st_shared_v4(stg_s + (uint32_t)lane * 128u + ((((uint32_t)q) ^ ((uint32_t)lane & 7u)) << 4),
                                          make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]));
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n\t"
                            "cp.async.bulk.commit_group;" ::"l"(&mapR),
                            "r"(f), "r"(y), "r"(stg_s)
                            : "memory");
                    busy = true;
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(acc_empty0 + 8u * a);
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc2<512>(tmem);
    }
}

__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// Per column (one warp): Phi at the column's (x, y), bf16 hi (+ lo) rows of the GEMM's A operand,
// and the output layer's Phi dot (fp32) into the record (same arithmetic as k_mlp_pair<COLS>).
template <bool X3>
__global__ void __launch_bounds__(256) k_cols_gather(FieldDev f, EvalJob cj, __nv_bfloat16* ah, __nv_bfloat16* al,
                                                     float* records, const float* wlast) {
    const unsigned base = cj.base ? *cj.base : 0u;
    const unsigned cnt = job_count(cj);
    const unsigned n = cnt > base ? cnt - base : 0u;
    const int lane = threadIdx.x & 31;
    const unsigned warp_g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    const int c0 = 4 * lane;  // channels {c0..c0+3, 128+c0..128+c0+3} (tg::tap_loads)
    float w5s[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w5s[i] = __ldg(&wlast[128 + c0 + (i & 3) + (i >> 2) * 128]);
    for (unsigned i0 = warp_g; i0 < n; i0 += 2 * nwarps) {
        const unsigned idx[2] = {i0, i0 + nwarps};
        float w[2][4];
        float4 tv[2][8];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            if (idx[p] >= n) continue;
            double pd[3];
            node_pos_d(job_node(cj, base + idx[p]), cj.cells, pd);
            const float pw[3] = {(float)pd[0], (float)pd[1], (float)pd[2]};
            float q[3];
            input_coords(f, pw, q);
            const float* m00;
            tg::tap_rows(f, q, m00, w[p]);
            tg::tap_loads(f, m00, c0, tv[p]);
        }
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            if (idx[p] >= n) continue;
            float val[8];
            tg::tap_blend(tv[p], w[p], val);
            uint32_t hp[4], lp[4];
            float dot = 0.0f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float a = val[2 * i], b = val[2 * i + 1];
                hp[i] = pack_bf2(a, b);
                lp[i] = pack_bf2(a - __uint_as_float(hp[i] << 16), b - __uint_as_float(hp[i] & 0xFFFF0000u));
                dot = fmaf(w5s[2 * i], a, dot);
                dot = fmaf(w5s[2 * i + 1], b, dot);
            }
            __nv_bfloat16* rh = ah + (size_t)idx[p] * 256;
            *reinterpret_cast<uint2*>(rh + c0) = make_uint2(hp[0], hp[1]);
            *reinterpret_cast<uint2*>(rh + 128 + c0) = make_uint2(hp[2], hp[3]);
            if (X3) {
                __nv_bfloat16* rl = al + (size_t)idx[p] * 256;
                *reinterpret_cast<uint2*>(rl + c0) = make_uint2(lp[0], lp[1]);
                *reinterpret_cast<uint2*>(rl + 128 + c0) = make_uint2(lp[2], lp[3]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            if (lane == 0) records[(size_t)(base + idx[p]) * kColRecord + 1920] = dot;
        }
    }
}

}  // namespace cg

// bf16 weights of the column GEMM: rows [layer-1 Phi part (1024) | layer 2 (512) | layer 3 (256) |
// layer 4 (128) | zero (128)] x the 256 Phi channels, as hi and lo
int cg_pack_weights(const float* const* w, __nv_bfloat16* hi, __nv_bfloat16* lo) {
    const int outs[4] = {1024, 512, 256, 128};
    int row = 0;
    for (int l = 0; l < 4; ++l) {
        const int prev = l ? outs[l - 1] : 0, in = prev + kGeoSkip;
        for (int o = 0; o < outs[l]; ++o, ++row)
            for (int k = 0; k < 256; ++k) {
                const float v = w[l][(size_t)o * in + prev + k];
                const __nv_bfloat16 h = __float2bfloat16_rn(v);
                hi[(size_t)row * 256 + k] = h;
                lo[(size_t)row * 256 + k] = __float2bfloat16_rn(v - __bfloat162float(h));
            }
    }
    for (; row < 2048; ++row)
        for (int k = 0; k < 256; ++k) {
            hi[(size_t)row * 256 + k] = __float2bfloat16_rn(0.0f);
            lo[(size_t)row * 256 + k] = __float2bfloat16_rn(0.0f);
        }
    return ICG_OK;
}

// bf16 (or fp32) row-major tensor map, boxes of box_cols x box_rows, 128-byte swizzle
int cg_make_tmap(const void* base, size_t rows, size_t cols, size_t row_bytes, unsigned box_cols, unsigned box_rows,
                 bool f32, void* out) {
    return make_tmap_2d(base, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rows, cols,
                        row_bytes, box_cols, box_rows, CU_TENSOR_MAP_SWIZZLE_128B, out);
}

// column records of the list window of `cj` (max_cols entries at most): gather + GEMM
int launch_cols_gemm(const FieldDev& f, const EvalJob& cj, const float* wlast, __nv_bfloat16* ah, __nv_bfloat16* al,
                     float* records, const void* mapAh, const void* mapAl, const void* mapWh, const void* mapWl,
                     const void* mapR, unsigned max_cols, bool x3, cudaStream_t s) {
    static PerDeviceOnce once;
    if (int r = once.run([] {
            ICG_CUDA_TRY(cudaFuncSetAttribute(cg::k_cols<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)cg::Cfg<true>::kSmem));
            ICG_CUDA_TRY(cudaFuncSetAttribute(cg::k_cols<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)cg::Cfg<false>::kSmem));
            return ICG_OK;
        }))
        return r;
    unsigned blocks = (max_cols + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks == 0) blocks = 1;
    if (x3)
        cg::k_cols_gather<true><<<blocks, 256, 0, s>>>(f, cj, ah, al, records, wlast);
    else
        cg::k_cols_gather<false><<<blocks, 256, 0, s>>>(f, cj, ah, al, records, wlast);
    ICG_CUDA_TRY(cudaGetLastError());
    cg::Params p{};
    p.count = cj.count;
    p.base = cj.base;
    p.n_static = cj.n_static;
    const unsigned tiles = (max_cols + 255) / 256 * cg::kNTiles;
    unsigned pairs = tiles < 74 ? tiles : 74;
    if (pairs == 0) pairs = 1;
    CUtensorMap a0, a1, w0, w1, rr;
    std::memcpy(&a0, mapAh, sizeof(CUtensorMap));
    std::memcpy(&a1, mapAl, sizeof(CUtensorMap));
    std::memcpy(&w0, mapWh, sizeof(CUtensorMap));
    std::memcpy(&w1, mapWl, sizeof(CUtensorMap));
    std::memcpy(&rr, mapR, sizeof(CUtensorMap));
    if (x3)
        cg::k_cols<true><<<2 * pairs, cg::kThreads, cg::Cfg<true>::kSmem, s>>>(a0, a1, w0, w1, rr, p);
    else
        cg::k_cols<false><<<2 * pairs, cg::kThreads, cg::Cfg<false>::kSmem, s>>>(a0, a1, w0, w1, rr, p);
    if (const cudaError_t e = cudaGetLastError()) {
        set_error(std::string("k_cols: ") + cudaGetErrorString(e));
        return ICG_ERUNTIME;
    }
    return ICG_OK;
}

}  // namespace icg

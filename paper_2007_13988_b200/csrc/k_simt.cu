// k_simt.cu — CUDA-core fp32 PIFu field (ICG_PREC_FP32_SIMT): the
// correctness cross-check for the tcgen05 path, and the feature-map layout pass.
//
// Per CTA tile of 16 points: pixel-aligned feature sampling Phi (bilinear over
// an H x W x C map: one thread per channel, so every tap of a point is one
// coalesced 1 KB row), then the skip-concat MLP with fp32 FFMA accumulation,
// activations resident in shared memory.  Geometry: 257->1024->512->256->128->1
// (+ bias - sdf_scale*sdf(P), sigmoid).  Texture: geometry layers 1-3 give h3,
// then 513->1024->512->256->128->3 over [Phi, h3, z], sigmoid.
#include "eval_common.cuh"

namespace icg {

constexpr int TP = 16;   // points per tile
constexpr int NT = 256;  // threads per CTA
constexpr int kFS = 272; // geometry skip stride (257 padded)
constexpr int kTS = 528; // texture skip stride (513 padded)

// ---- feature map CHW -> HWC ---------------------------------------------
__global__ void k_chw_to_hwc(const float* __restrict__ chw, float* __restrict__ hwc, int C, int HW) {
    __shared__ float tile[32][33];
    int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        int c = c0 + r, p = p0 + tx;
        tile[r][tx] = (c < C && p < HW) ? chw[(size_t)c * HW + p] : 0.0f;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        int p = p0 + r, c = c0 + tx;
        if (c < C && p < HW) hwc[(size_t)p * C + c] = tile[tx][r];
    }
}

// 64 x 64 tiles, 8-byte loads and stores (C and H*W multiples of 64, 8-byte aligned maps)
__global__ void __launch_bounds__(256) k_chw_to_hwc64(const float* __restrict__ chw, float* __restrict__ hwc, int C,
                                                      int HW) {
    __shared__ float tile[64][65];
    const int p0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
#pragma unroll
    for (int r = ty; r < 64; r += 8) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(chw + (size_t)(c0 + r) * HW + p0 + 2 * tx));
        tile[r][2 * tx] = v.x;
        tile[r][2 * tx + 1] = v.y;
    }
    __syncthreads();
#pragma unroll
    for (int r = ty; r < 64; r += 8)
        *reinterpret_cast<float2*>(hwc + (size_t)(p0 + r) * C + c0 + 2 * tx) = make_float2(tile[2 * tx][r], tile[2 * tx + 1][r]);
}

int launch_fmap_chw_to_hwc(const float* chw, float* hwc, int C, int H, int W, cudaStream_t s) {
    int HW = H * W;
    if (C % 64 == 0 && HW % 64 == 0 && !((uintptr_t)chw & 7u) && !((uintptr_t)hwc & 7u)) {
        k_chw_to_hwc64<<<dim3(HW / 64, C / 64), dim3(32, 8), 0, s>>>(chw, hwc, C, HW);
        ICG_CUDA_TRY(cudaGetLastError());
        return ICG_OK;
    }
    dim3 grid((HW + 31) / 32, (C + 31) / 32), block(32, 8);
    k_chw_to_hwc<<<grid, block, 0, s>>>(chw, hwc, C, HW);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// ---- Phi: bilinear sample of all channels at P_xy ------------------------
// u = (x+1)/2 (W-1), v = (1-y)/2 (H-1): align-corners, image row 0 at y = +1.
__device__ __forceinline__ void sample_setup(const FieldDev& f, float x, float y, size_t& o00, float* w) {
    float u = (x + 1.0f) * 0.5f * (float)(f.W - 1);
    float v = (1.0f - y) * 0.5f * (float)(f.H - 1);
    u = fminf(fmaxf(u, 0.0f), (float)(f.W - 1));
    v = fminf(fmaxf(v, 0.0f), (float)(f.H - 1));
    int x0 = min((int)floorf(u), f.W - 2), y0 = min((int)floorf(v), f.H - 2);
    float ax = u - (float)x0, ay = v - (float)y0;
    w[0] = (1.0f - ax) * (1.0f - ay);
    w[1] = ax * (1.0f - ay);
    w[2] = (1.0f - ax) * ay;
    w[3] = ax * ay;
    o00 = ((size_t)y0 * f.W + x0) * (size_t)f.C;
}

// one dense layer: hout[p][o] = act(b[o] + sum_k Wt[k][o] * [hin, skip][p][k])
template <int R>
__device__ __forceinline__ void simt_layer(const float* __restrict__ Wt, const float* __restrict__ bias, int Kh,
                                           int Ks, int O, const float* hin, int hin_stride, const float* skip,
                                           int skip_stride, float* hout, int hout_stride, bool leaky, float slope) {
    const int t = threadIdx.x;
    float acc[R][TP];
    int o[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        o[r] = t + r * NT;
        float b = o[r] < O ? bias[o[r]] : 0.0f;
#pragma unroll
        for (int p = 0; p < TP; ++p) acc[r][p] = b;
    }
    for (int k = 0; k < Kh; ++k) {
        float w[R];
#pragma unroll
        for (int r = 0; r < R; ++r) w[r] = o[r] < O ? __ldg(&Wt[(size_t)k * O + o[r]]) : 0.0f;
#pragma unroll
        for (int p = 0; p < TP; ++p) {
            float x = hin[p * hin_stride + k];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r][p] = fmaf(w[r], x, acc[r][p]);
        }
    }
    for (int k = 0; k < Ks; ++k) {
        float w[R];
#pragma unroll
        for (int r = 0; r < R; ++r) w[r] = o[r] < O ? __ldg(&Wt[(size_t)(Kh + k) * O + o[r]]) : 0.0f;
#pragma unroll
        for (int p = 0; p < TP; ++p) {
            float x = skip[p * skip_stride + k];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r][p] = fmaf(w[r], x, acc[r][p]);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (o[r] >= O) continue;
#pragma unroll
        for (int p = 0; p < TP; ++p) {
            float v = acc[r][p];
            if (leaky && v < 0.0f) v *= slope;
            hout[p * hout_stride + o[r]] = v;
        }
    }
}

__device__ __forceinline__ void run_layer(const SimtMlp& m, int l, const float* hin, int hin_stride,
                                          const float* skip, int skip_stride, float* hout, int hout_stride) {
    int Kh = l ? m.out[l - 1] : 0;
    int O = m.out[l];
    if (O > 2 * NT)
        simt_layer<4>(m.wt[l], m.b[l], Kh, m.skip, O, hin, hin_stride, skip, skip_stride, hout, hout_stride, true, m.slope);
    else if (O > NT)
        simt_layer<2>(m.wt[l], m.b[l], Kh, m.skip, O, hin, hin_stride, skip, skip_stride, hout, hout_stride, true, m.slope);
    else
        simt_layer<1>(m.wt[l], m.b[l], Kh, m.skip, O, hin, hin_stride, skip, skip_stride, hout, hout_stride, true, m.slope);
}

// Final narrow layer (1 or 3 outputs): one warp per (point, output) dot product.
__device__ __forceinline__ void last_layer(const SimtMlp& m, const float* hin, int hin_stride, const float* skip,
                                           int skip_stride, float* out /* [TP][4] */) {
    const int l = 4, O = m.out[4], Kh = m.out[3], K = Kh + m.skip;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int job = warp; job < TP * O; job += NT / 32) {
        int p = job / O, c = job % O;
        float acc = 0.0f;
        for (int k = lane; k < K; k += 32) {
            float x = k < Kh ? hin[p * hin_stride + k] : skip[p * skip_stride + (k - Kh)];
            acc = fmaf(__ldg(&m.wt[l][(size_t)k * O + c]), x, acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[p * 4 + c] = acc + m.b[l][c];
    }
}

struct SimtSmem {
    float f[TP][kFS];
    float hA[TP][1024];
    float hB[TP][512];
    float pos[TP][3];
    double posd[TP][3];
    float outv[TP][4];
};

__device__ void load_tile(const FieldDev& f, const EvalJob& job, unsigned base, unsigned n, SimtSmem& sm) {
    if (threadIdx.x < TP) {
        unsigned t = base + threadIdx.x;
        double p[3] = {0.0, 0.0, 0.0};
        if (t < n) field_point_d(f, job, t, p);
        const float pw[3] = {(float)p[0], (float)p[1], (float)p[2]};
        float q[3];
        input_coords(f, pw, q);  // Phi at q.xy, depth feature q.z; the sdf bias at the world point
        for (int d = 0; d < 3; ++d) {
            sm.posd[threadIdx.x][d] = p[d];
            sm.pos[threadIdx.x][d] = q[d];
        }
    }
    __syncthreads();
    // Phi + z into the skip buffer; thread = channel (C == 256 == NT)
    for (int p = 0; p < TP; ++p) {
        size_t o00;
        float w[4];
        sample_setup(f, sm.pos[p][0], sm.pos[p][1], o00, w);
        const float* m = f.fmap_hwc;
        size_t rowW = (size_t)f.W * f.C;
        for (int c = threadIdx.x; c < f.C; c += NT) {
            float v = w[0] * __ldg(&m[o00 + c]) + w[1] * __ldg(&m[o00 + f.C + c]) + w[2] * __ldg(&m[o00 + rowW + c]) +
                      w[3] * __ldg(&m[o00 + rowW + f.C + c]);
            sm.f[p][c] = v;
        }
        if (threadIdx.x < kFS - kC) sm.f[p][kC + threadIdx.x] = threadIdx.x == 0 ? sm.pos[p][2] : 0.0f;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(NT, 1) k_pifu_simt_eval(FieldDev f, SimtMlp geo, EvalJob job) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    SimtSmem& sm = *reinterpret_cast<SimtSmem*>(smem_raw);
    __shared__ DevScene scene;
    if (blockIdx.x * TP >= job_count(job)) {
        job_account(job);
        return;
    }
    for (int i = threadIdx.x; i < (int)(sizeof(DevScene) / 8); i += blockDim.x)
        reinterpret_cast<double*>(&scene)[i] = reinterpret_cast<const double*>(f.scene)[i];
    __syncthreads();
    job_account(job);
    unsigned n = job_count(job);
    for (unsigned base = blockIdx.x * TP; base < n; base += gridDim.x * TP) {
        load_tile(f, job, base, n, sm);
        run_layer(geo, 0, nullptr, 0, &sm.f[0][0], kFS, &sm.hA[0][0], 1024);
        __syncthreads();
        run_layer(geo, 1, &sm.hA[0][0], 1024, &sm.f[0][0], kFS, &sm.hB[0][0], 512);
        __syncthreads();
        run_layer(geo, 2, &sm.hB[0][0], 512, &sm.f[0][0], kFS, &sm.hA[0][0], 1024);
        __syncthreads();
        run_layer(geo, 3, &sm.hA[0][0], 1024, &sm.f[0][0], kFS, &sm.hB[0][0], 512);
        __syncthreads();
        last_layer(geo, &sm.hB[0][0], 512, &sm.f[0][0], kFS, &sm.outv[0][0]);
        __syncthreads();
        if (threadIdx.x < TP) {
            unsigned t = base + threadIdx.x;
            if (t < n) {
                double sdf = scene_sdf(scene, sm.posd[threadIdx.x]);
                float logit = sm.outv[threadIdx.x][0] + (float)(-scene.sdf_scale * sdf);
                float v = 1.0f / (1.0f + expf(-logit));
                if (job_is_grid(job))
                    grid_epilogue(job, job_node(job, t), v);
                else
                    job.out[t] = v;
            }
        }
        __syncthreads();
    }
}

struct SimtTexSmem {
    SimtSmem g;
    float t[TP][kTS];
};

__global__ void __launch_bounds__(NT, 1) k_pifu_simt_texture(FieldDev f, SimtMlp geo, SimtMlp tex, EvalJob job) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    SimtTexSmem& sm = *reinterpret_cast<SimtTexSmem*>(smem_raw);
    unsigned n = job_count(job);
    for (unsigned base = blockIdx.x * TP; base < n; base += gridDim.x * TP) {
        load_tile(f, job, base, n, sm.g);
        // geometry prefix: layers 1-3 -> h3 (256-d)
        run_layer(geo, 0, nullptr, 0, &sm.g.f[0][0], kFS, &sm.g.hA[0][0], 1024);
        __syncthreads();
        run_layer(geo, 1, &sm.g.hA[0][0], 1024, &sm.g.f[0][0], kFS, &sm.g.hB[0][0], 512);
        __syncthreads();
        run_layer(geo, 2, &sm.g.hB[0][0], 512, &sm.g.f[0][0], kFS, &sm.t[0][kC], kTS);
        // texture skip = [Phi (256), h3 (256), z, pad]
        for (int p = 0; p < TP; ++p) {
            for (int c = threadIdx.x; c < kC; c += NT) sm.t[p][c] = sm.g.f[p][c];
            if (threadIdx.x < kTS - 2 * kC) sm.t[p][2 * kC + threadIdx.x] = threadIdx.x == 0 ? sm.g.pos[p][2] : 0.0f;
        }
        __syncthreads();
        run_layer(tex, 0, nullptr, 0, &sm.t[0][0], kTS, &sm.g.hA[0][0], 1024);
        __syncthreads();
        run_layer(tex, 1, &sm.g.hA[0][0], 1024, &sm.t[0][0], kTS, &sm.g.hB[0][0], 512);
        __syncthreads();
        run_layer(tex, 2, &sm.g.hB[0][0], 512, &sm.t[0][0], kTS, &sm.g.hA[0][0], 1024);
        __syncthreads();
        run_layer(tex, 3, &sm.g.hA[0][0], 1024, &sm.t[0][0], kTS, &sm.g.hB[0][0], 512);
        __syncthreads();
        last_layer(tex, &sm.g.hB[0][0], 512, &sm.t[0][0], kTS, &sm.g.outv[0][0]);
        __syncthreads();
        if (threadIdx.x < TP * 3) {
            int p = threadIdx.x / 3, c = threadIdx.x % 3;
            unsigned t = base + p;
            if (t < n) {
                float v = 1.0f / (1.0f + expf(-sm.g.outv[p][c]));
                if (job.out_pixel) {
                    v = fminf(fmaxf(v, 0.0f), 1.0f);  // clamp01, render.hpp:276
                    job.out[(size_t)job.out_pixel[t] * 3 + c] = v;
                } else {
                    job.out[(size_t)t * 3 + c] = v;
                }
            }
        }
        __syncthreads();
    }
}

int launch_pifu_simt_eval(const FieldDev& f, const SimtMlp& geo, const EvalJob& job, unsigned int max_points,
                          cudaStream_t s) {
    static PerDeviceOnce once;
    const size_t smem = sizeof(SimtSmem);
    if (int r = once.run([&] {
            ICG_CUDA_TRY(cudaFuncSetAttribute(k_pifu_simt_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            return ICG_OK;
        }))
        return r;
    unsigned blocks = (max_points + TP - 1) / TP;
    if (blocks > 148) blocks = 148;
    if (blocks == 0) blocks = 1;
    k_pifu_simt_eval<<<blocks, NT, smem, s>>>(f, geo, job);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

int launch_pifu_simt_texture(const FieldDev& f, const SimtMlp& geo, const SimtMlp& tex, const EvalJob& job,
                             unsigned int max_points, cudaStream_t s) {
    static PerDeviceOnce once;
    const size_t smem = sizeof(SimtTexSmem);
    if (int r = once.run([&] {
            ICG_CUDA_TRY(cudaFuncSetAttribute(k_pifu_simt_texture, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            return ICG_OK;
        }))
        return r;
    unsigned blocks = (max_points + TP - 1) / TP;
    if (blocks > 148) blocks = 148;
    if (blocks == 0) blocks = 1;
    k_pifu_simt_texture<<<blocks, NT, smem, s>>>(f, geo, tex, job);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

}  // namespace icg

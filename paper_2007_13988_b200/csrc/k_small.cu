// k_small.cu — latency path of the PIFu geometry field for small point batches
// (the tail of the conflict loop, localize.hpp:338-353, is a chain of dependent
// batches of ~10-1000 nodes).  The tensor-core kernel streams every weight
// tile through one SM per 64-point tile, so a tiny batch costs a full tile
// latency; here each LAYER is spread over the whole GPU instead: one
// cooperative kernel, grid-wide barrier between layers, every thread owning
// one output feature of PG points (fp32 FFMA, k-ordered, so a point's value
// does not depend on the batch it is evaluated in).  Activations live in a
// small global scratch (L2-resident).  Decides on device whether to run:
// batches above `max_count` exit immediately (the tensor-core kernel takes
// them), so both can be enqueued without a host round-trip.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "eval_common.cuh"

namespace cg = cooperative_groups;

namespace icg {

constexpr int kSmallThreads = 256;
constexpr int kPG = 8;        // points per warp-item
constexpr int kSkipS = 264;   // skip stride (257 padded)

__device__ __forceinline__ void small_gather(const FieldDev& f, const EvalJob& job, unsigned n, float* skip,
                                             double* pos) {
    // one warp per point: 256 channels, 8 per lane, rows coalesced
    const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (unsigned p = gw; p < n; p += nw) {
        double pd[3];
        job_point_d(job, p, pd);
        if (lane < 3) pos[3 * (size_t)p + lane] = pd[lane];
        const float x = (float)pd[0], y = (float)pd[1];
        float u = (x + 1.0f) * 0.5f * (float)(f.W - 1);
        float v = (1.0f - y) * 0.5f * (float)(f.H - 1);
        u = fminf(fmaxf(u, 0.0f), (float)(f.W - 1));
        v = fminf(fmaxf(v, 0.0f), (float)(f.H - 1));
        const int x0 = min((int)floorf(u), f.W - 2), y0 = min((int)floorf(v), f.H - 2);
        const float ax = u - (float)x0, ay = v - (float)y0;
        const float w00 = (1.0f - ax) * (1.0f - ay), w10 = ax * (1.0f - ay), w01 = (1.0f - ax) * ay, w11 = ax * ay;
        const float* m = f.fmap_hwc + ((size_t)y0 * f.W + x0) * (size_t)f.C;
        const size_t rowW = (size_t)f.W * f.C;
        float* out = skip + (size_t)p * kSkipS;
        for (int c = lane; c < f.C; c += 32)
            out[c] = w00 * __ldg(&m[c]) + w10 * __ldg(&m[f.C + c]) + w01 * __ldg(&m[rowW + c]) +
                     w11 * __ldg(&m[rowW + f.C + c]);
        if (lane < kSkipS - kC) out[kC + lane] = lane == 0 ? (float)pd[2] : 0.0f;
    }
}

// hout[p][o] = act(b[o] + sum_k W[o][k] * [hin[p], skip[p]][k]).  One BLOCK
// per (output o, group of kPG points): the 8 warps take contiguous K slices,
// lanes stride inside a slice with every load issued before the FMAs, so a
// layer costs ~one L2 round trip per item round; partial sums combine in
// shared memory in a fixed order (deterministic, batch-independent).
constexpr int kSliceMax = 8;  // per-lane elements per slice (K <= 8 warps * 32 lanes * 8)

__device__ __forceinline__ void small_layer(const SimtMlp& m, const float* const* wrow, int l, const float* hin,
                                            int hin_s, const float* skip, unsigned n, float* hout, int hout_s,
                                            float (*red)[kPG]) {
    const int O = m.out[l], Kh = l ? m.out[l - 1] : 0, Ks = m.skip, K = Kh + Ks;
    const float* __restrict__ W = wrow[l];
    const unsigned groups = (n + kPG - 1) / kPG;
    const unsigned items = groups * (unsigned)O;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = kSmallThreads / 32;
    const int slice = (K + nwarps - 1) / nwarps;
    const int k0 = warp * slice, k1 = min(K, k0 + slice);
    for (unsigned it = blockIdx.x; it < items; it += gridDim.x) {
        const int o = (int)(it % (unsigned)O);
        const unsigned p0 = (it / (unsigned)O) * kPG;
        const float* wr = W + (size_t)o * K;
        float w[kSliceMax], x[kSliceMax][kPG];
#pragma unroll
        for (int u = 0; u < kSliceMax; ++u) {
            const int k = k0 + lane + 32 * u;
            const bool ok = k < k1;
            w[u] = ok ? __ldg(&wr[k]) : 0.0f;
#pragma unroll
            for (int q = 0; q < kPG; ++q) {
                const float* src = k < Kh ? hin + (size_t)(p0 + q) * hin_s + k : skip + (size_t)(p0 + q) * kSkipS + (k - Kh);
                x[u][q] = ok ? *src : 0.0f;
            }
        }
        float acc[kPG];
#pragma unroll
        for (int q = 0; q < kPG; ++q) {
            float a = 0.0f;
#pragma unroll
            for (int u = 0; u < kSliceMax; ++u) a = fmaf(w[u], x[u][q], a);
            acc[q] = a;
        }
#pragma unroll
        for (int q = 0; q < kPG; ++q)
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], s);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < kPG; ++q) red[warp][q] = acc[q];
        __syncthreads();
        if (threadIdx.x < kPG && p0 + threadIdx.x < n) {
            float v = 0.0f;
            for (int w2 = 0; w2 < nwarps; ++w2) v += red[w2][threadIdx.x];
            v += __ldg(&m.b[l][o]);
            if (v < 0.0f) v *= m.slope;
            hout[(size_t)(p0 + threadIdx.x) * hout_s + o] = v;
        }
        __syncthreads();
    }
}

struct RowWeights {
    const float* w[5];  // row-major [out][in] fp32 copies of the geometry MLP
};

__device__ __forceinline__ unsigned long long sg_time() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kSmallThreads) k_small_mlp(FieldDev f, SimtMlp geo, RowWeights rw, EvalJob job,
                                                             float* scratch, unsigned cap, unsigned max_count,
                                                             unsigned long long* trace) {
    const unsigned n = job_count(job);
    if (n == 0 || n > max_count || n > cap) return;  // grid-uniform decision
    cg::grid_group grid = cg::this_grid();
    job_account(job);
    const unsigned capr = (cap + kPG - 1) / kPG * kPG;
    float* skip = scratch;
    float* hA = skip + (size_t)capr * kSkipS;
    float* hB = hA + (size_t)capr * 1024;
    double* pos = reinterpret_cast<double*>(hB + (size_t)capr * 512);
    __shared__ float red[kSmallThreads / 32][kPG];
    const bool tr = trace && blockIdx.x == 0 && threadIdx.x == 0;
    int ti = 0;
    if (tr) trace[ti++] = sg_time();
    small_gather(f, job, n, skip, pos);
    grid.sync();
    if (tr) trace[ti++] = sg_time();
    small_layer(geo, rw.w, 0, nullptr, 0, skip, n, hA, 1024, red);
    grid.sync();
    if (tr) trace[ti++] = sg_time();
    small_layer(geo, rw.w, 1, hA, 1024, skip, n, hB, 512, red);
    grid.sync();
    if (tr) trace[ti++] = sg_time();
    small_layer(geo, rw.w, 2, hB, 512, skip, n, hA, 1024, red);
    grid.sync();
    if (tr) trace[ti++] = sg_time();
    small_layer(geo, rw.w, 3, hA, 1024, skip, n, hB, 512, red);
    grid.sync();
    if (tr) trace[ti++] = sg_time();
    // final 385 -> 1 layer: one warp per point, lanes split K, fixed reduction order
    const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int Kh = geo.out[3], K = Kh + geo.skip;
    for (unsigned p = gw; p < n; p += nw) {
        float acc = 0.0f;
        for (int k = lane; k < K; k += 32) {
            const float x = k < Kh ? hB[(size_t)p * 512 + k] : skip[(size_t)p * kSkipS + (k - Kh)];
            acc = fmaf(__ldg(&rw.w[4][k]), x, acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            const double* pd = pos + 3 * (size_t)p;
            const double sdf = scene_sdf(*f.scene, pd);
            const float logit = acc + __ldg(&geo.b[4][0]) + (float)(-f.scene->sdf_scale * sdf);
            const float v = 1.0f / (1.0f + expf(-logit));
            if (job_is_grid(job))
                grid_epilogue(job, job_node(job, p), v);
            else
                job.out[p] = v;
        }
    }
    if (tr) {
        trace[ti++] = sg_time();
        trace[15] = n;
    }
}

size_t small_scratch_bytes(unsigned cap) {
    const size_t capr = (cap + kPG - 1) / kPG * kPG;
    return capr * (kSkipS + 1024 + 512) * sizeof(float) + capr * 3 * sizeof(double);
}

int launch_small_mlp(const FieldDev& f, const SimtMlp& geo, const float* const* wrow, const EvalJob& job,
                     float* scratch, unsigned cap, unsigned max_count, cudaStream_t s) {
    static int grid = 0;
    if (grid == 0) {
        int per_sm = 0, sms = 0, dev = 0;
        ICG_CUDA_TRY(cudaGetDevice(&dev));
        ICG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        ICG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_small_mlp, kSmallThreads, 0));
        const char* g = getenv("ICG_SMALL_BPS");
        const int bps = g ? atoi(g) : 4;
        grid = sms * (per_sm < bps ? per_sm : bps);
        if (grid <= 0) grid = sms;
    }
    FieldDev fa = f;
    SimtMlp ga = geo;
    RowWeights rw;
    for (int l = 0; l < 5; ++l) rw.w[l] = wrow[l];
    EvalJob ja = job;
    static unsigned long long* trace = nullptr;
    static int tron = -1;
    if (tron < 0) {
        const char* e = getenv("ICG_TC_TRACE");
        tron = e && e[0] == '1';
        if (tron) cudaMallocManaged(&trace, 16 * sizeof(unsigned long long));
    }
    unsigned long long* tp = tron ? trace : nullptr;
    if (tp) cudaMemsetAsync(tp, 0, 16 * 8, s);
    void* args[] = {&fa, &ga, &rw, &ja, &scratch, &cap, &max_count, &tp};
    ICG_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_small_mlp, grid, kSmallThreads, args, 0, s));
    if (tp) {
        cudaStreamSynchronize(s);
        if (tp[0])
            fprintf(stderr, "[small-trace] n=%llu gather %.1f L1 %.1f L2 %.1f L3 %.1f L4 %.1f final %.1f us\n", tp[15],
                    (tp[1] - tp[0]) * 1e-3, (tp[2] - tp[1]) * 1e-3, (tp[3] - tp[2]) * 1e-3, (tp[4] - tp[3]) * 1e-3,
                    (tp[5] - tp[4]) * 1e-3, (tp[6] - tp[5]) * 1e-3);
    }
    return ICG_OK;
}

}  // namespace icg

// k_render.cu — mesh-free first-crossing renderer on sm_100a
// (conventions of render.hpp:140-206 and 264-278).
//
// One thread per pixel.  Pixel (col, row) is the view ray x = -1 + 2 col/(W-1),
// y = 1 - 2 row/(H-1) (row 0 at the top, render.hpp:48-49); sample k sits at
// view z = 1 - 2k/R (k = 0 nearest, grid.hpp:50-53) and is mapped to the world
// grid with view_to_world (render.hpp:29-32) in double, rounded once to fp32
// grid coordinates, then trilinearly interpolated in fp32 in a fixed order.
// The first sample with value >= 0.5f is the crossing (argmax of the binarised
// column with the smallest-index tie rule, grid.hpp:173-197); the bracket
// (k1-1, k1) gives s = clamp((0.5-v0)/(v1-v0), 0, 1) (s = 1 when k1 == 0 or
// the bracket is degenerate) and depth = 1 - 2(k1-1+s)/R (render.hpp:190-204).
// Every operation is an explicit round-to-nearest intrinsic, so the CPU oracle
// (oracle/isocull_oracle.c, -ffp-contract=off) reproduces each crossing index
// bit-exactly.  Covered pixels append their world surface point to a compact
// list consumed by the texture MLP.
//
// Speed without changing a single rounding: the per-pixel parts of
// view_to_world (x/scale, y/scale and the first two products of each row) and
// the view depth of every sample (1 - 2k/R, a shared table) are computed once,
// and a warp walks one ray 32 samples at a time (coalesced corner loads).
// Rays along grid x (the yaw-90 view) skip empty space exactly: a sample whose
// cell corners are all 0.0f interpolates to exactly 0 (no crossing, not
// grazing), so only the samples whose cell meets the nonzero extent of the 4
// x-lines around the ray (k_xline_extents) are evaluated.
#include <algorithm>

#include "eval_common.cuh"

namespace icg {

__device__ __forceinline__ float lerp_rn(float a, float b, float t) {
    return __fadd_rn(a, __fmul_rn(t, __fsub_rn(b, a)));
}

__device__ __forceinline__ float sample_grid(const float* __restrict__ V, int R, float gx, float gy, float gk) {
    float fR = (float)R;
    if (!(gx >= 0.0f && gx <= fR && gy >= 0.0f && gy <= fR && gk >= 0.0f && gk <= fR)) return 0.0f;
    int i0 = min((int)floorf(gx), R - 1), j0 = min((int)floorf(gy), R - 1), k0 = min((int)floorf(gk), R - 1);
    float fx = __fsub_rn(gx, (float)i0), fy = __fsub_rn(gy, (float)j0), fk = __fsub_rn(gk, (float)k0);
    size_t n = (size_t)R + 1, sj = n, sk = n * n;
    size_t b = (size_t)i0 + n * ((size_t)j0 + n * (size_t)k0);
    float c00 = lerp_rn(__ldg(&V[b]), __ldg(&V[b + 1]), fx);
    float c10 = lerp_rn(__ldg(&V[b + sj]), __ldg(&V[b + sj + 1]), fx);
    float c01 = lerp_rn(__ldg(&V[b + sk]), __ldg(&V[b + sk + 1]), fx);
    float c11 = lerp_rn(__ldg(&V[b + sj + sk]), __ldg(&V[b + sj + sk + 1]), fx);
    float c0 = lerp_rn(c00, c10, fy);
    float c1 = lerp_rn(c01, c11, fy);
    return lerp_rn(c0, c1, fk);
}

// view_to_world, render.hpp:29-32: R^T (v - t), v = (x/scale, y/scale, z)
__device__ __forceinline__ void view_to_world_d(const RenderJob& r, double x, double y, double z, double* w) {
    double v0 = __dsub_rn(__ddiv_rn(x, r.scale), r.trans[0]);
    double v1 = __dsub_rn(__ddiv_rn(y, r.scale), r.trans[1]);
    double v2 = __dsub_rn(z, r.trans[2]);
    const double* m = r.rot;
    w[0] = __dadd_rn(__dadd_rn(__dmul_rn(m[0], v0), __dmul_rn(m[3], v1)), __dmul_rn(m[6], v2));
    w[1] = __dadd_rn(__dadd_rn(__dmul_rn(m[1], v0), __dmul_rn(m[4], v1)), __dmul_rn(m[7], v2));
    w[2] = __dadd_rn(__dadd_rn(__dmul_rn(m[2], v0), __dmul_rn(m[5], v1)), __dmul_rn(m[8], v2));
}

constexpr int kMaxRenderCells = 1024;
constexpr int kRenderThreads = 256;

// One WARP per pixel ray: lane l evaluates sample k = kb + l of the current
// 32-sample chunk.  Consecutive samples sit one cell apart along the ray, so
// the lanes' corner loads are spatially coherent (fully coalesced when the ray
// runs along the x-fastest memory axis, as for yaw 90).  The first crossing is
// the lowest lane whose value is >= 0.5f (ballot); every value is computed with
// the same operations as the per-thread formulation, so results are unchanged.
__global__ void __launch_bounds__(kRenderThreads, 6) k_render(RenderJob r) {
    __shared__ double vz_tab[kMaxRenderCells + 1];
    const int W = r.width, H = r.height, R = r.cells;
    for (int k = threadIdx.x; k <= R; k += blockDim.x)
        vz_tab[k] = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, (double)k), (double)R));
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const size_t npx = (size_t)W * H;
    const size_t nwarps = (size_t)gridDim.x * (kRenderThreads / 32);
    unsigned long long n_cov = 0, n_deg = 0, n_graz = 0;
    const double* m = r.rot;
    const double hr = __dmul_rn(0.5, (double)R);
    const float fR = (float)R;
    for (size_t px = (size_t)blockIdx.x * (kRenderThreads / 32) + (threadIdx.x >> 5); px < npx; px += nwarps) {
        const int col = (int)(px % W), row = (int)(px / W);
        const double vx = __dadd_rn(-1.0, __ddiv_rn(__dmul_rn(2.0, (double)col), (double)(W - 1)));
        const double vy = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, (double)row), (double)(H - 1)));
        // view_to_world (render.hpp:29-32) with the per-pixel terms hoisted (same operations, same order)
        const double v0 = __dsub_rn(__ddiv_rn(vx, r.scale), r.trans[0]);
        const double v1 = __dsub_rn(__ddiv_rn(vy, r.scale), r.trans[1]);
        const double c0 = __dadd_rn(__dmul_rn(m[0], v0), __dmul_rn(m[3], v1));
        const double c1 = __dadd_rn(__dmul_rn(m[1], v0), __dmul_rn(m[4], v1));
        const double c2 = __dadd_rn(__dmul_rn(m[2], v0), __dmul_rn(m[5], v1));
        int k1 = -1;
        float vprev = 0.0f, vhit = 0.0f, last = 0.0f;
        bool grazing = false;
        // Rays that run along grid x (the yaw-90 view): every grid coordinate of a sample is a
        // monotone function of k (each step a correctly rounded op with fixed operands), so if gy
        // and gk agree at k = 0 and k = R they are the SAME for every sample.  Those rays hoist
        // the y/z part of the coordinates and of the trilinear setup out of the sample loop, and a
        // sample with fx == 0 skips its x+1 corners (lerp_rn(a, b, 0) == a exactly for finite
        // values).  Every arithmetic result is unchanged.
        float gyc = 0.0f, gkc = 0.0f;
        if (lane < 2) {
            const double v2 = __dsub_rn(vz_tab[lane == 0 ? 0 : R], r.trans[2]);
            gyc = (float)__dmul_rn(__dadd_rn(__dadd_rn(c1, __dmul_rn(m[7], v2)), 1.0), hr);
            gkc = (float)__dmul_rn(__dsub_rn(1.0, __dadd_rn(c2, __dmul_rn(m[8], v2))), hr);
        }
        const float gy_a = __shfl_sync(0xffffffffu, gyc, 0), gy_b = __shfl_sync(0xffffffffu, gyc, 1);
        const float gk_a = __shfl_sync(0xffffffffu, gkc, 0), gk_b = __shfl_sync(0xffffffffu, gkc, 1);
        const bool xray = gy_a == gy_b && gk_a == gk_b;
        const bool yz_in = gy_a >= 0.0f && gy_a <= fR && gk_a >= 0.0f && gk_a <= fR;
        const int j0 = min((int)floorf(gy_a), R - 1), kk0 = min((int)floorf(gk_a), R - 1);
        const float fy = __fsub_rn(gy_a, (float)j0), fk = __fsub_rn(gk_a, (float)kk0);
        const size_t nn = (size_t)R + 1;
        const size_t byz = nn * ((size_t)j0 + nn * (size_t)kk0);
        // samples [k_lo, k_hi] may be nonzero; outside it every sample is exactly 0
        int k_lo = 0, k_hi = R;
        if (xray && r.xext) {
            if (!yz_in) {
                k_hi = -1;
            } else {
                const int2 e00 = __ldg(&r.xext[(size_t)j0 + nn * (size_t)kk0]);
                const int2 e10 = __ldg(&r.xext[(size_t)j0 + 1 + nn * (size_t)kk0]);
                const int2 e01 = __ldg(&r.xext[(size_t)j0 + nn * (size_t)(kk0 + 1)]);
                const int2 e11 = __ldg(&r.xext[(size_t)j0 + 1 + nn * (size_t)(kk0 + 1)]);
                const int lo = min(min(e00.x, e10.x), min(e01.x, e11.x));
                const int hi = max(max(e00.y, e10.y), max(e01.y, e11.y));
                if (lo > hi) {
                    k_hi = -1;  // all four lines are zero: the ray misses
                } else {
                    // gx(k) = A + B k up to roundings (sample_at); cells lo-1 .. hi <=> gx in [lo-1, hi+1]
                    const double B = -m[6];
                    if (fabs(B) > 0.25) {
                        const double A = (c0 + m[6] * (1.0 - r.trans[2]) + 1.0) * hr;
                        const double ka = ((double)(lo - 1) - A) / B, kb = ((double)(hi + 1) - A) / B;
                        const double kmin = fmin(ka, kb), kmax = fmax(ka, kb);
                        k_lo = kmin < 0.0 ? 0 : (kmin > (double)R ? R + 1 : (int)floor(kmin) - 2);
                        k_hi = kmax > (double)R ? R : (kmax < 0.0 ? -1 : (int)ceil(kmax) + 2);
                        k_lo = max(k_lo, 0);
                        k_hi = min(k_hi, R);
                    }
                }
            }
        }
        auto sample_at = [&](int k) -> float {
            float v = 0.0f;
            if (k <= R) {
                const double v2 = __dsub_rn(vz_tab[k], r.trans[2]);
                const double w0 = __dadd_rn(c0, __dmul_rn(m[6], v2));
                const float gx = (float)__dmul_rn(__dadd_rn(w0, 1.0), hr);
                if (xray) {
                    if (yz_in && gx >= 0.0f && gx <= fR) {
                        const int i0 = min((int)floorf(gx), R - 1);
                        const float fx = __fsub_rn(gx, (float)i0);
                        const float* V = r.values + byz + (size_t)i0;
                        const size_t sj = nn, sk = nn * nn;
                        float c00, c10, c01, c11;
                        if (fx == 0.0f) {
                            c00 = __ldg(&V[0]);
                            c10 = __ldg(&V[sj]);
                            c01 = __ldg(&V[sk]);
                            c11 = __ldg(&V[sj + sk]);
                        } else {
                            c00 = lerp_rn(__ldg(&V[0]), __ldg(&V[1]), fx);
                            c10 = lerp_rn(__ldg(&V[sj]), __ldg(&V[sj + 1]), fx);
                            c01 = lerp_rn(__ldg(&V[sk]), __ldg(&V[sk + 1]), fx);
                            c11 = lerp_rn(__ldg(&V[sj + sk]), __ldg(&V[sj + sk + 1]), fx);
                        }
                        const float cy0 = lerp_rn(c00, c10, fy);
                        const float cy1 = lerp_rn(c01, c11, fy);
                        v = lerp_rn(cy0, cy1, fk);
                    }
                } else {
                    const double w1 = __dadd_rn(c1, __dmul_rn(m[7], v2));
                    const double w2 = __dadd_rn(c2, __dmul_rn(m[8], v2));
                    const float gy = (float)__dmul_rn(__dadd_rn(w1, 1.0), hr);
                    const float gk = (float)__dmul_rn(__dsub_rn(1.0, w2), hr);
                    v = sample_grid(r.values, R, gx, gy, gk);
                }
            }
            return v;
        };
        // kBatch 32-sample chunks per iteration (measured: batching chunks so more corner loads are
        // in flight costs more in registers and discarded samples than it hides; 1 is fastest)
        constexpr int kBatch = 1;
        for (int kb2 = k_lo; kb2 <= k_hi; kb2 += 32 * kBatch) {
            float vv[kBatch];
#pragma unroll
            for (int h = 0; h < kBatch; ++h)
                vv[h] = kb2 + 32 * h + lane <= k_hi ? sample_at(kb2 + 32 * h + lane) : 0.0f;
            bool done = false;
#pragma unroll
            for (int h = 0; h < kBatch; ++h) {
            const int kb = kb2 + 32 * h;
            if (done || kb > k_hi) break;
            const int k = kb + lane;
            const float v = vv[h];
            const unsigned hit = __ballot_sync(0xffffffffu, k <= R && v >= 0.5f);
            const int first = hit ? __ffs(hit) - 1 : 32;
            // samples before the crossing: grazing (0 < v < 1), render.hpp:180-188
            grazing |= __ballot_sync(0xffffffffu, lane < first && k <= R && v > 0.0f && v < 1.0f) != 0u;
            const float prev_in_chunk = __shfl_up_sync(0xffffffffu, v, 1);
            if (hit) {
                k1 = kb + first;
                vhit = __shfl_sync(0xffffffffu, v, first);
                const float pv = __shfl_sync(0xffffffffu, prev_in_chunk, first);
                vprev = first > 0 ? pv : last;
                done = true;
                break;
            }
            last = __shfl_sync(0xffffffffu, v, 31);
            }
            if (done) break;
        }
        if (lane == 0) {
            r.rgb[3 * px + 0] = r.bg[0];
            r.rgb[3 * px + 1] = r.bg[1];
            r.rgb[3 * px + 2] = r.bg[2];
            if (k1 < 0) {
                r.depth[px] = -2.0f;  // kInvalidDepth, render.hpp:72
                r.mask[px] = 0;
                if (r.surface_k) r.surface_k[px] = -1;
                n_graz += grazing ? 1 : 0;
            } else {
                ++n_cov;
                double s = 1.0;
                if (k1 > 0) {
                    double v1d = (double)vhit, v0d = (double)vprev;
                    double denom = __dsub_rn(v1d, v0d);
                    if (denom > 0.0) {
                        s = __ddiv_rn(__dsub_rn(0.5, v0d), denom);
                        s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
                    } else {
                        ++n_deg;
                    }
                }
                double depth =
                    __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, __dadd_rn(__dsub_rn((double)k1, 1.0), s)), (double)R));
                r.depth[px] = (float)depth;
                r.mask[px] = 1;
                if (r.surface_k) r.surface_k[px] = k1;
                double w[3];
                view_to_world_d(r, vx, vy, depth, w);
                unsigned pos = atomicAdd(&r.ctr->surface_count, 1u);
                r.surface_pts[3 * (size_t)pos + 0] = w[0];
                r.surface_pts[3 * (size_t)pos + 1] = w[1];
                r.surface_pts[3 * (size_t)pos + 2] = w[2];
                r.surface_px[pos] = (uint32_t)px;
            }
        }
    }
    (void)fR;
    if (lane == 0) {
        if (n_cov) atomicAdd(&r.ctr->covered, n_cov);
        if (n_deg) atomicAdd(&r.ctr->degenerate, n_deg);
        if (n_graz) atomicAdd(&r.ctr->grazing, n_graz);
    }
}

// one warp per x-line (j, k): first and last i with values[i + n (j + n k)] != 0 ({n, -1} if none)
__global__ void __launch_bounds__(256) k_xline_extents(const float* __restrict__ V, int R, int2* __restrict__ ext) {
    const int n = R + 1;
    const size_t lines = (size_t)n * n;
    const int lane = threadIdx.x & 31;
    for (size_t L = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; L < lines;
         L += ((size_t)gridDim.x * blockDim.x) >> 5) {
        const float* row = V + L * (size_t)n;
        int first = n, last = -1;
        for (int i0 = 0; i0 < n; i0 += 32) {
            const int i = i0 + lane;
            const unsigned nz = __ballot_sync(0xffffffffu, i < n && __ldg(&row[i]) != 0.0f);
            if (nz) {
                if (first == n) first = i0 + __ffs(nz) - 1;
                last = i0 + 31 - __clz(nz);
            }
        }
        if (lane == 0) ext[L] = make_int2(first, last);
    }
}

int launch_xline_extents(const float* values, int cells, int2* ext, cudaStream_t s) {
    const size_t lines = ((size_t)cells + 1) * ((size_t)cells + 1);
    const unsigned blocks = (unsigned)std::min<size_t>((lines + 7) / 8, 148 * 16);
    k_xline_extents<<<blocks, 256, 0, s>>>(values, cells, ext);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

int launch_render_first_crossing(const RenderJob& r, cudaStream_t s) {
    if (r.cells > kMaxRenderCells) {
        set_error("render: grid larger than 1024 cells");
        return ICG_EINVAL;
    }
    const size_t npx = (size_t)r.width * r.height;
    const size_t blocks = std::min<size_t>((npx + kRenderThreads / 32 - 1) / (kRenderThreads / 32), 148 * 16);
    k_render<<<(unsigned)blocks, kRenderThreads, 0, s>>>(r);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

}  // namespace icg

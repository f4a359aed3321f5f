// k_depth.cu — the level-L half of render_view's view-space depth pass (detail::depth_pass,
// render.hpp:105-206), exact: compiled without FMA contraction, fp64 where the reference uses
// double.  The grid is the view-space grid (node (i, j, k) at view NDC (-1+2i/R, -1+2j/R,
// 1-2k/R), k = 0 nearest); a column (i, j) is one pixel.  One thread per column walks k with
// coalesced accesses (consecutive threads = consecutive i).
//
//   k_depth_shadow  : argmax of the tentative (upsampled binarized) column (render.hpp:118-127):
//                     when its maximum is exactly 1, every non-evaluated node behind the first
//                     such k becomes a shadow node; the surviving fractional candidates
//                     (tent in (0,1), state interpolated, :131-137) are flagged for evaluation;
//   k_depth_bracket : argmax on the binarized updated column (:140-146) -> the bracket nodes
//                     k1-1, k1 that are not evaluated yet (:156-173);
//   k_depth_final   : per pixel: k1, bracket fraction s, depth = 1 - 2(k1 - 1 + s)/R, the
//                     degenerate / grazing counters (:175-206); image row = n-1-j
//                     (render.hpp:222-226, 266-272); covered pixels append their world surface
//                     point for the texture field.
#include "eval_common.cuh"

namespace icg {

__device__ __forceinline__ bool dbit(const uint32_t* b, size_t i) { return (b[i >> 5] >> (i & 31)) & 1u; }

// tentative value of fine node (i, j, k) as (ones, count) over its 1/2/4/8 coarse parents
// (upsample_interpolate of the binarized grid, grid.hpp:87-120): tent = ones / count exactly
__device__ __forceinline__ void tent_parts(const uint32_t* cbin, unsigned cn, unsigned i, unsigned j, unsigned k,
                                           int& ones, int& cnt) {
    const unsigned i0 = i >> 1, i1 = (i + 1) >> 1, j0 = j >> 1, j1 = (j + 1) >> 1, k0 = k >> 1, k1 = (k + 1) >> 1;
    ones = 0;
    cnt = 0;
    for (unsigned kk = k0; kk <= k1; ++kk)
        for (unsigned jj = j0; jj <= j1; ++jj)
            for (unsigned ii = i0; ii <= i1; ++ii) {
                ones += dbit(cbin, ii + (size_t)cn * (jj + (size_t)cn * kk));
                ++cnt;
            }
}

__global__ void __launch_bounds__(256) k_depth_shadow(const uint32_t* __restrict__ cbin, int rc, uint8_t* fs,
                                                      uint32_t* sel) {
    const unsigned fn = 2u * rc + 1u, cn = rc + 1u;
    const unsigned col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= fn * fn) return;
    const unsigned i = col % fn, j = col / fn;
    const size_t plane = (size_t)fn * fn;
    int kfull = -1;  // first k with tent == 1 (the column's argmax when its maximum is 1)
    for (unsigned k = 0; k < fn && kfull < 0; ++k) {
        int o, c;
        tent_parts(cbin, cn, i, j, k, o, c);
        if (o == c) kfull = (int)k;
    }
    for (unsigned k = 0; k < fn; ++k) {
        const size_t idx = col + plane * k;
        const uint8_t st = fs[idx];
        if (kfull >= 0 && (int)k > kfull) {
            if (st != ICG_STATE_EVALUATED) fs[idx] = ICG_STATE_SHADOW;
            continue;  // shadow (no candidate) or evaluated (not interpolated)
        }
        if (st != ICG_STATE_INTERPOLATED) continue;
        int o, c;
        tent_parts(cbin, cn, i, j, k, o, c);
        if (o > 0 && o < c) atomicOr(&sel[idx >> 5], 1u << (idx & 31));
    }
}

// first k of a column with a binarized value of 1 (argmax_z of the binarized grid), or -1
__device__ __forceinline__ int first_inside(const float* fv, size_t col, size_t plane, unsigned fn) {
    for (unsigned k = 0; k < fn; ++k)
        if (fv[col + plane * k] >= 0.5f) return (int)k;
    return -1;
}

// k1 of every column is kept (colk): the per-pixel pass uses the argmax taken BEFORE the bracket
// nodes are evaluated (final_pass, render.hpp:140-146), even if an evaluated bracket node k1-1
// turns out inside (then s clamps to 0)
__global__ void __launch_bounds__(256) k_depth_bracket(const float* __restrict__ fv, const uint8_t* __restrict__ fs,
                                                       int rc, uint32_t* sel, int* __restrict__ colk) {
    const unsigned fn = 2u * rc + 1u;
    const unsigned col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= fn * fn) return;
    const size_t plane = (size_t)fn * fn;
    const int k1 = first_inside(fv, col, plane, fn);
    colk[col] = k1;
    if (k1 < 0) return;
    for (int k = k1 > 0 ? k1 - 1 : 0; k <= k1; ++k) {
        const size_t idx = col + plane * (size_t)k;
        if (fs[idx] != ICG_STATE_EVALUATED) atomicOr(&sel[idx >> 5], 1u << (idx & 31));
    }
}

struct FinalArgs {
    const float* fv;
    const int* colk;
    int rc;
    double vr[9], vt[3], vs;
    float bg[3];
    float* depth;
    float* rgb;
    uint8_t* mask;
    int32_t* surface_k;
    double* surface_pts;
    uint32_t* surface_px;
    DevCounters* ctr;
};

__global__ void __launch_bounds__(256) k_depth_final(FinalArgs a) {
    const unsigned fn = 2u * a.rc + 1u, cells = 2u * a.rc;
    const unsigned col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= fn * fn) return;
    const size_t plane = (size_t)fn * fn;
    const unsigned i = col % fn, j = col / fn;
    const size_t px = i + (size_t)fn * (fn - 1 - j);  // image row = n-1-j, column = i
    const int k1 = a.colk[col];
    if (k1 < 0) {
        for (unsigned k = 0; k < fn; ++k) {
            const float v = a.fv[col + plane * k];
            if (v > 0.0f && v < 1.0f) {
                atomicAdd(&a.ctr->grazing, 1ull);
                break;
            }
        }
        a.depth[px] = -2.0f;
        a.mask[px] = 0;
        a.surface_k[px] = -1;
        a.rgb[3 * px] = a.bg[0];
        a.rgb[3 * px + 1] = a.bg[1];
        a.rgb[3 * px + 2] = a.bg[2];
        return;
    }
    double s = 1.0;
    if (k1 > 0) {
        const double v1 = (double)a.fv[col + plane * (size_t)k1];
        const double v0 = (double)a.fv[col + plane * (size_t)(k1 - 1)];
        const double denom = __dsub_rn(v1, v0);
        if (denom > 0.0) {
            const double x = __ddiv_rn(__dsub_rn(0.5, v0), denom);
            s = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
        } else {
            atomicAdd(&a.ctr->degenerate, 1ull);
        }
    }
    const double R = (double)cells;
    const double depth = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, __dadd_rn(__dsub_rn((double)k1, 1.0), s)), R));
    a.depth[px] = (float)depth;
    a.mask[px] = 1;
    a.surface_k[px] = k1;
    atomicAdd(&a.ctr->covered, 1ull);
    // surface point: view (x = -1 + 2 col / R, y = -1 + 2 (n-1-row) / R, depth) -> world
    // (render.hpp:271-276; n-1-row = j)
    const double vx = __dadd_rn(-1.0, __ddiv_rn(__dmul_rn(2.0, (double)i), R));
    const double vy = __dadd_rn(-1.0, __ddiv_rn(__dmul_rn(2.0, (double)j), R));
    const double w0 = __dsub_rn(__ddiv_rn(vx, a.vs), a.vt[0]);
    const double w1 = __dsub_rn(__ddiv_rn(vy, a.vs), a.vt[1]);
    const double w2 = __dsub_rn(depth, a.vt[2]);
    const double* m = a.vr;
    const unsigned slot = atomicAdd(&a.ctr->surface_count, 1u);
    double* sp = a.surface_pts + 3 * (size_t)slot;
    sp[0] = __dadd_rn(__dadd_rn(__dmul_rn(m[0], w0), __dmul_rn(m[3], w1)), __dmul_rn(m[6], w2));
    sp[1] = __dadd_rn(__dadd_rn(__dmul_rn(m[1], w0), __dmul_rn(m[4], w1)), __dmul_rn(m[7], w2));
    sp[2] = __dadd_rn(__dadd_rn(__dmul_rn(m[2], w0), __dmul_rn(m[5], w1)), __dmul_rn(m[8], w2));
    a.surface_px[slot] = (uint32_t)px;
    // covered pixels take the texture (written by the texture job); until then the background
    a.rgb[3 * px] = a.bg[0];
    a.rgb[3 * px + 1] = a.bg[1];
    a.rgb[3 * px + 2] = a.bg[2];
}

static unsigned column_blocks(int rc) {
    const size_t fn = 2 * (size_t)rc + 1;
    return (unsigned)((fn * fn + 255) / 256);
}

int launch_depth_shadow(const DepthJob& j, cudaStream_t s) {
    k_depth_shadow<<<column_blocks(j.rc), 256, 0, s>>>(j.cbin, j.rc, j.fs, j.sel);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

int launch_depth_bracket(const DepthJob& j, cudaStream_t s) {
    k_depth_bracket<<<column_blocks(j.rc), 256, 0, s>>>(j.fv, j.fs, j.rc, j.sel, j.colk);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

int launch_depth_final(const DepthJob& j, cudaStream_t s) {
    FinalArgs a{};
    a.fv = j.fv;
    a.colk = j.colk;
    a.rc = j.rc;
    for (int k = 0; k < 9; ++k) a.vr[k] = j.vr[k];
    for (int k = 0; k < 3; ++k) {
        a.vt[k] = j.vt[k];
        a.bg[k] = j.bg[k];
    }
    a.vs = j.vs;
    a.depth = j.depth;
    a.rgb = j.rgb;
    a.mask = j.mask;
    a.surface_k = j.surface_k;
    a.surface_pts = j.surface_pts;
    a.surface_px = j.surface_px;
    a.ctr = j.ctr;
    k_depth_final<<<column_blocks(j.rc), 256, 0, s>>>(a);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

}  // namespace icg

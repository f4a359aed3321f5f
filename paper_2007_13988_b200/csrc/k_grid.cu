// k_grid.cu — per-level dense passes of progressive localization on sm_100a.
//
// Replaces, per refinement level (localize.hpp:325-356):
//   binarize (grid.hpp:122-130) + upsample_interpolate (grid.hpp:87-120)
//   + boundary_candidates (grid.hpp:133-140) + dilate_1ring (grid.hpp:144-163)
//   + carry_scalars (localize.hpp:110-122) + mask_to_unevaluated_list
//   (localize.hpp:124-129), and the conflict expansion
//   collect_unevaluated_neighbors (localize.hpp:160-177).
//
// Layout (HBM): values fp32 and states u8, x-fastest idx = i + n(j + n k)
// (grid.hpp:45-48); every per-node mask is a flat bitset (bit idx of word idx/32).
//
// The dilated candidate mask is computed without materialising candidates:
// a fine node's tentative value is fractional iff its parent box (1, 2, 4 or 8
// coarse nodes) is not uniform after binarisation; the 26-ring dilation of
// that set is exactly "some adjacent coarse cell has mixed binarised corners",
// where the adjacent cells of fine index i along one axis are {(i-1)/2} for
// odd i and {i/2-1, i/2} (clipped) for even i.  The mixed-cell set is the
// refined-cell output of the level.  Checked bit-exactly against the
// reference by tests/test_gpu_parity.py.
#include <cuda_runtime.h>

#include "icg_internal.h"

namespace icg {

__device__ __forceinline__ bool test_bit(const uint32_t* bits, size_t idx) {
    return (bits[idx >> 5] >> (idx & 31)) & 1u;
}

// ---- coarse binarised bits ------------------------------------------------
__global__ void k_coarse_bits(const float* __restrict__ cv, size_t n, uint32_t* __restrict__ bits) {
    size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool b = idx < n && cv[idx] >= 0.5f;  // binarize_value, grid.hpp:122
    unsigned m = __ballot_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0 && idx < n) bits[idx >> 5] = m;
}

// ---- coarse cells with mixed binarised corners (refined-cell set) ---------
__global__ void k_mixed_cells(const uint32_t* __restrict__ cbin, int rc, uint32_t* __restrict__ mixed,
                              unsigned long long* refined) {
    const unsigned ncell = (unsigned)rc * rc * rc;
    const unsigned idx = blockIdx.x * blockDim.x + threadIdx.x;
    bool m = false;
    if (idx < ncell) {
        const unsigned jk = idx / (unsigned)rc;
        const unsigned ci = idx - jk * rc, ck = jk / (unsigned)rc, cj = jk - ck * rc;
        const unsigned cn = rc + 1u;
        const unsigned base = ci + cn * (cj + cn * ck);
        int ones = 0;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            unsigned o = base + (d & 1) + cn * (((d >> 1) & 1) + cn * (d >> 2));
            ones += test_bit(cbin, o);
        }
        m = ones != 0 && ones != 8;
    }
    unsigned w = __ballot_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) {
        if (idx < ncell) mixed[idx >> 5] = w;
        if (w) atomicAdd(refined, (unsigned long long)__popc(w));
    }
}

// ---- fine pass: tent / carry / tentbin / selection + block counts ---------
constexpr int kClassifyBlock = 1024;

__device__ __forceinline__ void adjacent_cells(int i, int rc, int& lo, int& hi) {
    if (i & 1) {
        lo = hi = (i - 1) >> 1;
    } else {
        lo = (i >> 1) - 1;
        hi = i >> 1;
        if (lo < 0) lo = 0;
        if (hi > rc - 1) hi = rc - 1;
    }
}

__global__ void __launch_bounds__(kClassifyBlock)
k_fine_classify(const float* __restrict__ cv, const uint8_t* __restrict__ cs, const uint32_t* __restrict__ cbin,
                const uint32_t* __restrict__ mixed, int rc, float* __restrict__ fv, uint8_t* __restrict__ fs,
                uint32_t* __restrict__ tentbin, uint32_t* __restrict__ sel, uint32_t* __restrict__ block_counts) {
    __shared__ unsigned warp_counts[kClassifyBlock / 32];
    const unsigned fn = 2u * rc + 1u, cn = rc + 1u;
    const unsigned nf = fn * fn * fn;
    const unsigned idx = blockIdx.x * kClassifyBlock + threadIdx.x;
    bool tb = false, s = false;
    if (idx < nf) {
        const unsigned jk = idx / fn;
        int i = (int)(idx - jk * fn);
        int k = (int)(jk / fn);
        int j = (int)(jk - (unsigned)k * fn);
        int i0 = i >> 1, i1 = (i + 1) >> 1, j0 = j >> 1, j1 = (j + 1) >> 1, k0 = k >> 1, k1 = (k + 1) >> 1;
        float v;
        uint8_t st;
        if (i0 == i1 && j0 == j1 && k0 == k1) {
            // even node: carry the coarse scalar and state (carry_scalars, localize.hpp:116-119)
            unsigned ci = (unsigned)i0 + cn * ((unsigned)j0 + cn * (unsigned)k0);
            v = cv[ci];
            st = cs[ci];
            tb = test_bit(cbin, ci);
        } else {
            // mean of the binarised parents (upsample_interpolate, grid.hpp:106-115)
            int ones = 0, cnt = 0;
            for (int kk = k0; kk <= k1; ++kk)
                for (int jj = j0; jj <= j1; ++jj)
                    for (int ii = i0; ii <= i1; ++ii) {
                        ones += test_bit(cbin, (unsigned)ii + cn * ((unsigned)jj + cn * (unsigned)kk));
                        ++cnt;
                    }
            v = (float)ones / (float)cnt;  // exact dyadic; equals (float)(double sum / cnt)
            st = ICG_STATE_INTERPOLATED;
            tb = 2 * ones >= cnt;          // tent >= 0.5f
        }
        fv[idx] = v;
        fs[idx] = st;
        // dilate_1ring(boundary_candidates(tent)) via adjacent mixed coarse cells
        int xl, xh, yl, yh, zl, zh;
        adjacent_cells(i, rc, xl, xh);
        adjacent_cells(j, rc, yl, yh);
        adjacent_cells(k, rc, zl, zh);
        bool flagged = false;
        for (int cz = zl; cz <= zh && !flagged; ++cz)
            for (int cy = yl; cy <= yh && !flagged; ++cy)
                for (int cx = xl; cx <= xh && !flagged; ++cx)
                    flagged = test_bit(mixed, (unsigned)cx + (unsigned)rc * ((unsigned)cy + (unsigned)rc * (unsigned)cz));
        s = flagged && st != ICG_STATE_EVALUATED;  // mask_to_unevaluated_list, localize.hpp:127
    }
    unsigned tbw = __ballot_sync(0xffffffffu, tb);
    unsigned sw = __ballot_sync(0xffffffffu, s);
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        if (idx < nf) {
            tentbin[idx >> 5] = tbw;
            sel[idx >> 5] = sw;
        }
        warp_counts[warp] = __popc(sw);
    }
    __syncthreads();
    if (warp == 0) {
        unsigned c = warp_counts[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) block_counts[blockIdx.x] = c;
    }
}

// ---- exclusive scan of block counts (single block) ------------------------
__global__ void __launch_bounds__(1024)
k_scan_blocks(uint32_t* __restrict__ counts, unsigned nblocks, DevCounters* ctr, int level) {
    __shared__ unsigned warp_sums[32];
    __shared__ unsigned carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (unsigned base = 0; base < nblocks; base += 1024) {
        unsigned idx = base + threadIdx.x;
        unsigned v = idx < nblocks ? counts[idx] : 0u;
        unsigned x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned w = warp_sums[lane];
            unsigned ws = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                unsigned y = __shfl_up_sync(0xffffffffu, ws, o);
                if (lane >= o) ws += y;
            }
            warp_sums[lane] = ws - w;  // exclusive
        }
        __syncthreads();
        unsigned excl = carry + warp_sums[warp] + x - v;
        if (idx < nblocks) counts[idx] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ctr->list_count = carry;
        ctr->evals[level] += carry;
        ctr->cf_count[0] = 0;
        ctr->cf_count[1] = 0;
        ctr->nx_count[0] = 0;
        ctr->nx_count[1] = 0;
    }
}

// ---- write the ascending E0 list -----------------------------------------
__global__ void __launch_bounds__(kClassifyBlock)
k_write_list(const uint32_t* __restrict__ sel, size_t nf, const uint32_t* __restrict__ offsets,
             uint32_t* __restrict__ list) {
    __shared__ unsigned warp_off[kClassifyBlock / 32];
    const size_t idx = (size_t)blockIdx.x * kClassifyBlock + threadIdx.x;
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned w = idx < nf ? sel[idx >> 5] : 0u;
    if (idx >= nf) w = 0u;
    if (lane == 0) warp_off[warp] = __popc(w);
    __syncthreads();
    if (warp == 0) {
        unsigned c = warp_off[lane], x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        warp_off[lane] = x - c;
    }
    __syncthreads();
    if (idx < nf && ((w >> lane) & 1u)) {
        unsigned pos = offsets[blockIdx.x] + warp_off[warp] + __popc(w & ((1u << lane) - 1u));
        list[pos] = (uint32_t)idx;
    }
}

int launch_level_classify(const LevelBufs& b, DevCounters* ctr, int level, cudaStream_t s) {
    const int rc = b.rc, cn = rc + 1, fn = 2 * rc + 1;
    size_t ncoarse = (size_t)cn * cn * cn, ncell = (size_t)rc * rc * rc, nf = (size_t)fn * fn * fn;
    k_coarse_bits<<<(unsigned)((ncoarse + 255) / 256), 256, 0, s>>>(b.cv, ncoarse, b.cbin);
    k_mixed_cells<<<(unsigned)((ncell + 255) / 256), 256, 0, s>>>(b.cbin, rc, b.mixed, &ctr->refined[level]);
    unsigned nblocks = (unsigned)((nf + kClassifyBlock - 1) / kClassifyBlock);
    k_fine_classify<<<nblocks, kClassifyBlock, 0, s>>>(b.cv, b.cs, b.cbin, b.mixed, rc, b.fv, b.fs, b.tentbin, b.sel,
                                                       b.block_counts);
    k_scan_blocks<<<1, 1024, 0, s>>>(b.block_counts, nblocks, ctr, level);
    k_write_list<<<nblocks, kClassifyBlock, 0, s>>>(b.sel, nf, b.block_counts, b.list);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// ---- conflict expansion (localize.hpp:338-353, 160-177) --------------------
// Iteration `iter` reads conflicts cf[iter&1], writes neighbours to next_list /
// nx[iter&1], and clears the buffers iteration iter+1 will fill.
__global__ void k_conflict_expand(uint32_t* __restrict__ queued, const uint8_t* __restrict__ fs, int fcells,
                                  const uint32_t* __restrict__ conflicts, DevCounters* ctr, int iter, int max_iters,
                                  uint32_t* __restrict__ next_list, unsigned cap) {
    const int p = iter & 1;
    unsigned ncf = ctr->cf_count[p];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr->cf_count[p ^ 1] = 0;
        ctr->nx_count[p ^ 1] = 0;
        if (ncf > 0 && iter >= max_iters) ctr->warning = 1;  // localize.hpp:343-346
    }
    if (ncf == 0 || iter >= max_iters) return;
    const int fn = fcells + 1;
    // one thread per (conflict, neighbour) pair, 26 neighbours in (dk, dj, di) order
    size_t total = (size_t)ncf * 26;
    for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
        unsigned c = (unsigned)(t / 26);
        int r = (int)(t % 26);
        if (r >= 13) ++r;  // skip the centre (di = dj = dk = 0)
        int di = r % 3 - 1, dj = (r / 3) % 3 - 1, dk = r / 9 - 1;
        size_t idx = conflicts[c];
        int i = (int)(idx % fn), j = (int)((idx / fn) % fn), k = (int)(idx / ((size_t)fn * fn));
        int ii = i + di, jj = j + dj, kk = k + dk;
        if (ii < 0 || jj < 0 || kk < 0 || ii >= fn || jj >= fn || kk >= fn) continue;
        size_t nb = (size_t)ii + (size_t)fn * ((size_t)jj + (size_t)fn * (size_t)kk);
        if (fs[nb] == ICG_STATE_EVALUATED) continue;
        unsigned bit = 1u << (nb & 31);
        unsigned old = atomicOr(&queued[nb >> 5], bit);
        if (old & bit) continue;
        unsigned pos = atomicAdd(&ctr->nx_count[p], 1u);
        if (pos < cap)
            next_list[pos] = (uint32_t)nb;
        else
            ctr->overflow = 1;
    }
}

int launch_conflict_expand(uint32_t* queued, const uint8_t* fs, int fcells, const uint32_t* conflicts,
                           DevCounters* ctr, int iter, int max_iters, uint32_t* next_list, unsigned cap,
                           cudaStream_t s) {
    k_conflict_expand<<<148, 256, 0, s>>>(queued, fs, fcells, conflicts, ctr, iter, max_iters, next_list, cap);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

__global__ void k_unroll_check(DevCounters* ctr, int parity, int level) {
    if (ctr->cf_count[parity] > 0) ctr->unroll_exhausted |= 1u << level;
}

int launch_unroll_check(DevCounters* ctr, int parity, int level, cudaStream_t s) {
    k_unroll_check<<<1, 1, 0, s>>>(ctr, parity, level);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// ---- binarized_volume (localize.hpp:154-158) --------------------------------
__global__ void k_binarize(const float* __restrict__ v, uint8_t* __restrict__ out, size_t n) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = v[i] >= 0.5f ? 1 : 0;
}

int launch_binarize(const float* v, uint8_t* out, size_t n, cudaStream_t s) {
    k_binarize<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(v, out, n);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// ---- compare_iou (localize.hpp:377-387) -------------------------------------
__global__ void k_iou(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, size_t n,
                      unsigned long long* iu) {
    unsigned long long inter = 0, uni = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        bool av = a[i] != 0, bv = b[i] != 0;
        inter += (av && bv);
        uni += (av || bv);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        inter += __shfl_xor_sync(0xffffffffu, inter, o);
        uni += __shfl_xor_sync(0xffffffffu, uni, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&iu[0], inter);
        atomicAdd(&iu[1], uni);
    }
}

int launch_iou(const uint8_t* a, const uint8_t* b, size_t n, unsigned long long* iu, cudaStream_t s) {
    k_iou<<<148 * 8, 256, 0, s>>>(a, b, n, iu);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

__global__ void k_fill_u8(uint8_t* p, size_t n, uint8_t v) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

int launch_fill_states(uint8_t* p, size_t n, uint8_t v, cudaStream_t s) {
    k_fill_u8<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n, v);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

}  // namespace icg

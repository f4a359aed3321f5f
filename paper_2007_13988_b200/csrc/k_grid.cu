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

#include <algorithm>

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

// the same, 128 nodes per warp step: lane l loads nodes 4l..4l+3 as one float4 (cv 16-byte aligned,
// the launcher checks), its 4 bits are OR-merged over groups of 8 lanes into the step's 4 words
__global__ void k_coarse_bits4(const float* __restrict__ cv, size_t n, uint32_t* __restrict__ bits) {
    const unsigned lane = threadIdx.x & 31u;
    const size_t nwarps = (size_t)gridDim.x * (blockDim.x >> 5);
    for (size_t q = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); 128 * q < n; q += nwarps) {
        const size_t i0 = 128 * q + 4 * lane;
        uint32_t nib = 0u;
        if (i0 + 3 < n) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(cv + i0));
            nib = (v.x >= 0.5f ? 1u : 0u) | (v.y >= 0.5f ? 2u : 0u) | (v.z >= 0.5f ? 4u : 0u) | (v.w >= 0.5f ? 8u : 0u);
        } else {
            for (int e = 0; e < 4; ++e)
                if (i0 + e < n && __ldg(&cv[i0 + e]) >= 0.5f) nib |= 1u << e;  // binarize_value, grid.hpp:122
        }
        uint32_t w = nib << (4u * (lane & 7u));
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        w |= __shfl_xor_sync(0xffffffffu, w, 4);
        if ((lane & 7u) == 0 && 128 * q + 4 * lane < n) bits[4 * q + (lane >> 3)] = w;
    }
}

static void launch_coarse_bits(const float* cv, size_t n, uint32_t* bits, cudaStream_t s) {
    if (((uintptr_t)cv & 15u) == 0) {
        const size_t steps = (n + 127) / 128;  // one per warp, 8 warps per block
        const unsigned blocks = (unsigned)std::min<size_t>((steps + 7) / 8, 148u * 16u);
        k_coarse_bits4<<<blocks, 256, 0, s>>>(cv, n, bits);
    } else {
        k_coarse_bits<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(cv, n, bits);
    }
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

// ---- fine pass: one WARP per fine row (j, k) ----------------------------------
// The row's parent information is staged per warp in shared memory as aligned
// bit rows: the (1, 2 or 4) coarse binarised rows (jj, kk) it interpolates
// from, and the OR of the (1..4) adjacent rows of mixed coarse cells.  A node
// then costs a handful of shared-memory bit tests; all index math is 32-bit.
// Values/states are stored coalesced along x; the flat tentbin / sel words
// (rows are not word-aligned) are merged with atomicOr (buffers cleared first).
constexpr int kFineThreads = 256;
constexpr int kRowWords = 17;  // >= (cn + 32) / 32 for cn <= 513

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

// word w of the bit row starting at flat bit `base` of g
__device__ __forceinline__ uint32_t row_word(const uint32_t* __restrict__ g, uint32_t base, int w) {
    const uint32_t b = base + 32u * (uint32_t)w, q = b >> 5, r = b & 31u;
    const uint32_t lo = __ldg(&g[q]);
    return r ? __funnelshift_r(lo, __ldg(&g[q + 1]), r) : lo;
}

// ---- the same cells 32 at a time (rc a multiple of 32: a word of the cell bitset is 32 cells of
// one cell row): per corner node row, the word of corners x and its shift by one (corners x + 1);
// a cell is mixed when the OR of its 8 corners is set and their AND is not
__global__ void k_mixed_words(const uint32_t* __restrict__ cbin, int rc, uint32_t* __restrict__ mixed,
                              unsigned long long* refined) {
    const unsigned wpr = (unsigned)rc >> 5, nw = (unsigned)rc * (unsigned)rc * wpr;
    const unsigned w = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned cnt = 0;
    if (w < nw) {
        const unsigned row = w / wpr, ci0 = (w - row * wpr) << 5;
        const unsigned ck = row / (unsigned)rc, cj = row - ck * (unsigned)rc, cn = (unsigned)rc + 1u;
        uint32_t any = 0u, all = ~0u;
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const uint32_t base = cn * ((cj + (d & 1)) + cn * (ck + (d >> 1))) + ci0;
            const uint32_t lo = row_word(cbin, base, 0);
            const uint32_t b32 = (__ldg(&cbin[(base + 32u) >> 5]) >> ((base + 32u) & 31u)) & 1u;
            const uint32_t x1 = (lo >> 1) | (b32 << 31);
            any |= lo | x1;
            all &= lo & x1;
        }
        const uint32_t mw = any & ~all;
        mixed[w] = mw;
        cnt = __popc(mw);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(refined, (unsigned long long)cnt);
}

static void launch_mixed(const uint32_t* cbin, int rc, uint32_t* mixed, unsigned long long* refined, cudaStream_t s) {
    if ((rc & 31) == 0) {
        const unsigned nw = (unsigned)rc * (unsigned)rc * ((unsigned)rc >> 5);
        k_mixed_words<<<(nw + 255) / 256, 256, 0, s>>>(cbin, rc, mixed, refined);
    } else {
        const size_t ncell = (size_t)rc * rc * rc;
        k_mixed_cells<<<(unsigned)((ncell + 255) / 256), 256, 0, s>>>(cbin, rc, mixed, refined);
    }
}



__global__ void __launch_bounds__(kFineThreads, 8)
k_fine_rows(const float* __restrict__ cv, const uint8_t* __restrict__ cs, const uint32_t* __restrict__ cbin,
            const uint32_t* __restrict__ mixed, int rc, float* __restrict__ fv, uint8_t* __restrict__ fs,
            uint32_t* __restrict__ tentbin, uint32_t* __restrict__ sel, int2* __restrict__ xext) {
    // per warp: one byte per coarse x of the row, (number of binarised parents set, bits 0-2) |
    // (coarse cell x mixed in an adjacent cell row, bit 4); built only for rows near the surface
    __shared__ uint8_t info_s[kFineThreads / 32][32 * kRowWords];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int fn = 2 * rc + 1, cn = rc + 1;
    const uint32_t nrows_total = (uint32_t)fn * (uint32_t)fn;
    const int cwords = (cn + 31) >> 5, mwords = (rc + 31) >> 5;
    uint8_t* inf = info_s[wl];
    // valid bits of this lane's word of a coarse node row (cn bits) and of a cell row (rc bits)
    const uint32_t valid = lane < cwords ? (lane == cwords - 1 && (cn & 31) ? (1u << (cn & 31)) - 1u : ~0u) : 0u;
    const uint32_t mvalid = lane < mwords ? (lane == mwords - 1 && (rc & 31) ? (1u << (rc & 31)) - 1u : ~0u) : 0u;
    for (uint32_t row = blockIdx.x * (kFineThreads / 32) + wl; row < nrows_total; row += gridDim.x * (kFineThreads / 32)) {
        const int k = (int)(row / (uint32_t)fn), j = (int)(row - (uint32_t)k * fn);
        const int j0 = j >> 1, j1 = (j + 1) >> 1, k0 = k >> 1, k1 = (k + 1) >> 1;
        const bool jy = j1 != j0, kz = k1 != k0;
        const int lgr = (int)jy + (int)kz;  // log2 of the parent rows (1, 2 or 4)
        int yl, yh, zl, zh;
        adjacent_cells(j, rc, yl, yh);
        adjacent_cells(k, rc, zl, zh);
        // lane w < cwords: word w of the bit-sliced sum of the (1, 2 or 4) parent bit rows
        // (upsample_interpolate, grid.hpp:106-115): count = p0 + 2 p1 + 4 p2 <= 4
        uint32_t p0 = 0u, p1 = 0u, p2 = 0u, m = 0u;
        if (lane < cwords) {
            const uint32_t a = row_word(cbin, (uint32_t)cn * ((uint32_t)j0 + (uint32_t)cn * (uint32_t)k0), lane);
            const uint32_t b = jy ? row_word(cbin, (uint32_t)cn * ((uint32_t)j1 + (uint32_t)cn * (uint32_t)k0), lane) : 0u;
            const uint32_t c = kz ? row_word(cbin, (uint32_t)cn * ((uint32_t)j0 + (uint32_t)cn * (uint32_t)k1), lane) : 0u;
            const uint32_t d = (jy && kz) ? row_word(cbin, (uint32_t)cn * ((uint32_t)j1 + (uint32_t)cn * (uint32_t)k1), lane) : 0u;
            const uint32_t ab0 = a ^ b, ab1 = a & b, cd0 = c ^ d, cd1 = c & d;
            const uint32_t carry = ab0 & cd0, t = ab1 ^ cd1;
            p0 = (ab0 ^ cd0) & valid;
            p1 = (t ^ carry) & valid;
            p2 = ((ab1 & cd1) | (t & carry)) & valid;
        }
        // lane w < mwords: word w of the OR of the adjacent mixed-cell rows (dilate_1ring of
        // boundary_candidates, as cells)
        if (lane < mwords) {  // (at most 2 x 2 rows: all loads issued before the ORs)
            const uint32_t r00 = (uint32_t)rc * ((uint32_t)yl + (uint32_t)rc * (uint32_t)zl);
            const uint32_t r10 = (uint32_t)rc * ((uint32_t)yh + (uint32_t)rc * (uint32_t)zl);
            const uint32_t r01 = (uint32_t)rc * ((uint32_t)yl + (uint32_t)rc * (uint32_t)zh);
            const uint32_t r11 = (uint32_t)rc * ((uint32_t)yh + (uint32_t)rc * (uint32_t)zh);
            const bool dy = yh != yl, dz = zh != zl;
            const uint32_t m00 = row_word(mixed, r00, lane);
            const uint32_t m10 = dy ? row_word(mixed, r10, lane) : 0u;
            const uint32_t m01 = dz ? row_word(mixed, r01, lane) : 0u;
            const uint32_t m11 = (dy && dz) ? row_word(mixed, r11, lane) : 0u;
            m = (m00 | m10 | m01 | m11) & mvalid;
        }
        const uint32_t rowbase = row * (uint32_t)fn;
        const bool even_jk = !((j | k) & 1);
        const uint32_t cbase = (uint32_t)cn * ((uint32_t)j0 + (uint32_t)cn * (uint32_t)k0);
        // rows away from the surface (most of them): no adjacent mixed cell and a uniform parent box
        // along the whole row -> every non-even node is the uniform value 0 or 1, nothing selected
        {
            const uint32_t full = lgr == 0 ? p0 : lgr == 1 ? p1 : p2;  // count == 2^lgr (all parents inside)
            const bool any_mixed = __any_sync(0xffffffffu, m != 0u);
            const bool all0 = !__any_sync(0xffffffffu, (p0 | p1 | p2) != 0u);
            const bool all1 = !__any_sync(0xffffffffu, lane < cwords && (full != valid || (lgr >= 1 && p0) ||
                                                                          (lgr == 2 && p1)));
            if (!any_mixed && (all0 || all1)) {
                const float u = all1 ? 1.0f : 0.0f;
                if (!even_jk) {
                    // every node is u / interpolated: 16-byte stores between a scalar head and tail
                    float* vrow = fv + rowbase;
                    const int hv = min((int)(((16u - ((uint32_t)(uintptr_t)vrow & 15u)) & 15u) >> 2), fn);
                    const int nv = (fn - hv) >> 2, tv = hv + 4 * nv;
                    if (lane < hv) vrow[lane] = u;
                    float4* v4 = reinterpret_cast<float4*>(vrow + hv);
                    for (int q = lane; q < nv; q += 32) v4[q] = make_float4(u, u, u, u);
                    if (tv + lane < fn) vrow[tv + lane] = u;
                    uint8_t* srow = fs + rowbase;
                    const int hs = min((int)((16u - ((uint32_t)(uintptr_t)srow & 15u)) & 15u), fn);
                    const int ns = (fn - hs) >> 4, ts = hs + 16 * ns;
                    constexpr uint32_t i4 = 0x01010101u * ICG_STATE_INTERPOLATED;
                    if (lane < hs) srow[lane] = ICG_STATE_INTERPOLATED;
                    uint4* s16 = reinterpret_cast<uint4*>(srow + hs);
                    for (int q = lane; q < ns; q += 32) s16[q] = make_uint4(i4, i4, i4, i4);
                    if (ts + lane < fn) srow[ts + lane] = ICG_STATE_INTERPOLATED;
                } else {
                    // even nodes carry the coarse row, odd ones are u: 4 nodes per lane (float4 +
                    // 4-byte state stores; the launcher checks fv 16-byte / fs 4-byte base alignment)
                    const int hv = min((int)((4u - (rowbase & 3u)) & 3u), fn);
                    const int nq = (fn - hv) >> 2, tq = hv + 4 * nq;
                    auto one = [&](int i) {
                        float v = u;
                        uint8_t st = ICG_STATE_INTERPOLATED;
                        if (!(i & 1)) {
                            v = __ldg(&cv[cbase + (i >> 1)]);
                            st = __ldg(&cs[cbase + (i >> 1)]);
                        }
                        fv[rowbase + i] = v;
                        fs[rowbase + i] = st;
                    };
                    if (lane < hv) one(lane);
                    if (tq + lane < fn) one(tq + lane);
                    const int par = hv & 1;  // group node e is even iff e == par (mod 2)
                    float4* v4 = reinterpret_cast<float4*>(fv + rowbase + hv);
                    uint32_t* s4 = reinterpret_cast<uint32_t*>(fs + rowbase + hv);
                    for (int q = lane; q < nq; q += 32) {
                        const uint32_t x0 = cbase + (uint32_t)((hv + par) >> 1) + 2u * (uint32_t)q;
                        const float c0 = __ldg(&cv[x0]), c1 = __ldg(&cv[x0 + 1]);
                        const uint32_t t0 = __ldg(&cs[x0]), t1 = __ldg(&cs[x0 + 1]);
                        constexpr uint32_t I = ICG_STATE_INTERPOLATED;
                        if (par == 0) {
                            v4[q] = make_float4(c0, u, c1, u);
                            s4[q] = t0 | (I << 8) | (t1 << 16) | (I << 24);
                        } else {
                            v4[q] = make_float4(u, c0, u, c1);
                            s4[q] = I | (t0 << 8) | (I << 16) | (t1 << 24);
                        }
                    }
                }
                if (xext) {  // the row's nonzero extent: u everywhere, or the carried even nodes
                    int first = fn, last = -1;
                    if (all1) {
                        first = (even_jk && __ldg(&cv[cbase]) == 0.0f) ? 1 : 0;
                        last = (even_jk && __ldg(&cv[cbase + (uint32_t)rc]) == 0.0f) ? fn - 2 : fn - 1;
                    } else if (even_jk) {
                        for (int x = lane; x <= rc; x += 32)
                            if (__ldg(&cv[cbase + (uint32_t)x]) != 0.0f) {
                                first = min(first, 2 * x);
                                last = max(last, 2 * x);
                            }
                        first = __reduce_min_sync(0xffffffffu, first);
                        last = __reduce_max_sync(0xffffffffu, last);
                    }
                    if (lane == 0) xext[row] = make_int2(first, last);
                }
                if (all1) {  // every tentative bit of the row is set: one OR per word
                    const uint32_t last = rowbase + (uint32_t)fn - 1u, w0 = rowbase >> 5, w1 = last >> 5;
                    for (uint32_t w = w0 + (uint32_t)lane; w <= w1; w += 32u) {
                        uint32_t mk = ~0u;
                        if (w == w0) mk &= ~0u << (rowbase & 31u);
                        if (w == w1) mk &= ~0u >> (31u - (last & 31u));
                        atomicOr(&tentbin[w], mk);
                    }
                }
                continue;
            }
        }
        // the per-x info bytes of this row (word t of the planes / mixed row from lane t)
        __syncwarp();  // the previous row's readers are done
        for (int t = 0; t < cwords; ++t) {
            const uint32_t q0 = __shfl_sync(0xffffffffu, p0, t), q1 = __shfl_sync(0xffffffffu, p1, t),
                           q2 = __shfl_sync(0xffffffffu, p2, t), qm = __shfl_sync(0xffffffffu, m, t);
            inf[32 * t + lane] = (uint8_t)(((q0 >> lane) & 1u) | (((q1 >> lane) & 1u) << 1) |
                                           (((q2 >> lane) & 1u) << 2) | (((qm >> lane) & 1u) << 4));
        }
        __syncwarp();
        int nz_first = fn, nz_last = -1;  // the row's nonzero extent (xext)
        for (int i0w = 0; i0w < fn; i0w += 32) {
            const int i = i0w + lane;
            bool tb = false, sl = false, nz = false;
            if (i < fn) {
                const int odd = i & 1, x0 = i >> 1;
                // node i interpolates coarse nodes x0 (and x0 + 1 if odd); its adjacent cells are x0
                // (odd) or x0 - 1 and x0, clamped to the grid (an unused x0 = rc cell bit is 0)
                const uint32_t ia = inf[x0], ib = inf[odd ? x0 + 1 : (x0 > 0 ? x0 - 1 : 0)];
                const int ones = (int)(ia & 7u) + (odd ? (int)(ib & 7u) : 0);
                const bool flagged = (((odd ? ia : (ia | ib)) >> 4) & 1u) != 0u;  // dilate_1ring(boundary_candidates)
                const int lg = lgr + odd;
                float v;
                uint8_t st;
                if (even_jk && !odd) {
                    // even node: carry the coarse scalar and state (carry_scalars, localize.hpp:116-119)
                    v = __ldg(&cv[cbase + x0]);
                    st = __ldg(&cs[cbase + x0]);
                } else {
                    // mean of the binarised parents: exact dyadic ones / 2^lg
                    v = (float)ones * __int_as_float((127 - lg) << 23);
                    st = ICG_STATE_INTERPOLATED;
                }
                // tent >= 0.5f (for an even node: its binarised coarse value)
                tb = 2 * ones >= (1 << lg);
                fv[rowbase + i] = v;
                fs[rowbase + i] = st;
                sl = flagged && st != ICG_STATE_EVALUATED;  // mask_to_unevaluated_list
                nz = v != 0.0f;
            }
            if (xext) {
                const unsigned nzw = __ballot_sync(0xffffffffu, nz);
                if (nzw) {
                    if (nz_first == fn) nz_first = i0w + __ffs(nzw) - 1;
                    nz_last = i0w + 31 - __clz(nzw);
                }
            }
            const unsigned tbw = __ballot_sync(0xffffffffu, tb), sw = __ballot_sync(0xffffffffu, sl);
            // lane 0 merges the tentative bits, lane 1 the selection bits (one code path)
            const unsigned bits = lane == 0 ? tbw : sw;
            if (lane < 2 && bits) {
                uint32_t* dst = lane == 0 ? tentbin : sel;
                const uint32_t first = rowbase + (uint32_t)i0w, sh = first & 31u, w = first >> 5;
                atomicOr(&dst[w], bits << sh);
                if (sh && (bits >> (32 - sh))) atomicOr(&dst[w + 1], bits >> (32 - sh));
            }
        }
        if (xext && lane == 0) xext[row] = make_int2(nz_first, nz_last);
    }
}

// per-CTA selection counts over the word partition used by k_write_words
constexpr int kWordsPerCta = 2048;
constexpr int kWriteThreads = 1024;

__global__ void __launch_bounds__(kWriteThreads)
k_count_words(const uint32_t* __restrict__ sel, unsigned nwords, uint32_t* __restrict__ counts) {
    __shared__ unsigned warp_counts[kWriteThreads / 32];
    unsigned c = 0;
    for (unsigned w = blockIdx.x * kWordsPerCta + threadIdx.x; w < min(nwords, (blockIdx.x + 1) * kWordsPerCta);
         w += kWriteThreads)
        c += __popc(__ldg(&sel[w]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) warp_counts[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned v = warp_counts[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) counts[blockIdx.x] = v;
    }
}

// ---- exclusive scan of the per-CTA counts (single block) -----------------------
// in place; returns the total (valid in every thread)
__device__ unsigned scan_block_counts(uint32_t* __restrict__ counts, unsigned nblocks) {
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
    return carry;
}

__global__ void __launch_bounds__(1024)
k_scan_blocks(uint32_t* __restrict__ counts, unsigned nblocks, DevCounters* ctr, int level) {
    const unsigned total = scan_block_counts(counts, nblocks);
    if (threadIdx.x == 0) {
        ctr->list_count = total;
        ctr->e0[level] = total;
        ctr->evals[level] += total;
        ctr->cf_count[0] = 0;
        ctr->cf_count[1] = 0;
        ctr->nx_count[0] = 0;
        ctr->nx_count[1] = 0;
    }
}

__global__ void __launch_bounds__(1024) k_scan_total(uint32_t* __restrict__ counts, unsigned nblocks, unsigned* total) {
    const unsigned t = scan_block_counts(counts, nblocks);
    if (threadIdx.x == 0) *total = t;
}

// ---- write the ascending E0 list: same CTA/word partition as k_fine_words -------
__global__ void __launch_bounds__(kWriteThreads)
k_write_words(const uint32_t* __restrict__ sel, unsigned long long nwords, const uint32_t* __restrict__ offsets,
              uint32_t* __restrict__ list) {
    __shared__ unsigned warp_sums[kWriteThreads / 32];
    const unsigned long long wbeg = (unsigned long long)blockIdx.x * kWordsPerCta;
    const int per = kWordsPerCta / kWriteThreads;  // consecutive words per thread
    const unsigned long long w0 = wbeg + (unsigned long long)threadIdx.x * per;
    uint32_t wv[kWordsPerCta / kWriteThreads];
    unsigned c = 0;
#pragma unroll
    for (int q = 0; q < per; ++q) {
        wv[q] = w0 + q < nwords ? __ldg(&sel[w0 + q]) : 0u;
        c += __popc(wv[q]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const unsigned w = warp_sums[lane];
        unsigned ws = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= o) ws += y;
        }
        warp_sums[lane] = ws - w;
    }
    __syncthreads();
    unsigned pos = offsets[blockIdx.x] + warp_sums[warp] + x - c;
#pragma unroll
    for (int q = 0; q < per; ++q) {
        uint32_t m = wv[q];
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            list[pos++] = (uint32_t)((w0 + q) * 32 + b);
        }
    }
}

// binarize + mixed cells + upsample/carry of one level (fine values/states, tentbin, sel) without
// the E0 compaction: the first half of launch_level_classify (also render_view's level-L pass)
int launch_level_carry(const LevelBufs& b, DevCounters* ctr, int level, cudaStream_t s) {
    const int rc = b.rc, cn = rc + 1, fn = 2 * rc + 1;
    if (cn + 32 > 32 * kRowWords) {
        set_error("level classify: grid too large");
        return ICG_ERUNTIME;
    }
    if (((uintptr_t)b.fv & 15u) || ((uintptr_t)b.fs & 3u)) {  // k_fine_rows' vector stores
        set_error("level classify: fine grid buffers not 16-byte (values) / 4-byte (states) aligned");
        return ICG_ERUNTIME;
    }
    size_t ncoarse = (size_t)cn * cn * cn, ncell = (size_t)rc * rc * rc, nf = (size_t)fn * fn * fn;
    const unsigned nwords = (unsigned)((nf + 31) / 32);
    launch_coarse_bits(b.cv, ncoarse, b.cbin, s);
    launch_mixed(b.cbin, rc, b.mixed, &ctr->refined[level], s);
    ICG_CUDA_TRY(cudaMemsetAsync(b.tentbin, 0, ((size_t)nwords + 1) * 4, s));
    ICG_CUDA_TRY(cudaMemsetAsync(b.sel, 0, ((size_t)nwords + 1) * 4, s));
    const unsigned rows = (unsigned)fn * fn;
    const unsigned fine_blocks = std::min<unsigned>((rows + kFineThreads / 32 - 1) / (kFineThreads / 32), 148u * 8u);
    k_fine_rows<<<fine_blocks, kFineThreads, 0, s>>>(b.cv, b.cs, b.cbin, b.mixed, rc, b.fv, b.fs, b.tentbin, b.sel, b.xext);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

int launch_level_classify(const LevelBufs& b, DevCounters* ctr, int level, cudaStream_t s) {
    const int rc = b.rc, cn = rc + 1, fn = 2 * rc + 1;
    if (cn + 32 > 32 * kRowWords) {
        set_error("level classify: grid too large");
        return ICG_ERUNTIME;
    }
    if (((uintptr_t)b.fv & 15u) || ((uintptr_t)b.fs & 3u)) {  // k_fine_rows' vector stores
        set_error("level classify: fine grid buffers not 16-byte (values) / 4-byte (states) aligned");
        return ICG_ERUNTIME;
    }
    size_t ncoarse = (size_t)cn * cn * cn, ncell = (size_t)rc * rc * rc, nf = (size_t)fn * fn * fn;
    const unsigned nwords = (unsigned)((nf + 31) / 32);
    const unsigned nblocks = (nwords + kWordsPerCta - 1) / kWordsPerCta;
    launch_coarse_bits(b.cv, ncoarse, b.cbin, s);
    launch_mixed(b.cbin, rc, b.mixed, &ctr->refined[level], s);
    ICG_CUDA_TRY(cudaMemsetAsync(b.tentbin, 0, ((size_t)nwords + 1) * 4, s));
    ICG_CUDA_TRY(cudaMemsetAsync(b.sel, 0, ((size_t)nwords + 1) * 4, s));
    const unsigned rows = (unsigned)fn * fn;
    const unsigned fine_blocks = std::min<unsigned>((rows + kFineThreads / 32 - 1) / (kFineThreads / 32), 148u * 8u);
    k_fine_rows<<<fine_blocks, kFineThreads, 0, s>>>(b.cv, b.cs, b.cbin, b.mixed, rc, b.fv, b.fs, b.tentbin, b.sel, b.xext);
    k_count_words<<<nblocks, kWriteThreads, 0, s>>>(b.sel, nwords, b.block_counts);
    k_scan_blocks<<<1, 1024, 0, s>>>(b.block_counts, nblocks, ctr, level);
    k_write_words<<<nblocks, kWriteThreads, 0, s>>>(b.sel, nwords, b.block_counts, b.list);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// ---- conflict expansion (localize.hpp:338-353, 160-177) --------------------
// Iteration `iter` reads conflicts cf[iter&1], writes neighbours to next_list /
// nx[iter&1], and clears the buffers iteration iter+1 will fill.
__device__ __forceinline__ int chain_class(unsigned n, const ChainClasses& cc) {
    return n == 0 ? 0 : ((cc.big_max && n > cc.big_max) ? 8 : (n > cc.mid_max ? 1 : (n > cc.tail_max ? 2 : 4)));
}
// the batch of host iteration `it` (count n) must have met one of the launched evaluators
__device__ __forceinline__ void check_class(DevCounters* ctr, const ChainClasses& cc, int it, unsigned n) {
    if (cc.prev_mask < 0) return;
    const int c = chain_class(n, cc);
    if (c == 0) return;  // empty, or evaluated by the tail (which clears the counts when done)
    if (!(c & cc.prev_mask)) ctr->mispredict |= 1u << cc.level;
    if (it >= 0 && it < kPredIters && c != 4) ctr->cls[cc.level][it] |= (uint8_t)c;
}

__global__ void k_conflict_expand(uint32_t* __restrict__ queued, const uint8_t* __restrict__ fs, int fcells,
                                  const uint32_t* __restrict__ conflicts, DevCounters* ctr, int iter, int max_iters,
                                  uint32_t* __restrict__ next_list, unsigned cap, ChainClasses cc) {
    const int p = iter & 1;
    unsigned ncf = ctr->cf_count[p];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (iter > 0) check_class(ctr, cc, iter - 1, ctr->nx_count[p ^ 1]);
        ctr->ncols_base = ctr->ncols;  // the column records this iteration's batch may add start here
        ctr->cf_count[p ^ 1] = 0;
        ctr->nx_count[p ^ 1] = 0;
        if (ncf > 0 && iter >= max_iters) ctr->warning = 1;  // localize.hpp:343-346
    }
    if (ncf == 0 || iter >= max_iters) return;
    const unsigned fn = (unsigned)fcells + 1u;  // fn^3 <= 1025^3 < 2^32: 32-bit node indices
    // one thread per (conflict, neighbour) pair, 26 neighbours in (dk, dj, di) order; the new
    // entries of a warp take one atomicAdd on the shared counter (warp-aggregated)
    const unsigned long long total = (unsigned long long)ncf * 26u;
    const unsigned lane = threadIdx.x & 31u;
    for (unsigned long long t0 = (unsigned long long)blockIdx.x * blockDim.x; t0 < total;
         t0 += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long t = t0 + threadIdx.x;
        bool add = false;
        uint32_t nb = 0;
        if (t < total) {
            const unsigned c = (unsigned)(t / 26u);
            unsigned r = (unsigned)(t - (unsigned long long)c * 26u);
            if (r >= 13u) ++r;  // skip the centre (di = dj = dk = 0)
            const int di = (int)(r % 3u) - 1, dj = (int)((r / 3u) % 3u) - 1, dk = (int)(r / 9u) - 1;
            const uint32_t idx = conflicts[c];
            const unsigned jk = idx / fn, i = idx - jk * fn, k = jk / fn, j = jk - k * fn;
            const int ii = (int)i + di, jj = (int)j + dj, kk = (int)k + dk;
            if (ii >= 0 && jj >= 0 && kk >= 0 && ii < (int)fn && jj < (int)fn && kk < (int)fn) {
                nb = (uint32_t)ii + fn * ((uint32_t)jj + fn * (uint32_t)kk);
                if (fs[nb] != ICG_STATE_EVALUATED) {
                    const unsigned bit = 1u << (nb & 31u);
                    add = !(atomicOr(&queued[nb >> 5], bit) & bit);
                }
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, add);
        if (m) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&ctr->nx_count[p], (unsigned)__popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (add) {
                const unsigned pos = base + __popc(m & ((1u << lane) - 1u));
                if (pos < cap)
                    next_list[pos] = nb;
                else
                    ctr->overflow = 1;
            }
        }
    }
}

#ifndef EXPAND_BLOCKS
#define EXPAND_BLOCKS (148 * 8)
#endif
// 8 blocks per SM: a thread's (conflict, neighbour) chain is a few dependent random accesses, so
// the big expansions (tens of thousands of conflicts) want many of them in flight
constexpr unsigned kExpandBlocks = EXPAND_BLOCKS;

int launch_conflict_expand(uint32_t* queued, const uint8_t* fs, int fcells, const uint32_t* conflicts,
                           DevCounters* ctr, int iter, int max_iters, uint32_t* next_list, unsigned cap,
                           cudaStream_t s) {
    ChainClasses cc{0, 0, 0, -1};
    k_conflict_expand<<<kExpandBlocks, 256, 0, s>>>(queued, fs, fcells, conflicts, ctr, iter, max_iters, next_list, cap, cc);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

int launch_conflict_expand_cls(uint32_t* queued, const uint8_t* fs, int fcells, const uint32_t* conflicts,
                               DevCounters* ctr, int iter, int max_iters, uint32_t* next_list, unsigned cap,
                               const ChainClasses& cc, cudaStream_t s) {
    k_conflict_expand<<<kExpandBlocks, 256, 0, s>>>(queued, fs, fcells, conflicts, ctr, iter, max_iters, next_list, cap, cc);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// ---- column claim (column-factored PIFu field) ------------------------------
// Slot order depends on atomic timing, but a column's record is a function of the column
// alone, so every node value is independent of it.
__global__ void k_col_claim(const uint32_t* __restrict__ list, const unsigned* __restrict__ count, int cells,
                            int* __restrict__ cmap, uint32_t* __restrict__ collist, DevCounters* ctr,
                            unsigned min_count) {
    const unsigned n = *count;
    // a conflict-loop batch claims columns only when it is the factored kernels' size class: which
    // kernel records a column (tensor-core COLS or the tail's CUDA-core pass) must not depend on
    // which evaluators the frame enqueued
    if (n < min_count) return;
    const uint32_t n1 = (uint32_t)cells + 1u, plane = n1 * n1;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t col = list[t] % plane;
        if (cmap[col] != -1) continue;  // cheap pre-check; the CAS decides
        if (atomicCAS(&cmap[col], -1, -2) == -1) {
            const unsigned slot = atomicAdd(&ctr->ncols, 1u);
            collist[slot] = col;
            cmap[col] = (int)slot;
        }
    }
}

int launch_col_claim(const uint32_t* list, const unsigned* count, int cells, int* cmap, uint32_t* collist,
                     DevCounters* ctr, unsigned max_points, cudaStream_t s, unsigned min_count) {
    const unsigned blocks = std::min<unsigned>((max_points + 255) / 256, 148u * 8u);
    k_col_claim<<<blocks ? blocks : 1, 256, 0, s>>>(list, count, cells, cmap, collist, ctr, min_count);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

__global__ void k_slot_count(const uint32_t* __restrict__ list, const unsigned* __restrict__ count, int cells,
                             const int* __restrict__ cmap, uint32_t* __restrict__ cnt, unsigned min_count) {
    const unsigned n = *count;
    if (n < min_count) return;  // below the size class its columns were not claimed
    const uint32_t n1 = (uint32_t)cells + 1u, plane = n1 * n1;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        atomicAdd(&cnt[cmap[list[t] % plane]], 1u);
}

// exclusive scan of cnt[0 .. *ncols) in place, in chunks of 8 K entries (1024 threads x 8): pass 1
// sums each chunk, pass 2 rescans it from the sum of the chunks before it (every block adds up the
// few chunk sums itself).  Both passes skip a batch below its size class (count < min_count).
constexpr unsigned kScanChunk = 8192;

__device__ __forceinline__ unsigned block_sum_1024(unsigned v, unsigned* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    unsigned t = lane < 32 ? red[lane] : 0u;
    if (warp == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

__global__ void __launch_bounds__(1024) k_scan_part(const uint32_t* __restrict__ cnt, const unsigned* __restrict__ ncols,
                                                    const unsigned* __restrict__ count, unsigned min_count,
                                                    unsigned* __restrict__ bsum) {
    __shared__ unsigned red[33];
    if (count && *count < min_count) return;
    const unsigned n = *ncols, b0 = blockIdx.x * kScanChunk;
    if (b0 >= n) return;
    unsigned v = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const unsigned i = b0 + q * 1024u + threadIdx.x;
        v += i < n ? cnt[i] : 0u;
    }
    v = block_sum_1024(v, red);
    if (threadIdx.x == 0) bsum[blockIdx.x] = v;
}

__global__ void __launch_bounds__(1024) k_scan_slots(uint32_t* __restrict__ cnt, const unsigned* __restrict__ ncols,
                                                     const unsigned* __restrict__ count, unsigned min_count,
                                                     const unsigned* __restrict__ bsum) {
    constexpr int kPer = 8;
    __shared__ unsigned warp_sums[33];
    __shared__ unsigned stage[1024 * kPer];  // coalesced loads, scanned per thread from shared memory
    if (count && *count < min_count) return;
    const unsigned n = *ncols, base = blockIdx.x * kScanChunk;
    if (base >= n) return;
    // the sum of the chunks before this one
    unsigned pre = 0;
    for (unsigned c = threadIdx.x; c < blockIdx.x; c += 1024u) pre += bsum[c];
    const unsigned carry = block_sum_1024(pre, warp_sums);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const unsigned i = base + q * 1024u + threadIdx.x;
        stage[q * 1024 + threadIdx.x] = i < n ? cnt[i] : 0u;
    }
    __syncthreads();
    unsigned v[kPer], sum = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        v[q] = stage[threadIdx.x * kPer + q];
        sum += v[q];
    }
    unsigned x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const unsigned w = warp_sums[lane];
        unsigned ws = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= o) ws += y;
        }
        warp_sums[lane] = ws - w;
    }
    __syncthreads();
    unsigned run = carry + warp_sums[warp] + x - sum;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        stage[threadIdx.x * kPer + q] = run;
        run += v[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
        const unsigned i = base + q * 1024u + threadIdx.x;
        if (i < n) cnt[i] = stage[q * 1024 + threadIdx.x];
    }
}

__global__ void k_slot_scatter(const uint32_t* __restrict__ list, const unsigned* __restrict__ count, int cells,
                               const int* __restrict__ cmap, uint32_t* __restrict__ off, uint32_t* __restrict__ sorted,
                               unsigned min_count) {
    const unsigned n = *count;
    if (n < min_count) return;
    const uint32_t n1 = (uint32_t)cells + 1u, plane = n1 * n1;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t node = list[t];
        sorted[atomicAdd(&off[cmap[node % plane]], 1u)] = node;
    }
}

int launch_sort_by_column(const uint32_t* list, const unsigned* count, int cells, const int* cmap, uint32_t* cnt,
                          DevCounters* ctr, uint32_t* sorted, unsigned* bsum, unsigned max_points, cudaStream_t s,
                          unsigned min_count) {
    const size_t plane = ((size_t)cells + 1) * ((size_t)cells + 1);
    ICG_CUDA_TRY(cudaMemsetAsync(cnt, 0, plane * 4, s));
    const unsigned blocks = std::max(1u, std::min<unsigned>((max_points + 255) / 256, 148u * 8u));
    k_slot_count<<<blocks, 256, 0, s>>>(list, count, cells, cmap, cnt, min_count);
    const unsigned chunks = (unsigned)((plane + kScanChunk - 1) / kScanChunk);
    k_scan_part<<<chunks, 1024, 0, s>>>(cnt, &ctr->ncols, count, min_count, bsum);
    k_scan_slots<<<chunks, 1024, 0, s>>>(cnt, &ctr->ncols, count, min_count, bsum);
    k_slot_scatter<<<blocks, 256, 0, s>>>(list, count, cells, cmap, cnt, sorted, min_count);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

__global__ void k_dense_column_list(int cells, uint32_t* __restrict__ list) {
    const uint32_t n1 = (uint32_t)cells + 1u, plane = n1 * n1, total = plane * n1;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x)
        list[t] = t / n1 + plane * (t % n1);
}

int launch_dense_column_list(int cells, uint32_t* list, cudaStream_t s) {
    const size_t total = ((size_t)cells + 1) * ((size_t)cells + 1) * ((size_t)cells + 1);
    const unsigned blocks = (unsigned)std::min<size_t>((total + 255) / 256, 148 * 16);
    k_dense_column_list<<<blocks, 256, 0, s>>>(cells, list);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// ---- octree baselines (extract_octree_binarized / _threshold, localize.hpp:199-306) -----------
// binarized octree: coarse nodes whose 6-neighbourhood crosses the binarized value (:214-228)
__global__ void k_interface_nodes(const uint32_t* __restrict__ cbin, int rc, uint32_t* __restrict__ iface) {
    const unsigned cn = rc + 1u;
    const unsigned long long n = (unsigned long long)cn * cn * cn;
    const unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool m = false;
    if (idx < n) {
        const unsigned jk = (unsigned)(idx / cn), i = (unsigned)(idx - (unsigned long long)jk * cn);
        const unsigned k = jk / cn, j = jk - k * cn;
        const bool b = test_bit(cbin, idx);
        const int st[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
#pragma unroll
        for (int s = 0; s < 6; ++s) {
            const int ii = (int)i + st[s][0], jj = (int)j + st[s][1], kk = (int)k + st[s][2];
            if (ii < 0 || jj < 0 || kk < 0 || ii >= (int)cn || jj >= (int)cn || kk >= (int)cn) continue;
            if (test_bit(cbin, (unsigned)ii + (unsigned long long)cn * ((unsigned)jj + (unsigned long long)cn * (unsigned)kk)) != b) {
                m = true;
                break;
            }
        }
    }
    const unsigned w = __ballot_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && idx < n) iface[idx >> 5] = w;
}

// cell marks: mode 0 (binarized) any corner is an interface node (:230-242); mode 1 (threshold)
// the spread of the corner values exceeds the threshold (:271-285)
__global__ void k_octree_cells(const uint32_t* __restrict__ iface, const float* __restrict__ cv, int rc, double thr,
                               int mode, uint32_t* __restrict__ marks, unsigned long long* refined) {
    const unsigned long long ncell = (unsigned long long)rc * rc * rc;
    const unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool m = false;
    if (idx < ncell) {
        const unsigned jk = (unsigned)(idx / rc), ci = (unsigned)(idx - (unsigned long long)jk * rc);
        const unsigned ck = jk / rc, cj = jk - ck * rc, cn = rc + 1u;
        float lo = 1.0f, hi = 0.0f;
        for (int d = 0; d < 8; ++d) {
            const unsigned long long o =
                (ci + (d & 1)) + (unsigned long long)cn * ((cj + ((d >> 1) & 1)) + (unsigned long long)cn * (ck + (d >> 2)));
            if (mode == 0) {
                m = m || test_bit(iface, o);
            } else {
                const float v = cv[o];
                lo = fminf(lo, v);
                hi = fmaxf(hi, v);
            }
        }
        if (mode == 1) m = (double)(hi - lo) > thr;
    }
    const unsigned w = __ballot_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) {
        if (idx < ncell) marks[idx >> 5] = w;
        if (w) atomicAdd(refined, (unsigned long long)__popc(w));
    }
}

// the octree's fine grid and the nodes of marked cells to evaluate (cell_nodes_to_evaluate,
// localize.hpp:131-151): mode 0 even nodes carry the coarse scalar and state, the rest take the
// binarized interpolant of the binarized coarse grid (:244-246); mode 1 upsample_interpolate of the
// continuous values (grid.hpp:87-120: double sum over the parents in (k, j, i) order / count)
__global__ void k_octree_fine(const float* __restrict__ cv, const uint8_t* __restrict__ cs,
                              const uint32_t* __restrict__ cbin, const uint32_t* __restrict__ marks, int rc, int mode,
                              float* __restrict__ fv, uint8_t* __restrict__ fs, uint32_t* __restrict__ sel) {
    const unsigned fn = 2u * rc + 1u, cn = rc + 1u;
    const unsigned long long nf = (unsigned long long)fn * fn * fn;
    const unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool pick = false;
    if (idx < nf) {
        const unsigned jk = (unsigned)(idx / fn), i = (unsigned)(idx - (unsigned long long)jk * fn);
        const unsigned k = jk / fn, j = jk - k * fn;
        const unsigned i0 = i >> 1, i1 = (i + 1) >> 1, j0 = j >> 1, j1 = (j + 1) >> 1, k0 = k >> 1, k1 = (k + 1) >> 1;
        float v;
        uint8_t st;
        if (i0 == i1 && j0 == j1 && k0 == k1) {
            const unsigned long long c = i0 + (unsigned long long)cn * (j0 + (unsigned long long)cn * k0);
            v = cv[c];
            st = cs[c];
        } else {
            st = ICG_STATE_INTERPOLATED;
            if (mode == 0) {
                int ones = 0, cnt = 0;
                for (unsigned kk = k0; kk <= k1; ++kk)
                    for (unsigned jj = j0; jj <= j1; ++jj)
                        for (unsigned ii = i0; ii <= i1; ++ii) {
                            ones += test_bit(cbin, ii + (unsigned long long)cn * (jj + (unsigned long long)cn * kk));
                            ++cnt;
                        }
                v = 2 * ones >= cnt ? 1.0f : 0.0f;  // binarize_value(ones / cnt), exact for cnt in {2, 4, 8}
            } else {
                double sum = 0.0;
                int cnt = 0;
                for (unsigned kk = k0; kk <= k1; ++kk)
                    for (unsigned jj = j0; jj <= j1; ++jj)
                        for (unsigned ii = i0; ii <= i1; ++ii) {
                            sum = __dadd_rn(sum, (double)cv[ii + (unsigned long long)cn * (jj + (unsigned long long)cn * kk)]);
                            ++cnt;
                        }
                v = (float)__ddiv_rn(sum, (double)cnt);
            }
        }
        fv[idx] = v;
        fs[idx] = st;
        if (st != ICG_STATE_EVALUATED) {
            // coarse cells whose 3x3x3 fine nodes include (i, j, k): ci in [ceil((i-2)/2), floor(i/2)]
            const int ca = i & 1 ? (int)i0 : (int)i0 - 1, cb = (int)i0 < rc ? (int)i0 : rc - 1;
            const int ja = j & 1 ? (int)j0 : (int)j0 - 1, jb = (int)j0 < rc ? (int)j0 : rc - 1;
            const int ka = k & 1 ? (int)k0 : (int)k0 - 1, kb = (int)k0 < rc ? (int)k0 : rc - 1;
            for (int ck = ka < 0 ? 0 : ka; ck <= kb && !pick; ++ck)
                for (int cj = ja < 0 ? 0 : ja; cj <= jb && !pick; ++cj)
                    for (int ci = ca < 0 ? 0 : ca; ci <= cb && !pick; ++ci)
                        pick = test_bit(marks, (unsigned)ci + (unsigned long long)rc * ((unsigned)cj + (unsigned long long)rc * (unsigned)ck));
        }
    }
    const unsigned w = __ballot_sync(0xffffffffu, pick);
    if ((threadIdx.x & 31) == 0 && idx < nf) sel[idx >> 5] = w;
}

int launch_octree_level(const LevelBufs& b, uint32_t* iface, int mode, double threshold, DevCounters* ctr, int level,
                        cudaStream_t s) {
    const int rc = b.rc, cn = rc + 1, fn = 2 * rc + 1;
    const size_t ncoarse = (size_t)cn * cn * cn, ncell = (size_t)rc * rc * rc, nf = (size_t)fn * fn * fn;
    if (mode == 0) {
        launch_coarse_bits(b.cv, ncoarse, b.cbin, s);
        k_interface_nodes<<<(unsigned)((ncoarse + 255) / 256), 256, 0, s>>>(b.cbin, rc, iface);
    }
    k_octree_cells<<<(unsigned)((ncell + 255) / 256), 256, 0, s>>>(iface, b.cv, rc, threshold, mode, b.mixed,
                                                                     &ctr->refined[level]);
    k_octree_fine<<<(unsigned)((nf + 255) / 256), 256, 0, s>>>(b.cv, b.cs, b.cbin, b.mixed, rc, mode, b.fv, b.fs, b.sel);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// ---- per-level sets kept for icg_level_set -------------
// nodes of the fine grid evaluated during this level: evaluated now, and not an even node that
// carried an evaluated coarse state (carry_scalars, localize.hpp:110-122)
__global__ void k_level_eval_bits(const uint8_t* __restrict__ fs, const uint8_t* __restrict__ cs, int rc,
                                  uint32_t* __restrict__ bits) {
    const unsigned fn = 2u * rc + 1u, cn = rc + 1u;
    const unsigned long long nf = (unsigned long long)fn * fn * fn;
    const unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool b = false;
    if (idx < nf) {
        b = fs[idx] == ICG_STATE_EVALUATED;
        if (b) {
            const unsigned jk = (unsigned)(idx / fn), i = (unsigned)(idx - (unsigned long long)jk * fn);
            const unsigned k = jk / fn, j = jk - k * fn;
            if (!((i | j | k) & 1u)) b = cs[(i >> 1) + cn * ((j >> 1) + (unsigned long long)cn * (k >> 1))] != ICG_STATE_EVALUATED;
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, b);
    if ((threadIdx.x & 31) == 0 && idx < nf) bits[idx >> 5] = m;
}

int launch_level_eval_bits(const uint8_t* fs, const uint8_t* cs, int rc, uint32_t* bits, cudaStream_t s) {
    const size_t fn = 2 * (size_t)rc + 1, nf = fn * fn * fn;
    k_level_eval_bits<<<(unsigned)((nf + 255) / 256), 256, 0, s>>>(fs, cs, rc, bits);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// every bit of a flat bitset of nbits bits set (the dense level-0 / brute-force evaluation)
__global__ void k_all_bits(uint32_t* __restrict__ bits, unsigned long long nbits) {
    const unsigned long long w = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x, nw = (nbits + 31) / 32;
    if (w < nw) bits[w] = (w + 1) * 32 <= nbits ? 0xffffffffu : (1u << (nbits & 31)) - 1u;
}

int launch_all_bits(uint32_t* bits, size_t nbits, cudaStream_t s) {
    const size_t nw = (nbits + 31) / 32;
    k_all_bits<<<(unsigned)((nw + 255) / 256), 256, 0, s>>>(bits, nbits);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

// in-place exclusive scan of n counts (one block), *total = their sum
int launch_exclusive_scan(uint32_t* counts, unsigned n, unsigned* total, cudaStream_t s) {
    k_scan_total<<<1, 1024, 0, s>>>(counts, n, total);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

size_t bits_to_list_scratch_words(size_t nbits) {
    const size_t nw = (nbits + 31) / 32;
    return (nw + kWordsPerCta - 1) / kWordsPerCta + 2;
}

// ascending list of the set bits of a flat bitset (count / scan / ordered write, the E0 compaction);
// *total (device) = number of set bits; list must hold them all
int launch_bits_to_list(const uint32_t* bits, size_t nbits, uint32_t* scratch, uint32_t* list, unsigned* total,
                        cudaStream_t s) {
    const unsigned nwords = (unsigned)((nbits + 31) / 32);
    const unsigned nblocks = (nwords + kWordsPerCta - 1) / kWordsPerCta;
    if (nblocks == 0) {
        ICG_CUDA_TRY(cudaMemsetAsync(total, 0, sizeof(unsigned), s));
        return ICG_OK;
    }
    k_count_words<<<nblocks, kWriteThreads, 0, s>>>(bits, nwords, scratch);
    k_scan_total<<<1, 1024, 0, s>>>(scratch, nblocks, total);
    if (list) k_write_words<<<nblocks, kWriteThreads, 0, s>>>(bits, nwords, scratch, list);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

__global__ void k_unroll_check(DevCounters* ctr, int parity, int level, ChainClasses cc, int last_iter) {
    if (ctr->cf_count[parity] > 0) ctr->unroll_exhausted |= 1u << level;
    if (last_iter >= 0) check_class(ctr, cc, last_iter, ctr->nx_count[last_iter & 1]);
}

int launch_unroll_check_cls(DevCounters* ctr, int parity, int level, const ChainClasses& cc, int last_iter,
                            cudaStream_t s) {
    k_unroll_check<<<1, 1, 0, s>>>(ctr, parity, level, cc, last_iter);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

int launch_unroll_check(DevCounters* ctr, int parity, int level, cudaStream_t s) {
    ChainClasses cc{0, 0, level, -1};
    k_unroll_check<<<1, 1, 0, s>>>(ctr, parity, level, cc, -1);
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

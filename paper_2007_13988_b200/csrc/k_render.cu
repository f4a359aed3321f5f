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

constexpr int kMaxRenderCells = 1024;
constexpr int kRenderThreads = 256;
constexpr int kLaneSamples = 8;  // samples each lane walks of its own ray before the warp walk

// The ray-independent double terms of view_to_world, each computed once per frame with the
// operations (and roundings) of the per-sample formulation:
//   tab[col]             = vx(col)/scale - t0     (v0 of render.hpp:29-32)
//   tab[W + row]         = vy(row)/scale - t1     (v1)
//   tab[W + H + 3k + a]  = m[6 + a] * (vz(k) - t2) (the view-depth products of sample k)
__global__ void k_render_setup(RenderJob r) {
    const int W = r.width, H = r.height, R = r.cells;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < W) {
        const double vx = __dadd_rn(-1.0, __ddiv_rn(__dmul_rn(2.0, (double)t), (double)(W - 1)));
        r.tab[t] = __dsub_rn(__ddiv_rn(vx, r.scale), r.trans[0]);
    } else if (t < W + H) {
        const double vy = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, (double)(t - W)), (double)(H - 1)));
        r.tab[t] = __dsub_rn(__ddiv_rn(vy, r.scale), r.trans[1]);
    } else if (t < W + H + R + 1) {
        const int k = t - W - H;
        const double vz = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, (double)k), (double)R));
        const double v2 = __dsub_rn(vz, r.trans[2]);
        for (int a = 0; a < 3; ++a) r.tab[W + H + 3 * k + a] = __dmul_rn(r.rot[6 + a], v2);
    }
}

// A warp renders 32 consecutive pixels.  Per-pixel work is lane-parallel (lane p owns
// pixel base + p): the view_to_world terms, the x-ray test and the empty-space
// window, then the output writes and the surface-point append (one atomic per
// warp).  Each ray is then walked by the whole warp: lane l evaluates sample
// k = kb + l of the current 32-sample chunk, so consecutive samples (one cell
// apart along the ray) make coalesced corner loads, and the first crossing is
// the lowest lane whose value is >= 0.5f (ballot).  Every value is computed
// with the same operations as the per-sample formulation.
__global__ void __launch_bounds__(kRenderThreads, 4) k_render(RenderJob r) {
    __shared__ double mv_tab[3][kMaxRenderCells + 1];  // m[6 + a] * (vz(k) - t2)
    const int W = r.width, H = r.height, R = r.cells;
    for (int e = threadIdx.x; e < 3 * (R + 1); e += blockDim.x) mv_tab[e % 3][e / 3] = r.tab[W + H + e];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned npx = (unsigned)W * (unsigned)H;
    const unsigned nwarps = gridDim.x * (kRenderThreads / 32);
    unsigned long long n_cov = 0, n_deg = 0, n_graz = 0;
    const double* m = r.rot;
    const double hr = __dmul_rn(0.5, (double)R);
    const float fR = (float)R;
    const size_t nn = (size_t)R + 1;
    // gx(k) = A + B k up to roundings: the empty-space window is estimated with B's inverse
    const double B = -m[6];
    const bool xwin = r.xext && fabs(B) > 0.25;
    const double invB = xwin ? 1.0 / B : 0.0;
    for (unsigned base = (blockIdx.x * (kRenderThreads / 32) + (threadIdx.x >> 5)) * 32u; base < npx;
         base += nwarps * 32u) {
        // ---------------- per-pixel setup, lane-parallel ----------------
        const unsigned px = base + (unsigned)lane;
        const bool valid = px < npx;
        const unsigned pxc = valid ? px : npx - 1;
        const unsigned row = pxc / (unsigned)W, col = pxc - row * (unsigned)W;
        // view_to_world (render.hpp:29-32) with the per-pixel terms hoisted (same operations, same order)
        const double v0 = __ldg(&r.tab[col]);
        const double v1 = __ldg(&r.tab[W + row]);
        const double c0 = __dadd_rn(__dmul_rn(m[0], v0), __dmul_rn(m[3], v1));
        const double c1 = __dadd_rn(__dmul_rn(m[1], v0), __dmul_rn(m[4], v1));
        const double c2 = __dadd_rn(__dmul_rn(m[2], v0), __dmul_rn(m[5], v1));
        // Rays that run along grid x (the yaw-90 view): every grid coordinate of a sample is a
        // monotone function of k (each step a correctly rounded op with fixed operands), so if gy
        // and gk agree at k = 0 and k = R they are the SAME for every sample.  Those rays hoist
        // the y/z part of the coordinates and of the trilinear setup out of the sample loop, and a
        // sample with fx == 0 skips its x+1 corners (lerp_rn(a, b, 0) == a exactly for finite
        // values).  Every arithmetic result is unchanged.
        const float gy_a = (float)__dmul_rn(__dadd_rn(__dadd_rn(c1, mv_tab[1][0]), 1.0), hr);
        const float gy_b = (float)__dmul_rn(__dadd_rn(__dadd_rn(c1, mv_tab[1][R]), 1.0), hr);
        const float gk_a = (float)__dmul_rn(__dsub_rn(1.0, __dadd_rn(c2, mv_tab[2][0])), hr);
        const float gk_b = (float)__dmul_rn(__dsub_rn(1.0, __dadd_rn(c2, mv_tab[2][R])), hr);
        const bool xray = gy_a == gy_b && gk_a == gk_b;
        const bool yz_in = gy_a >= 0.0f && gy_a <= fR && gk_a >= 0.0f && gk_a <= fR;
        const int j0 = min(max((int)floorf(gy_a), 0), R - 1), kk0 = min(max((int)floorf(gk_a), 0), R - 1);
        const float fy = __fsub_rn(gy_a, (float)j0), fk = __fsub_rn(gk_a, (float)kk0);
        // samples [k_lo, k_hi] may be nonzero; outside it every sample is exactly 0: a sample whose
        // cell corners are all 0.0f interpolates to exactly 0 (no crossing, not grazing)
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
                } else if (xwin) {
                    // cells lo-1 .. hi <=> gx in [lo-1, hi+1]; 2 samples of margin for the roundings
                    const double A = (c0 + m[6] * (1.0 - r.trans[2]) + 1.0) * hr;
                    const double ka = ((double)(lo - 1) - A) * invB, kb = ((double)(hi + 1) - A) * invB;
                    const double kmin = fmin(ka, kb), kmax = fmax(ka, kb);
                    k_lo = kmin < 0.0 ? 0 : (kmin > (double)R ? R + 1 : (int)floor(kmin) - 2);
                    k_hi = kmax > (double)R ? R : (kmax < 0.0 ? -1 : (int)ceil(kmax) + 2);
                    k_lo = max(k_lo, 0);
                    k_hi = min(k_hi, R);
                }
            }
        }
        // ---------------- first samples of every ray, lane-parallel ----------------
        // Most rays cross within a few samples of their window start: each lane walks the first
        // kLaneSamples samples of its own ray (independent loads in flight), with the same per-
        // sample arithmetic and the same scan order as the warp walk below, which takes over
        // (from sample k_lo + kLaneSamples, carrying the last value and the grazing flag) only for
        // the rays still unresolved.
        int my_k1 = -1;
        float my_vhit = 0.0f, my_vprev = 0.0f;
        bool my_graz = false;
        float my_last = 0.0f;  // the sample before the warp walk's start (the one before k_lo is exactly 0)
        int k_lo2 = k_lo;
        if (valid && k_lo <= k_hi) {
            const size_t byz = nn * ((size_t)j0 + nn * (size_t)kk0);
            auto sample_own = [&](int k) -> float {
                float v = 0.0f;
                const double w0 = __dadd_rn(c0, mv_tab[0][k]);
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
                    const double w1 = __dadd_rn(c1, mv_tab[1][k]);
                    const double w2 = __dadd_rn(c2, mv_tab[2][k]);
                    const float gy = (float)__dmul_rn(__dadd_rn(w1, 1.0), hr);
                    const float gk = (float)__dmul_rn(__dsub_rn(1.0, w2), hr);
                    v = sample_grid(r.values, R, gx, gy, gk);
                }
                return v;
            };
            bool done = false;
#pragma unroll
            for (int g = 0; g < kLaneSamples; g += 4) {
                if (!done) {
                    float v[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int k = k_lo + g + e;
                        v[e] = k <= k_hi ? sample_own(k) : 0.0f;
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int k = k_lo + g + e;
                        if (!done && k <= k_hi) {
                            if (v[e] >= 0.5f) {
                                my_k1 = k;
                                my_vhit = v[e];
                                my_vprev = my_last;
                                done = true;
                            } else {
                                my_graz |= v[e] > 0.0f && v[e] < 1.0f;  // render.hpp:180-188
                                my_last = v[e];
                            }
                        }
                    }
                }
            }
            k_lo2 = done ? k_hi + 1 : k_lo + kLaneSamples;
        }
        // ---------------- the remaining rays, one at a time across the warp ----------------
        unsigned todo = __ballot_sync(0xffffffffu, valid && k_lo2 <= k_hi);
        while (todo) {
            const int p = __ffs(todo) - 1;
            todo &= todo - 1;
            const double pc0 = __shfl_sync(0xffffffffu, c0, p);
            const double pc1 = __shfl_sync(0xffffffffu, c1, p);
            const double pc2 = __shfl_sync(0xffffffffu, c2, p);
            const bool pxray = __shfl_sync(0xffffffffu, (int)xray, p) != 0;
            const bool pyz_in = __shfl_sync(0xffffffffu, (int)yz_in, p) != 0;
            const int pj0 = __shfl_sync(0xffffffffu, j0, p), pkk0 = __shfl_sync(0xffffffffu, kk0, p);
            const float pfy = __shfl_sync(0xffffffffu, fy, p), pfk = __shfl_sync(0xffffffffu, fk, p);
            const int plo = __shfl_sync(0xffffffffu, k_lo2, p), phi = __shfl_sync(0xffffffffu, k_hi, p);
            const float plast = __shfl_sync(0xffffffffu, my_last, p);
            const bool pgraz = __shfl_sync(0xffffffffu, (int)my_graz, p) != 0;
            const size_t byz = nn * ((size_t)pj0 + nn * (size_t)pkk0);
            auto sample_at = [&](int k) -> float {
                float v = 0.0f;
                const double w0 = __dadd_rn(pc0, mv_tab[0][k]);
                const float gx = (float)__dmul_rn(__dadd_rn(w0, 1.0), hr);
                if (pxray) {
                    if (pyz_in && gx >= 0.0f && gx <= fR) {
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
                        const float cy0 = lerp_rn(c00, c10, pfy);
                        const float cy1 = lerp_rn(c01, c11, pfy);
                        v = lerp_rn(cy0, cy1, pfk);
                    }
                } else {
                    const double w1 = __dadd_rn(pc1, mv_tab[1][k]);
                    const double w2 = __dadd_rn(pc2, mv_tab[2][k]);
                    const float gy = (float)__dmul_rn(__dadd_rn(w1, 1.0), hr);
                    const float gk = (float)__dmul_rn(__dsub_rn(1.0, w2), hr);
                    v = sample_grid(r.values, R, gx, gy, gk);
                }
                return v;
            };
            int k1 = -1;
            float vprev = 0.0f, vhit = 0.0f, last = plast;  // the lane-parallel samples' last value
            bool grazing = pgraz;
            for (int kb = plo; kb <= phi; kb += 32) {
                const int k = kb + lane;
                const float v = k <= phi ? sample_at(k) : 0.0f;
                const unsigned hit = __ballot_sync(0xffffffffu, k <= phi && v >= 0.5f);
                const int first = hit ? __ffs(hit) - 1 : 32;
                // samples before the crossing: grazing (0 < v < 1), render.hpp:180-188
                grazing |= __ballot_sync(0xffffffffu, lane < first && k <= phi && v > 0.0f && v < 1.0f) != 0u;
                const float prev_in_chunk = __shfl_up_sync(0xffffffffu, v, 1);
                if (hit) {
                    k1 = kb + first;
                    vhit = __shfl_sync(0xffffffffu, v, first);
                    const float pv = __shfl_sync(0xffffffffu, prev_in_chunk, first);
                    vprev = first > 0 ? pv : last;
                    break;
                }
                last = __shfl_sync(0xffffffffu, v, 31);
            }
            if (lane == p) {
                my_k1 = k1;
                my_vhit = vhit;
                my_vprev = vprev;
                my_graz = grazing;
            }
        }
        // ---------------- outputs, lane-parallel ----------------
        const bool cov = valid && my_k1 >= 0;
        const unsigned covm = __ballot_sync(0xffffffffu, cov);
        unsigned pos0 = 0;
        if (covm) {  // the warp's surface points take one contiguous range of the compact list
            if (lane == 0) pos0 = atomicAdd(&r.ctr->surface_count, (unsigned)__popc(covm));
            pos0 = __shfl_sync(0xffffffffu, pos0, 0);
        }
        if (valid) {
            r.rgb[3 * (size_t)px + 0] = r.bg[0];
            r.rgb[3 * (size_t)px + 1] = r.bg[1];
            r.rgb[3 * (size_t)px + 2] = r.bg[2];
            if (!cov) {
                r.depth[px] = -2.0f;  // kInvalidDepth, render.hpp:72
                r.mask[px] = 0;
                if (r.surface_k) r.surface_k[px] = -1;
                n_graz += my_graz ? 1 : 0;
            } else {
                ++n_cov;
                double sv = 1.0;
                if (my_k1 > 0) {
                    const double v1d = (double)my_vhit, v0d = (double)my_vprev;
                    const double denom = __dsub_rn(v1d, v0d);
                    if (denom > 0.0) {
                        sv = __ddiv_rn(__dsub_rn(0.5, v0d), denom);
                        sv = sv < 0.0 ? 0.0 : (sv > 1.0 ? 1.0 : sv);
                    } else {
                        ++n_deg;
                    }
                }
                const double depth =
                    __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, __dadd_rn(__dsub_rn((double)my_k1, 1.0), sv)), (double)R));
                r.depth[px] = (float)depth;
                r.mask[px] = 1;
                if (r.surface_k) r.surface_k[px] = my_k1;
                // view_to_world(vx, vy, depth) = c + m[6..8] (depth - t2): the hoisted terms again
                const double v2 = __dsub_rn(depth, r.trans[2]);
                const unsigned pos = pos0 + (unsigned)__popc(covm & ((1u << lane) - 1u));
                r.surface_pts[3 * (size_t)pos + 0] = __dadd_rn(c0, __dmul_rn(m[6], v2));
                r.surface_pts[3 * (size_t)pos + 1] = __dadd_rn(c1, __dmul_rn(m[7], v2));
                r.surface_pts[3 * (size_t)pos + 2] = __dadd_rn(c2, __dmul_rn(m[8], v2));
                r.surface_px[pos] = px;
            }
        }
    }
    // block-level counter totals
    for (int o = 16; o > 0; o >>= 1) {
        n_cov += __shfl_xor_sync(0xffffffffu, n_cov, o);
        n_deg += __shfl_xor_sync(0xffffffffu, n_deg, o);
        n_graz += __shfl_xor_sync(0xffffffffu, n_graz, o);
    }
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
        for (int g0 = 0; g0 < n; g0 += 32 * 8) {  // 8 chunks of 32 in flight per lane
            float v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int i = g0 + 32 * c + lane;
                v[c] = i < n ? __ldg(&row[i]) : 0.0f;
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const unsigned nz = __ballot_sync(0xffffffffu, v[c] != 0.0f);
                if (nz) {
                    const int i0 = g0 + 32 * c;
                    if (first == n) first = i0 + __ffs(nz) - 1;
                    last = i0 + 31 - __clz(nz);
                }
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
    if (npx >= (1ull << 32)) {
        set_error("render: too many pixels");
        return ICG_EINVAL;
    }
    const int nt = r.width + r.height + r.cells + 1;
    k_render_setup<<<(nt + 255) / 256, 256, 0, s>>>(r);
    const size_t warps = (npx + 31) / 32;  // 32 pixels per warp
    // one 32-pixel group per warp (up to 64 blocks per SM): the hardware block scheduler balances the
    // groups' very different ray walks (a grid-stride loop over one resident wave left ~half of the
    // warps idle at the end)
    const size_t blocks = std::min<size_t>((warps + kRenderThreads / 32 - 1) / (kRenderThreads / 32), 148 * 64);
    k_render<<<(unsigned)blocks, kRenderThreads, 0, s>>>(r);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

}  // namespace icg

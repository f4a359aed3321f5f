// k_tail.cu — the tail of the conflict loop (localize.hpp:334-354) as ONE persistent kernel.
//
// After its first few iterations the conflict loop of a level is a chain of
// dependent batches of ~10-500 nodes (256^3 level 3: ~17 of its 22 iterations).
// Launched per iteration, each link pays several kernel launches and a full
// MLP latency.  This cooperative kernel (one CTA per SM) instead runs every
// remaining iteration of the level itself:
//
//   expand   collect_unevaluated_neighbors (localize.hpp:160-177) of the conflict
//            list into the next batch (queued bitmask dedupe, as k_conflict_expand)
//            and claims a column record for every column not seen before
//   columns  Phi gather + the Phi part of every layer for the new columns (the
//            COLS record of k_mlp_pair.cu, here on CUDA cores)
//   h1       act(S1[col] + w1z z + b1): layer 1 of the column-factored field
//   L2..L4   layer-parallel fp32: CTA c owns output rows r = c (mod grid) of
//            each layer, their hidden-input weights resident in shared memory;
//            a warp computes all owned rows of one point (lanes split K, fixed
//            order: a node's value does not depend on its batch)
//   final    output dot + Phi dot + z + bias - sdf_scale * sdf, sigmoid, the
//            grid epilogue of evaluate_nodes fused with the conflict test
//            (localize.hpp:86-88, 341-342)
//
// with grid barriers between phases and no host involvement until the chain
// ends.  The kernel only starts when the current batch is small (the CTA-pair
// tensor-core kernel takes large ones); once started it finishes the level,
// then clears the loop's counters so the launches the host unrolled after it
// find nothing to do.  Evaluation counts and iteration counts follow the
// reference exactly (evals += batch, iters += 1 per non-empty batch).
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "eval_common.cuh"

namespace cg = cooperative_groups;

namespace icg {

namespace tail {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRec = 1936;  // column record floats (k_mlp_pair.cu kSRow)
// Grid size: every activation is read by every CTA (rows are partitioned), so more CTAs mean
// less work but more broadcast per CTA.  The kernel is cooperative and holds its SMs for the whole
// chain while doing little: with other frames in flight on the device a 64-CTA grid leaves SMs to
// them (222 vs 191 frames/s with 3 in flight), while a frame alone on the device takes the
// 148-CTA grid (lower latency).  Both are instantiated; launch_tail picks.
constexpr int kSRows = 1921;  // Phi rows of a record: 1024 + 512 + 256 + 128 + final dot
constexpr int kPB = 16;       // points per staged activation block

template <int G>
struct TailCfg {
    static constexpr int kMaxOwn2 = (512 + G - 1) / G, kMaxOwn3 = (256 + G - 1) / G, kMaxOwn4 = (128 + G - 1) / G;
    static constexpr int kMaxOwnS = (kSRows + G - 1) / G;
    // double-buffer the staged activations when the resident weights leave room for it
    static constexpr size_t kWeightBytes =
        4 * ((size_t)kMaxOwn2 * 1024 + (size_t)kMaxOwn3 * 512 + (size_t)kMaxOwn4 * 256 + (size_t)kMaxOwnS * 256 + 128);
    static constexpr int kStageBufs = kWeightBytes + 2 * (size_t)kPB * 1024 * 4 <= 220 * 1024 ? 2 : 1;
    struct Smem {
        float w2[kMaxOwn2][1024];
        float w3[kMaxOwn3][512];
        float w4[kMaxOwn4][256];
        float wphi[kMaxOwnS][256];
        float wlast[128];
        alignas(16) float stage[kStageBufs][kPB * 1024];  // activations of kPB points (layer input)
    };
};

__host__ __device__ constexpr int rec_row_layer(int r) { return r < 1024 ? 0 : r < 1536 ? 1 : r < 1792 ? 2 : r < 1920 ? 3 : 4; }

__device__ __forceinline__ float leaky(float x, float s) { return x < 0.0f ? x * s : x; }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int kG>
__global__ void __launch_bounds__(kThreads, 1) k_tail(TailParams P) {
    using TC = TailCfg<kG>;
    using Smem = typename TC::Smem;
    constexpr int kMaxOwn2 = TC::kMaxOwn2, kMaxOwn3 = TC::kMaxOwn3, kMaxOwn4 = TC::kMaxOwn4, kMaxOwnS = TC::kMaxOwnS;
    constexpr int kStageBufs = TC::kStageBufs;
    DevCounters* ctr = P.ctr;
    {  // grid-uniform start decision: the batch of host iteration it0 is nx[it0 & 1]
        const unsigned n0 = ctr->nx_count[P.it0 & 1];
        if (n0 == 0 || n0 > P.max_start) return;
    }
    cg::grid_group grid = cg::this_grid();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr->tail_start[P.level] = (unsigned)P.it0 + 1u;
        if (P.it0 < kPredIters) ctr->cls[P.level][P.it0] |= 4u;
    }
    int ntr = 0;  // trace (block 0): (tag, globaltimer) pairs
    auto tr = [&](unsigned tag) {
        if (P.trace && blockIdx.x == 0 && threadIdx.x == 0 && ntr < 1000) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            P.trace[2 * ntr] = tag;
            P.trace[2 * ntr + 1] = t;
            ++ntr;
        }
    };
    tr(1);
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    constexpr int G = kG;
    const int cta = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gwarp = cta * kWarps + warp, nwarps = G * kWarps;
    const unsigned gtid = cta * kThreads + tid, nthreads = G * kThreads;
    const float slope = P.slope;
    const int fn = P.cells + 1;
    const uint32_t plane = (uint32_t)fn * (uint32_t)fn;
    const double dcells = (double)P.cells;

    // ---- resident weights: this CTA's rows of layers 2-4 (hidden inputs) and record rows ----
#pragma unroll 8
    for (int i = tid; i < kMaxOwn2 * 1024; i += kThreads) {
        const int a = i / 1024, k = i % 1024, r = cta + a * G;
        sm.w2[a][k] = r < 512 ? __ldg(&P.w[1][(size_t)r * (1024 + kGeoSkip) + k]) : 0.0f;
    }
#pragma unroll 8
    for (int i = tid; i < kMaxOwn3 * 512; i += kThreads) {
        const int a = i / 512, k = i % 512, r = cta + a * G;
        sm.w3[a][k] = r < 256 ? __ldg(&P.w[2][(size_t)r * (512 + kGeoSkip) + k]) : 0.0f;
    }
    for (int i = tid; i < kMaxOwn4 * 256; i += kThreads) {
        const int a = i / 256, k = i % 256, r = cta + a * G;
        sm.w4[a][k] = r < 128 ? __ldg(&P.w[3][(size_t)r * (256 + kGeoSkip) + k]) : 0.0f;
    }
#pragma unroll 8
    for (int i = tid; i < kMaxOwnS * 256; i += kThreads) {
        const int a = i / 256, k = i % 256, r = cta + a * G;
        float v = 0.0f;
        if (r < kSRows) {
            const int l = rec_row_layer(r);
            if (l == 0) v = __ldg(&P.w[0][(size_t)r * kGeoSkip + k]);
            else if (l == 1) v = __ldg(&P.w[1][(size_t)(r - 1024) * (1024 + kGeoSkip) + 1024 + k]);
            else if (l == 2) v = __ldg(&P.w[2][(size_t)(r - 1536) * (512 + kGeoSkip) + 512 + k]);
            else if (l == 3) v = __ldg(&P.w[3][(size_t)(r - 1792) * (256 + kGeoSkip) + 256 + k]);
            else v = __ldg(&P.wlast[128 + k]);
        }
        sm.wphi[a][k] = v;
    }
    for (int i = tid; i < 128; i += kThreads) sm.wlast[i] = __ldg(&P.wlast[i]);

    const float* b1 = P.bias;
    const float* b2 = b1 + 2 * 1024;
    const float* b3 = b2 + 2 * 512;
    const float* b4 = b3 + 2 * 256;
    const float* b5 = b4 + 2 * 128;
    const float w5z = __ldg(&P.wlast[128 + kGeoSkip - 1]);

    // claim a record slot for column col (cmap[col] == -1: new); new slots are listed in P.newcols
    auto claim = [&](uint32_t col) {
        if (P.cmap[col] != -1) return;
        if (atomicCAS(&P.cmap[col], -1, -2) == -1) {
            const unsigned slot = atomicAdd(&ctr->ncols, 1u);
            const unsigned k = atomicAdd(P.nnew, 1u);
            P.newcols[k] = slot;
            P.collist[slot] = col;
            __threadfence();
            atomicExch(&P.cmap[col], (int)slot);
        }
    };

    // entry: the host's expand of iteration it0 produced nx[it0 & 1]; claim its columns
    if (gtid == 0) *P.nnew = 0u;
    grid.sync();
    {
        const int q = P.it0 & 1;
        const unsigned n = __ldcg(&ctr->nx_count[q]);
        for (unsigned t = gtid; t < n; t += nthreads) claim(__ldcg(&P.nx[q][t]) % plane);
    }
    grid.sync();

    tr(2);
    for (int it = P.it0;; ++it) {
        const int q = it & 1;
        const unsigned n = __ldcg(&ctr->nx_count[q]);
        tr(1000000u + n);
        if (n == 0) break;
        const uint32_t* list = P.nx[q];
        // ---- new columns (chunks of the Phi scratch): Phi gather, then their records ----
        const unsigned m = __ldcg(P.nnew);
        for (unsigned c0 = 0; c0 < m; c0 += P.cap_new) {
            const unsigned mc = min(P.cap_new, m - c0);
            for (unsigned c = gwarp; c < mc; c += nwarps) {
                const unsigned slot = __ldcg(&P.newcols[c0 + c]);
                const uint32_t col = __ldcg(&P.collist[slot]);
                const int i = (int)(col % (uint32_t)fn), j = (int)(col / (uint32_t)fn);
                const float x = (float)__dadd_rn(-1.0, __ddiv_rn(2.0 * (double)i, dcells));
                const float y = (float)__dadd_rn(-1.0, __ddiv_rn(2.0 * (double)j, dcells));
                const FieldDev& f = P.f;
                float u = (x + 1.0f) * 0.5f * (float)(f.W - 1);
                float v = (1.0f - y) * 0.5f * (float)(f.H - 1);
                u = fminf(fmaxf(u, 0.0f), (float)(f.W - 1));
                v = fminf(fmaxf(v, 0.0f), (float)(f.H - 1));
                const int x0 = min((int)floorf(u), f.W - 2), y0 = min((int)floorf(v), f.H - 2);
                const float ax = u - (float)x0, ay = v - (float)y0;
                const float w00 = (1.0f - ax) * (1.0f - ay), w10 = ax * (1.0f - ay), w01 = (1.0f - ax) * ay,
                            w11 = ax * ay;
                const float* m00 = f.fmap_hwc + ((size_t)y0 * f.W + x0) * (size_t)f.C;
                const size_t rowW = (size_t)f.W * f.C;
                for (int ch = lane; ch < kC; ch += 32)
                    P.phi[(size_t)c * kC + ch] = w00 * __ldg(&m00[ch]) + w10 * __ldg(&m00[f.C + ch]) +
                                                 w01 * __ldg(&m00[rowW + ch]) + w11 * __ldg(&m00[rowW + f.C + ch]);
            }
            grid.sync();
            tr(3);
            // this CTA's record rows of each new column (warp per column, lanes split the channels)
            for (unsigned c = warp; c < mc; c += kWarps) {
                const unsigned slot = __ldcg(&P.newcols[c0 + c]);
                float ph[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) ph[e] = __ldcg(&P.phi[(size_t)c * kC + lane + 32 * e]);
                for (int a = 0; a < kMaxOwnS; ++a) {
                    const int r = cta + a * G;
                    if (r >= kSRows) break;
                    float acc = 0.0f;
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc = fmaf(sm.wphi[a][lane + 32 * e], ph[e], acc);
                    acc = warp_sum(acc);
                    if (lane == 0) P.colrec[(size_t)slot * kRec + r] = acc;
                }
            }
            grid.sync();
        }
        // every CTA read *P.nnew before the record phase's barriers; the claims that count it
        // again come after this iteration's layer barriers
        if (m > 0 && gtid == 0) *P.nnew = 0u;
        // ---- process the batch in chunks of the scratch capacity ----
        for (unsigned base = 0; base < n; base += P.cap_pts) {
            const unsigned nc = min(P.cap_pts, n - base);
            // h1 = act(S1 + w1z z + b1), per point: node info
            for (unsigned e = gtid; e < nc * 1024u; e += nthreads) {
                const unsigned t = e / 1024u, k = e % 1024u;
                const uint32_t node = __ldcg(&list[base + t]);
                const uint32_t col = node % plane;
                const int slot = __ldcg(&P.cmap[col]);
                const int kk = (int)(node / plane);
                const float z = (float)__dsub_rn(1.0, __ddiv_rn(2.0 * (double)kk, dcells));
                P.h1[(size_t)t * 1024 + k] =
                    leaky(__ldcg(&P.colrec[(size_t)slot * kRec + k]) + fmaf(__ldg(&b1[1024 + k]), z, __ldg(&b1[k])), slope);
                if (k == 0) {
                    P.pslot[t] = slot;
                    P.pz[t] = z;
                }
            }
            grid.sync();
            // layers 2-4: this CTA's rows for every point of the chunk.  Activations arriving from
            // other CTAs are staged per block of kPB points in shared memory (coalesced L2 loads,
            // all in flight), then a warp computes (owned row, point) dot products from it.
            auto layer = [&](const float* hin, int K, const float* wrows, int nown, int rows, int soff,
                             const float* bl, float* hout) {
                // double-buffered: the next block's copies are in flight while this one is computed
                auto issue = [&](unsigned pb, int buf) {
                    const unsigned np = min((unsigned)kPB, nc - pb);
                    const float4* src = reinterpret_cast<const float4*>(hin + (size_t)pb * K);
                    float4* dst = reinterpret_cast<float4*>(sm.stage[buf]);
                    const unsigned nv = np * (unsigned)K / 4u;
                    for (unsigned e = tid; e < nv; e += kThreads) {  // 16-byte copies, L2 only
                        const uint32_t d = (uint32_t)__cvta_generic_to_shared(&dst[e]);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(&src[e]) : "memory");
                    }
                    asm volatile("cp.async.commit_group;" ::: "memory");
                };
                issue(0, 0);
                int b = 0;
                static_assert(kStageBufs == 1 || kStageBufs == 2, "stage buffers");
                for (unsigned pb = 0; pb < nc; pb += kPB, ++b) {
                    const unsigned np = min((unsigned)kPB, nc - pb);
                    if (kStageBufs == 2 && pb + kPB < nc) {
                        issue(pb + kPB, (b + 1) & 1);
                        asm volatile("cp.async.wait_group 1;" ::: "memory");
                    } else {
                        asm volatile("cp.async.wait_group 0;" ::: "memory");
                    }
                    __syncthreads();
                    const float* stage = sm.stage[kStageBufs == 2 ? (b & 1) : 0];
                    for (unsigned t = warp; t < np; t += kWarps) {
                        const float* h = stage + (size_t)t * K;
                        const unsigned tt = pb + t;
                        // this point's per-row epilogue operands (lane a < nown: row a), loaded before
                        // the dot so their latency overlaps it
                        const int r_l = cta + lane * G;
                        float pre_s = 0.0f, pre_b = 0.0f, pre_w = 0.0f, z = 0.0f;
                        {
                            const int slot = __ldcg(&P.pslot[tt]);
                            z = __ldcg(&P.pz[tt]);
                            if (lane < nown && r_l < rows) {
                                pre_s = __ldcg(&P.colrec[(size_t)slot * kRec + soff + r_l]);
                                pre_b = __ldg(&bl[r_l]);
                                pre_w = __ldg(&bl[rows + r_l]);
                            }
                        }
                        float acc[kMaxOwn2];
#pragma unroll
                        for (int a = 0; a < kMaxOwn2; ++a) acc[a] = 0.0f;
                        // the rows' (absent rows: zero weights) dots with one point, lanes split K
#pragma unroll 2
                        for (int k = lane; k < K; k += 32) {
                            const float x = h[k];
#pragma unroll
                            for (int a = 0; a < kMaxOwn2; ++a)
                                if (a < nown) acc[a] = fmaf(wrows[(size_t)a * K + k], x, acc[a]);
                        }
                        float mine = 0.0f;
#pragma unroll
                        for (int a = 0; a < kMaxOwn2; ++a) {
                            if (a >= nown) break;
                            const float sum = warp_sum(acc[a]);
                            if (lane == a) mine = sum;
                        }
                        if (lane < nown && r_l < rows)
                            hout[(size_t)tt * rows + r_l] = leaky(mine + pre_s + fmaf(pre_w, z, pre_b), slope);
                    }
                    __syncthreads();
                    if (kStageBufs == 1 && pb + kPB < nc) issue(pb + kPB, 0);  // single buffer: refill now
                }
            };
            tr(5);
            layer(P.h1, 1024, &sm.w2[0][0], kMaxOwn2, 512, 1024, b2, P.h2);
            grid.sync();
            tr(6);
            layer(P.h2, 512, &sm.w3[0][0], kMaxOwn3, 256, 1536, b3, P.h3);
            grid.sync();
            tr(7);
            layer(P.h3, 256, &sm.w4[0][0], kMaxOwn4, 128, 1792, b4, P.h4);
            grid.sync();
            tr(8);
            // final layer + sdf bias + sigmoid + grid epilogue with the conflict test
            for (unsigned t = gwarp; t < nc; t += nwarps) {
                const float* h = P.h4 + (size_t)t * 128;
                float acc = 0.0f;
#pragma unroll
                for (int e = 0; e < 4; ++e) acc = fmaf(sm.wlast[lane + 32 * e], __ldcg(&h[lane + 32 * e]), acc);
                acc = warp_sum(acc);
                const uint32_t node = __ldcg(&list[base + t]);
                float pos[3];
                node_pos_f(node, P.cells, pos);
                // union sdf: lane i takes primitives i, i + 32, ... (same per-primitive arithmetic)
                float d = 3.0e38f;
                const int nprim = __ldg(&P.f.fscene->n_prims);
                for (int i = lane; i < nprim; i += 32) d = fminf(d, prim_sdf_f(&P.f.fscene->prims[i], pos));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) d = fminf(d, __shfl_xor_sync(0xffffffffu, d, o));
                if (lane == 0) {
                    const int slot = __ldcg(&P.pslot[t]);
                    const float sdf = nprim > 0 ? d : 0.0f;
                    const float s = acc + __ldcg(&P.colrec[(size_t)slot * kRec + 1920]) +
                                    (__ldg(&b5[0]) + w5z * __ldcg(&P.pz[t]) - __ldg(&P.f.fscene->sdf_scale) * sdf);
                    const float v = 1.0f / (1.0f + expf(-s));
                    EvalJob j{};
                    j.cells = P.cells;
                    j.xext = P.xext;
                    j.values = P.fv;
                    j.states = P.fs;
                    j.tentbin = P.tentbin;
                    j.conflicts = P.cf[q ^ 1];
                    j.conflict_count = &ctr->cf_count[q ^ 1];
                    j.conflict_cap = P.cap;
                    j.overflow = &ctr->overflow;
                    grid_epilogue(j, node, v);
                }
            }
            grid.sync();
        }
        tr(9);
        if (gtid == 0) {
            ctr->evals[P.level] += n;
            ctr->conflict_iters[P.level] += 1u;
        }
        // ---- expand for iteration it + 1 (k_conflict_expand with p = (it + 1) & 1) ----
        const int p = q ^ 1;
        const unsigned ncf = __ldcg(&ctr->cf_count[p]);
        // the counters reset here (cf / nx of parity q) were last read before earlier barriers
        if (gtid == 0) {
            ctr->cf_count[p ^ 1] = 0;
            ctr->nx_count[p ^ 1] = 0;
            if (ncf > 0 && it + 1 >= P.max_iters) ctr->warning = 1;  // localize.hpp:343-346
        }
        tr(2000000u + ncf);
        if (ncf == 0 || it + 1 >= P.max_iters) break;
        const uint32_t* conf = P.cf[p];
        const size_t total = (size_t)ncf * 26;
        for (size_t e = gtid; e < total; e += nthreads) {
            const unsigned c = (unsigned)(e / 26);
            int r = (int)(e % 26);
            if (r >= 13) ++r;
            const int di = r % 3 - 1, dj = (r / 3) % 3 - 1, dk = r / 9 - 1;
            const uint32_t idx = __ldcg(&conf[c]);
            const int i = (int)(idx % (uint32_t)fn), j = (int)((idx / (uint32_t)fn) % (uint32_t)fn),
                      k = (int)(idx / plane);
            const int ii = i + di, jj = j + dj, kk = k + dk;
            if (ii < 0 || jj < 0 || kk < 0 || ii >= fn || jj >= fn || kk >= fn) continue;
            const uint32_t nb = (uint32_t)ii + (uint32_t)fn * ((uint32_t)jj + (uint32_t)fn * (uint32_t)kk);
            if (__ldcg(&P.fs[nb]) == ICG_STATE_EVALUATED) continue;
            const unsigned bit = 1u << (nb & 31);
            if (atomicOr(&P.queued[nb >> 5], bit) & bit) continue;
            const unsigned pos = atomicAdd(&ctr->nx_count[p], 1u);
            if (pos < P.cap)
                P.nx[p][pos] = nb;
            else
                ctr->overflow = 1;
            claim(nb % plane);
        }
        grid.sync();
    }
    // the chain is finished: the host-unrolled launches after this one must find nothing to do
    tr(10);
    grid.sync();
    if (gtid == 0) {
        ctr->cf_count[0] = ctr->cf_count[1] = 0;
        ctr->nx_count[0] = ctr->nx_count[1] = 0;
    }
}

}  // namespace tail

size_t tail_smem_bytes() { return sizeof(tail::TailCfg<148>::Smem); }

// scratch: per-point activations for cap_pts points, Phi of cap_new columns, the new-column list
// (up to max_cols entries: every column of the level)
size_t tail_scratch_bytes(unsigned cap_pts, unsigned cap_new, unsigned max_cols) {
    return (size_t)cap_pts * (1024 + 512 + 256 + 128 + 2) * 4 + (size_t)cap_new * kC * 4 + (size_t)max_cols * 4 + 256;
}

template <int G>
static int tail_setup(int sms) {
    const size_t smem = sizeof(typename tail::TailCfg<G>::Smem);
    ICG_CUDA_TRY(cudaFuncSetAttribute(tail::k_tail<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per = 0;
    ICG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tail::k_tail<G>, tail::kThreads, smem));
    if (per < 1 || sms < G) {
        set_error("k_tail: does not fit the device");
        return ICG_ERUNTIME;
    }
    return ICG_OK;
}

// CTAs of the tail when other frames share the device (ICG_TAIL_SHARED=32|64, default 32: the
// cooperative kernel holds its SMs for the whole chain; 32 CTAs gave 375 vs 363 frames/s at 4 in flight)
static int shared_width() {
    static const int w = [] {
        const char* e = getenv("ICG_TAIL_SHARED");
        return e && atoi(e) == 64 ? 64 : 32;
    }();
    return w;
}

// wide: the frame is alone on the device (148-CTA grid, lower latency); otherwise 64 CTAs
int launch_tail(TailParams p, uint8_t* scratch, unsigned cap_pts, unsigned cap_new, unsigned max_cols, cudaStream_t s,
                bool wide) {
    static PerDeviceOnce once;
    if (int r = once.run([] {
            int dev = 0, sms = 0;
            ICG_CUDA_TRY(cudaGetDevice(&dev));
            ICG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            if (int e = tail_setup<32>(sms)) return e;
            if (int e = tail_setup<64>(sms)) return e;
            return tail_setup<148>(sms);
        }))
        return r;
    uint8_t* q = scratch;
    p.h1 = reinterpret_cast<float*>(q);
    q += (size_t)cap_pts * 1024 * 4;
    p.h2 = reinterpret_cast<float*>(q);
    q += (size_t)cap_pts * 512 * 4;
    p.h3 = reinterpret_cast<float*>(q);
    q += (size_t)cap_pts * 256 * 4;
    p.h4 = reinterpret_cast<float*>(q);
    q += (size_t)cap_pts * 128 * 4;
    p.pz = reinterpret_cast<float*>(q);
    q += (size_t)cap_pts * 4;
    p.pslot = reinterpret_cast<int*>(q);
    q += (size_t)cap_pts * 4;
    p.phi = reinterpret_cast<float*>(q);
    q += (size_t)cap_new * kC * 4;
    p.newcols = reinterpret_cast<unsigned*>(q);
    q += (size_t)max_cols * 4;
    p.nnew = reinterpret_cast<unsigned*>(q);
    p.cap_pts = cap_pts;
    p.cap_new = cap_new;
    // dev trace buffer (ICG_TAIL_TRACE=1), created once (thread-safe static initialisation)
    static unsigned long long* const trace = [] {
        const char* e = getenv("ICG_TAIL_TRACE");
        unsigned long long* t = nullptr;
        if (e && e[0] == '1' && cudaMallocManaged(&t, 2000 * sizeof(unsigned long long)) != cudaSuccess) t = nullptr;
        return t;
    }();
    p.trace = trace;
    if (p.trace) cudaMemsetAsync(p.trace, 0, 2000 * 8, s);
    void* args[] = {&p};
    if (wide)
        ICG_CUDA_TRY(cudaLaunchCooperativeKernel((void*)tail::k_tail<148>, 148, tail::kThreads, args,
                                                 sizeof(tail::TailCfg<148>::Smem), s));
    else if (shared_width() == 32)
        ICG_CUDA_TRY(cudaLaunchCooperativeKernel((void*)tail::k_tail<32>, 32, tail::kThreads, args,
                                                 sizeof(tail::TailCfg<32>::Smem), s));
    else
        ICG_CUDA_TRY(cudaLaunchCooperativeKernel((void*)tail::k_tail<64>, 64, tail::kThreads, args,
                                                 sizeof(tail::TailCfg<64>::Smem), s));
    if (p.trace) {
        cudaStreamSynchronize(s);
        if (trace[1]) {
            fprintf(stderr, "[tail-trace level %d it0 %d]", p.level, p.it0);
            for (int i = 1; i < 1000 && trace[2 * i + 1]; ++i) {
                const unsigned long long tag = trace[2 * i];
                const double dt = (trace[2 * i + 1] - trace[2 * i - 1]) * 1e-3;
                if (tag >= 2000000ull) fprintf(stderr, " |cf=%llu", tag - 2000000ull);
                else if (tag >= 1000000ull) fprintf(stderr, "\n   n=%llu(+%.1f)", tag - 1000000ull, dt);
                else fprintf(stderr, " %llu:%.1f", tag, dt);
            }
            fprintf(stderr, "\n");
        }
    }
    return ICG_OK;
}

}  // namespace icg

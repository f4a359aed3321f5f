// k_mc.cu — marching cubes over a localized grid on the GPU (the reference's
// marching_cubes, mesh.hpp:75-156, and export_obj, :159-172).
//
// Same lattice conventions as the reference: cell corners in the Bourke order (mesh.hpp:36-40),
// a cell edge keyed by its lower endpoint node and axis (:42-46) so neighbouring cells share one
// vertex per crossed grid edge, corner bit set where v < iso, vertex = lerp(node_a, node_b, t)
// with t = clamp((iso - v0) / (v1 - v0), 0, 1) in fp64 (0.5 for a zero denominator), vertices at
// bit-identical positions welded (on a grid edge that happens only at t = 0 or 1, i.e. at a
// node, so the weld key is the node), degenerate (repeated-vertex or < 1e-12 area) triangles
// dropped and vertices numbered in order of first use.
//
// The triangulation table is NOT the reference's (its Bourke table is not copied): it is
// generated at load time by walking the cube faces.  On every face the crossed edges are
// paired so that each maximal run of below-iso corners is cut off on its own (the same rule on
// both sides of a shared face keeps the mesh watertight); the oriented face segments chain into
// closed loops, each fanned into triangles.  Crossed edges -- hence the vertex set -- are the
// reference's; the triangles of a polygon may differ.
//
// Device passes: per cell the case and its triangle count (block totals), a scan, the emit pass
// writing each triangle as three weld keys (cell order), key marking, the ordered key list,
// per-triangle degenerate test, first-use ordering of the surviving vertices.
#include <cstring>
#include <vector>

#include "icg_internal.h"

namespace icg {

namespace mc {

// Bourke corner offsets and edges (corner pairs); the edge's lower endpoint and axis
constexpr int kCorner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
constexpr int kEdgeEnds[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6}, {6, 7}, {7, 4},
                                  {0, 4}, {1, 5}, {2, 6}, {3, 7}};
constexpr int kEdgeBase[12] = {0, 1, 3, 0, 4, 5, 7, 4, 0, 1, 2, 3};
constexpr int kEdgeAxis[12] = {0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2};

// device copies of the lattice conventions
__constant__ int8_t d_corner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
__constant__ int8_t d_edge_base[12] = {0, 1, 3, 0, 4, 5, 7, 4, 0, 1, 2, 3};
__constant__ int8_t d_edge_axis[12] = {0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2};

struct Tables {
    int8_t tri[256][16];  // edge indices, 3 per triangle, -1 terminated
    uint8_t ntri[256];
};

__constant__ Tables c_tables;

// faces as corner cycles, counter-clockwise seen from outside the cube
constexpr int kFace[6][4] = {{0, 3, 2, 1}, {4, 5, 6, 7}, {0, 1, 5, 4}, {2, 3, 7, 6}, {0, 4, 7, 3}, {1, 2, 6, 5}};

int edge_of(int a, int b) {
    for (int e = 0; e < 12; ++e)
        if ((kEdgeEnds[e][0] == a && kEdgeEnds[e][1] == b) || (kEdgeEnds[e][0] == b && kEdgeEnds[e][1] == a)) return e;
    return -1;
}

// triangulation of every case (bit c set: corner c below iso)
int build_tables(Tables& t) {
    std::memset(&t, 0xFF, sizeof(t));
    for (int cs = 0; cs < 256; ++cs) {
        // next[e]: the crossed edge a segment from e leads to (each crossed edge starts one segment)
        int next[12];
        for (int& x : next) x = -1;
        for (const auto& f : kFace) {
            for (int s = 0; s < 4; ++s) {
                const int a = f[s], b = f[(s + 1) % 4];
                const bool ba = (cs >> a) & 1, bb = (cs >> b) & 1;
                if (!(!ba && bb)) continue;  // a run of below corners starts at b
                // walk the run to its end
                int q = (s + 1) % 4;
                while ((cs >> f[(q + 1) % 4]) & 1) q = (q + 1) % 4;
                const int e0 = edge_of(a, b), e1 = edge_of(f[q], f[(q + 1) % 4]);
                if (next[e0] != -1) return ICG_ERUNTIME;
                next[e0] = e1;
            }
        }
        int n = 0;
        bool seen[12] = {};
        for (int e = 0; e < 12; ++e) {
            if (next[e] < 0 || seen[e]) continue;
            int loop[12], len = 0;
            for (int x = e; !seen[x]; x = next[x]) {
                if (x < 0 || len >= 12) return ICG_ERUNTIME;
                seen[x] = true;
                loop[len++] = x;
            }
            for (int v = 1; v + 1 < len; ++v) {  // fan, wound like the reference's table
                if (n >= 5) return ICG_ERUNTIME;
                t.tri[cs][3 * n] = (int8_t)loop[0];
                t.tri[cs][3 * n + 1] = (int8_t)loop[v + 1];
                t.tri[cs][3 * n + 2] = (int8_t)loop[v];
                ++n;
            }
        }
        t.ntri[cs] = (uint8_t)n;
    }
    return ICG_OK;
}

// pass 1: triangles per cell, summed per block of 1024 cells
__global__ void __launch_bounds__(1024) k_mc_count(const float* __restrict__ v, int cells, double iso,
                                                   uint32_t* __restrict__ block_tris) {
    __shared__ unsigned ws[32];
    const unsigned long long ncell = (unsigned long long)cells * cells * cells;
    const unsigned long long c = (unsigned long long)blockIdx.x * 1024 + threadIdx.x;
    unsigned nt = 0;
    if (c < ncell) {
        const unsigned jk = (unsigned)(c / cells), i = (unsigned)(c - (unsigned long long)jk * cells);
        const unsigned k = jk / cells, j = jk - k * cells;
        unsigned cs = 0;
        const unsigned n = cells + 1;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const size_t idx = (i + d_corner[q][0]) + (size_t)n * ((j + d_corner[q][1]) + (size_t)n * (k + d_corner[q][2]));
            if ((double)v[idx] < iso) cs |= 1u << q;
        }
        nt = c_tables.ntri[cs];
    }
    unsigned s = nt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned x = ws[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (threadIdx.x == 0) block_tris[blockIdx.x] = x;
    }
}

// grid.hpp:50-53 node position and lerp (geom.hpp:39), reference operation order
__device__ __forceinline__ double node_coord(unsigned i, double r, bool flip) {
    const double q = __ddiv_rn(__dmul_rn(2.0, (double)i), r);
    return flip ? __dsub_rn(1.0, q) : __dadd_rn(-1.0, q);
}

// weld key of the vertex on edge e of cell (i, j, k): 4 * node + axis, or 4 * node + 3 when the
// interpolant lands on a node (t = 0 or 1)
__device__ __forceinline__ uint32_t edge_key(const float* __restrict__ v, unsigned i, unsigned j, unsigned k,
                                                       unsigned n, int e, double iso) {
    const int8_t* o = d_corner[d_edge_base[e]];
    const unsigned a0 = i + o[0], a1 = j + o[1], a2 = k + o[2];
    const int ax = d_edge_axis[e];
    const unsigned long long na = a0 + (unsigned long long)n * (a1 + (unsigned long long)n * a2);
    const unsigned long long nb = na + (ax == 0 ? 1ull : ax == 1 ? (unsigned long long)n : (unsigned long long)n * n);
    const double v0 = (double)v[na], v1 = (double)v[nb];
    const double den = __dsub_rn(v1, v0);
    double t = fabs(den) < 1e-300 ? 0.5 : __ddiv_rn(__dsub_rn(iso, v0), den);
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    if (t == 0.0) return (uint32_t)(4ull * na + 3ull);
    if (t == 1.0) return (uint32_t)(4ull * nb + 3ull);
    return (uint32_t)(4ull * na + (unsigned long long)ax);
}

// pass 2: each cell's triangles as weld keys at the cell's offset (cell order, deterministic);
// offsets: exclusive block totals, then the in-block scan
__global__ void __launch_bounds__(1024) k_mc_emit(const float* __restrict__ v, int cells, double iso,
                                                  const uint32_t* __restrict__ block_off,
                                                  uint32_t* __restrict__ tri_keys,
                                                  uint32_t* __restrict__ key_bits) {
    __shared__ unsigned ws[32];
    const unsigned long long ncell = (unsigned long long)cells * cells * cells;
    const unsigned long long c = (unsigned long long)blockIdx.x * 1024 + threadIdx.x;
    const unsigned n = cells + 1;
    unsigned cs = 0, nt = 0, i = 0, j = 0, k = 0;
    if (c < ncell) {
        const unsigned jk = (unsigned)(c / cells);
        i = (unsigned)(c - (unsigned long long)jk * cells);
        k = jk / cells;
        j = jk - k * cells;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const size_t idx = (i + d_corner[q][0]) + (size_t)n * ((j + d_corner[q][1]) + (size_t)n * (k + d_corner[q][2]));
            if ((double)v[idx] < iso) cs |= 1u << q;
        }
        nt = c_tables.ntri[cs];
    }
    // exclusive scan of nt over the block
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned x = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        const unsigned t = ws[lane];
        unsigned s = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        ws[lane] = s - t;
    }
    __syncthreads();
    if (!nt) return;
    const unsigned long long base = (unsigned long long)block_off[blockIdx.x] + ws[w] + x - nt;
    for (unsigned t = 0; t < nt; ++t)
        for (int q = 0; q < 3; ++q) {
            const uint32_t key = edge_key(v, i, j, k, n, c_tables.tri[cs][3 * t + q], iso);
            tri_keys[3 * (base + t) + q] = key;
            atomicOr(&key_bits[key >> 5], 1u << (key & 31));
        }
}

__device__ unsigned find_key(const uint32_t* __restrict__ keys, unsigned n, uint32_t k) {
    unsigned lo = 0, hi = n;
    while (lo < hi) {
        const unsigned mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// position of a weld key (fp64, reference operation order)
__device__ void key_position(uint32_t key, const float* __restrict__ v, int cells, double iso, double* p) {
    const unsigned n = cells + 1;
    const unsigned long long node = key >> 2;
    const int ax = (int)(key & 3u);
    const unsigned jk = (unsigned)(node / n), i = (unsigned)(node - (unsigned long long)jk * n);
    const unsigned k = jk / n, j = jk - k * n;
    const double r = (double)cells;
    const double a[3] = {node_coord(i, r, false), node_coord(j, r, false), node_coord(k, r, true)};
    if (ax == 3) {
        p[0] = a[0];
        p[1] = a[1];
        p[2] = a[2];
        return;
    }
    const unsigned i1 = i + (ax == 0), j1 = j + (ax == 1), k1 = k + (ax == 2);
    const double b[3] = {node_coord(i1, r, false), node_coord(j1, r, false), node_coord(k1, r, true)};
    const unsigned long long nb = i1 + (unsigned long long)n * (j1 + (unsigned long long)n * k1);
    const double v0 = (double)v[node], v1 = (double)v[nb];
    const double den = __dsub_rn(v1, v0);
    double t = fabs(den) < 1e-300 ? 0.5 : __ddiv_rn(__dsub_rn(iso, v0), den);
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    for (int d = 0; d < 3; ++d) p[d] = __dadd_rn(a[d], __dmul_rn(t, __dsub_rn(b[d], a[d])));
}

// pass 3: per triangle: the weld ids, the degenerate test (repeated vertex or area < 1e-12,
// mesh.hpp:138-142), keep bit; surviving triangles mark each vertex's first use (atomicMin of
// the corner slot)
__global__ void k_mc_filter(const uint32_t* __restrict__ tri_keys, unsigned ntri,
                            const uint32_t* __restrict__ keys, unsigned nkeys, const float* __restrict__ v,
                            int cells, double iso, uint32_t* __restrict__ tri_ids, uint32_t* __restrict__ keep,
                            uint32_t* __restrict__ first_use) {
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = false;
    if (t < ntri) {
        unsigned id[3];
        double p[3][3];
        for (int q = 0; q < 3; ++q) {
            const uint32_t key = tri_keys[3 * (size_t)t + q];
            id[q] = find_key(keys, nkeys, key);
            key_position(key, v, cells, iso, p[q]);
            tri_ids[3 * (size_t)t + q] = id[q];
        }
        ok = id[0] != id[1] && id[1] != id[2] && id[0] != id[2];
        if (ok) {
            // triangle_area (mesh.hpp:29-31): 0.5 |(b - a) x (c - a)|
            const double u[3] = {__dsub_rn(p[1][0], p[0][0]), __dsub_rn(p[1][1], p[0][1]), __dsub_rn(p[1][2], p[0][2])};
            const double w[3] = {__dsub_rn(p[2][0], p[0][0]), __dsub_rn(p[2][1], p[0][1]), __dsub_rn(p[2][2], p[0][2])};
            const double cx = __dsub_rn(__dmul_rn(u[1], w[2]), __dmul_rn(u[2], w[1]));
            const double cy = __dsub_rn(__dmul_rn(u[2], w[0]), __dmul_rn(u[0], w[2]));
            const double cz = __dsub_rn(__dmul_rn(u[0], w[1]), __dmul_rn(u[1], w[0]));
            const double area = __dmul_rn(0.5, sqrt(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz))));
            ok = !(area < 1e-12);
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    if ((threadIdx.x & 31) == 0 && t < ntri) keep[t >> 5] = m;
    if (ok)
        for (int q = 0; q < 3; ++q) atomicMin(&first_use[tri_ids[3 * (size_t)t + q]], 3u * t + (unsigned)q);
}

// pass 4: mark every surviving vertex's first-use slot
__global__ void k_mc_mark_first(const uint32_t* __restrict__ first_use, unsigned nkeys, uint32_t* __restrict__ slot_bits) {
    const unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nkeys && first_use[k] != 0xFFFFFFFFu) atomicOr(&slot_bits[first_use[k] >> 5], 1u << (first_use[k] & 31));
}

// pass 5: vertex i of the output = the key whose first use is the i-th marked slot
__global__ void k_mc_vertices(const uint32_t* __restrict__ slots, unsigned nv, const uint32_t* __restrict__ tri_ids,
                              const uint32_t* __restrict__ keys, const float* __restrict__ v, int cells,
                              double iso, uint32_t* __restrict__ new_id, double* __restrict__ out_v) {
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nv) return;
    const unsigned id = tri_ids[slots[i]];
    new_id[id] = i;
    key_position(keys[id], v, cells, iso, out_v + 3 * (size_t)i);
}

// pass 6: surviving triangles in order, renumbered
__global__ void k_mc_triangles(const uint32_t* __restrict__ tri_list, unsigned nt, const uint32_t* __restrict__ tri_ids,
                               const uint32_t* __restrict__ new_id, int32_t* __restrict__ out_t) {
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nt) return;
    const unsigned t = tri_list[i];
    for (int q = 0; q < 3; ++q) out_t[3 * (size_t)i + q] = (int32_t)new_id[tri_ids[3 * (size_t)t + q]];
}

}  // namespace mc

int mc_init_tables() {
    static PerDeviceOnce once;
    return once.run([] {
        static mc::Tables host;
        static const int built = mc::build_tables(host);  // once per process (thread-safe)
        if (built != ICG_OK) {
            set_error("marching cubes: triangulation table generation failed");
            return ICG_ERUNTIME;
        }
        ICG_CUDA_TRY(cudaMemcpyToSymbol(mc::c_tables, &host, sizeof(host)));
        return ICG_OK;
    });
}

int mc_table_row(int cs, int8_t* out16, int* ntri) {
    mc::Tables t;
    if (int r = mc::build_tables(t)) return r;
    std::memcpy(out16, t.tri[cs & 255], 16);
    *ntri = t.ntri[cs & 255];
    return ICG_OK;
}

}  // namespace icg

extern "C" int icg_mc_case(int cs, int8_t* edges16, int* ntri) {
    if (cs < 0 || cs > 255 || !edges16 || !ntri) {
        icg::set_error("mc_case: bad arguments");
        return ICG_EINVAL;
    }
    return icg::mc_table_row(cs, edges16, ntri);
}

namespace icg {

// launchers (buffers owned by the host runtime)
int launch_mc_count(const float* v, int cells, double iso, uint32_t* block_tris, unsigned nblocks, cudaStream_t s) {
    mc::k_mc_count<<<nblocks, 1024, 0, s>>>(v, cells, iso, block_tris);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}
int launch_mc_emit(const float* v, int cells, double iso, const uint32_t* block_off, unsigned nblocks,
                   uint32_t* tri_keys, uint32_t* key_bits, cudaStream_t s) {
    mc::k_mc_emit<<<nblocks, 1024, 0, s>>>(v, cells, iso, block_off, tri_keys, key_bits);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}
int launch_mc_filter(const uint32_t* tri_keys, unsigned ntri, const uint32_t* keys, unsigned nkeys,
                     const float* v, int cells, double iso, uint32_t* tri_ids, uint32_t* keep, uint32_t* first_use,
                     cudaStream_t s) {
    if (!ntri) return ICG_OK;
    mc::k_mc_filter<<<(ntri + 255) / 256, 256, 0, s>>>(tri_keys, ntri, keys, nkeys, v, cells, iso, tri_ids, keep, first_use);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}
int launch_mc_mark_first(const uint32_t* first_use, unsigned nkeys, uint32_t* slot_bits, cudaStream_t s) {
    if (!nkeys) return ICG_OK;
    mc::k_mc_mark_first<<<(nkeys + 255) / 256, 256, 0, s>>>(first_use, nkeys, slot_bits);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}
int launch_mc_vertices(const uint32_t* slots, unsigned nv, const uint32_t* tri_ids, const uint32_t* keys,
                       const float* v, int cells, double iso, uint32_t* new_id, double* out_v, cudaStream_t s) {
    if (!nv) return ICG_OK;
    mc::k_mc_vertices<<<(nv + 255) / 256, 256, 0, s>>>(slots, nv, tri_ids, keys, v, cells, iso, new_id, out_v);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}
int launch_mc_triangles(const uint32_t* tri_list, unsigned nt, const uint32_t* tri_ids, const uint32_t* new_id,
                        int32_t* out_t, cudaStream_t s) {
    if (!nt) return ICG_OK;
    mc::k_mc_triangles<<<(nt + 255) / 256, 256, 0, s>>>(tri_list, nt, tri_ids, new_id, out_t);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

}  // namespace icg

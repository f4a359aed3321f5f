// eval_common.cuh — shared pieces of every field-evaluation kernel: where the
// points come from (a level's node list, or explicit points) and what happens
// to each result (the grid epilogue of evaluate_nodes, localize.hpp:76-90,
// fused with the conflict test of localize.hpp:341-342).
#pragma once

#include <cuda_runtime.h>

#include "icg_internal.h"

namespace icg {

__device__ __forceinline__ unsigned job_count(const EvalJob& j) { return j.count ? *j.count : j.n_static; }

__device__ __forceinline__ uint32_t job_node(const EvalJob& j, unsigned t) { return j.list ? j.list[t] : t; }

__device__ __forceinline__ bool job_is_grid(const EvalJob& j) { return j.points == nullptr; }

// grid.hpp:50-53 node_position, in double, same operation order.
__device__ __forceinline__ void node_pos_d(uint32_t idx, int cells, double* p) {
    unsigned n = (unsigned)cells + 1u;
    unsigned jk = idx / n, i = idx - jk * n, k = jk / n, j = jk - k * n;
    double r = (double)cells;
    p[0] = __dadd_rn(-1.0, __ddiv_rn(2.0 * (double)i, r));
    p[1] = __dadd_rn(-1.0, __ddiv_rn(2.0 * (double)j, r));
    p[2] = __dsub_rn(1.0, __ddiv_rn(2.0 * (double)k, r));
}

// The same position in fp32: exact, because node coordinates are dyadic
// (2i/R with R a power of two <= 1024).
__device__ __forceinline__ void node_pos_f(uint32_t idx, int cells, float* p) {
    unsigned n = (unsigned)cells + 1u;
    unsigned jk = idx / n, i = idx - jk * n, k = jk / n, j = jk - k * n;
    float r = (float)cells;
    p[0] = -1.0f + (2.0f * (float)i) / r;
    p[1] = -1.0f + (2.0f * (float)j) / r;
    p[2] = 1.0f - (2.0f * (float)k) / r;
}

__device__ __forceinline__ void job_point_d(const EvalJob& j, unsigned t, double* p) {
    if (j.points) {
        p[0] = j.points[3 * (size_t)t];
        p[1] = j.points[3 * (size_t)t + 1];
        p[2] = j.points[3 * (size_t)t + 2];
    } else {
        node_pos_d(job_node(j, t), j.cells, p);
    }
}

// CameraSpec::view_to_world (render.hpp:29-32): R^T ({p.x / s, p.y / s, p.z} - t), Mat3::apply's
// operation order (geom.hpp:64-68) with explicit roundings (bit-exact against the reference)
__device__ __forceinline__ void view_to_world_d(const FieldDev& f, double* p) {
    const double w0 = __dsub_rn(__ddiv_rn(p[0], f.vs), f.vt[0]);
    const double w1 = __dsub_rn(__ddiv_rn(p[1], f.vs), f.vt[1]);
    const double w2 = __dsub_rn(p[2], f.vt[2]);
    const double* m = f.vr;
    p[0] = __dadd_rn(__dadd_rn(__dmul_rn(m[0], w0), __dmul_rn(m[3], w1)), __dmul_rn(m[6], w2));
    p[1] = __dadd_rn(__dadd_rn(__dmul_rn(m[1], w0), __dmul_rn(m[4], w1)), __dmul_rn(m[7], w2));
    p[2] = __dadd_rn(__dadd_rn(__dmul_rn(m[2], w0), __dmul_rn(m[5], w1)), __dmul_rn(m[8], w2));
}

// world position of point t of a job: grid nodes of a view-space field go through view_to_world
// (the render_view wrap, render.hpp:98-99); explicit points are world points already
__device__ __forceinline__ void field_point_d(const FieldDev& f, const EvalJob& j, unsigned t, double* p) {
    job_point_d(j, t, p);
    if (f.view && !j.points) view_to_world_d(f, p);
}

// input-camera coordinates of a world point: Phi is sampled at (q.x, q.y), the depth feature is
// q.z (CameraSpec::world_to_view, render.hpp:23-26; identity without an input camera)
__device__ __forceinline__ void input_coords(const FieldDev& f, const float* w, float* q) {
    if (!f.icam) {
        q[0] = w[0];
        q[1] = w[1];
        q[2] = w[2];
        return;
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) q[r] = f.ic[4 * r] * w[0] + f.ic[4 * r + 1] * w[1] + f.ic[4 * r + 2] * w[2] + f.ic[4 * r + 3];
}

// evaluate_nodes write-back (localize.hpp:86-88) + conflict detection
// (localize.hpp:341-342): bin(oracle value) != bin(tentative value).
__device__ __forceinline__ void grid_epilogue(const EvalJob& j, uint32_t idx, float v) {
    j.values[idx] = v;
    j.states[idx] = ICG_STATE_EVALUATED;
    if (j.xext && v != 0.0f) {  // (a superset of the final extent is still exact for the renderer)
        const uint32_t fn = (uint32_t)j.cells + 1u, line = idx / fn;
        const int i = (int)(idx - line * fn);
        atomicMin(&j.xext[line].x, i);
        atomicMax(&j.xext[line].y, i);
    }
    if (j.tentbin) {
        bool tb = (j.tentbin[idx >> 5] >> (idx & 31)) & 1u;
        bool vb = v >= 0.5f;
        if (tb != vb) {
            unsigned pos = atomicAdd(j.conflict_count, 1u);
            if (pos < j.conflict_cap)
                j.conflicts[pos] = idx;
            else
                *j.overflow = 1u;
        }
    }
}

__device__ __forceinline__ void job_account(const EvalJob& j) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned n = job_count(j);
        if (j.evals) *j.evals += n;
        if (j.iters && n > 0) *j.iters += 1u;
    }
}

// Union SDF of the analytic scene (scene.hpp:60-103, 130-146) in double,
// reference operation order; compiled without FMA contraction.
__device__ __forceinline__ double d_dot3(const double* a, const double* b) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}

__device__ __forceinline__ double prim_sdf(const DevPrim& pr, const double* p) {
    double l[3] = {__dsub_rn(p[0], pr.c[0]), __dsub_rn(p[1], pr.c[1]), __dsub_rn(p[2], pr.c[2])};
    if (pr.rotated) {
        const double* m = pr.inv;
        double r0[3] = {m[0], m[1], m[2]}, r1[3] = {m[3], m[4], m[5]}, r2[3] = {m[6], m[7], m[8]};
        double l2[3] = {d_dot3(r0, l), d_dot3(r1, l), d_dot3(r2, l)};
        l[0] = l2[0];
        l[1] = l2[1];
        l[2] = l2[2];
    }
    switch (pr.kind) {
        case ICG_PRIM_SPHERE: return __dsub_rn(sqrt(d_dot3(l, l)), pr.radius);
        case ICG_PRIM_BOX: {
            double q[3] = {__dsub_rn(fabs(l[0]), pr.half[0]), __dsub_rn(fabs(l[1]), pr.half[1]),
                           __dsub_rn(fabs(l[2]), pr.half[2])};
            double qp[3] = {q[0] < 0.0 ? 0.0 : q[0], q[1] < 0.0 ? 0.0 : q[1], q[2] < 0.0 ? 0.0 : q[2]};
            double m12 = q[1] < q[2] ? q[2] : q[1];
            double m = q[0] < m12 ? m12 : q[0];
            double mn = 0.0 < m ? 0.0 : m;
            return __dadd_rn(sqrt(d_dot3(qp, qp)), mn);
        }
        case ICG_PRIM_CAPSULE: {
            double pa[3] = {__dsub_rn(p[0], pr.a[0]), __dsub_rn(p[1], pr.a[1]), __dsub_rn(p[2], pr.a[2])};
            double ba[3] = {__dsub_rn(pr.b[0], pr.a[0]), __dsub_rn(pr.b[1], pr.a[1]), __dsub_rn(pr.b[2], pr.a[2])};
            double den = d_dot3(ba, ba);
            double h = 0.0;
            if (den > 0.0) {
                h = __ddiv_rn(d_dot3(pa, ba), den);
                h = h < 0.0 ? 0.0 : (h > 1.0 ? 1.0 : h);
            }
            double v[3] = {__dsub_rn(pa[0], __dmul_rn(h, ba[0])), __dsub_rn(pa[1], __dmul_rn(h, ba[1])),
                           __dsub_rn(pa[2], __dmul_rn(h, ba[2]))};
            return __dsub_rn(sqrt(d_dot3(v, v)), pr.radius);
        }
        case ICG_PRIM_TORUS: {
            double qx = __dsub_rn(sqrt(__dadd_rn(__dmul_rn(l[0], l[0]), __dmul_rn(l[2], l[2]))), pr.major);
            return __dsub_rn(sqrt(__dadd_rn(__dmul_rn(qx, qx), __dmul_rn(l[1], l[1]))), pr.minor);
        }
    }
    return 1e300;
}

__device__ __forceinline__ double scene_sdf(const DevScene& s, const double* p) {
    double acc = 0.0;
    for (int i = 0; i < s.n_prims; ++i) {
        double d = prim_sdf(s.prims[i], p);
        acc = (i == 0) ? d : (d < acc ? d : acc);
    }
    return acc;
}

// SceneSpec::texture_color (scene.hpp:105-127) in fp64, reference operation order (lerp:
// a + t (b - a), geom.hpp:39; per primitive: the first primitive of minimum distance)
__device__ __forceinline__ void scene_texture(const DevScene& s, const double* p, double* rgb) {
    if (s.tex_kind == ICG_TEXTURE_CONSTANT) {
        rgb[0] = s.tex_color[0];
        rgb[1] = s.tex_color[1];
        rgb[2] = s.tex_color[2];
    } else if (s.tex_kind == ICG_TEXTURE_GRADIENT) {
        const double c = p[s.tex_axis];
        const double t = __dmul_rn(0.5, __dadd_rn(c, 1.0));
        for (int d = 0; d < 3; ++d) rgb[d] = __dadd_rn(s.tex_from[d], __dmul_rn(t, __dsub_rn(s.tex_to[d], s.tex_from[d])));
    } else {
        double best = 1.0 / 0.0;
        int bi = 0;
        for (int i = 0; i < s.n_prims; ++i) {
            const double d = prim_sdf(s.prims[i], p);
            if (d < best) {
                best = d;
                bi = i;
            }
        }
        rgb[0] = s.tex_colors[bi][0];
        rgb[1] = s.tex_colors[bi][1];
        rgb[2] = s.tex_colors[bi][2];
    }
}

// fp32 union SDF (same formulas; the PIFu capsule bias is tolerance-bound)
__device__ __forceinline__ float prim_sdf_f(const FPrim* pr, const float* p) {
    const int kind = __ldg(&pr->kind);
    float l[3] = {p[0] - __ldg(&pr->c[0]), p[1] - __ldg(&pr->c[1]), p[2] - __ldg(&pr->c[2])};
    if (__ldg(&pr->rotated)) {
        float l2[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
            l2[r] = __ldg(&pr->inv[3 * r]) * l[0] + __ldg(&pr->inv[3 * r + 1]) * l[1] + __ldg(&pr->inv[3 * r + 2]) * l[2];
        l[0] = l2[0];
        l[1] = l2[1];
        l[2] = l2[2];
    }
    if (kind == ICG_PRIM_CAPSULE) {
        const float pa[3] = {p[0] - __ldg(&pr->a[0]), p[1] - __ldg(&pr->a[1]), p[2] - __ldg(&pr->a[2])};
        const float ba[3] = {__ldg(&pr->b[0]) - __ldg(&pr->a[0]), __ldg(&pr->b[1]) - __ldg(&pr->a[1]),
                             __ldg(&pr->b[2]) - __ldg(&pr->a[2])};
        const float den = ba[0] * ba[0] + ba[1] * ba[1] + ba[2] * ba[2];
        float h = 0.0f;
        if (den > 0.0f) h = fminf(fmaxf((pa[0] * ba[0] + pa[1] * ba[1] + pa[2] * ba[2]) / den, 0.0f), 1.0f);
        const float v[3] = {pa[0] - h * ba[0], pa[1] - h * ba[1], pa[2] - h * ba[2]};
        return sqrtf(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]) - __ldg(&pr->radius);
    }
    if (kind == ICG_PRIM_SPHERE) return sqrtf(l[0] * l[0] + l[1] * l[1] + l[2] * l[2]) - __ldg(&pr->radius);
    if (kind == ICG_PRIM_BOX) {
        const float q[3] = {fabsf(l[0]) - __ldg(&pr->half[0]), fabsf(l[1]) - __ldg(&pr->half[1]),
                            fabsf(l[2]) - __ldg(&pr->half[2])};
        const float qp[3] = {fmaxf(q[0], 0.0f), fmaxf(q[1], 0.0f), fmaxf(q[2], 0.0f)};
        return sqrtf(qp[0] * qp[0] + qp[1] * qp[1] + qp[2] * qp[2]) + fminf(fmaxf(q[0], fmaxf(q[1], q[2])), 0.0f);
    }
    if (kind == ICG_PRIM_TORUS) {
        const float qx = sqrtf(l[0] * l[0] + l[2] * l[2]) - __ldg(&pr->major);
        return sqrtf(qx * qx + l[1] * l[1]) - __ldg(&pr->minor);
    }
    return 1e30f;
}

__device__ __forceinline__ float scene_sdf_f(const FScene* s, const float* p) {
    const int n = __ldg(&s->n_prims);
    float acc = 0.0f;
    for (int i = 0; i < n; ++i) {
        const float d = prim_sdf_f(&s->prims[i], p);
        acc = (i == 0) ? d : fminf(d, acc);
    }
    return acc;
}

// Warp-cooperative scene_sdf: lane i evaluates primitives i, i+32, ...; the
// union keeps the first minimum in primitive order, exactly as the serial loop
// (every lane returns the result).
__device__ __forceinline__ double scene_sdf_warp(const DevScene& s, const double* p) {
    const int lane = threadIdx.x & 31;
    double best = 0.0;
    int bi = 0x7fffffff;
    for (int i = lane; i < s.n_prims; i += 32) {
        const double d = prim_sdf(s.prims[i], p);
        if (bi == 0x7fffffff || d < best) {
            best = d;
            bi = i;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        // a wins if strictly smaller, or equal and earlier in primitive order
        const bool take = oi != 0x7fffffff && (bi == 0x7fffffff || ob < best || (!(best < ob) && oi < bi));
        if (take) {
            best = ob;
            bi = oi;
        }
    }
    return best;
}

}  // namespace icg

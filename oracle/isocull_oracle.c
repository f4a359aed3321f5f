/*
 * isocull_oracle.c — CPU ORACLE: TEST INFRASTRUCTURE ONLY (see isocull_oracle.h).
 *
 * Compiled with -ffp-contract=off: every fp32/fp64 operation below rounds once,
 * in the written order, so the restatement is deterministic and the render
 * sampling arithmetic is bit-reproducible by the CUDA kernel that mirrors it.
 */
#include "isocull_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ======================================================================== */
/* Rng: std::mt19937_64 (the C++ standard's fixed algorithm) with the        */
/* reference's hand-rolled transforms, random.hpp:16-43.                      */
/* ======================================================================== */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

uint64_t orc_rng_raw(orc_rng* r) {
    if (r->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            uint64_t x = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* random.hpp:22 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_raw(r) >> 11) * 0x1.0p-53; }

/* random.hpp:25 */
static double rng_uniform_range(orc_rng* r, double lo, double hi) {
    return lo + (hi - lo) * orc_rng_uniform(r);
}

/* random.hpp:33-38 */
double orc_rng_normal(orc_rng* r) {
    double u1 = orc_rng_uniform(r);
    while (u1 <= 0.0) u1 = orc_rng_uniform(r);
    double u2 = orc_rng_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

void orc_rng_uniforms(uint64_t seed, size_t n, double* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = orc_rng_uniform(&r);
}

void orc_rng_normals(uint64_t seed, size_t n, double* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = orc_rng_normal(&r);
}

/* ======================================================================== */
/* Parallel for (parallel.hpp:12-30 semantics: contiguous chunks).           */
/* ======================================================================== */
typedef void (*range_fn)(void* ctx, size_t b, size_t e);
typedef struct {
    range_fn f;
    void* ctx;
    size_t b, e;
} pf_job;

static void* pf_thread(void* arg) {
    pf_job* j = (pf_job*)arg;
    j->f(j->ctx, j->b, j->e);
    return NULL;
}

static void parallel_for(size_t count, int workers, range_fn f, void* ctx) {
    if (workers <= 1 || count < 64) {
        f(ctx, 0, count);
        return;
    }
    size_t n = (size_t)workers;
    if (n > count) n = count;
    if (n > 256) n = 256;
    size_t chunk = (count + n - 1) / n;
    pthread_t th[256];
    pf_job jobs[256];
    size_t started = 0;
    for (size_t w = 0; w < n; ++w) {
        size_t b = w * chunk, e = b + chunk < count ? b + chunk : count;
        if (b >= e) break;
        jobs[w].f = f;
        jobs[w].ctx = ctx;
        jobs[w].b = b;
        jobs[w].e = e;
        if (pthread_create(&th[w], NULL, pf_thread, &jobs[w]) != 0) {
            f(ctx, b, e);
            jobs[w].f = NULL;
        }
        started = w + 1;
    }
    for (size_t w = 0; w < started; ++w)
        if (jobs[w].f) pthread_join(th[w], NULL);
}

/* ======================================================================== */
/* Analytic SDFs: scene.hpp:60-103, union scene.hpp:130-146                  */
/* ======================================================================== */
static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static double norm3(const double* a) { return sqrt(dot3(a, a)); }
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }
static double maxd(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double mind(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* scene.hpp:68-73 */
static double sd_capsule(const double* p, const double* a, const double* b, double r) {
    double pa[3] = {p[0] - a[0], p[1] - a[1], p[2] - a[2]};
    double ba[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    double denom = dot3(ba, ba);
    double h = denom > 0.0 ? clampd(dot3(pa, ba) / denom, 0.0, 1.0) : 0.0;
    double hb[3] = {h * ba[0], h * ba[1], h * ba[2]};
    double v[3] = {pa[0] - hb[0], pa[1] - hb[1], pa[2] - hb[2]};
    return norm3(v) - r;
}

/* scene.hpp:85-101 */
static double prim_distance(const icg_primitive* pr, const double* p) {
    double local[3] = {p[0] - pr->center[0], p[1] - pr->center[1], p[2] - pr->center[2]};
    if (pr->rotated) {
        const double* m = pr->inv_rotation;
        double l2[3] = {m[0] * local[0] + m[1] * local[1] + m[2] * local[2],
                        m[3] * local[0] + m[4] * local[1] + m[5] * local[2],
                        m[6] * local[0] + m[7] * local[1] + m[8] * local[2]};
        local[0] = l2[0];
        local[1] = l2[1];
        local[2] = l2[2];
    }
    switch (pr->kind) {
        case ICG_PRIM_SPHERE: return norm3(local) - pr->radius; /* scene.hpp:60 */
        case ICG_PRIM_BOX: {                                     /* scene.hpp:62-66 */
            double q[3] = {fabs(local[0]) - pr->half[0], fabs(local[1]) - pr->half[1],
                           fabs(local[2]) - pr->half[2]};
            double qp[3] = {maxd(q[0], 0.0), maxd(q[1], 0.0), maxd(q[2], 0.0)};
            return norm3(qp) + mind(maxd(q[0], maxd(q[1], q[2])), 0.0);
        }
        case ICG_PRIM_CAPSULE: return sd_capsule(p, pr->a, pr->b, pr->radius);
        case ICG_PRIM_TORUS: { /* scene.hpp:75-78 */
            double qx = sqrt(local[0] * local[0] + local[2] * local[2]) - pr->major;
            return sqrt(qx * qx + local[1] * local[1]) - pr->minor;
        }
    }
    return INFINITY;
}

double orc_scene_sdf(const icg_primitive* prims, int n, const double p[3]) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
        double d = prim_distance(&prims[i], p);
        acc = (i == 0) ? d : mind(acc, d);
    }
    return acc;
}

/* field.hpp:81 */
double orc_occupancy_from_distance(double d, double tau) { return 1.0 / (1.0 + exp(d / tau)); }

typedef struct {
    const icg_primitive* prims;
    int n;
    double tau;
    const double* pts;
    double* out;
} an_ctx;

static void an_range(void* c, size_t b, size_t e) {
    an_ctx* a = (an_ctx*)c;
    for (size_t i = b; i < e; ++i)
        a->out[i] = orc_occupancy_from_distance(orc_scene_sdf(a->prims, a->n, a->pts + 3 * i), a->tau);
}

void orc_analytic_occupancy_batch(const icg_primitive* prims, int n, double tau, const double* pts,
                                  size_t npts, double* out, int threads) {
    an_ctx c = {prims, n, tau, pts, out};
    parallel_for(npts, threads, an_range, &c);
}

/* ======================================================================== */
/* PIFu field restatement (BASELINE.json configs[1-3])  */
/* ======================================================================== */
void orc_sample_features(const orc_pifu* m, const double p[3], double* out) {
    double u = (p[0] + 1.0) * 0.5 * (double)(m->W - 1);
    double v = (1.0 - p[1]) * 0.5 * (double)(m->H - 1);
    u = clampd(u, 0.0, (double)(m->W - 1));
    v = clampd(v, 0.0, (double)(m->H - 1));
    int x0 = (int)floor(u), y0 = (int)floor(v);
    if (x0 > m->W - 2) x0 = m->W - 2;
    if (y0 > m->H - 2) y0 = m->H - 2;
    double ax = u - (double)x0, ay = v - (double)y0;
    double w00 = (1.0 - ax) * (1.0 - ay), w10 = ax * (1.0 - ay), w01 = (1.0 - ax) * ay, w11 = ax * ay;
    size_t plane = (size_t)m->H * (size_t)m->W;
    size_t o00 = (size_t)y0 * m->W + x0;
    for (int c = 0; c < m->C; ++c) {
        const float* f = m->fmap + (size_t)c * plane;
        out[c] = w00 * (double)f[o00] + w10 * (double)f[o00 + 1] + w01 * (double)f[o00 + m->W] +
                 w11 * (double)f[o00 + m->W + 1];
    }
}

/* CameraSpec::world_to_view (render.hpp:23-26) of the PIFu input view; identity without one */
static void pifu_input(const orc_pifu* m, const double* P, double* q) {
    if (!m->has_cam) {
        q[0] = P[0];
        q[1] = P[1];
        q[2] = P[2];
        return;
    }
    const double* R = m->cam_rot;
    double v[3];
    for (int r = 0; r < 3; ++r) v[r] = R[3 * r] * P[0] + R[3 * r + 1] * P[1] + R[3 * r + 2] * P[2] + m->cam_t[r];
    q[0] = m->cam_scale * v[0];
    q[1] = m->cam_scale * v[1];
    q[2] = v[2];
}

#define PB 32 /* points per vector block; per-point arithmetic is independent of PB */

/* One dense layer over a block of PB points: out[o][p] = b[o] + sum_k W[o][k] in[k][p]
 * with in = [prev (prev_dim rows), skip (skip_dim rows)], k ascending.  Each
 * point's sum is accumulated in the same order regardless of PB. */
static void layer_block(const float* W, const float* b, int out_dim, const double* prev, int prev_dim,
                        const double* skip, int skip_dim, double* out, int leaky, double slope) {
    int in_dim = prev_dim + skip_dim;
    for (int o = 0; o < out_dim; ++o) {
        double acc[PB];
        for (int p = 0; p < PB; ++p) acc[p] = (double)b[o];
        const float* wr = W + (size_t)o * in_dim;
        for (int k = 0; k < prev_dim; ++k) {
            double w = (double)wr[k];
            const double* x = prev + (size_t)k * PB;
            for (int p = 0; p < PB; ++p) acc[p] += w * x[p];
        }
        wr += prev_dim;
        for (int k = 0; k < skip_dim; ++k) {
            double w = (double)wr[k];
            const double* x = skip + (size_t)k * PB;
            for (int p = 0; p < PB; ++p) acc[p] += w * x[p];
        }
        for (int p = 0; p < PB; ++p) {
            double v = acc[p];
            if (leaky && v < 0.0) v = v * slope;
            out[(size_t)o * PB + p] = v;
        }
    }
}

/* Runs layers [0, upto) of an MLP.  skip: [skip_dim][PB].  Returns the
 * activations of layer upto-1 (in bufA or bufB, [out_dims[upto-1]][PB]). */
static void mlp_block(const orc_mlp* net, const double* skip, int upto, double* bufA, double* bufB,
                      double** result) {
    const double* prev = NULL;
    int prev_dim = 0;
    double* cur = bufA;
    double* other = bufB;
    for (int l = 0; l < upto; ++l) {
        int leaky = (l < net->n_layers - 1);
        layer_block(net->w[l], net->b[l], net->out_dims[l], prev, prev_dim, skip, net->skip_dim, cur, leaky,
                    net->slope);
        prev = cur;
        prev_dim = net->out_dims[l];
        double* t = cur;
        cur = other;
        other = t;
    }
    *result = (double*)prev;
}

/* Single-point variants (the FieldOracle per-point shape): 8 output rows at a
 * time for instruction-level parallelism; each output still accumulates in k
 * order, so results equal the blocked path bit-for-bit. */
static void layer_point(const float* W, const float* b, int out_dim, const double* prev, int prev_dim,
                        const double* skip, int skip_dim, double* out, int leaky, double slope) {
    int in_dim = prev_dim + skip_dim;
    int o = 0;
    for (; o + 8 <= out_dim; o += 8) {
        double acc[8];
        const float* wr[8];
        for (int r = 0; r < 8; ++r) {
            acc[r] = (double)b[o + r];
            wr[r] = W + (size_t)(o + r) * in_dim;
        }
        for (int k = 0; k < prev_dim; ++k) {
            double x = prev[k];
            for (int r = 0; r < 8; ++r) acc[r] += (double)wr[r][k] * x;
        }
        for (int k = 0; k < skip_dim; ++k) {
            double x = skip[k];
            for (int r = 0; r < 8; ++r) acc[r] += (double)wr[r][prev_dim + k] * x;
        }
        for (int r = 0; r < 8; ++r) {
            double v = acc[r];
            if (leaky && v < 0.0) v = v * slope;
            out[o + r] = v;
        }
    }
    for (; o < out_dim; ++o) {
        double acc = (double)b[o];
        const float* wr = W + (size_t)o * in_dim;
        for (int k = 0; k < prev_dim; ++k) acc += (double)wr[k] * prev[k];
        for (int k = 0; k < skip_dim; ++k) acc += (double)wr[prev_dim + k] * skip[k];
        if (leaky && acc < 0.0) acc = acc * slope;
        out[o] = acc;
    }
}

static const double* mlp_point(const orc_mlp* net, const double* skip, int upto, double* bufA, double* bufB) {
    const double* prev = NULL;
    int prev_dim = 0;
    double* cur = bufA;
    double* other = bufB;
    for (int l = 0; l < upto; ++l) {
        layer_point(net->w[l], net->b[l], net->out_dims[l], prev, prev_dim, skip, net->skip_dim, cur,
                    l < net->n_layers - 1, net->slope);
        prev = cur;
        prev_dim = net->out_dims[l];
        double* t = cur;
        cur = other;
        other = t;
    }
    return prev;
}

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

typedef struct {
    const orc_pifu* m;
    const double* pts;
    size_t n;
    double* out;
    int mode; /* 0 occupancy, 1 logit, 2 texture */
} pifu_ctx;

static void pifu_range(void* c, size_t b, size_t e) {
    pifu_ctx* a = (pifu_ctx*)c;
    const orc_pifu* m = a->m;
    size_t nblocks = (e - b + PB - 1) / PB;
    int C = m->C;
    double* feat = (double*)malloc(sizeof(double) * (size_t)C);
    double* gskip = (double*)calloc((size_t)m->geo.skip_dim * PB, sizeof(double));
    double* tskip = m->has_texture ? (double*)calloc((size_t)m->tex.skip_dim * PB, sizeof(double)) : NULL;
    double* bufA = (double*)malloc(sizeof(double) * 1024 * PB);
    double* bufB = (double*)malloc(sizeof(double) * 1024 * PB);
    for (size_t blk = 0; blk < nblocks; ++blk) {
        size_t p0 = b + blk * PB;
        int np = (int)((e - p0) < PB ? (e - p0) : PB);
        /* skip features [Phi (C), z] per point (padding lanes repeat point 0) */
        for (int p = 0; p < PB; ++p) {
            double q[3];
            pifu_input(m, a->pts + 3 * (p0 + (size_t)(p < np ? p : 0)), q);
            orc_sample_features(m, q, feat);
            for (int c = 0; c < C; ++c) gskip[(size_t)c * PB + p] = feat[c];
            gskip[(size_t)C * PB + p] = q[2];
            if (tskip) {
                for (int c = 0; c < C; ++c) tskip[(size_t)c * PB + p] = feat[c];
                tskip[(size_t)(m->tex.skip_dim - 1) * PB + p] = q[2];
            }
        }
        if (a->mode == 2) {
            /* geometry prefix: layers 1-3 -> h3 (256-d), texture skip = [Phi, h3, z] */
            double* h3;
            mlp_block(&m->geo, gskip, 3, bufA, bufB, &h3);
            int hd = m->geo.out_dims[2];
            for (int k = 0; k < hd; ++k)
                for (int p = 0; p < PB; ++p) tskip[(size_t)(C + k) * PB + p] = h3[(size_t)k * PB + p];
            double* o;
            mlp_block(&m->tex, tskip, m->tex.n_layers, bufA, bufB, &o);
            for (int p = 0; p < np; ++p)
                for (int ch = 0; ch < 3; ++ch) a->out[(p0 + p) * 3 + ch] = sigmoid(o[(size_t)ch * PB + p]);
        } else {
            double* o;
            mlp_block(&m->geo, gskip, m->geo.n_layers, bufA, bufB, &o);
            for (int p = 0; p < np; ++p) {
                const double* P = a->pts + 3 * (p0 + p);
                double sdf = orc_scene_sdf(m->prims, m->n_prims, P);
                double logit = o[p] - m->sdf_scale * sdf;
                a->out[p0 + p] = a->mode == 1 ? logit : sigmoid(logit);
            }
        }
    }
    free(feat);
    free(gskip);
    free(tskip);
    free(bufA);
    free(bufB);
}

static void pifu_one(const orc_pifu* m, const double* P, double* out, int mode) {
    double gskip[257 + 8], tskip[513 + 8], bufA[1024], bufB[1024];
    int C = m->C;
    double q[3];
    pifu_input(m, P, q);
    orc_sample_features(m, q, gskip);
    gskip[C] = q[2];
    if (mode == 2) {
        for (int c = 0; c < C; ++c) tskip[c] = gskip[c];
        const double* h3 = mlp_point(&m->geo, gskip, 3, bufA, bufB);
        for (int k = 0; k < m->geo.out_dims[2]; ++k) tskip[C + k] = h3[k];
        tskip[m->tex.skip_dim - 1] = q[2];
        const double* o = mlp_point(&m->tex, tskip, m->tex.n_layers, bufA, bufB);
        for (int ch = 0; ch < 3; ++ch) out[ch] = sigmoid(o[ch]);
    } else {
        const double* o = mlp_point(&m->geo, gskip, m->geo.n_layers, bufA, bufB);
        double logit = o[0] - m->sdf_scale * orc_scene_sdf(m->prims, m->n_prims, P);
        out[0] = mode == 1 ? logit : sigmoid(logit);
    }
}

static void pifu_run(const orc_pifu* m, const double* pts, size_t n, double* out, int threads, int mode) {
    if (n == 1 && m->C == 256) {
        pifu_one(m, pts, out, mode);
        return;
    }
    pifu_ctx c = {m, pts, n, out, mode};
    if (threads <= 1 || n < 2 * PB) {
        pifu_range(&c, 0, n);
        return;
    }
    /* chunk in PB multiples so block boundaries do not depend on thread count */
    size_t nb = (n + PB - 1) / PB;
    size_t nt = (size_t)threads;
    if (nt > nb) nt = nb;
    size_t per = (nb + nt - 1) / nt;
    pthread_t th[256];
    pf_job jobs[256];
    size_t started = 0;
    for (size_t w = 0; w < nt && w < 256; ++w) {
        size_t bb = w * per * PB, ee = (w + 1) * per * PB;
        if (ee > n) ee = n;
        if (bb >= ee) break;
        jobs[w].f = pifu_range;
        jobs[w].ctx = &c;
        jobs[w].b = bb;
        jobs[w].e = ee;
        pthread_create(&th[w], NULL, pf_thread, &jobs[w]);
        started = w + 1;
    }
    for (size_t w = 0; w < started; ++w) pthread_join(th[w], NULL);
}

void orc_pifu_occupancy_batch(const orc_pifu* m, const double* pts, size_t n, double* out, int threads) {
    pifu_run(m, pts, n, out, threads, 0);
}
void orc_pifu_logit_batch(const orc_pifu* m, const double* pts, size_t n, double* out, int threads) {
    pifu_run(m, pts, n, out, threads, 1);
}
void orc_pifu_texture_batch(const orc_pifu* m, const double* pts, size_t n, double* rgb, int threads) {
    pifu_run(m, pts, n, rgb, threads, 2);
}

/* ---- callbacks -------------------------------------------------------- */
void orc_cb_analytic(void* user, const double* pts, size_t n, double* out) {
    orc_analytic* a = (orc_analytic*)user;
    orc_analytic_occupancy_batch(a->prims, a->n_prims, a->tau, pts, n, out, a->threads);
}
void orc_cb_pifu_occ(void* user, const double* pts, size_t n, double* out) {
    orc_pifu_cb* c = (orc_pifu_cb*)user;
    orc_pifu_occupancy_batch(c->model, pts, n, out, c->threads);
}
void orc_cb_pifu_tex(void* user, const double* pts, size_t n, double* rgb) {
    orc_pifu_cb* c = (orc_pifu_cb*)user;
    orc_pifu_texture_batch(c->model, pts, n, rgb, c->threads);
}
double orc_pt_analytic(void* user, const double* p) {
    orc_analytic* a = (orc_analytic*)user;
    return orc_occupancy_from_distance(orc_scene_sdf(a->prims, a->n_prims, p), a->tau);
}
double orc_pt_pifu_occ(void* user, const double* p) {
    orc_pifu_cb* c = (orc_pifu_cb*)user;
    double out;
    pifu_run(c->model, p, 1, &out, 1, 0);
    return out;
}
void orc_pt_pifu_tex(void* user, const double* p, double* rgb) {
    orc_pifu_cb* c = (orc_pifu_cb*)user;
    pifu_run(c->model, p, 1, rgb, 1, 2);
}

static long replay_index(const orc_replay* r, const double* p) {
    int n = r->cells + 1;
    double fi = (p[0] + 1.0) * 0.5 * r->cells, fj = (p[1] + 1.0) * 0.5 * r->cells,
           fk = (1.0 - p[2]) * 0.5 * r->cells;
    long i = lround(fi), j = lround(fj), k = lround(fk);
    if (i < 0 || j < 0 || k < 0 || i >= n || j >= n || k >= n) return -1;
    if (fabs(fi - (double)i) > 1e-9 || fabs(fj - (double)j) > 1e-9 || fabs(fk - (double)k) > 1e-9) return -1;
    return i + (long)n * (j + (long)n * k);
}

double orc_pt_replay(void* user, const double* p) {
    orc_replay* r = (orc_replay*)user;
    __atomic_fetch_add(&r->calls, 1, __ATOMIC_RELAXED);
    long idx = replay_index(r, p);
    if (idx < 0 || r->states[idx] != ICG_STATE_EVALUATED) {
        __atomic_fetch_add(&r->misses, 1, __ATOMIC_RELAXED);
        return 0.0;
    }
    return (double)r->values[idx];
}

void orc_cb_replay(void* user, const double* pts, size_t n, double* out) {
    for (size_t i = 0; i < n; ++i) out[i] = orc_pt_replay(user, pts + 3 * i);
}

/* ======================================================================== */
/* Grid primitives, grid.hpp:84-197                                          */
/* ======================================================================== */
static size_t gidx(int n, int i, int j, int k) { return (size_t)i + (size_t)n * ((size_t)j + (size_t)n * (size_t)k); }

/* grid.hpp:87-120 */
void orc_upsample_interpolate(int coarse_cells, const float* cv, const uint8_t* cs, float* fv, uint8_t* fs) {
    int cn = coarse_cells + 1, fn = 2 * coarse_cells + 1;
    for (int k = 0; k < fn; ++k) {
        int k0 = k / 2, k1 = (k + 1) / 2;
        for (int j = 0; j < fn; ++j) {
            int j0 = j / 2, j1 = (j + 1) / 2;
            for (int i = 0; i < fn; ++i) {
                int i0 = i / 2, i1 = (i + 1) / 2;
                size_t fi = gidx(fn, i, j, k);
                if (i0 == i1 && j0 == j1 && k0 == k1) {
                    size_t ci = gidx(cn, i0, j0, k0);
                    fv[fi] = cv[ci];
                    fs[fi] = cs[ci];
                    continue;
                }
                double sum = 0.0;
                int cnt = 0;
                for (int kk = k0; kk <= k1; ++kk)
                    for (int jj = j0; jj <= j1; ++jj)
                        for (int ii = i0; ii <= i1; ++ii) {
                            sum += cv[gidx(cn, ii, jj, kk)];
                            ++cnt;
                        }
                fv[fi] = (float)(sum / cnt);
                fs[fi] = ICG_STATE_INTERPOLATED;
            }
        }
    }
}

/* grid.hpp:144-163 */
void orc_dilate_1ring(int n, const uint8_t* mask, uint8_t* out) {
    memset(out, 0, (size_t)n * n * n);
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                if (!mask[gidx(n, i, j, k)]) continue;
                int klo = k > 0 ? k - 1 : 0, khi = k < n - 1 ? k + 1 : n - 1;
                int jlo = j > 0 ? j - 1 : 0, jhi = j < n - 1 ? j + 1 : n - 1;
                int ilo = i > 0 ? i - 1 : 0, ihi = i < n - 1 ? i + 1 : n - 1;
                for (int kk = klo; kk <= khi; ++kk)
                    for (int jj = jlo; jj <= jhi; ++jj)
                        for (int ii = ilo; ii <= ihi; ++ii) out[gidx(n, ii, jj, kk)] = 1;
            }
}

/* grid.hpp:173-197 */
void orc_argmax_z(int n, const float* values, float* max_value, int* max_index) {
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            size_t px = (size_t)i + (size_t)n * j;
            float best = values[gidx(n, i, j, 0)];
            int bk = 0;
            for (int k = 1; k < n; ++k) {
                float v = values[gidx(n, i, j, k)];
                if (v > best) {
                    best = v;
                    bk = k;
                }
            }
            max_value[px] = best;
            max_index[px] = bk;
        }
}

/* ======================================================================== */
/* Localization, localize.hpp:66-193,315-363                                 */
/* ======================================================================== */
static float binarize_value(float v) { return v >= 0.5f ? 1.0f : 0.0f; } /* grid.hpp:122 */

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* grid.hpp:50-53 */
static void node_position(int cells, size_t idx, double* p) {
    size_t n = (size_t)cells + 1;
    int i = (int)(idx % n), j = (int)((idx / n) % n), k = (int)(idx / (n * n));
    double r = (double)cells;
    p[0] = -1.0 + 2.0 * i / r;
    p[1] = -1.0 + 2.0 * j / r;
    p[2] = 1.0 - 2.0 * k / r;
}

/* localize.hpp:76-90 */
static uint64_t evaluate_nodes(orc_occ_batch_fn occ, void* user, int cells, float* values, uint8_t* states,
                               const size_t* list, size_t n) {
    if (n == 0) return 0;
    double* pts = (double*)malloc(sizeof(double) * 3 * n);
    double* out = (double*)malloc(sizeof(double) * n);
    for (size_t t = 0; t < n; ++t) node_position(cells, list[t], pts + 3 * t);
    occ(user, pts, n, out);
    for (size_t t = 0; t < n; ++t) {
        values[list[t]] = (float)out[t];
        states[list[t]] = ICG_STATE_EVALUATED;
    }
    free(pts);
    free(out);
    return n;
}

/* localize.hpp:93-104 (via a full index list) */
static uint64_t evaluate_full(orc_occ_batch_fn occ, void* user, int cells, float* values, uint8_t* states) {
    size_t n = (size_t)(cells + 1);
    size_t count = n * n * n;
    size_t* list = (size_t*)malloc(sizeof(size_t) * count);
    for (size_t i = 0; i < count; ++i) list[i] = i;
    uint64_t r = evaluate_nodes(occ, user, cells, values, states, list, count);
    free(list);
    return r;
}

typedef struct {
    size_t* v;
    size_t n, cap;
} vec_sz;
static void vpush(vec_sz* v, size_t x) {
    if (v->n == v->cap) {
        v->cap = v->cap ? 2 * v->cap : 1024;
        v->v = (size_t*)realloc(v->v, sizeof(size_t) * v->cap);
    }
    v->v[v->n++] = x;
}

/* record the level of every node of a level-l list in the final-grid eval_level map */
static void mark_level(orc_extract_out* out, int l, int target_level, int cells, const size_t* list, size_t n) {
    if (!out->eval_level) return;
    const size_t nn = (size_t)cells + 1, fn = ((size_t)cells << (target_level - l)) + 1;
    const int sh = target_level - l;
    for (size_t t = 0; t < n; ++t) {
        size_t idx = list[t], i = idx % nn, j = (idx / nn) % nn, k = idx / (nn * nn);
        out->eval_level[(i << sh) + fn * ((j << sh) + fn * (k << sh))] = (uint8_t)l;
    }
}

int orc_extract_progressive(orc_occ_batch_fn occ, void* user, int coarsest_cells, int target_level,
                            int max_conflict_iters, int conflict_pass, orc_extract_out* out) {
    /* validate_config, localize.hpp:47-55 */
    if (coarsest_cells < 2 || target_level < 0 || (coarsest_cells << target_level) > 1024 || target_level > 15)
        return ICG_EINVAL;
    double t0 = now_s();
    memset(out->evals_per_level, 0, sizeof(out->evals_per_level));
    memset(out->refined_cells_per_level, 0, sizeof(out->refined_cells_per_level));
    memset(out->conflict_iters_per_level, 0, sizeof(out->conflict_iters_per_level));
    out->conflict_warning = 0;
    int cells = coarsest_cells;
    size_t n = (size_t)cells + 1, count = n * n * n;
    float* gv = (float*)malloc(sizeof(float) * count);
    uint8_t* gs = (uint8_t*)malloc(count);
    memset(gs, ICG_STATE_UNKNOWN, count);
    out->evals_per_level[0] = evaluate_full(occ, user, cells, gv, gs);
    if (out->eval_level) {
        size_t fnodes = ((size_t)coarsest_cells << target_level) + 1;
        memset(out->eval_level, 0xFF, fnodes * fnodes * fnodes);
        size_t* all = (size_t*)malloc(sizeof(size_t) * count);
        for (size_t i = 0; i < count; ++i) all[i] = i;
        mark_level(out, 0, target_level, cells, all, count);
        free(all);
    }

    for (int l = 1; l <= target_level; ++l) {
        int cc = cells, cn = cc + 1;
        int fcells = 2 * cc, fn = fcells + 1;
        size_t fcount = (size_t)fn * fn * fn;
        /* refined cells (new output): coarse cells whose 8 binarized corners disagree */
        uint64_t refined = 0;
        for (int k = 0; k < cc; ++k)
            for (int j = 0; j < cc; ++j)
                for (int i = 0; i < cc; ++i) {
                    int ones = 0;
                    for (int d = 0; d < 8; ++d)
                        ones += gv[gidx(cn, i + (d & 1), j + ((d >> 1) & 1), k + (d >> 2))] >= 0.5f;
                    refined += (ones != 0 && ones != 8);
                    if (out->refined_cells[l])
                        out->refined_cells[l][(size_t)i + (size_t)cc * ((size_t)j + (size_t)cc * k)] = ones != 0 && ones != 8;
                }
        out->refined_cells_per_level[l] = refined;
        /* bin = binarize(grid); tent = upsample_interpolate(bin) */
        float* bin = (float*)malloc(sizeof(float) * (size_t)cn * cn * cn);
        for (size_t i = 0; i < (size_t)cn * cn * cn; ++i) bin[i] = binarize_value(gv[i]);
        float* tv = (float*)malloc(sizeof(float) * fcount);
        uint8_t* ts = (uint8_t*)malloc(fcount);
        orc_upsample_interpolate(cc, bin, gs, tv, ts);
        /* flagged = dilate_1ring(boundary_candidates(tent)) */
        uint8_t* cand = (uint8_t*)malloc(fcount);
        for (size_t i = 0; i < fcount; ++i) cand[i] = (tv[i] > 0.0f && tv[i] < 1.0f);
        uint8_t* flagged = (uint8_t*)malloc(fcount);
        orc_dilate_1ring(fn, cand, flagged);
        /* fine = carry_scalars(grid, tent), localize.hpp:110-122 */
        float* fv = (float*)malloc(sizeof(float) * fcount);
        uint8_t* fs = (uint8_t*)malloc(fcount);
        memcpy(fv, tv, sizeof(float) * fcount);
        memcpy(fs, ts, fcount);
        for (int k = 0; k < cn; ++k)
            for (int j = 0; j < cn; ++j)
                for (int i = 0; i < cn; ++i) {
                    size_t fi = gidx(fn, 2 * i, 2 * j, 2 * k), ci = gidx(cn, i, j, k);
                    fv[fi] = gv[ci];
                    fs[fi] = gs[ci];
                }
        /* to_eval = mask_to_unevaluated_list(flagged, fine), localize.hpp:124-129 */
        vec_sz to_eval = {0};
        for (size_t i = 0; i < fcount; ++i)
            if (flagged[i] && fs[i] != ICG_STATE_EVALUATED) vpush(&to_eval, i);
        out->evals_per_level[l] += evaluate_nodes(occ, user, fcells, fv, fs, to_eval.v, to_eval.n);
        mark_level(out, l, target_level, fcells, to_eval.v, to_eval.n);
        /* conflict pass, localize.hpp:333-354 */
        uint8_t* queued = (uint8_t*)calloc(fcount, 1);
        vec_sz newly = {0};
        if (conflict_pass) newly = to_eval;
        else free(to_eval.v);
        int max_iters = max_conflict_iters > 0 ? max_conflict_iters : fcells;
        for (int iter = 0;; ++iter) {
            vec_sz conflicts = {0};
            for (size_t t = 0; t < newly.n; ++t) {
                size_t idx = newly.v[t];
                if (binarize_value(fv[idx]) != binarize_value(tv[idx])) vpush(&conflicts, idx);
            }
            if (conflicts.n == 0) {
                free(conflicts.v);
                break;
            }
            if (iter >= max_iters) {
                out->conflict_warning = 1;
                free(conflicts.v);
                break;
            }
            vec_sz next = {0};
            for (size_t t = 0; t < conflicts.n; ++t) {
                /* collect_unevaluated_neighbors, localize.hpp:160-177 */
                size_t idx = conflicts.v[t];
                int i = (int)(idx % fn), j = (int)((idx / fn) % fn), k = (int)(idx / ((size_t)fn * fn));
                for (int dk = -1; dk <= 1; ++dk)
                    for (int dj = -1; dj <= 1; ++dj)
                        for (int di = -1; di <= 1; ++di) {
                            if (!di && !dj && !dk) continue;
                            int ii = i + di, jj = j + dj, kk = k + dk;
                            if (ii < 0 || jj < 0 || kk < 0 || ii >= fn || jj >= fn || kk >= fn) continue;
                            size_t nb = gidx(fn, ii, jj, kk);
                            if (queued[nb] || fs[nb] == ICG_STATE_EVALUATED) continue;
                            queued[nb] = 1;
                            vpush(&next, nb);
                        }
            }
            const uint64_t conflicts_n_dump = conflicts.n;
            if (getenv("ORC_CHAIN_DUMP")) {
                FILE* df = fopen(getenv("ORC_CHAIN_DUMP"), "ab");
                if (df) {
                    uint64_t hdr[4] = {(uint64_t)l, (uint64_t)iter | (1ull << 32), conflicts.n, 0};
                    fwrite(hdr, 8, 4, df);
                    fwrite(conflicts.v, sizeof(size_t), conflicts.n, df);
                    fclose(df);
                }
            }
            free(conflicts.v);
            if (next.n == 0) {
                free(next.v);
                break;
            }
            if (getenv("ORC_CHAIN_DUMP")) {  /* dev aid: per-iteration conflict / next lists */
                FILE* df = fopen(getenv("ORC_CHAIN_DUMP"), "ab");
                if (df) {
                    uint64_t hdr[4] = {(uint64_t)l, (uint64_t)iter, conflicts_n_dump, next.n};
                    fwrite(hdr, 8, 4, df);
                    fwrite(next.v, sizeof(size_t), next.n, df);
                    fclose(df);
                }
            }
            out->evals_per_level[l] += evaluate_nodes(occ, user, fcells, fv, fs, next.v, next.n);
            mark_level(out, l, target_level, fcells, next.v, next.n);
            out->conflict_iters_per_level[l] += 1;
            free(newly.v);
            newly = next;
        }
        free(newly.v);
        free(queued);
        free(bin);
        free(tv);
        free(ts);
        free(cand);
        free(flagged);
        free(gv);
        free(gs);
        gv = fv;
        gs = fs;
        cells = fcells;
    }
    size_t fcount = (size_t)(cells + 1) * (cells + 1) * (cells + 1);
    out->total_evals = 0;
    for (int l = 0; l <= target_level; ++l) out->total_evals += out->evals_per_level[l];
    memcpy(out->values, gv, sizeof(float) * fcount);
    memcpy(out->states, gs, fcount);
    if (out->binarized)
        for (size_t i = 0; i < fcount; ++i) out->binarized[i] = gv[i] >= 0.5f ? 1 : 0;
    free(gv);
    free(gs);
    out->wall_seconds = now_s() - t0;
    return ICG_OK;
}

/* localize.hpp:181-193 */
int orc_extract_brute(orc_occ_batch_fn occ, void* user, int coarsest_cells, int target_level, orc_extract_out* out) {
    if (coarsest_cells < 2 || target_level < 0 || (coarsest_cells << target_level) > 1024) return ICG_EINVAL;
    double t0 = now_s();
    memset(out->evals_per_level, 0, sizeof(out->evals_per_level));
    memset(out->refined_cells_per_level, 0, sizeof(out->refined_cells_per_level));
    memset(out->conflict_iters_per_level, 0, sizeof(out->conflict_iters_per_level));
    out->conflict_warning = 0;
    int cells = coarsest_cells << target_level;
    size_t n = (size_t)cells + 1, count = n * n * n;
    out->evals_per_level[target_level] = evaluate_full(occ, user, cells, out->values, out->states);
    out->total_evals = out->evals_per_level[target_level];
    if (out->binarized)
        for (size_t i = 0; i < count; ++i) out->binarized[i] = out->values[i] >= 0.5f ? 1 : 0;
    out->wall_seconds = now_s() - t0;
    return ICG_OK;
}

static void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        c[1] = (uint32_t)p1;
        c[3] = (uint32_t)p0;
        c[0] = n0;
        c[2] = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

void orc_feature_normals(uint64_t seed, size_t n, float* out) {
    for (size_t e = 0; e < n; ++e) {
        uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), 0u, 0u};
        philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
        double a = (double)((((uint64_t)c[0] << 32) | c[1]) >> 11) * 0x1.0p-53;
        const double b = (double)((((uint64_t)c[2] << 32) | c[3]) >> 11) * 0x1.0p-53;
        if (a <= 0.0) a = 0x1.0p-53;
        out[e] = (float)(sqrt(-2.0 * log(a)) * cos(2.0 * 3.14159265358979323846 * b));
    }
}

/* localize.hpp:377-387 */
double orc_compare_iou(const uint8_t* a, const uint8_t* b, size_t n) {
    uint64_t inter = 0, uni = 0;
    for (size_t i = 0; i < n; ++i) {
        int av = a[i] != 0, bv = b[i] != 0;
        inter += (av && bv);
        uni += (av || bv);
    }
    if (uni == 0) return 1.0;
    return (double)inter / (double)uni;
}

/* ======================================================================== */
/* Render: first-crossing through the world grid    */
/* ======================================================================== */

/* CameraSpec::from_angles, render.hpp:36-45; Mat3 rotations geom.hpp:46-73 */
void orc_camera_from_angles(double yaw_deg, double pitch_deg, double dist, double scale, icg_camera* out) {
    const double kPi = 3.14159265358979323846;
    double yaw = fmod(yaw_deg, 360.0), pitch = fmod(pitch_deg, 360.0);
    double ry = yaw * kPi / 180.0, rx = pitch * kPi / 180.0;
    double cx = cos(rx), sx = sin(rx), cy = cos(ry), sy = sin(ry);
    double A[9] = {1, 0, 0, 0, cx, -sx, 0, sx, cx};  /* rotation_x */
    double B[9] = {cy, 0, sy, 0, 1, 0, -sy, 0, cy};  /* rotation_y */
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int k = 0; k < 3; ++k) s += A[3 * i + k] * B[3 * k + j];
            out->rotation[3 * i + j] = s;
        }
    out->translation[0] = 0.0;
    out->translation[1] = 0.0;
    out->translation[2] = -dist;
    out->scale = scale;
}

/* view_to_world, render.hpp:29-32: R^T (v - t) with v = (x/scale, y/scale, z) */
static void view_to_world(const icg_camera* c, const double* p, double* w) {
    double v[3] = {p[0] / c->scale - c->translation[0], p[1] / c->scale - c->translation[1],
                   p[2] - c->translation[2]};
    const double* m = c->rotation;
    w[0] = m[0] * v[0] + m[3] * v[1] + m[6] * v[2];
    w[1] = m[1] * v[0] + m[4] * v[1] + m[7] * v[2];
    w[2] = m[2] * v[0] + m[5] * v[1] + m[8] * v[2];
}

static float lerpf(float a, float b, float t) { return a + t * (b - a); }

/* Trilinear sample of the world grid at grid coordinates (gx, gy, gk) in
 * [0, R]^3 (gk = depth index, k = 0 at world z = +1); 0 outside. */
static float sample_grid(const float* V, int R, float gx, float gy, float gk) {
    float fR = (float)R;
    if (!(gx >= 0.0f && gx <= fR && gy >= 0.0f && gy <= fR && gk >= 0.0f && gk <= fR)) return 0.0f;
    int i0 = (int)floorf(gx), j0 = (int)floorf(gy), k0 = (int)floorf(gk);
    if (i0 > R - 1) i0 = R - 1;
    if (j0 > R - 1) j0 = R - 1;
    if (k0 > R - 1) k0 = R - 1;
    float fx = gx - (float)i0, fy = gy - (float)j0, fk = gk - (float)k0;
    size_t n = (size_t)R + 1;
    size_t b = (size_t)i0 + n * ((size_t)j0 + n * (size_t)k0);
    size_t sj = n, sk = n * n;
    float c00 = lerpf(V[b], V[b + 1], fx);
    float c10 = lerpf(V[b + sj], V[b + sj + 1], fx);
    float c01 = lerpf(V[b + sk], V[b + sk + 1], fx);
    float c11 = lerpf(V[b + sj + sk], V[b + sj + sk + 1], fx);
    float c0 = lerpf(c00, c10, fy);
    float c1 = lerpf(c01, c11, fy);
    return lerpf(c0, c1, fk);
}

/* Grid coordinates of view sample (vx, vy, k): world = view_to_world(vx, vy,
 * 1 - 2k/R); gx = (wx+1)*R/2, gy = (wy+1)*R/2, gk = (1-wz)*R/2, each in
 * double, rounded once to float. */
static void ray_coords(const icg_camera* c, int R, double vx, double vy, int k, float* g) {
    double vz = 1.0 - 2.0 * (double)k / (double)R;
    double p[3] = {vx, vy, vz}, w[3];
    view_to_world(c, p, w);
    double hr = 0.5 * (double)R;
    g[0] = (float)((w[0] + 1.0) * hr);
    g[1] = (float)((w[1] + 1.0) * hr);
    g[2] = (float)((1.0 - w[2]) * hr);
}

int orc_render_first_crossing(const float* values, int cells, const icg_camera* cam, int width, int height,
                              const float* background, orc_tex_batch_fn tex, void* tex_user,
                              orc_render_out* out) {
    if (width < 2 || height < 2 || cells < 1) return ICG_EINVAL;
    int R = cells;
    size_t npx = (size_t)width * height;
    double* spts = (double*)malloc(sizeof(double) * 3 * npx);
    size_t* spx = (size_t*)malloc(sizeof(size_t) * npx);
    size_t ns = 0;
    out->covered = out->degenerate = out->grazing = 0;
    for (int row = 0; row < height; ++row)
        for (int col = 0; col < width; ++col) {
            size_t px = (size_t)row * width + col;
            double vx = -1.0 + 2.0 * (double)col / (double)(width - 1);
            double vy = 1.0 - 2.0 * (double)row / (double)(height - 1);
            int k1 = -1, grazing = 0;
            float vprev = 0.0f, vhit = 0.0f;
            for (int k = 0; k <= R; ++k) {
                float g[3];
                ray_coords(cam, R, vx, vy, k, g);
                float v = sample_grid(values, R, g[0], g[1], g[2]);
                if (v >= 0.5f) {
                    k1 = k;
                    vhit = v;
                    break;
                }
                if (v > 0.0f && v < 1.0f) grazing = 1;
                vprev = v;
            }
            out->rgb[3 * px + 0] = background[0];
            out->rgb[3 * px + 1] = background[1];
            out->rgb[3 * px + 2] = background[2];
            if (k1 < 0) {
                out->depth[px] = -2.0f;
                out->mask[px] = 0;
                if (out->surface_k) out->surface_k[px] = -1;
                out->grazing += (uint64_t)grazing;
                continue;
            }
            /* bracket, render.hpp:190-204 */
            double s = 1.0;
            if (k1 > 0) {
                double v1 = (double)vhit, v0 = (double)vprev;
                double denom = v1 - v0;
                if (denom > 0.0)
                    s = clampd((0.5 - v0) / denom, 0.0, 1.0);
                else
                    out->degenerate += 1;
            }
            double depth = 1.0 - 2.0 * ((double)k1 - 1.0 + s) / (double)R;
            out->depth[px] = (float)depth;
            out->mask[px] = 1;
            if (out->surface_k) out->surface_k[px] = k1;
            out->covered += 1;
            double vp[3] = {vx, vy, depth};
            view_to_world(cam, vp, spts + 3 * ns);
            if (out->surface_pts) memcpy(out->surface_pts + 3 * px, spts + 3 * ns, sizeof(double) * 3);
            spx[ns++] = px;
        }
    if (tex && ns) {
        double* rgb = (double*)malloc(sizeof(double) * 3 * ns);
        tex(tex_user, spts, ns, rgb);
        for (size_t t = 0; t < ns; ++t)
            for (int ch = 0; ch < 3; ++ch) out->rgb[3 * spx[t] + ch] = (float)clampd(rgb[3 * t + ch], 0.0, 1.0);
        free(rgb);
    }
    free(spts);
    free(spx);
    return ICG_OK;
}

/* ======================================================================== */
/* Seeded inputs                                                             */
/* ======================================================================== */
void orc_gen_capsules(uint64_t seed, int n, icg_primitive* out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (int c = 0; c < n; ++c) {
        memset(&out[c], 0, sizeof(icg_primitive));
        out[c].kind = ICG_PRIM_CAPSULE;
        for (int d = 0; d < 3; ++d) out[c].a[d] = rng_uniform_range(&r, -0.5, 0.5);
        for (int d = 0; d < 3; ++d) out[c].b[d] = rng_uniform_range(&r, -0.5, 0.5);
        out[c].radius = rng_uniform_range(&r, 0.03, 0.08);
        out[c].inv_rotation[0] = out[c].inv_rotation[4] = out[c].inv_rotation[8] = 1.0;
    }
}

static const int kGeoOut[5] = {1024, 512, 256, 128, 1};
static const int kTexOut[5] = {1024, 512, 256, 128, 3};

void orc_gen_mlp(uint64_t seed, int which, float* w, float* b) {
    const int* outs = which == ICG_MLP_TEXTURE ? kTexOut : kGeoOut;
    int skip = which == ICG_MLP_TEXTURE ? 513 : 257;
    double slope = 0.02;
    double gain = sqrt(2.0 / (1.0 + slope * slope));
    orc_rng r;
    orc_rng_seed(&r, seed);
    size_t wo = 0, bo = 0;
    for (int l = 0; l < 5; ++l) {
        int in = (l ? outs[l - 1] : 0) + skip;
        double bound = gain * sqrt(3.0 / (double)in);
        for (size_t i = 0; i < (size_t)outs[l] * in; ++i) w[wo + i] = (float)rng_uniform_range(&r, -bound, bound);
        double bb = 1.0 / sqrt((double)in);
        for (int o = 0; o < outs[l]; ++o) b[bo + o] = (float)rng_uniform_range(&r, -bb, bb);
        wo += (size_t)outs[l] * in;
        bo += (size_t)outs[l];
    }
}

/*
 * rt_oracle.c — CPU restatement of emtrace's propagation hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2303_11103_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path never links or calls it.
 *
 * It restates (does not copy) the reference algorithm in plain C, operation by
 * operation where IEEE rounding decides a discrete outcome:
 *   - median-split BVH build        /root/reference/pkg/src/emtrace/bvh.py:33-79
 *   - stack traversal + slab + MT    bvh.py:117-177 (right child popped first)
 *   - intersect / occluded           bvh.py:83-115
 *   - Fibonacci launch               tracer.py:217-244 (directions come from the
 *                                    caller, produced by numpy as geometry.py:62-76)
 *   - image solve + validity         tracer.py:71-183
 *   - path assembly                  tracer.py:105-133
 *   - coincident-path merge          tracer.py:247-265
 *   - polarized transfer             em.py:42-171, 291-312
 *   - probe path gain / coverage     channel.py:190-253
 *
 * numpy's 1-D `a @ b` on 3-vectors dispatches to OpenBLAS ddot, which on the
 * machine the golden vectors were generated on evaluates
 * fma(a2,b2, fma(a1,b1, a0*b0)); `dot_blas` reproduces that.  Python-float
 * expressions (`t_dot`) are left-to-right without contraction: this file must
 * be compiled with -ffp-contract=off.
 *
 * Parallelism: OpenMP over rays (launch) and over cells / receivers (coverage,
 * paths).  Each work item is independent, as the reference's SPEC allows.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LEAF_SIZE 4            /* bvh.py:16 */
#define RAY_EPS 1e-4           /* bvh.py:17 */
#define DET_EPS 1e-12          /* bvh.py:18 */
#define BARY_EPS 1e-12         /* bvh.py:19 */
#define MERGE_TOL 1e-6         /* tracer.py:30 */
#define INSIDE_TOL 1e-9        /* tracer.py:31 */
#define SIDE_TOL 1e-12         /* tracer.py:32 */
#define SPEED_OF_LIGHT 299792458.0
#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#define TWO_PI (2.0 * M_PI)

/* ------------------------------------------------------------------------ */
/* small vector helpers                                                       */

static inline double tdot(const double* a, const double* b) {  /* geometry.py t_dot */
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
static inline double dot_blas(const double* a, const double* b) {  /* numpy 1-D @ */
    return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}

/* ------------------------------------------------------------------------ */
/* BVH                                                                         */

typedef struct {
    double lo[3], hi[3];
    int a, b, leaf;
} onode;

typedef struct {
    int64_t n;
    const double *v0, *e1, *e2;     /* [n*3] in _gather order (bvh.py:180-197) */
    onode* nodes;
    int64_t n_nodes, cap_nodes;
    int64_t* order;                 /* traversal order -> prim id */
    int64_t cursor;
    double* cent; double* lo; double* hi;
    /* per-slot copies in traversal order (bvh.py:54-55) */
    double* tri;                    /* [n*9] v0,e1,e2 */
    int64_t* tri_prim;
} obvh;

typedef struct { double key; int64_t pos; } skey;

static int cmp_skey(const void* x, const void* y) {
    const skey* a = (const skey*)x; const skey* b = (const skey*)y;
    if (a->key < b->key) return -1;
    if (a->key > b->key) return 1;
    return (a->pos < b->pos) ? -1 : (a->pos > b->pos);   /* stable */
}
static int cmp_i64(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    return (a > b) - (a < b);
}

static int64_t push_node(obvh* t) {
    if (t->n_nodes == t->cap_nodes) {
        t->cap_nodes = t->cap_nodes ? 2 * t->cap_nodes : 64;
        t->nodes = (onode*)realloc(t->nodes, sizeof(onode) * t->cap_nodes);
    }
    return t->n_nodes++;
}

/* bvh.py:59-79 — returns node id; idx is owned scratch of length m */
static int64_t build_rec(obvh* t, int64_t* idx, int64_t m) {
    int64_t id = push_node(t);
    double bmin[3], bmax[3];
    for (int k = 0; k < 3; ++k) { bmin[k] = INFINITY; bmax[k] = -INFINITY; }
    for (int64_t i = 0; i < m; ++i) {
        for (int k = 0; k < 3; ++k) {
            double l = t->lo[idx[i] * 3 + k], h = t->hi[idx[i] * 3 + k];
            /* numpy min/max reduce: NaN-free inputs, plain compare */
            if (l < bmin[k]) bmin[k] = l;
            if (h > bmax[k]) bmax[k] = h;
        }
    }
    if (m <= LEAF_SIZE) {
        int64_t* s = (int64_t*)malloc(sizeof(int64_t) * m);
        memcpy(s, idx, sizeof(int64_t) * m);
        qsort(s, m, sizeof(int64_t), cmp_i64);                /* np.sort(idx) */
        for (int64_t i = 0; i < m; ++i) t->order[t->cursor + i] = s[i];
        free(s);
        onode* nd = &t->nodes[id];
        memcpy(nd->lo, bmin, sizeof bmin); memcpy(nd->hi, bmax, sizeof bmax);
        nd->a = (int)t->cursor; nd->b = (int)(t->cursor + m); nd->leaf = 1;
        t->cursor += m;
        return id;
    }
    double cmin[3], cmax[3];
    for (int k = 0; k < 3; ++k) { cmin[k] = INFINITY; cmax[k] = -INFINITY; }
    for (int64_t i = 0; i < m; ++i)
        for (int k = 0; k < 3; ++k) {
            double c = t->cent[idx[i] * 3 + k];
            if (c < cmin[k]) cmin[k] = c;
            if (c > cmax[k]) cmax[k] = c;
        }
    int axis = 0; double best = cmax[0] - cmin[0];          /* np.argmax: first max */
    for (int k = 1; k < 3; ++k) if (cmax[k] - cmin[k] > best) { best = cmax[k] - cmin[k]; axis = k; }
    skey* ks = (skey*)malloc(sizeof(skey) * m);
    for (int64_t i = 0; i < m; ++i) { ks[i].key = t->cent[idx[i] * 3 + axis]; ks[i].pos = i; }
    qsort(ks, m, sizeof(skey), cmp_skey);                     /* stable argsort */
    int64_t* sorted = (int64_t*)malloc(sizeof(int64_t) * m);
    for (int64_t i = 0; i < m; ++i) sorted[i] = idx[ks[i].pos];
    free(ks);
    int64_t half = m / 2;
    int64_t left = build_rec(t, sorted, half);
    int64_t right = build_rec(t, sorted + half, m - half);
    free(sorted);
    onode* nd = &t->nodes[id];
    memcpy(nd->lo, bmin, sizeof bmin); memcpy(nd->hi, bmax, sizeof bmax);
    nd->a = (int)left; nd->b = (int)right; nd->leaf = 0;
    return id;
}

void* orc_bvh_build(const double* v0, const double* e1, const double* e2, int64_t n) {
    obvh* t = (obvh*)calloc(1, sizeof(obvh));
    t->n = n; t->v0 = v0; t->e1 = e1; t->e2 = e2;
    t->order = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    if (n) {
        t->cent = (double*)malloc(sizeof(double) * 3 * n);
        t->lo = (double*)malloc(sizeof(double) * 3 * n);
        t->hi = (double*)malloc(sizeof(double) * 3 * n);
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) {
                double a = v0[i * 3 + k], b = e1[i * 3 + k], c = e2[i * 3 + k];
                t->cent[i * 3 + k] = a + (b + c) / 3.0;       /* bvh.py:49 */
                double p1 = a + b, p2 = a + c;
                double l = fmin(fmin(a, p1), p2), h = fmax(fmax(a, p1), p2);
                t->lo[i * 3 + k] = l; t->hi[i * 3 + k] = h;
            }
        int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * n);
        for (int64_t i = 0; i < n; ++i) idx[i] = i;
        build_rec(t, idx, n);
        free(idx);
        t->tri = (double*)malloc(sizeof(double) * 9 * n);
        t->tri_prim = (int64_t*)malloc(sizeof(int64_t) * n);
        for (int64_t s = 0; s < n; ++s) {
            int64_t p = t->order[s];
            for (int k = 0; k < 3; ++k) {
                t->tri[s * 9 + k] = v0[p * 3 + k];
                t->tri[s * 9 + 3 + k] = e1[p * 3 + k];
                t->tri[s * 9 + 6 + k] = e2[p * 3 + k];
            }
            t->tri_prim[s] = p;
        }
    }
    return t;
}

void orc_bvh_free(void* h) {
    obvh* t = (obvh*)h;
    if (!t) return;
    free(t->nodes); free(t->order); free(t->cent); free(t->lo); free(t->hi);
    free(t->tri); free(t->tri_prim); free(t);
}

int64_t orc_bvh_num_nodes(void* h) { return ((obvh*)h)->n_nodes; }

/* Python's builtin max/min: first argument seeds, later ones replace only on a
 * strict comparison, so NaNs behave exactly as in bvh.py:141-142. */
static inline double pymax4(double a, double b, double c, double d) {
    double m = a; if (b > m) m = b; if (c > m) m = c; if (d > m) m = d; return m;
}
static inline double pymin4(double a, double b, double c, double d) {
    double m = a; if (b < m) m = b; if (c < m) m = c; if (d < m) m = d; return m;
}

/* bvh.py:117-177; returns prim id or -1, *t_out the hit distance */
static int64_t trace(const obvh* t, double ox, double oy, double oz,
                     double dx, double dy, double dz, double t_min, double t_max,
                     int any_hit, double* t_out) {
    if (t->n_nodes == 0) return -1;
    double inv_x = dx != 0.0 ? 1.0 / dx : INFINITY;
    double inv_y = dy != 0.0 ? 1.0 / dy : INFINITY;
    double inv_z = dz != 0.0 ? 1.0 / dz : INFINITY;
    double best_t = t_max; int64_t best_prim = -1;
    int stack[256]; int sp = 0;
    stack[sp++] = 0;
    while (sp) {
        const onode* nd = &t->nodes[stack[--sp]];
        double tx1 = (nd->lo[0] - ox) * inv_x, tx2 = (nd->hi[0] - ox) * inv_x;
        if (tx1 > tx2) { double s = tx1; tx1 = tx2; tx2 = s; }
        double ty1 = (nd->lo[1] - oy) * inv_y, ty2 = (nd->hi[1] - oy) * inv_y;
        if (ty1 > ty2) { double s = ty1; ty1 = ty2; ty2 = s; }
        double tz1 = (nd->lo[2] - oz) * inv_z, tz2 = (nd->hi[2] - oz) * inv_z;
        if (tz1 > tz2) { double s = tz1; tz1 = tz2; tz2 = s; }
        double near = pymax4(tx1, ty1, tz1, t_min);
        double far = pymin4(tx2, ty2, tz2, best_t);
        if (near > far) continue;
        if (!nd->leaf) { stack[sp++] = nd->a; stack[sp++] = nd->b; continue; }
        for (int k = nd->a; k < nd->b; ++k) {
            const double* T = &t->tri[(int64_t)k * 9];
            double v0x = T[0], v0y = T[1], v0z = T[2];
            double e1x = T[3], e1y = T[4], e1z = T[5];
            double e2x = T[6], e2y = T[7], e2z = T[8];
            double px = dy * e2z - dz * e2y;
            double py = dz * e2x - dx * e2z;
            double pz = dx * e2y - dy * e2x;
            double det = e1x * px + e1y * py + e1z * pz;
            if (-DET_EPS < det && det < DET_EPS) continue;
            double inv_det = 1.0 / det;
            double tx = ox - v0x, ty = oy - v0y, tz = oz - v0z;
            double u = (tx * px + ty * py + tz * pz) * inv_det;
            if (u < -BARY_EPS || u > 1.0 + BARY_EPS) continue;
            double qx = ty * e1z - tz * e1y;
            double qy = tz * e1x - tx * e1z;
            double qz = tx * e1y - ty * e1x;
            double v = (dx * qx + dy * qy + dz * qz) * inv_det;
            if (v < -BARY_EPS || u + v > 1.0 + BARY_EPS) continue;
            double tt = (e2x * qx + e2y * qy + e2z * qz) * inv_det;
            if (t_min < tt && tt < best_t) {
                best_t = tt; best_prim = t->tri_prim[k];
                if (any_hit) { *t_out = best_t; return best_prim; }
            }
        }
    }
    *t_out = best_t;
    return best_prim;
}

/* batch intersect: bvh.py:83-101 (t, prim); any_hit selects bvh.py:103-115 semantics */
void orc_trace(void* h, const double* o, const double* d, const double* tmin,
               const double* tmax, int64_t n, int any_hit, double* t_out, int64_t* prim_out) {
    const obvh* t = (const obvh*)h;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        double tt = 0.0;
        int64_t p = trace(t, o[3 * i], o[3 * i + 1], o[3 * i + 2], d[3 * i], d[3 * i + 1],
                          d[3 * i + 2], tmin[i], tmax[i], any_hit, &tt);
        prim_out[i] = p; t_out[i] = p >= 0 ? tt : INFINITY;
    }
}

/* bvh.py:103-115; returns 1 occluded, 0 clear, -1 coincident endpoints */
static int occluded(const obvh* t, const double* p, const double* q, double eps) {
    double dx = q[0] - p[0], dy = q[1] - p[1], dz = q[2] - p[2];
    double dist = sqrt(dx * dx + dy * dy + dz * dz);
    if (dist == 0.0) return -1;
    double inv = 1.0 / dist;
    double tt;
    return trace(t, p[0], p[1], p[2], dx * inv, dy * inv, dz * inv, eps, dist - eps, 1, &tt) >= 0;
}

int orc_occluded(void* h, const double* p, const double* q) {
    return occluded((const obvh*)h, p, q, RAY_EPS);
}

/* ------------------------------------------------------------------------ */
/* launch: tracer.py:217-244                                                   */

/* For each direction: up to max_depth closest hits; seq_out[i*max_depth + k]
 * holds the k-th hit prim (-1 after the ray escapes).  bounces_out[i] counts
 * intersect calls, including the final miss (SURVEY §8d unit). */
void orc_launch(void* h, const double* normals, const double* tx, const double* dirs,
                int64_t n, int max_depth, int32_t* seq_out, int32_t* bounces_out) {
    const obvh* t = (const obvh*)h;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
        double o[3] = {tx[0], tx[1], tx[2]};
        double d[3] = {dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
        int32_t* seq = seq_out + i * max_depth;
        for (int k = 0; k < max_depth; ++k) seq[k] = -1;
        int nb = 0;
        for (int k = 0; k < max_depth; ++k) {
            double tt;
            ++nb;
            int64_t p = trace(t, o[0], o[1], o[2], d[0], d[1], d[2], RAY_EPS, INFINITY, 0, &tt);
            if (p < 0) break;
            seq[k] = (int32_t)p;
            double nrm[3] = {normals[3 * p], normals[3 * p + 1], normals[3 * p + 2]};
            if (dot_blas(nrm, d) > 0.0) { nrm[0] = -nrm[0]; nrm[1] = -nrm[1]; nrm[2] = -nrm[2]; }
            double pt[3] = {o[0] + tt * d[0], o[1] + tt * d[1], o[2] + tt * d[2]};
            double kk = 2.0 * dot_blas(d, nrm);
            for (int c = 0; c < 3; ++c) d[c] = d[c] - kk * nrm[c];
            o[0] = pt[0]; o[1] = pt[1]; o[2] = pt[2];
        }
        bounces_out[i] = nb;
    }
}

/* ------------------------------------------------------------------------ */
/* image method: tracer.py:71-183                                              */

typedef struct {
    const obvh* bvh;
    const double* normals;       /* [n*3] */
    const double* plane_offset;  /* [n]   */
} oscene;

static inline void mirror(const double* p, const double* n, double c, double* out) {
    double k = 2.0 * (tdot(p, n) - c);                        /* tracer.py:71-73 */
    out[0] = p[0] - n[0] * k; out[1] = p[1] - n[1] * k; out[2] = p[2] - n[2] * k;
}

static int inside_triangle(const obvh* b, int64_t prim, const double* p) {  /* tracer.py:136-147 */
    const double* v0 = b->v0 + 3 * prim; const double* e1 = b->e1 + 3 * prim;
    const double* e2 = b->e2 + 3 * prim;
    double w[3] = {p[0] - v0[0], p[1] - v0[1], p[2] - v0[2]};
    double d11 = dot_blas(e1, e1), d12 = dot_blas(e1, e2), d22 = dot_blas(e2, e2);
    double w1 = dot_blas(w, e1), w2 = dot_blas(w, e2);
    double den = d11 * d22 - d12 * d12;
    double u = (d22 * w1 - d12 * w2) / den;
    double v = (d11 * w2 - d12 * w1) / den;
    return u >= -INSIDE_TOL && v >= -INSIDE_TOL && u + v <= 1.0 + INSIDE_TOL;
}

/* Returns 1 when valid; pts_out [k*3] the interaction points. */
static int image_solve(const oscene* sc, const double* tx, const double* rx,
                       const int32_t* seq, int k, double* pts) {
    double images[16][3];
    memcpy(images[0], tx, 3 * sizeof(double));
    for (int j = 0; j < k; ++j)
        mirror(images[j], sc->normals + 3 * seq[j], sc->plane_offset[seq[j]], images[j + 1]);
    double cur[3] = {rx[0], rx[1], rx[2]};
    double params[16];
    for (int j = k - 1; j >= 0; --j) {
        const double* n = sc->normals + 3 * seq[j]; double c = sc->plane_offset[seq[j]];
        double seg[3] = {images[j + 1][0] - cur[0], images[j + 1][1] - cur[1], images[j + 1][2] - cur[2]};
        double denom = tdot(seg, n);
        if (fabs(denom) < 1e-15) return 0;
        double s = (c - tdot(cur, n)) / denom;
        double* p = pts + 3 * j;
        p[0] = cur[0] + seg[0] * s; p[1] = cur[1] + seg[1] * s; p[2] = cur[2] + seg[2] * s;
        params[j] = s;
        cur[0] = p[0]; cur[1] = p[1]; cur[2] = p[2];
    }
    for (int j = 0; j < k; ++j)
        if (!(1e-12 < params[j] && params[j] < 1.0 - 1e-12)) return 0;
    for (int j = 0; j < k; ++j)
        if (!inside_triangle(sc->bvh, seq[j], pts + 3 * j)) return 0;
    const double* chain[18];
    chain[0] = tx;
    for (int j = 0; j < k; ++j) chain[j + 1] = pts + 3 * j;
    chain[k + 1] = rx;
    for (int j = 0; j < k; ++j) {
        const double* n = sc->normals + 3 * seq[j]; double c = sc->plane_offset[seq[j]];
        double before = tdot(chain[j], n) - c;
        double after = tdot(chain[j + 2], n) - c;
        if (before * after <= SIDE_TOL) return 0;
    }
    for (int j = 0; j <= k; ++j) {
        const double* a = chain[j]; const double* b = chain[j + 1];
        double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
        double d = sqrt(dx * dx + dy * dy + dz * dz);        /* math.dist */
        if (d <= 2 * RAY_EPS) return 0;
        if (occluded(sc->bvh, a, b, RAY_EPS) != 0) return 0;
    }
    return 1;
}

int orc_image_solve(void* h, const double* normals, const double* poff, const double* tx,
                    const double* rx, const int32_t* seq, int k, double* pts_out) {
    oscene sc = {(const obvh*)h, normals, poff};
    return image_solve(&sc, tx, rx, seq, k, pts_out);
}

/* ------------------------------------------------------------------------ */
/* paths between one tx and one probe / rx: tracer.py:268-295                 */

typedef struct {
    int32_t cand;        /* -1 for LOS */
    int32_t order;
    double pts[16 * 3];
} opath;

static int allclose3(const double* a, const double* b) {        /* np.allclose */
    for (int c = 0; c < 3; ++c)
        if (!(fabs(a[c] - b[c]) <= 1e-8 + 1e-5 * fabs(b[c]))) return 0;
    return 1;
}

/* Candidates are given sorted by (length, lexicographic sequence): for equal
 * length this is Python's tuple order, which is all the merge and the final
 * (los, order, seq) sort depend on.  Returns the number of kept paths or -1
 * when tx and rx coincide (tracer.py:188-189). */
static int paths_between(const oscene* sc, const double* tx, const double* rx,
                         const int32_t* cands, const int8_t* lens, int64_t n_cand,
                         int max_len, opath* out, int cap) {
    if (allclose3(tx, rx)) return -1;
    int np_ = 0;
    if (!(sc->bvh->n && occluded(sc->bvh, tx, rx, RAY_EPS) == 1)) {
        out[np_].cand = -1; out[np_].order = 0; ++np_;
    }
    double pts[16 * 3];
    for (int64_t c = 0; c < n_cand; ++c) {
        int k = lens[c];
        const int32_t* seq = cands + c * max_len;
        if (!image_solve(sc, tx, rx, seq, k, pts)) continue;
        /* _merge_coincident: tracer.py:247-265 (kept-list greedy) */
        int merged = 0;
        for (int q = 0; q < np_; ++q) {
            if (out[q].order != k || k == 0) continue;
            double mx = 0.0;
            for (int j = 0; j < 3 * k; ++j) {
                double dd = fabs(pts[j] - out[q].pts[j]);
                if (dd > mx) mx = dd;
            }
            if (mx < MERGE_TOL) { merged = 1; break; }
        }
        if (merged) continue;
        if (np_ == cap) return -2;
        out[np_].cand = (int32_t)c; out[np_].order = k;
        memcpy(out[np_].pts, pts, sizeof(double) * 3 * k);
        ++np_;
    }
    return np_;
}

/* Batched over receivers.  out_* are [n_rx * cap]; counts_out[r] the number of
 * kept paths (or -1 coincident, -2 overflow).  Paths are emitted in candidate
 * order per receiver: LOS first, then (order, seq) since candidates are sorted. */
void orc_paths(void* h, const double* normals, const double* poff, const double* tx,
               const double* rx, int64_t n_rx, const int32_t* cands, const int8_t* lens,
               int64_t n_cand, int max_len, int cap, int32_t* cand_out, double* pts_out,
               int32_t* counts_out) {
    oscene sc = {(const obvh*)h, normals, poff};
#pragma omp parallel
    {
        opath* buf = (opath*)malloc(sizeof(opath) * cap);
#pragma omp for schedule(dynamic, 1)
        for (int64_t r = 0; r < n_rx; ++r) {
            int np_ = paths_between(&sc, tx, rx + 3 * r, cands, lens, n_cand, max_len, buf, cap);
            counts_out[r] = np_;
            for (int q = 0; q < np_; ++q) {
                cand_out[r * cap + q] = buf[q].cand;
                memcpy(pts_out + (r * cap + q) * max_len * 3, buf[q].pts,
                       sizeof(double) * 3 * buf[q].order);
            }
        }
        free(buf);
    }
}

/* ------------------------------------------------------------------------ */
/* electromagnetics: em.py                                                     */

typedef struct { double re, im; } cplx;
static inline cplx cmul(cplx a, cplx b) {  /* autodiff.py DiffComplex.__mul__ */
    cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; return r;
}
static inline cplx cdiv(cplx a, cplx o) {  /* DiffComplex.__truediv__ */
    double d = o.re * o.re + o.im * o.im;
    cplx r = {(a.re * o.re + a.im * o.im) / d, (a.im * o.re - a.re * o.im) / d}; return r;
}
static inline cplx cscale(cplx a, double s) { cplx r = {a.re * s, a.im * s}; return r; }
static inline cplx cadd(cplx a, cplx b) { cplx r = {a.re + b.re, a.im + b.im}; return r; }
static inline cplx csub(cplx a, cplx b) { cplx r = {a.re - b.re, a.im - b.im}; return r; }

enum { PAT_ISO = 0, PAT_DIPOLE = 1, PAT_TR38901 = 2, PAT_PROBE_THETA = 3, PAT_PROBE_PHI = 4 };

static void pattern(int id, double theta, double phi, double* eth, double* eph) {  /* em.py:42-75 */
    *eth = 0.0; *eph = 0.0;
    switch (id) {
    case PAT_ISO: *eth = 1.0; break;
    case PAT_DIPOLE: {
        double s = sin(theta);
        if (s < 1e-9) return;
        *eth = sqrt(1.643) * cos(1.5707963267948966 * cos(theta)) / s;
        break;
    }
    case PAT_TR38901: {
        double deg = 180.0 / M_PI;
        double tilt = theta * deg - 90.0, pan = phi * deg;
        double av = 12.0 * (tilt / 65.0) * (tilt / 65.0); if (!(av <= 30.0)) av = 30.0;
        double ah = 12.0 * (pan / 65.0) * (pan / 65.0); if (!(ah <= 30.0)) ah = 30.0;
        double s = av + ah; if (!(s <= 30.0)) s = 30.0;
        *eth = exp((8.0 - s) * (log(10.0) / 20.0));
        break;
    }
    case PAT_PROBE_THETA: *eth = 1.0; break;
    case PAT_PROBE_PHI: *eph = 1.0; break;
    }
}

/* em.py:98-118; rows is the 3x3 row-major device rotation */
static void element_field(int pat, double slant, const double* R, const double* k, double* out) {
    double kb[3] = {R[0] * k[0] + R[3] * k[1] + R[6] * k[2],
                    R[1] * k[0] + R[4] * k[1] + R[7] * k[2],
                    R[2] * k[0] + R[5] * k[1] + R[8] * k[2]};
    double cz = cos(slant), sz = sin(slant);
    double ke[3] = {kb[0], cz * kb[1] + sz * kb[2], -sz * kb[1] + cz * kb[2]};
    double theta = atan2(sqrt(ke[0] * ke[0] + ke[1] * ke[1]), ke[2]);
    double phi = atan2(ke[1], ke[0]);
    double eth, eph;
    pattern(pat, theta, phi, &eth, &eph);
    double ct = cos(theta), st = sin(theta), cp = cos(phi), sp = sin(phi);
    double ee[3] = {eth * (ct * cp) + eph * (-sp), eth * (ct * sp) + eph * cp, eth * (-st)};
    double eb[3] = {ee[0], cz * ee[1] - sz * ee[2], sz * ee[1] + cz * ee[2]};
    out[0] = R[0] * eb[0] + R[1] * eb[1] + R[2] * eb[2];
    out[1] = R[3] * eb[0] + R[4] * eb[1] + R[5] * eb[2];
    out[2] = R[6] * eb[0] + R[7] * eb[1] + R[8] * eb[2];
}

static cplx csqrt_posreal(cplx z) {  /* autodiff.py:365-382 */
    double m = sqrt(z.re * z.re + z.im * z.im);
    double u2 = (m + z.re) * 0.5, v2 = (m - z.re) * 0.5;
    double u = u2 > 0.0 ? sqrt(u2) : u2 * 0.0;
    double v = v2 > 0.0 ? sqrt(v2) : v2 * 0.0;
    if (z.im < 0.0) v = -v;
    cplx r = {u, v}; return r;
}

static void fresnel(cplx eta, double ci, cplx* rte, cplx* rtm) {  /* em.py:123-141 */
    double sin2 = 1.0 - ci * ci;
    cplx arg = {eta.re - sin2, eta.im};
    cplx w = csqrt_posreal(arg);
    cplx c = {ci, 0.0};
    *rte = cdiv(csub(c, w), cadd(c, w));
    cplx ec = cscale(eta, ci);
    *rtm = cdiv(csub(w, ec), cadd(w, ec));
}

static inline void cross3(const double* a, const double* b, double* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
static inline void normalize3(double* a) {
    double n = sqrt(tdot(a, a));
    a[0] /= n; a[1] /= n; a[2] /= n;
}

static void reflect_field(cplx* f, const double* kin, const double* kout, const double* n,
                          cplx rte, cplx rtm) {  /* em.py:144-171 */
    double ep[3];
    cross3(kin, n, ep);
    if (tdot(ep, ep) < 1e-16) {
        double a0 = fabs(kin[0]), a1 = fabs(kin[1]), a2 = fabs(kin[2]);
        int ax = 0; double mn = a0;
        if (a1 < mn) { mn = a1; ax = 1; }
        if (a2 < mn) { mn = a2; ax = 2; }
        double axis[3] = {0.0, 0.0, 0.0}; axis[ax] = 1.0;
        cross3(kin, axis, ep);
    }
    normalize3(ep);
    double epi[3], epr[3];
    cross3(kin, ep, epi);
    cross3(ep, kout, epr);
    cplx fp = cadd(cadd(cscale(f[0], ep[0]), cscale(f[1], ep[1])), cscale(f[2], ep[2]));
    cplx fa = cadd(cadd(cscale(f[0], epi[0]), cscale(f[1], epi[1])), cscale(f[2], epi[2]));
    cplx gp = cmul(rte, fp), ga = cmul(rtm, fa);
    for (int c = 0; c < 3; ++c) f[c] = cadd(cscale(gp, ep[c]), cscale(ga, epr[c]));
}

typedef struct {
    double wavelength, frequency;
    const double* eta;        /* [n_mat*2] */
    const int32_t* prim_mat;  /* [n_prims] */
    const double* normals;
} oem;

/* Path geometry as geometry_from_path (em.py:246-255) from vertices [k+2] and
 * the incidence-oriented normals/cosines of path_from_points (tracer.py:105-133). */
typedef struct {
    int k;
    double verts[18][3];
    double dirs[17][3];
    double nrm[16][3];
    double cosi[16];
    double length, delay;
} ogeom;

static void make_geom(const oem* em, const double* tx, const double* rx, const int32_t* seq,
                      int k, const double* pts, ogeom* g) {
    g->k = k;
    memcpy(g->verts[0], tx, 24);
    for (int j = 0; j < k; ++j) memcpy(g->verts[j + 1], pts + 3 * j, 24);
    memcpy(g->verts[k + 1], rx, 24);
    double total = 0.0;
    double ndirs[17][3];
    for (int j = 0; j <= k; ++j) {
        double s[3] = {g->verts[j + 1][0] - g->verts[j][0], g->verts[j + 1][1] - g->verts[j][1],
                       g->verts[j + 1][2] - g->verts[j][2]};
        double l = sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);   /* np.linalg.norm axis=1 */
        total += l;                                                   /* lens.sum() */
        for (int c = 0; c < 3; ++c) ndirs[j][c] = s[c] / l;          /* numpy dirs */
        double t[3] = {s[0], s[1], s[2]};                            /* t_normalize */
        double tn = sqrt(tdot(t, t));
        for (int c = 0; c < 3; ++c) g->dirs[j][c] = t[c] / tn;
    }
    for (int j = 0; j < k; ++j) {
        const double* n = em->normals + 3 * seq[j];
        double ci = -dot_blas(ndirs[j], n);
        double sgn = 1.0;
        if (ci < 0.0) { sgn = -1.0; ci = -ci; }
        for (int c = 0; c < 3; ++c) g->nrm[j][c] = sgn * n[c];
        g->cosi[j] = ci;
    }
    g->length = total;
    g->delay = total / SPEED_OF_LIGHT;
}

/* em.py:291-312 */
static cplx transfer(const oem* em, const ogeom* g, const int32_t* seq, int tx_pat,
                     double tx_slant, const double* Rtx, int rx_pat, double rx_slant,
                     const double* Rrx) {
    double ef[3];
    element_field(tx_pat, tx_slant, Rtx, g->dirs[0], ef);
    cplx f[3] = {{ef[0], 0.0}, {ef[1], 0.0}, {ef[2], 0.0}};
    for (int j = 0; j < g->k; ++j) {
        int m = em->prim_mat[seq[j]];
        cplx eta = {em->eta[2 * m], em->eta[2 * m + 1]};
        cplx rte, rtm;
        fresnel(eta, g->cosi[j], &rte, &rtm);
        reflect_field(f, g->dirs[j], g->dirs[j + 1], g->nrm[j], rte, rtm);
    }
    double karr[3] = {g->dirs[g->k][0] * -1.0, g->dirs[g->k][1] * -1.0, g->dirs[g->k][2] * -1.0};
    double rf[3];
    element_field(rx_pat, rx_slant, Rrx, karr, rf);
    cplx coup = cadd(cadd(cscale(f[0], rf[0]), cscale(f[1], rf[1])), cscale(f[2], rf[2]));
    double amp = em->wavelength / (2.0 * TWO_PI * g->length);
    double phase = -TWO_PI * em->frequency * g->delay;
    cplx ph = {cos(phase), sin(phase)};
    return cmul(cscale(coup, amp), ph);
}

/* One transfer per path given its vertices; used for compute_gains parity. */
void orc_transfer(const double* normals, const int32_t* prim_mat, const double* eta,
                  double wavelength, double frequency, const double* tx, const double* rx,
                  const int32_t* seq, int k, const double* pts, int tx_pat, double tx_slant,
                  const double* Rtx, int rx_pat, double rx_slant, const double* Rrx,
                  double* out_re_im) {
    oem em = {wavelength, frequency, eta, prim_mat, normals};
    ogeom g;
    make_geom(&em, tx, rx, seq, k, pts, &g);
    cplx a = transfer(&em, &g, seq, tx_pat, tx_slant, Rtx, rx_pat, rx_slant, Rrx);
    out_re_im[0] = a.re; out_re_im[1] = a.im;
}

/* point_path_gain (channel.py:190-233) over many probe points; tx_mode 0 =
 * central element, 1 = coherent array sum with element offsets (already
 * rotated to world, em.py:373-374) and per-element slants. */
void orc_coverage(void* h, const double* normals, const double* poff, const int32_t* prim_mat,
                  const double* eta, double wavelength, double frequency, const double* tx,
                  const double* Rtx, int tx_pat, const double* slants, const double* offsets_w,
                  int n_el, int tx_mode, const double* Rprobe, const double* points, int64_t n_pts,
                  const int32_t* cands, const int8_t* lens, int64_t n_cand, int max_len,
                  int cap, double* gains_out, int32_t* counts_out) {
    oscene sc = {(const obvh*)h, normals, poff};
    oem em = {wavelength, frequency, eta, prim_mat, normals};
#pragma omp parallel
    {
        opath* buf = (opath*)malloc(sizeof(opath) * cap);
#pragma omp for schedule(dynamic, 1)
        for (int64_t r = 0; r < n_pts; ++r) {
            const double* rx = points + 3 * r;
            int np_ = paths_between(&sc, tx, rx, cands, lens, n_cand, max_len, buf, cap);
            counts_out[r] = np_;
            double gain = 0.0;
            for (int q = 0; q < np_; ++q) {
                const int32_t* seq = buf[q].cand >= 0 ? cands + (int64_t)buf[q].cand * max_len : NULL;
                ogeom g;
                make_geom(&em, tx, rx, seq, buf[q].order, buf[q].pts, &g);
                for (int pol = 0; pol < 2; ++pol) {
                    int rp = pol == 0 ? PAT_PROBE_THETA : PAT_PROBE_PHI;
                    cplx a;
                    if (tx_mode == 0) {
                        a = transfer(&em, &g, seq, tx_pat, slants[0], Rtx, rp, 0.0, Rprobe);
                    } else {
                        a.re = 0.0; a.im = 0.0;
                        for (int e = 0; e < n_el; ++e) {
                            cplx el = transfer(&em, &g, seq, tx_pat, slants[e], Rtx, rp, 0.0, Rprobe);
                            double ph = TWO_PI * tdot(g.dirs[0], offsets_w + 3 * e) / wavelength;
                            cplx z = {cos(ph), sin(ph)};
                            a = cadd(a, cmul(el, z));
                        }
                    }
                    gain = gain + (a.re * a.re + a.im * a.im);
                }
            }
            gains_out[r] = np_ >= 0 ? gain : NAN;
        }
        free(buf);
    }
}

/* ------------------------------------------------------------------------ */
/* prefix set: the `found` set of tracer.py:232-243 (every prefix of every    */
/* ray's hit history) for launches too large for Python tuples.  Keys are     */
/* prefixes padded with -1 to L entries; open addressing, FNV-1a hash.        */

typedef struct {
    int L;
    int64_t cap, n;
    int32_t* keys;   /* cap * L; slot empty when keys[s*L] == INT32_MIN */
} opset;

static uint64_t pset_hash(const int32_t* k, int L) {
    uint64_t h = 1469598103934665603ULL;
    for (int i = 0; i < L; ++i) {
        h ^= (uint32_t)k[i];
        h *= 1099511628211ULL;
    }
    return h ^ (h >> 29);
}

static void pset_alloc(opset* s, int64_t cap) {
    s->cap = cap;
    s->keys = (int32_t*)malloc(sizeof(int32_t) * cap * s->L);
    for (int64_t i = 0; i < cap; ++i) s->keys[i * s->L] = INT32_MIN;
}

static int pset_insert(opset* s, const int32_t* k) {
    uint64_t m = (uint64_t)s->cap - 1, h = pset_hash(k, s->L) & m;
    for (;;) {
        int32_t* slot = s->keys + h * s->L;
        if (slot[0] == INT32_MIN) {
            memcpy(slot, k, sizeof(int32_t) * s->L);
            s->n++;
            return 1;
        }
        if (memcmp(slot, k, sizeof(int32_t) * s->L) == 0) return 0;
        h = (h + 1) & m;
    }
}

void* orc_pset_new(int L) {
    opset* s = (opset*)calloc(1, sizeof(opset));
    s->L = L;
    pset_alloc(s, 1 << 16);
    return s;
}

void orc_pset_free(void* h) {
    opset* s = (opset*)h;
    free(s->keys);
    free(s);
}

/* add every prefix of each row of seq [n, L] (rows end at the first -1) */
void orc_pset_add(void* h, const int32_t* seq, int64_t n) {
    opset* s = (opset*)h;
    int L = s->L;
    int32_t key[16];
    for (int64_t i = 0; i < n; ++i) {
        const int32_t* r = seq + i * L;
        for (int k = 0; k < L && r[k] >= 0; ++k) {
            for (int j = 0; j < L; ++j) key[j] = j <= k ? r[j] : -1;
            if (2 * (s->n + 1) > s->cap) {   /* grow: keep the load below 1/2 */
                opset t = {L, 0, 0, NULL};
                pset_alloc(&t, s->cap * 4);
                for (int64_t q = 0; q < s->cap; ++q)
                    if (s->keys[q * L] != INT32_MIN) pset_insert(&t, s->keys + q * L);
                free(s->keys);
                *s = t;
            }
            pset_insert(s, key);
        }
    }
}

int64_t orc_pset_size(void* h) { return ((opset*)h)->n; }

/* the set's keys [n, L] in slot order (the caller sorts) */
void orc_pset_export(void* h, int32_t* out) {
    opset* s = (opset*)h;
    int64_t w = 0;
    for (int64_t q = 0; q < s->cap; ++q)
        if (s->keys[q * s->L] != INT32_MIN) memcpy(out + (w++) * s->L, s->keys + q * s->L, sizeof(int32_t) * s->L);
}

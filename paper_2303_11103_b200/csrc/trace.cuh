// trace.cuh — BVH traversal with the reference's FP64 Moller-Trumbore test.
//
// Semantics (bvh.py:117-177 restated as a closest-hit query): the hit is the
// triangle with the smallest t in (t_min, t_max) among all triangles whose
// FP64 Moller-Trumbore test (two-sided, det window 1e-12, barycentric
// tolerance 1e-12, operation order of bvh.py:151-170) accepts the ray; equal
// t resolves to the lower global prim id (the reference's brute-force oracle,
// tests/conftest.py:45-80).  Node boxes are conservative (inflated, rounded
// outward to float) so the tree never culls a triangle the exact test accepts.

#pragma once
#include "rt_common.cuh"

// The per-push stack bound check is compiled out when the builder verified
// that the tree depth fits the stack (PLOC build: rt_bvh_build fails loudly
// otherwise; at most one entry per ancestor is ever on the stack).
// Measured on C3 (launch ms): unchecked 22.40 vs checked 21.96 (code layout),
// so the check stays on by default; the depth is still verified and reported
// (C3 tree depth 25, C5 30).
#ifndef RT_STACK_CHECK
#define RT_STACK_CHECK 1
#endif

// per-prim skip of the subtree behind the wall a ray leaves (bvh_ploc.cuh
// k_skip_table).  Measured on C3: 19.2 -> 16.2 node visits and 2.9 -> 1.75
// triangle tests per bounce, launch 14.3 -> 13.0 ms.
#ifndef RT_ORIGIN_SKIP
#define RT_ORIGIN_SKIP 1
#endif
#ifndef RT_END_SKIP
#define RT_END_SKIP 0   // measured on C3: validate 3.01 (on) vs 2.99 ms (off); kept as an A/B
#endif
#if RT_ORIGIN_SKIP
#define RT_SKIPPED(ref) ((ref) == skip || (ANY && RT_END_SKIP && (ref) == skip_end))
#else
#define RT_SKIPPED(ref) false
#endif

namespace rt {

struct Ray {
    double ox, oy, oz, dx, dy, dz;
    float fix, fiy, fiz;      // FP32 1/d for the box filter
    float oix, oiy, oiz;      // FP32 -(o * (1/d)): slab planes are fma(bound, inv, oi)
};

// 1/d, +inf where d == 0 (bvh.py:120-122)
__device__ __forceinline__ double inv_dir(double d) {
    return d != 0.0 ? 1.0 / d : __longlong_as_double(0x7ff0000000000000LL);
}

// FP32 reciprocal for the box filter.  RT_RCP_APPROX: one MUFU.RCP
// (rcp.approx.ftz, <= 1 ulp = 2^-23 relative) instead of the correctly rounded
// __frcp_rn (a ~10-instruction sequence per axis); the box inflation eps_box
// doubles to cover the extra ulp (slab32's error budget below).
__device__ __forceinline__ float rcp32(float x) {
#if RT_RCP_APPROX
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
#else
    return __frcp_rn(x);
#endif
}

__device__ inline Ray make_ray(d3 o, d3 d) {
    Ray r;
    r.ox = o.x; r.oy = o.y; r.oz = o.z;
    r.dx = d.x; r.dy = d.y; r.dz = d.z;
    // clamp 1/d to +-1e30: with an infinite inverse the fma form yields
    // inf - inf = NaN on one plane and +-inf on the other, which mis-culls a
    // slab the ray lies inside; a 1e-30 direction component moves the ray by
    // < 1e-25 m over any scene, far inside eps_box.
    // FP32 reciprocal of the FP32-rounded component: 1 + 2 units of 2^-24
    // relative (rounding of d, then the approximate reciprocal) instead of the
    // FP64 quotient's one, which the slab32 error budget absorbs; no FP64
    // divides per bounce.
    // d = +-0 gives +-inf -> +-1e30: min/max over the two planes is symmetric.
    r.fix = fminf(fmaxf(rcp32(__double2float_rn(d.x)), -1e30f), 1e30f);
    r.fiy = fminf(fmaxf(rcp32(__double2float_rn(d.y)), -1e30f), 1e30f);
    r.fiz = fminf(fmaxf(rcp32(__double2float_rn(d.z)), -1e30f), 1e30f);
    r.oix = -((float)o.x * r.fix); r.oiy = -((float)o.y * r.fiy); r.oiz = -((float)o.z * r.fiz);
    return r;
}

// FP32 box filter, one FFMA per slab plane: t = bound * inv - o * inv.
// Conservative by construction: node boxes are inflated by eps_box = 2^-19 S
// (S = max |scene coordinate|; 2^-20 S with the correctly rounded
// reciprocal).  For |o| <= 2S the spatial error of a plane distance is
// <= 2^-24 (|o| [origin rounding] + |o| [o*inv rounding] + 3 |bound - o|
// [1/d: d rounded to FP32 (1 unit), then rcp.approx (<= 2 units)] + |t d|
// [fma rounding]) <= (2 + 2 + 9 + 3) * 2^-24 S = 16 * 2^-24 S < eps_box =
// 32 * 2^-24 S (with __frcp_rn: 13 units < 16).
// tmin is rounded down and tmax up by the caller; 1/d is clamped (make_ray)
// so no plane distance is NaN.
// both planes of one slab in one packed FFMA2 (sm_100): (lo, hi) * inv + oi,
// inv and oi broadcast; per lane an IEEE fma, bit-identical to two FFMAs
__device__ __forceinline__ float2 slab_planes(float2 lohi, float inv, float oi) {
    unsigned long long x, s, t, o;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(lohi.x), "f"(lohi.y));
    asm("mov.b64 %0, {%1, %1};" : "=l"(s) : "f"(inv));
    asm("mov.b64 %0, {%1, %1};" : "=l"(t) : "f"(oi));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(o) : "l"(x), "l"(s), "l"(t));
    float2 v;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(o));
    return v;
}

__device__ __forceinline__ bool slab32(const Ray& r, float2 x, float2 y, float2 z, float tmin, float tmax,
                                       float& tnear) {
    float2 tx = slab_planes(x, r.fix, r.oix), ty = slab_planes(y, r.fiy, r.oiy),
           tz = slab_planes(z, r.fiz, r.oiz);
    float n = fmaxf(fmaxf(fminf(tx.x, tx.y), fminf(ty.x, ty.y)), fmaxf(fminf(tz.x, tz.y), tmin));
    float f = fminf(fminf(fmaxf(tx.x, tx.y), fmaxf(ty.x, ty.y)), fminf(fmaxf(tz.x, tz.y), tmax));
    tnear = n;
    return n <= f;
}

// slab32 for a ray whose direction signs are fixed at compile time (bit a of
// OCT set: 1/d_a < 0, so the hi plane is the entry plane of axis a): the six
// per-axis min / max of slab32 become register choices.  Same result bits:
// fma(b, inv, oi) is monotonic in b, so min / max pick exactly these planes.
template <int OCT>
__device__ __forceinline__ bool slab32_oct(const Ray& r, float2 x, float2 y, float2 z, float tmin, float tmax,
                                           float& tnear) {
    float2 tx = slab_planes(x, r.fix, r.oix), ty = slab_planes(y, r.fiy, r.oiy),
           tz = slab_planes(z, r.fiz, r.oiz);
    float nx = (OCT & 1) ? tx.y : tx.x, fx = (OCT & 1) ? tx.x : tx.y;
    float ny = (OCT & 2) ? ty.y : ty.x, fy = (OCT & 2) ? ty.x : ty.y;
    float nz = (OCT & 4) ? tz.y : tz.x, fz = (OCT & 4) ? tz.x : tz.y;
    float n = fmaxf(fmaxf(nx, ny), fmaxf(nz, tmin));
    float f = fminf(fminf(fx, fy), fminf(fz, tmax));
    tnear = n;
    return n <= f;
}

// FP64 slab test (origins beyond the FP32 filter's range); NaN never culls.
__device__ __forceinline__ bool slab(const Ray& r, float lx, float ly, float lz, float hx,
                                     float hy, float hz, double tmin, double tmax,
                                     double& tnear) {
    double ix = inv_dir(r.dx), iy = inv_dir(r.dy), iz = inv_dir(r.dz);
    double t0x = ((double)lx - r.ox) * ix, t1x = ((double)hx - r.ox) * ix;
    double t0y = ((double)ly - r.oy) * iy, t1y = ((double)hy - r.oy) * iy;
    double t0z = ((double)lz - r.oz) * iz, t1z = ((double)hz - r.oz) * iz;
    double n = fmax(fmax(fmin(t0x, t1x), fmin(t0y, t1y)), fmax(fmin(t0z, t1z), tmin));
    double f = fmin(fmin(fmax(t0x, t1x), fmax(t0y, t1y)), fmin(fmax(t0z, t1z), tmax));
    tnear = n;
    return n <= f;
}

// a child box as its three (lo, hi) pairs (BNode layout)
__device__ __forceinline__ bool box_hit(const Ray& r, bool fast, float2 x, float2 y, float2 z, double tmin,
                                        double tmax, float tmin_f, float tmax_f, float& tn) {
    if (fast) return slab32(r, x, y, z, tmin_f, tmax_f, tn);
    double d;
    bool h = slab(r, x.x, y.x, z.x, x.y, y.y, z.y, tmin, tmax, d);
    tn = __double2float_rd(d);
    return h;
}

// bvh.py:151-170 in operation order; returns true and t when accepted.
//
// The reference divides once (inv_det = 1/det) and multiplies: u = u_num *
// inv_det etc.  The computed u is within 2^-52 relative of the exact quotient
// u_num/det, so a test whose outcome is already certain from the exact
// numerator (rejected with a 1e-6 relative margin) skips the division; every
// other case runs the reference's arithmetic verbatim.  Decisions are
// therefore identical to the reference's, and the FP64 divide only runs for
// near-hits.  `tmax` is the current closest hit for the t-window quick reject.
__device__ __forceinline__ bool mt_test(const Ray& r, const TriRec* __restrict__ tp, double tmin,
                                        double tmax, double& t) {
    const double2* q = reinterpret_cast<const double2*>(tp);
    double2 a = __ldg(q + 0), b = __ldg(q + 1), c = __ldg(q + 2), dd = __ldg(q + 3),
            e = __ldg(q + 4);
    double v0x = a.x, v0y = a.y, v0z = b.x, e1x = b.y, e1y = c.x, e1z = c.y;
    double e2x = dd.x, e2y = dd.y, e2z = e.x;
    double px = r.dy * e2z - r.dz * e2y;
    double py = r.dz * e2x - r.dx * e2z;
    double pz = r.dx * e2y - r.dy * e2x;
    double det = e1x * px + e1y * py + e1z * pz;
    if (-DET_EPS < det && det < DET_EPS) return false;
    double s = det > 0.0 ? 1.0 : -1.0, ad = fabs(det);
    double tx = r.ox - v0x, ty = r.oy - v0y, tz = r.oz - v0z;
    double un = tx * px + ty * py + tz * pz;
    double us = un * s;   // sign(u) * |u| * |det|, exact
    if (us < -1.000001e-12 * ad || us > (1.0 + 2e-6) * ad) return false;   // certain u reject
    double qx = ty * e1z - tz * e1y;
    double qy = tz * e1x - tx * e1z;
    double qz = tx * e1y - ty * e1x;
    double vn = r.dx * qx + r.dy * qy + r.dz * qz;
    double vs = vn * s;
    if (vs < -1.000001e-12 * ad || us + vs > (1.0 + 2e-6) * ad) return false;   // certain v reject
    double tn = e2x * qx + e2y * qy + e2z * qz;
    double ts = tn * s;
    if (ts < tmin * ad * (1.0 - 1e-6) || ts > tmax * ad * (1.0 + 1e-6)) return false;   // certain t reject
    double inv_det = 1.0 / det;   // the reference's arithmetic from here on
    double u = un * inv_det;
    if (u < -BARY_EPS || u > 1.0 + BARY_EPS) return false;
    double v = vn * inv_det;
    if (v < -BARY_EPS || u + v > 1.0 + BARY_EPS) return false;
    t = tn * inv_det;
    return true;
}

struct Bvh {
    const BNode* __restrict__ nodes;
    const TriRec* __restrict__ tris;
    const int* __restrict__ skip;   // origin skip table [2 * n_prims] (bvh_ploc.cuh) or null
    int n_prims;
    const double* origin_limit;   // device: |o_i| bound for the FP32 filter (else the FP64 one)
    int* err;              // device error word: bit 0 = traversal stack overflow
};

// rays leaving a prim at |n.d| >= SKIP_MIN_COS: t_min |n.d| (5e-6 m) clears the
// table's 1e-7 m margin and the origin's rounding off the plane
constexpr double SKIP_MIN_COS = 0.05;

// the child ref a ray leaving `prim` (normal n as stored, direction d) may skip
__device__ __forceinline__ int origin_skip(const Bvh& bvh, int prim, double n_dot_d) {
    if (!bvh.skip || prim < 0 || fabs(n_dot_d) < SKIP_MIN_COS) return EMPTY_REF;
    return __ldg(bvh.skip + 2 * (long long)prim + (n_dot_d > 0.0 ? 1 : 0));
}

// the FP32 filter is valid for origins within origin_limit (slab32)
__device__ __forceinline__ bool ray_fast(const Bvh& bvh, const Ray& r) {
    // max |o_i| <= L as three compares (sm_100 has no FP64 min / max instruction)
    const double L = __ldg(bvh.origin_limit);
    return fabs(r.ox) <= L && fabs(r.oy) <= L && fabs(r.oz) <= L;
}

// FP32 lower bound of t_min for the box filter.  The common t_min = RAY_EPS is
// a literal (float RD of 1e-4, 0x38D1B717) so the compiler folds it into the
// FMNMX immediate instead of keeping or rematerialising it per node.
__device__ __forceinline__ float ray_tmin_f(double tmin) {
    return tmin == RAY_EPS ? __int_as_float(0x38D1B717) : __double2float_rd(tmin);
}

// compare-exchange on (t, ref) pairs, ascending t
__device__ __forceinline__ void cx(float& ta, int& ra, float& tb, int& rb) {
    if (tb < ta) {
        float t = ta; ta = tb; tb = t;
        int r = ra; ra = rb; rb = r;
    }
}

// Closest (ANY=false) or first (ANY=true) hit with t in (tmin, tmax).
// Returns the global prim id, -1 on a miss, -2 on stack overflow; *t_out
// the hit distance.  Children are visited nearest-first.
template <bool ANY, int MODE = 0>
__device__ int trace(const Bvh& bvh, const Ray& r, double tmin, double tmax, double* t_out,
                     int* visits = nullptr, int* tests = nullptr, int* hit_pos = nullptr,
                     int skip = EMPTY_REF, int skip_end = EMPTY_REF) {
    if (bvh.n_prims == 0) return -1;
    int2 stack[STACK_SIZE];   // (node ref, entry t bits): one 8-byte local access per push / pop
    int sp = 0;
    double best_t = tmax;
    float best_tf = __double2float_ru(tmax);
    const float tmin_f = ray_tmin_f(tmin);
    const bool fast = MODE == 1 ? true : MODE == 2 ? false : ray_fast(bvh, r);
    int best_prim = -1;
    int cur = 0;   // root node 0
    int nv = 0, nt = 0;
    while (true) {
        if (!ref_is_leaf(cur)) {
            ++nv;
            const float4* np = reinterpret_cast<const float4*>(bvh.nodes + cur);
            float4 a = __ldg(np), b = __ldg(np + 1), c = __ldg(np + 2);
            int4 ch = __ldg(reinterpret_cast<const int4*>(np + 3));
            float tn0, tn1;
            bool h0 = box_hit(r, fast, make_float2(a.x, a.y), make_float2(a.z, a.w), make_float2(b.x, b.y), tmin,
                              best_t, tmin_f, best_tf, tn0) &&
                      !RT_SKIPPED(ch.x);   // the subtree behind the ray's own wall (origin skip table)
            bool h1 = box_hit(r, fast, make_float2(b.z, b.w), make_float2(c.x, c.y), make_float2(c.z, c.w), tmin,
                              best_t, tmin_f, best_tf, tn1) &&
                      !RT_SKIPPED(ch.y);
            if (h0 && h1) {
                int nearc = ch.x, farc = ch.y;
                float tf = tn1;
                if (tn1 < tn0) { nearc = ch.y; farc = ch.x; tf = tn0; }
                if (RT_STACK_CHECK && sp >= STACK_SIZE) goto overflow;   // reported as an error
                stack[sp] = make_int2(farc, __float_as_int(tf));
                ++sp;
                cur = nearc;
                continue;
            } else if (h0) {
                cur = ch.x;
                continue;
            } else if (h1) {
                cur = ch.y;
                continue;
            }
        } else {
            int first = leaf_first(cur), cnt = leaf_count(cur);
            nt += cnt;
            for (int k = 0; k < cnt; ++k) {
                const TriRec* tp = bvh.tris + first + k;
                double t;
                if (mt_test(r, tp, tmin, best_t, t)) {
                    int prim = __ldg(&tp->prim);
                    if (tmin < t && (t < best_t || (t == best_t && best_prim >= 0 && prim < best_prim))) {
                        best_t = t;
                        best_tf = __double2float_ru(t);
                        best_prim = prim;
                        if (ANY) {
                            *t_out = t;
                            if (visits) *visits = nv;
                            if (tests) *tests = nt;
                            if (hit_pos) *hit_pos = first + k;
                            return prim;
                        }
                    }
                }
            }
        }
        // pop the next subtree whose entry distance still beats the best hit
        bool found = false;
        while (sp > 0) {
            --sp;
            int2 e = stack[sp];
                    if (__int_as_float(e.y) <= best_tf) { cur = e.x; found = true; break; }
        }
        if (!found) break;
    }
    *t_out = best_t;
    if (visits) *visits = nv;
    if (tests) *tests = nt;
    return best_prim;
overflow:
    *t_out = -1.0;
    return -2;
}

// "while-while" form of the binary traversal (Aila & Laine 2009): a lane
// descends internal nodes until it reaches a leaf, then the warp runs leaf
// tests together, instead of alternating node and FP64 triangle work per
// iteration.  Same visit order and results as trace<>.
// The octant copies only for the closest-hit traversal (k_launch): in the
// occlusion kernels the eight extra descents overflow the instruction cache
// (k_solve_validate: 20 % of stall samples "no_instructions"); C3 fused pass
// 2.52 -> 2.22 ms with the generic descent there.
#ifndef RT_OCTANT_ANY
#define RT_OCTANT_ANY 0
#endif
#ifndef RT_OCTANT
#define RT_OCTANT 1
#endif

// The descent of trace_ww: a lane walks internal nodes until it reaches a leaf
// (cur) or its stack runs empty (returns false).  OCT >= 0: FP32 filter with
// the ray's octant fixed at compile time (slab32_oct); OCT < 0: box_hit.
template <bool ANY, int OCT>
__device__ __forceinline__ bool ww_descend(const Bvh& bvh, const Ray& r, bool fast, double tmin, double best_t,
                                           float tmin_f, float best_tf, int& cur, int2* stack, int& sp, int& nv,
                                           bool& overflow, int skip, int skip_end) {
    while (!ref_is_leaf(cur)) {
        ++nv;
        const float4* np = reinterpret_cast<const float4*>(bvh.nodes + cur);
        float4 a = __ldg(np), b = __ldg(np + 1), c = __ldg(np + 2);
        int4 ch = __ldg(reinterpret_cast<const int4*>(np + 3));
        float tn0, tn1;
        bool h0, h1;
        if (OCT >= 0) {
            h0 = slab32_oct<(OCT < 0 ? 0 : OCT)>(r, make_float2(a.x, a.y), make_float2(a.z, a.w),
                                                 make_float2(b.x, b.y), tmin_f, best_tf, tn0) &&
                 !RT_SKIPPED(ch.x);
            h1 = slab32_oct<(OCT < 0 ? 0 : OCT)>(r, make_float2(b.z, b.w), make_float2(c.x, c.y),
                                                 make_float2(c.z, c.w), tmin_f, best_tf, tn1) &&
                 !RT_SKIPPED(ch.y);
        } else {
            h0 = box_hit(r, fast, make_float2(a.x, a.y), make_float2(a.z, a.w), make_float2(b.x, b.y), tmin,
                         best_t, tmin_f, best_tf, tn0) &&
                 !RT_SKIPPED(ch.x);   // the subtree behind the ray's own wall (origin skip table)
            h1 = box_hit(r, fast, make_float2(b.z, b.w), make_float2(c.x, c.y), make_float2(c.z, c.w), tmin,
                         best_t, tmin_f, best_tf, tn1) &&
                 !RT_SKIPPED(ch.y);
        }
        if (h0 && h1) {
            int nearc = ch.x, farc = ch.y;
            float tf = tn1;
            if (tn1 < tn0) { nearc = ch.y; farc = ch.x; tf = tn0; }
            if (RT_STACK_CHECK && sp >= STACK_SIZE) { overflow = true; return false; }   // reported as an error
            stack[sp] = make_int2(farc, __float_as_int(tf));
            ++sp;
            cur = nearc;
        } else if (h0) {
            cur = ch.x;
        } else if (h1) {
            cur = ch.y;
        } else {
            bool found = false;
            while (sp > 0) {
                --sp;
                int2 e = stack[sp];
                if (__int_as_float(e.y) <= best_tf) { cur = e.x; found = true; break; }
            }
            if (!found) return false;
        }
    }
    return true;
}

// "while-while" form of the binary traversal (Aila & Laine 2009): a lane
// descends internal nodes until it reaches a leaf, then the warp runs leaf
// tests together, instead of alternating node and FP64 triangle work per
// iteration.  Same visit order and results as trace<>.  With RT_OCTANT the
// descent of an FP32-filtered ray runs in the copy specialised for its
// octant (one switch per leaf visit; coherent warps share one copy).
template <bool ANY, int MODE = 0>
__device__ int trace_ww(const Bvh& bvh, const Ray& r, double tmin, double tmax, double* t_out,
                        int* visits = nullptr, int* tests = nullptr, int* hit_pos = nullptr,
                        int skip = EMPTY_REF, int skip_end = EMPTY_REF) {
    if (bvh.n_prims == 0) return -1;
    int2 stack[STACK_SIZE];   // (node ref, entry t bits): one 8-byte local access per push / pop
    int sp = 0;
    double best_t = tmax;
    float best_tf = __double2float_ru(tmax);
    const float tmin_f = ray_tmin_f(tmin);
    const bool fast = MODE == 1 ? true : MODE == 2 ? false : ray_fast(bvh, r);
    const int oct = (RT_OCTANT && (!ANY || RT_OCTANT_ANY) && fast)
                        ? ((r.fix < 0.f) | ((r.fiy < 0.f) << 1) | ((r.fiz < 0.f) << 2)) : -1;
    int best_prim = -1;
    int cur = 0;
    int nv = 0, nt = 0;
    bool overflow = false;
    for (;;) {
        bool more;
#define RT_WW_DESCEND(O) ww_descend<ANY, O>(bvh, r, fast, tmin, best_t, tmin_f, best_tf, cur, stack, sp, nv, \
                                            overflow, skip, skip_end)
        switch (oct) {
            case 0: more = RT_WW_DESCEND(0); break;
            case 1: more = RT_WW_DESCEND(1); break;
            case 2: more = RT_WW_DESCEND(2); break;
            case 3: more = RT_WW_DESCEND(3); break;
            case 4: more = RT_WW_DESCEND(4); break;
            case 5: more = RT_WW_DESCEND(5); break;
            case 6: more = RT_WW_DESCEND(6); break;
            case 7: more = RT_WW_DESCEND(7); break;
            default: more = RT_WW_DESCEND(-1); break;
        }
#undef RT_WW_DESCEND
        if (overflow) goto overflow;
        if (!more) break;
        int first = leaf_first(cur), cnt = leaf_count(cur);
        nt += cnt;
        for (int k = 0; k < cnt; ++k) {
            const TriRec* tp = bvh.tris + first + k;
            double t;
            if (mt_test(r, tp, tmin, best_t, t)) {
                int prim = __ldg(&tp->prim);
                if (tmin < t && (t < best_t || (t == best_t && best_prim >= 0 && prim < best_prim))) {
                    best_t = t;
                    best_tf = __double2float_ru(t);
                    best_prim = prim;
                    if (ANY) {
                        *t_out = t;
                        if (visits) *visits = nv;
                        if (tests) *tests = nt;
                        if (hit_pos) *hit_pos = first + k;
                        return prim;
                    }
                }
            }
        }
        bool found = false;
        while (sp > 0) {
            --sp;
            int2 e = stack[sp];
            if (__int_as_float(e.y) <= best_tf) { cur = e.x; found = true; break; }
        }
        if (!found) break;
    }
    *t_out = best_t;
    if (visits) *visits = nv;
    if (tests) *tests = nt;
    return best_prim;
overflow:
    *t_out = -1.0;
    return -2;
}

// measured on C3: while-while wins for the any-hit occlusion queries (7.4 vs
// 8.4 ms) and, since the origin skip table and the FFMA2 box filter, for the
// launch's closest-hit too (12.00 vs 12.27 ms; it lost 36.0 vs 35.3 before)
#ifndef RT_WW_ANY
#define RT_WW_ANY 1
#endif
#ifndef RT_WW_CLOSEST
#define RT_WW_CLOSEST 1
#endif
#ifndef RT_HOIST_FAST_ANY
#define RT_HOIST_FAST_ANY 1   // 0: one any-hit loop with a per-node FP32 / FP64 choice (C3 fused pass 2.22 -> 2.51 ms)
#endif
#ifndef RT_HOIST_FAST
#define RT_HOIST_FAST 1   // measured on C3: launch 25.8 vs 26.8 ms, validate 5.5 vs 6.3 ms
#endif

// the traversal the kernels call
template <bool ANY>
__device__ __forceinline__ int trace_ray(const Bvh& bvh, const Ray& r, double tmin, double tmax,
                                         double* t_out, int* visits = nullptr, int* tests = nullptr,
                                         int* hit_pos = nullptr, int skip = EMPTY_REF,
                                         int skip_end = EMPTY_REF) {
#if RT_HOIST_FAST
    // one FP32-only and one FP64-only copy of the loop: no per-node filter test
    if (ANY && !RT_HOIST_FAST_ANY && RT_WW_ANY)
        return trace_ww<ANY>(bvh, r, tmin, tmax, t_out, visits, tests, hit_pos, skip, skip_end);
    if ((ANY && RT_WW_ANY) || (!ANY && RT_WW_CLOSEST)) {
        if (ray_fast(bvh, r)) return trace_ww<ANY, 1>(bvh, r, tmin, tmax, t_out, visits, tests, hit_pos, skip, skip_end);
        return trace_ww<ANY, 2>(bvh, r, tmin, tmax, t_out, visits, tests, hit_pos, skip, skip_end);
    }
    if (ray_fast(bvh, r)) return trace<ANY, 1>(bvh, r, tmin, tmax, t_out, visits, tests, hit_pos, skip, skip_end);
    return trace<ANY, 2>(bvh, r, tmin, tmax, t_out, visits, tests, hit_pos, skip, skip_end);
#else
    if ((ANY && RT_WW_ANY) || (!ANY && RT_WW_CLOSEST))
        return trace_ww<ANY>(bvh, r, tmin, tmax, t_out, visits, tests, hit_pos, skip, skip_end);
    return trace<ANY>(bvh, r, tmin, tmax, t_out, visits, tests, hit_pos, skip, skip_end);
#endif
}

// Bvh.occluded (bvh.py:103-115): 1 blocked, 0 clear, -1 coincident endpoints.
// *hit_pos (optional) receives the blocker's TriRec index.
// from_prim >= 0: p lies on that prim (an interaction point) and the subtree
// behind it is skipped (origin_skip; nrm = the scene's stored normals);
// to_prim >= 0: q lies on that prim and the subtree beyond it, seen from p, is
// skipped too (the segment stops eps short of it: t_max = dist - eps).
__device__ inline int occluded(const Bvh& bvh, d3 p, d3 q, double eps = RAY_EPS, int* hit_pos = nullptr,
                               int from_prim = -1, const double* nrm = nullptr, int to_prim = -1) {
    double dx = q.x - p.x, dy = q.y - p.y, dz = q.z - p.z;
    double dist = sqrt(dx * dx + dy * dy + dz * dz);
    if (dist == 0.0) return -1;
    double inv = 1.0 / dist;
    d3 d = d3{dx * inv, dy * inv, dz * inv};
    Ray r = make_ray(p, d);
    int skip = EMPTY_REF;
    if (from_prim >= 0) {
        d3 n = d3{__ldg(nrm + 3 * (long long)from_prim), __ldg(nrm + 3 * (long long)from_prim + 1),
                  __ldg(nrm + 3 * (long long)from_prim + 2)};
        skip = origin_skip(bvh, from_prim, n.x * d.x + n.y * d.y + n.z * d.z);
    }
    int skip_end = EMPTY_REF;
    if (RT_END_SKIP && to_prim >= 0) {   // the ray arrives from the side -sign(n.d): skip what lies beyond
        d3 n = d3{__ldg(nrm + 3 * (long long)to_prim), __ldg(nrm + 3 * (long long)to_prim + 1),
                  __ldg(nrm + 3 * (long long)to_prim + 2)};
        skip_end = origin_skip(bvh, to_prim, -(n.x * d.x + n.y * d.y + n.z * d.z));
    }
    double t;
    int h = trace_ray<true>(bvh, r, eps, dist - eps, &t, nullptr, nullptr, hit_pos, skip, skip_end);
    if (h == -2) {   // stack overflow: the answer is unknown, so the call fails (flag bit 0)
        if (bvh.err) atomicOr(bvh.err, 1);
        return 1;
    }
    return h >= 0 ? 1 : 0;
}

#ifndef RT_HINT_R
#define RT_HINT_R 1   // C3 validate ms: R0 5.85, R1 3.89, R2 3.84, R4 4.47; with the skip table R1 2.88 vs R2 2.95
#endif
// Occluder cache: does one of the TriRecs pos-R..pos+R block segment p->q?
// Exactly the acceptance test the traversal applies (mt_test + the window
// (eps, dist - eps)), so a "yes" is the answer occluded() would give; a "no"
// decides nothing.  Coincident endpoints count as blocked, as in occluded().
__device__ inline bool hint_blocks(const Bvh& bvh, int pos, d3 p, d3 q, double eps = RAY_EPS) {
    double dx = q.x - p.x, dy = q.y - p.y, dz = q.z - p.z;
    double dist = sqrt(dx * dx + dy * dy + dz * dz);
    if (dist == 0.0) return true;
    double inv = 1.0 / dist;
    d3 d = d3{dx * inv, dy * inv, dz * inv};
    Ray r;
    r.ox = p.x; r.oy = p.y; r.oz = p.z;
    r.dx = d.x; r.dy = d.y; r.dz = d.z;
    double tmax = dist - eps;
#pragma unroll
    for (int k = 0; k < 2 * RT_HINT_R + 1; ++k) {
        int i = pos + ((k & 1) ? (k + 1) / 2 : -(k / 2));   // pos, pos+1, pos-1, pos+2, ...
        if (i < 0 || i >= bvh.n_prims) continue;
        double t;
        if (mt_test(r, bvh.tris + i, eps, tmax, t) && eps < t && t < tmax) return true;
    }
    return false;
}

}  // namespace rt

// solve.cuh — image-method solve, validity, occlusion, merge, coverage.
//
// Restates tracer.py:71-183 (_mirror, solve_points, _inside_triangle,
// image_solve), tracer.py:186-193 (los_path), tracer.py:247-295 (merge and
// ordering) and channel.py:190-253 (probe path gain per cell) as a
// candidate-major pipeline:
//   1. k_images      per candidate: the image chain I_1..I_K of the tx
//                     (identical floats to solve_points' images).
//   2. k_halfplanes + k_segments   per candidate: a valid receiver lies in
//                     every cone from I_K through the forward-mirrored
//                     interaction triangles (conservative half-planes on the
//                     grid plane); per row, the x-interval of cell centers
//                     inside all of them, one work item per cell.
//   3. k_solve_validate  per work item (warp chunks of consecutive cells) or
//                     per (candidate, rx): back-substitution + the geometric
//                     tests, the candidate's receiver-side occluder hint, then
//                     occlusion of every segment (any-hit traversals); thin
//                     warps' open items go to
//   4. k_validate    (deferred list, warm occluder cache); both emit records
//                     keyed (receiver, order, candidate rank).
//                     (RT_FUSED_SV=0: separate k_solve -> k_validate passes.)
//   5. sort records (CUB) and merge coincident paths per receiver in the
//      reference's greedy order, then accumulate / materialize.
#pragma once
#include "em.cuh"
#include "trace.cuh"

namespace rt {

struct SceneDev {
    const double* v0;
    const double* e1;
    const double* e2;
    const double* nrm;
    const double* poff;
    const int* prim_mat;
    int n;
};

struct Cands {
    const int* seq;
    const signed char* len;
    int max_len;
    long long n;
};

__device__ inline d3 mirror(d3 p, d3 n, double c) {   // tracer.py:71-73
    double k = 2.0 * (tdot(p, n) - c);
    return d3{p.x - n.x * k, p.y - n.y * k, p.z - n.z * k};
}

__global__ void k_images(Cands C, SceneDev S, d3 tx, double* images /*[n*max_len*3]*/) {
    long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= C.n) return;
    int K = C.len[c];
    d3 p = tx;
    for (int j = 0; j < K; ++j) {
        int prim = C.seq[c * C.max_len + j];
        p = mirror(p, ld3(S.nrm + 3 * (long long)prim), S.poff[prim]);
        st3(images + (c * C.max_len + j) * 3, p);
    }
}

// solve_points back-substitution (tracer.py:88-102) + the geometric part of
// image_solve (tracer.py:164-180).  Returns true when every test passes; the
// interaction points land in pts[0..K).
//
// rx_hint (optional): the candidate's receiver-side occluder-cache slot.  The
// back-substitution yields the last interaction point first; when the cached
// occluder blocks the segment from it to the receiver, the path cannot be
// valid whatever the remaining levels give (image_solve's conjunction,
// tracer.py:164-182), so the solve stops there and returns false.
__device__ inline bool solve_geometric(const Cands& C, const SceneDev& S, const double* images,
                                       long long c, d3 tx, d3 rx, d3* pts, const Bvh* bvh = nullptr,
                                       const int* rx_hint = nullptr) {
    int K = C.len[c];
    const int* seq = C.seq + c * C.max_len;
    d3 cur = rx;
    for (int j = K - 1; j >= 0; --j) {
        int prim = seq[j];
        d3 n = ld3(S.nrm + 3 * (long long)prim);
        double cc = S.poff[prim];
        d3 target = ld3(images + (c * C.max_len + j) * 3);
        d3 seg = sub(target, cur);
        double denom = tdot(seg, n);
        if (fabs(denom) < 1e-15) return false;
        double s = (cc - tdot(cur, n)) / denom;
        d3 p = d3{cur.x + seg.x * s, cur.y + seg.y * s, cur.z + seg.z * s};
        // early outs: image_solve applies the same tests after the loop
        // (tracer.py:164-169); the conjunction does not depend on the order
        if (!(1e-12 < s && s < 1.0 - 1e-12)) return false;
        {   // _inside_triangle (tracer.py:136-147)
            d3 v0 = ld3(S.v0 + 3 * (long long)prim), e1 = ld3(S.e1 + 3 * (long long)prim),
               e2 = ld3(S.e2 + 3 * (long long)prim);
            d3 w = sub(p, v0);
            double d11 = dot_blas(e1, e1), d12 = dot_blas(e1, e2), d22 = dot_blas(e2, e2);
            double w1 = dot_blas(w, e1), w2 = dot_blas(w, e2);
            double den = d11 * d22 - d12 * d12;
            double u = (d22 * w1 - d12 * w2) / den;
            double v = (d11 * w2 - d12 * w1) / den;
            if (!(u >= -INSIDE_TOL && v >= -INSIDE_TOL && u + v <= 1.0 + INSIDE_TOL)) return false;
        }
        pts[j] = p;
        cur = p;
        if (rx_hint && j == K - 1) {
            int h = __ldcg(rx_hint);
            if (h >= 0 && hint_blocks(*bvh, h, p, rx)) return false;
        }
    }
    for (int j = 0; j < K; ++j) {   // same-side reflection (tracer.py:170-176)
        int prim = seq[j];
        d3 n = ld3(S.nrm + 3 * (long long)prim);
        double cc = S.poff[prim];
        d3 before = j == 0 ? tx : pts[j - 1];
        d3 after = j == K - 1 ? rx : pts[j + 1];
        double b = tdot(before, n) - cc, a = tdot(after, n) - cc;
        if (b * a <= SIDE_TOL) return false;
    }
    d3 a = tx;
    for (int j = 0; j <= K; ++j) {   // minimum segment length (tracer.py:178-180)
        d3 b = j < K ? pts[j] : rx;
        double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
        // the square root only near the threshold: above (2 eps)^2 (1 + 1e-9) the
        // correctly rounded root exceeds 2 eps (a 5e-10 relative gap >> 1 ulp)
        double d2 = dx * dx + dy * dy + dz * dz;
        if (d2 <= (2 * RAY_EPS) * (2 * RAY_EPS) * (1.0 + 1e-9) && sqrt(d2) <= 2 * RAY_EPS) return false;
        a = b;
    }
    return true;
}

// occlusion of every segment (tracer.py:181-182); the conjunction is order-free,
// so the receiver-side segment (most often blocked near the ground) goes first
// (a segment from an interaction point skips the subtree behind its wall)
__device__ inline bool segments_clear(const Bvh& bvh, d3 tx, const d3* pts, int K, d3 rx, const int* seq,
                                      const double* nrm) {
    for (int j = K; j >= 0; --j) {
        d3 a = j == 0 ? tx : pts[j - 1];
        d3 b = j == K ? rx : pts[j];
        if (occluded(bvh, a, b, RAY_EPS, nullptr, j == 0 ? -1 : seq[j - 1], nrm, j == K ? -1 : seq[j]) != 0)
            return false;
    }
    return true;
}

// The same conjunction with an occluder cache per (candidate, segment):
// neighbouring cells of one candidate are mostly blocked by the same building,
// so the last blocker found for segment j of this candidate is tried first
// (hint_blocks: the traversal's own acceptance test, so the answer is the
// same).  hints[j] holds a TriRec index or -1; races only make hints stale.
#ifdef RT_VALIDATE_STATS
__device__ unsigned long long g_vstats[8];   // items, hint hits, traversals, blocked by traversal
#define VSTAT(i) atomicAdd(&g_vstats[i], 1ULL)
#else
#define VSTAT(i) ((void)0)
#endif

__device__ inline bool segments_clear_hinted(const Bvh& bvh, d3 tx, const d3* pts, int K, d3 rx,
                                             int* hints, const int* seq, const double* nrm, int skip = -1) {
    int h[MAX_DEPTH + 1];
    for (int j = 0; j <= K; ++j) h[j] = __ldcg(hints + j);
    for (int j = K; j >= 0; --j) {
        if (h[j] < 0 || j == skip) continue;
        d3 a = j == 0 ? tx : pts[j - 1];
        d3 b = j == K ? rx : pts[j];
        if (hint_blocks(bvh, h[j], a, b)) { VSTAT(4); return false; }
    }
    for (int j = K; j >= 0; --j) {
        d3 a = j == 0 ? tx : pts[j - 1];
        d3 b = j == K ? rx : pts[j];
        int pos = -1;
        VSTAT(2);
        if (occluded(bvh, a, b, RAY_EPS, &pos, j == 0 ? -1 : seq[j - 1], nrm, j == K ? -1 : seq[j]) != 0) {
            VSTAT(3);
            if (pos >= 0 && pos != h[j]) __stcg(hints + j, pos);
            return false;
        }
    }
    return true;
}

// ---- receivers: an explicit list or the cells of a grid --------------------------------

struct Receivers {
    const double* pts;   // list mode [n*3]; NULL for grid mode
    double ox, oy, cell, height;
    long long nx, ny;
    long long n;         // list: n rx; grid: nx*ny
};

// GridSpec.cell_center (channel.py:146-149)
__device__ inline d3 receiver_pos(const Receivers& R, long long r) {
    if (R.pts) return ld3(R.pts + 3 * r);
    long long iy = r / R.nx, ix = r - iy * R.nx;
    return d3{R.ox + ((double)ix + 0.5) * R.cell, R.oy + ((double)iy + 0.5) * R.cell, R.height};
}

// ---- footprints ---------------------------------------------------------------------------
//
// A receiver R is reachable by candidate (t_0..t_{K-1}) only if R lies in every
// cone {A + mu (x - A) : x in T'_j, mu > 0} with apex A = I_K (the last
// image) through the forward-mirrored interaction triangles T'_j =
// M_{K-1}...M_{j+1}(T_j), and beyond each T'_j's plane (segment fractions in
// (0,1), tracer.py:164-166).  Each cone is 3 half-spaces, each "beyond" one
// more; on the grid plane z = height they are half-planes.  Triangles are
// inflated by 1e-6 about their centroid first (the reference accepts
// barycentric -1e-9), so the half-planes are conservative.  Cells are then
// enumerated row by row inside the clipped polygon (rows padded by one; the
// x-intervals are exact up to a 1e-7-cell rounding allowance, row_interval).

constexpr int HP_PER_TRI = 4;
constexpr int HP_MAX = HP_PER_TRI * MAX_DEPTH;
#ifndef RT_POLY_CAP
#define RT_POLY_CAP 12
#endif
#ifndef RT_POLY_SMEM
#define RT_POLY_SMEM 1
#endif

// Half-plane a x + b y + c >= 0 on the grid plane (c widened by the rounding
// margin), stored in cell-index row form for row_interval: at the center of
// cell (u, iy) it reads A u + B iy + C >= 0; for A != 0 one bound u >= / <=
// P iy + Q (kind +1 / -1), else B iy + C >= 0 (kind 0).  The rewrite's
// rounding is far inside the 1e-9 margin.
__device__ inline void add_hp(double* hp, int& m, const Receivers& R, double a, double b, double c) {
    c += 1e-9 * (fabs(a) + fabs(b) + fabs(c));   // rounding margin
    double A = a * R.cell, B = b * R.cell;
    double C = a * (R.ox + 0.5 * R.cell) + b * (R.oy + 0.5 * R.cell) + c;
    if (A != 0.0) {
        double inv = 1.0 / A;
        hp[3 * m] = A > 0.0 ? 1.0 : -1.0;
        hp[3 * m + 1] = -B * inv;
        hp[3 * m + 2] = -C * inv;
    } else {
        hp[3 * m] = 0.0;
        hp[3 * m + 1] = B;
        hp[3 * m + 2] = C;
    }
    ++m;
}

// the row form as a half-plane a u + b iy + c >= 0 in cell-index space
__device__ inline void hp_line(const double* hp, double& a, double& b, double& c) {
    double k = hp[0];
    if (k != 0.0) { a = k; b = -k * hp[1]; c = -k * hp[2]; }
    else { a = 0.0; b = hp[1]; c = hp[2]; }
}

// clip a convex polygon by a x + b y + c >= 0 (Sutherland-Hodgman); vertex k
// at [k * PS]; the output has at most n + 1 vertices
template <int PS>
__device__ inline int clip_poly(const double* px, const double* py, int n, double a, double b,
                                double c, double* qx, double* qy) {
    int m = 0;
    for (int i = 0; i < n; ++i) {
        int j = i + 1 == n ? 0 : i + 1;
        double xi = px[i * PS], yi = py[i * PS], xj = px[j * PS], yj = py[j * PS];
        double fi = a * xi + b * yi + c, fj = a * xj + b * yj + c;
        if (fi >= 0.0) { qx[m * PS] = xi; qy[m * PS] = yi; ++m; }
        if ((fi >= 0.0) != (fj >= 0.0)) {
            double t = fi / (fi - fj);
            qx[m * PS] = xi + t * (xj - xi);
            qy[m * PS] = yi + t * (yj - yi);
            ++m;
        }
    }
    return m;
}

// Stage-2 row shards: blocks of RT_ROW_BLOCK grid rows go round-robin to the
// shard_count ranks (row iy belongs to shard (iy / RB) % count).  Measured per
// rank at 8 ranks (tools/scale_estimate.py --ranks): C5 rows 6.9-7.1 ms with
// single rows vs 6.1-7.6 ms with 8-row blocks (the city's 25 m street period
// beats against the block pattern), C3 unchanged; warmer occluder hints in
// larger blocks do not pay for the imbalance.
#ifndef RT_ROW_BLOCK
#define RT_ROW_BLOCK 1
#endif
__host__ __device__ inline bool row_in_shard(long long iy, int index, int count) {
    return (iy / RT_ROW_BLOCK) % count == index;
}

// rows of [0, x] owned by the shard
__host__ __device__ inline long long shard_rows_upto(long long x, int index, int count) {
    long long n = x + 1, nb = n / RT_ROW_BLOCK, rem = n - nb * RT_ROW_BLOCK;
    long long full = nb > index ? (nb - index + count - 1) / count : 0;
    return full * RT_ROW_BLOCK + ((nb % count == index) ? rem : 0);
}

// the s-th owned row at or after `first` (an owned row)
__host__ __device__ inline long long shard_row(long long first, long long s, int count) {
    long long bf = first / RT_ROW_BLOCK, off = first - bf * RT_ROW_BLOCK;
    if (s < RT_ROW_BLOCK - off) return first + s;
    long long t = s - (RT_ROW_BLOCK - off);
    return (bf + (t / RT_ROW_BLOCK + 1) * count) * RT_ROW_BLOCK + t % RT_ROW_BLOCK;
}

// launched with 128-thread blocks: the shared clip lists are laid out [.][.][128]
__global__ void __launch_bounds__(128) k_halfplanes(Cands C, SceneDev S, const double* images, Receivers R,
                                                    int shard_index, int shard_count,
                                                    double* hps /*[n*HP_MAX*3]*/, int* nhp, int* row0,
                                                    long long* seg_counts /*[n+1]*/) {
    long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (c >= C.n) {
        if (c == C.n) seg_counts[c] = 0;
        return;
    }
    int K = C.len[c];
    const int* seq = C.seq + c * C.max_len;
    d3 A = ld3(images + (c * C.max_len + K - 1) * 3);
    double hA = R.height - A.z;
    double* hp = hps + c * HP_MAX * 3;
    int m = 0;
    for (int j = 0; j < K; ++j) {
        int prim = seq[j];
        d3 v0 = ld3(S.v0 + 3 * (long long)prim), e1 = ld3(S.e1 + 3 * (long long)prim),
           e2 = ld3(S.e2 + 3 * (long long)prim);
        d3 x[3] = {v0, add(v0, e1), add(v0, e2)};
        d3 ctr = d3{(x[0].x + x[1].x + x[2].x) / 3.0, (x[0].y + x[1].y + x[2].y) / 3.0,
                    (x[0].z + x[1].z + x[2].z) / 3.0};
        for (int q = 0; q < 3; ++q) x[q] = add(ctr, scale(sub(x[q], ctr), 1.0 + 1e-6));
        for (int q = j + 1; q < K; ++q) {
            int pq = seq[q];
            d3 n = ld3(S.nrm + 3 * (long long)pq);
            double cc = S.poff[pq];
            for (int u = 0; u < 3; ++u) x[u] = mirror(x[u], n, cc);
        }
        // three side half-spaces of the cone through A
        for (int e = 0; e < 3; ++e) {
            d3 va = sub(x[e], A), vb = sub(x[(e + 1) % 3], A), vc = sub(x[(e + 2) % 3], A);
            d3 n = cross(va, vb);
            double sgn = tdot(n, vc);
            if (sgn == 0.0) continue;   // degenerate cone: no constraint
            if (sgn < 0.0) n = d3{-n.x, -n.y, -n.z};
            add_hp(hp, m, R, n.x, n.y, n.z * hA - n.x * A.x - n.y * A.y);
        }
        // beyond the (mirrored) triangle's plane, on the side away from A
        d3 nt = cross(sub(x[1], x[0]), sub(x[2], x[0]));
        double sA = tdot(nt, sub(A, x[0]));
        if (sA != 0.0) {
            double s = sA > 0.0 ? -1.0 : 1.0;
            add_hp(hp, m, R, s * nt.x, s * nt.y, s * (nt.z * R.height - tdot(nt, x[0])));
        }
    }
    nhp[c] = m;
    // clip the grid rectangle, padded one cell, in cell-index space (u, iy)
    // The polygon only bounds the rows (row_interval applies every half-plane
    // per row), so clipping may stop early: a polygon about to outgrow
    // RT_POLY_CAP vertices keeps its current, larger, shape.  The vertex lists
    // live in shared memory (RT_POLY_SMEM): as per-thread local arrays they
    // outgrow L1 and the clip loop waits on L2.
#if RT_POLY_SMEM
    __shared__ double sbuf[4][RT_POLY_CAP][128];
    double* px = &sbuf[0][0][threadIdx.x];
    double* py = &sbuf[1][0][threadIdx.x];
    double* qx = &sbuf[2][0][threadIdx.x];
    double* qy = &sbuf[3][0][threadIdx.x];
    constexpr int PS = 128;   // element stride
#else
    double bx[2][RT_POLY_CAP], by[2][RT_POLY_CAP];
    double *px = bx[0], *py = by[0], *qx = bx[1], *qy = by[1];
    constexpr int PS = 1;
#endif
    double x0 = -1.5, x1 = R.nx + 0.5, y0 = -1.5, y1 = R.ny + 0.5;
    px[0] = x0; py[0] = y0; px[PS] = x1; py[PS] = y0; px[2 * PS] = x1; py[2 * PS] = y1; px[3 * PS] = x0; py[3 * PS] = y1;
    int n = 4;
    for (int i = 0; i < m && n > 0 && n < RT_POLY_CAP; ++i) {
        double la, lb, lc;
        hp_line(hp + 3 * i, la, lb, lc);
        n = clip_poly<PS>(px, py, n, la, lb, lc, qx, qy);
        double* t = px; px = qx; qx = t;
        t = py; py = qy; qy = t;
    }
    long long rows = 0, first = 0;
    if (n > 0) {
        double ylo = py[0], yhi = py[0];
        for (int k = 1; k < n; ++k) { ylo = fmin(ylo, py[k * PS]); yhi = fmax(yhi, py[k * PS]); }
        long long iy0 = (long long)fmax(floor(ylo) - 1.0, 0.0);
        long long iy1 = (long long)fmin(ceil(yhi) + 1.0, (double)(R.ny - 1));
        if (iy0 <= iy1) {
            long long b0 = iy0 / RT_ROW_BLOCK;
            long long bf = b0 + ((shard_index - b0 % shard_count) + shard_count) % shard_count;
            first = bf == b0 ? iy0 : bf * RT_ROW_BLOCK;
            rows = first <= iy1 ? shard_rows_upto(iy1, shard_index, shard_count) -
                                      shard_rows_upto(first - 1, shard_index, shard_count)
                                : 0;
        }
    }
    row0[c] = (int)first;
    seg_counts[c] = rows;
}

// x-interval of cell centers inside every half-plane on row iy.  The
// half-planes are conservative already (inflated triangles, a rounding margin
// per half-plane), so the interval is not padded by whole cells, only by
// RT_FP_EPS cells against rounding.  hp is in k_halfplanes' row form: one
// FMA per half-plane per row.
// Measured at C3 (512^2 cells, depth 5): a one-cell pad each side made 37.5M
// items, none 29.1M; the stage-2 pass went 4.92 -> 4.19 ms, map bit-identical.
#ifndef RT_FP_PAD
#define RT_FP_PAD 0.0
#endif
#ifndef RT_FP_EPS
#define RT_FP_EPS 1e-7
#endif
__device__ inline void row_interval(const double* hp, int m, const Receivers& R, long long iy,
                                    long long& ix0, long long& ix1) {
    double y = (double)iy;
    double lo = -INFINITY, hi = INFINITY;
    for (int i = 0; i < m; ++i) {
        double k = hp[3 * i], v = fma(hp[3 * i + 1], y, hp[3 * i + 2]);
        if (k > 0.0) lo = fmax(lo, v);
        else if (k < 0.0) hi = fmin(hi, v);
        else if (v < 0.0) { lo = INFINITY; hi = -INFINITY; }
    }
    if (!(lo <= hi)) { ix0 = 0; ix1 = -1; return; }
    double flo = isinf(lo) ? -1.0 : fmax(ceil(lo - RT_FP_EPS) - RT_FP_PAD, 0.0);
    double fhi = isinf(hi) ? (double)(R.nx - 1) : fmin(floor(hi + RT_FP_EPS) + RT_FP_PAD, (double)(R.nx - 1));
    ix0 = (long long)fmax(flo, 0.0);
    ix1 = fhi < 0.0 ? -1 : (long long)fhi;
}

// largest s with off[s] <= w (off nondecreasing, off[0] = 0)
__device__ inline long long upper_index(const long long* off, long long n, long long w) {
    long long lo = 0, hi = n;
    while (hi - lo > 1) {
        long long mid = (lo + hi) >> 1;
        if (off[mid] <= w) lo = mid; else hi = mid;
    }
    return lo;
}

// one thread per row segment (cand, iy, ix0, count): candidates own from 0 to
// hundreds of rows, so rows, not candidates, are the parallel unit.  One
// binary search per warp finds the first lane's candidate; lanes walk forward.
__global__ void k_segments(long long n_cand, long long n_seg, const double* hps, const int* nhp,
                           const int* row0, const long long* seg_off, Receivers R, int shard_count,
                           int* seg_cand, int* seg_iy, int* seg_ix0, long long* seg_cnt) {
    const unsigned FULL = 0xffffffffu;
    int lane = threadIdx.x & 31;
    long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    long long s_w = s - lane;
    long long c0 = 0;
    if (lane == 0 && s_w < n_seg) c0 = upper_index(seg_off, n_cand, s_w);
    c0 = __shfl_sync(FULL, c0, 0);
    if (s >= n_seg) return;
    long long c = c0;
    while (seg_off[c + 1] <= s) ++c;
    long long iy = shard_row(row0[c], s - seg_off[c], shard_count);
    long long ix0, ix1;
    row_interval(hps + c * HP_MAX * 3, nhp[c], R, iy, ix0, ix1);
    seg_cand[s] = (int)c;
    seg_iy[s] = (int)iy;
    seg_ix0[s] = (int)ix0;
    seg_cnt[s] = ix1 >= ix0 ? ix1 - ix0 + 1 : 0;
}

// survivor of the geometric tests; carries its last interaction point so the
// validation can try the receiver-side occluder hint before re-solving
struct Pending {
    long long rx;
    int cand;
    int order;
    double lx, ly, lz;
};

struct Segs {
    const long long* item_off;   // [S+1]
    const int* cand;
    const int* iy;
    const int* ix0;
    const int* chunk_seg;        // [ceil(W/32)]: segment holding item 32q
    long long n;
};

// chunk_seg[q] = the segment whose item range holds item 32q: one thread per
// segment writes the 32-item chunk starts that fall inside it, so k_solve's
// warps find their first segment with one load instead of a binary search
// (a chain of ~22 dependent L2 loads).
__global__ void k_chunk_starts(long long n_seg, const long long* item_off, int* chunk_seg) {
    long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    long long a = item_off[s], b = item_off[s + 1];
    for (long long q = (a + 31) >> 5; (q << 5) < b; ++q) chunk_seg[q] = (int)s;
}

#ifndef RT_SOLVE_MINB
#define RT_SOLVE_MINB 5   // C3 solve 2.01 ms vs 2.16 (no minB), 2.10 (minB 6)
#endif
template <bool GRID>
__global__ void __launch_bounds__(256, RT_SOLVE_MINB) k_solve(Cands C, SceneDev S, const double* images,
                                               Receivers R, d3 tx, long long W, Segs G,
                                               Pending* out, unsigned long long* n_out,
                                               unsigned long long cap) {
    const unsigned FULL = 0xffffffffu;
    long long stride = (long long)gridDim.x * blockDim.x;
    long long iters = (W + stride - 1) / stride;
    int lane = threadIdx.x & 31;
    for (long long it = 0; it < iters; ++it) {
        long long w = it * stride + blockIdx.x * (long long)blockDim.x + threadIdx.x;
        bool ok = false;
        long long rxi = 0;
        int c = 0;
        if (GRID) {
            // one binary search per warp, then a short walk per lane
            long long w0 = w - lane;
            long long s0 = w0 < W ? G.chunk_seg[w0 >> 5] : 0;   // w0 is a multiple of 32
            if (w < W) {
                long long s = s0;
                while (G.item_off[s + 1] <= w) ++s;
                c = G.cand[s];
                long long iy = G.iy[s], ix = G.ix0[s] + (w - G.item_off[s]);
                rxi = iy * R.nx + ix;
            }
        } else if (w < W) {
            c = (int)(w % C.n);
            rxi = w / C.n;
        }
        d3 last = d3{0, 0, 0};
        int K = 0;
        if (w < W) {
            d3 pts[MAX_DEPTH];
            ok = solve_geometric(C, S, images, c, tx, receiver_pos(R, rxi), pts);
            K = C.len[c];
            if (ok) last = pts[K - 1];
        }
        unsigned m = __ballot_sync(FULL, ok);
        if (m) {
            unsigned long long base = 0;
            int leader = __ffs(m) - 1;
            if (lane == leader) base = atomicAdd(n_out, (unsigned long long)__popc(m));
            base = __shfl_sync(FULL, base, leader);
            if (ok) {
                unsigned long long slot = base + __popc(m & ((1u << lane) - 1u));
                if (slot < cap) {
                    Pending q;
                    q.rx = rxi; q.cand = c; q.order = K;
                    q.lx = last.x; q.ly = last.y; q.lz = last.z;
                    out[slot] = q;
                }
            }
        }
    }
}

// A valid path (after occlusion) of one receiver.
struct Rec {
    double p_theta, p_phi;   // probe powers (coverage) — unused for paths
    double p0x, p0y, p0z;    // first interaction point (merge pre-check)
    long long rx;
    int cand;
    int order;
};

struct EmParams {
    const double* eta;
    const double* tx_rows;     // 9
    const double* probe_rows;  // 9
    const double* slants;      // [n_el]
    const double* offsets_w;   // [n_el*3]
    int n_el;
    int tx_pattern;
    int tx_mode;               // 0 central, 1 array
    double wavelength, frequency;
};

// coverage power of one path: sum over the theta / phi probes (channel.py:214-232)
__device__ inline void probe_powers(const Geom& g, const EmParams& E, double& pt, double& pp) {
    d3 rft = rx_field(g, RT_PAT_PROBE_THETA_ID, 0.0, E.probe_rows);
    d3 rfp = rx_field(g, RT_PAT_PROBE_PHI_ID, 0.0, E.probe_rows);
    c2 at, ap;
    if (E.tx_mode == 0) {
        c3 f = transport(g, E.tx_pattern, E.slants[0], E.tx_rows, E.eta);
        at = finish(f, rft, g, E.wavelength, E.frequency);
        ap = finish(f, rfp, g, E.wavelength, E.frequency);
    } else {
        at = c2{0.0, 0.0};
        ap = c2{0.0, 0.0};
        // the element transfer depends on the element only through its slant
        double s_prev = 0.0;
        c2 bt = c2{0.0, 0.0}, bp = c2{0.0, 0.0};
        for (int e = 0; e < E.n_el; ++e) {
            double sl = E.slants[e];
            if (e == 0 || sl != s_prev) {
                c3 f = transport(g, E.tx_pattern, sl, E.tx_rows, E.eta);
                bt = finish(f, rft, g, E.wavelength, E.frequency);
                bp = finish(f, rfp, g, E.wavelength, E.frequency);
                s_prev = sl;
            }
            d3 off = ld3(E.offsets_w + 3 * e);
            double ph = TWO_PI * tdot(g.dir[0], off) / E.wavelength;   // em.py:174-181
            double s, c;
            sincos(ph, &s, &c);
            at = cadd(at, cmul(bt, c2{c, s}));
            ap = cadd(ap, cmul(bp, c2{c, s}));
        }
    }
    pt = at.re * at.re + at.im * at.im;
    pp = ap.re * ap.re + ap.im * ap.im;
}

#ifndef RT_VAL_PREFETCH
#define RT_VAL_PREFETCH 1
#endif
#ifndef RT_VAL_MINB
#define RT_VAL_MINB 8   // 64 registers: C3 validate 3.60 ms vs 4.65 (minB 1, 110 regs), 3.84 (minB 6)
#endif
// Deferral (RT_VAL_DEFER = d > 0): a warp whose receiver-side hints leave
// fewer than d of its lanes unresolved does not traverse for them; their
// items go to a deferred list that a second launch (items = that list)
// validates after this one has warmed the occluder cache.
#ifndef RT_VAL_DEFER
#define RT_VAL_DEFER 12   // C3 validate 2.84 -> 2.75 ms (8: 2.77, 16: 2.76)
#endif
template <bool POWER>
__global__ void __launch_bounds__(128, RT_VAL_MINB) k_validate(Cands C, SceneDev S, const double* images,
                                                  Receivers R, d3 tx, Bvh bvh,
                                                  const Pending* pend, long long n_pend,
                                                  EmParams E, Rec* recs,
                                                  unsigned long long* n_out, int* hints,
                                                  const int* items = nullptr, int defer_min = 0,
                                                  int* deferred = nullptr,
                                                  unsigned long long* n_deferred = nullptr) {
    const unsigned FULL = 0xffffffffu;
    long long stride = (long long)gridDim.x * blockDim.x;
    long long iters = (n_pend + stride - 1) / stride;
    int lane = threadIdx.x & 31;
    for (long long it = 0; it < iters; ++it) {
        long long i = it * stride + blockIdx.x * (long long)blockDim.x + threadIdx.x;
        bool ok = false;
        Rec rec;
#if RT_VAL_PREFETCH
        // the next iteration's item streams from HBM: start pulling it into L2 now
        if (i + stride < n_pend) asm volatile("prefetch.global.L2 [%0];" ::"l"(pend + i + stride));
#endif
        bool open_ = false;
        long long item = i;
        if (i < n_pend && items) item = items[i];
        Pending pd;
        d3 rx = d3{0, 0, 0};
        int K = 0;
        int* hc = nullptr;
        if (i < n_pend) {
            pd = pend[item];
            rx = receiver_pos(R, pd.rx);
            K = pd.order;
            hc = hints ? hints + (long long)pd.cand * (MAX_DEPTH + 1) : nullptr;
            VSTAT(0);
            // receiver-side occluder hint first: it needs only the stored last point
            int hK = hc ? __ldcg(hc + K) : -1;
            open_ = !(hK >= 0 && hint_blocks(bvh, hK, d3{pd.lx, pd.ly, pd.lz}, rx));
        }
        if (defer_min > 0) {   // too few open lanes to fill the warp's traversals: later
            unsigned om = __ballot_sync(FULL, open_);
            if (om && __popc(om) < defer_min) {
                unsigned long long base = 0;
                int leader = __ffs(om) - 1;
                if (lane == leader) base = atomicAdd(n_deferred, (unsigned long long)__popc(om));
                base = __shfl_sync(FULL, base, leader);
                if (open_) deferred[base + __popc(om & ((1u << lane) - 1u))] = (int)item;
                open_ = false;
            }
        }
        if (i < n_pend) {
            d3 pts[MAX_DEPTH];
            if (!open_) {
                VSTAT(1);
                ok = false;
            } else {
                solve_geometric(C, S, images, pd.cand, tx, rx, pts);   // recompute points
                const int* sq = C.seq + (long long)pd.cand * C.max_len;
                ok = hc ? segments_clear_hinted(bvh, tx, pts, K, rx, hc, sq, S.nrm, K)
                        : segments_clear(bvh, tx, pts, K, rx, sq, S.nrm);
            }
            if (ok) {
                rec.rx = pd.rx;
                rec.cand = pd.cand;
                rec.order = K;
                rec.p0x = pts[0].x; rec.p0y = pts[0].y; rec.p0z = pts[0].z;
                rec.p_theta = 0.0;
                rec.p_phi = 0.0;
                if (POWER) {
                    Geom g;
                    geom_from_points(tx, pts, K, rx, C.seq + (long long)pd.cand * C.max_len, S.nrm,
                                     S.prim_mat, g);
                    probe_powers(g, E, rec.p_theta, rec.p_phi);
                }
            }
        }
        unsigned m = __ballot_sync(FULL, ok);
        if (m) {
            unsigned long long base = 0;
            int leader = __ffs(m) - 1;
            if (lane == leader) base = atomicAdd(n_out, (unsigned long long)__popc(m));
            base = __shfl_sync(FULL, base, leader);
            if (ok) recs[base + __popc(m & ((1u << lane) - 1u))] = rec;
        }
    }
}

// Solve and validation in one pass (RT_FUSED_SV): each item is solved; a
// geometric survivor is first tried against the receiver-side occluder hint
// of its candidate (the common exit), and the warp's remaining open items
// are validated in place when at least defer_min of them are open, otherwise
// deferred as Pending records for a k_validate pass over the deferred list
// (full warps, warm occluder cache).  No Pending record per survivor, no
// re-solve of the items validated here.  Capacity overflow of the record or
// deferred list is counted (the host grows the buffers and reruns).
// ctr: [0] survivors, [1] records, [2] deferred.
#ifndef RT_SV_CHUNK
#define RT_SV_CHUNK 8
#endif
template <bool GRID>
__global__ void __launch_bounds__(128, RT_VAL_MINB) k_solve_validate(Cands C, SceneDev S, const double* images,
                                                        Receivers R, d3 tx, long long W, Segs G, Bvh bvh,
                                                        int* hints, int defer_min, Rec* recs,
                                                        unsigned long long rec_cap, Pending* deferred,
                                                        unsigned long long def_cap, unsigned long long* ctr) {
    const unsigned FULL = 0xffffffffu;
    int lane = threadIdx.x & 31;
    auto item = [&](long long w) {
        long long rxi = 0;
        int c = 0;
        d3 rx = d3{0, 0, 0};
        if (GRID) {
            long long w0 = w - lane;
            long long s0 = w0 < W ? G.chunk_seg[w0 >> 5] : 0;
            if (w < W) {
                long long sg = s0;
                while (G.item_off[sg + 1] <= w) ++sg;
                c = G.cand[sg];
                long long iy = G.iy[sg], ix = G.ix0[sg] + (w - G.item_off[sg]);
                rxi = iy * R.nx + ix;
                // GridSpec.cell_center from (ix, iy) directly (receiver_pos's arithmetic,
                // without dividing the flat index back)
                rx = d3{R.ox + ((double)ix + 0.5) * R.cell, R.oy + ((double)iy + 0.5) * R.cell, R.height};
            }
        } else if (w < W) {
            c = (int)(w % C.n);
            rxi = w / C.n;
            rx = receiver_pos(R, rxi);
        }
        d3 pts[MAX_DEPTH];
        int K = 0;
        bool geo = false;
        int* hc = hints + (long long)c * (MAX_DEPTH + 1);
        if (w < W) {
            K = C.len[c];
            // the receiver-side occluder hint is tried as soon as the solve has the
            // last interaction point: a blocked item skips the remaining levels
            geo = solve_geometric(C, S, images, c, tx, rx, pts, &bvh, hc + K);
            VSTAT(5);
            if (geo) VSTAT(6);
        }
        // geometric survivors not blocked by the receiver-side hint
        unsigned gm = __ballot_sync(FULL, geo);
        if (gm && lane == __ffs(gm) - 1) atomicAdd(ctr, (unsigned long long)__popc(gm));
        bool open_ = geo;
        unsigned om = __ballot_sync(FULL, open_);
        if (om && __popc(om) < defer_min) {   // too few to fill the warp's traversals: later
            unsigned long long base = 0;
            int leader = __ffs(om) - 1;
            if (lane == leader) base = atomicAdd(ctr + 2, (unsigned long long)__popc(om));
            base = __shfl_sync(FULL, base, leader);
            if (open_) {
                unsigned long long slot = base + __popc(om & ((1u << lane) - 1u));
                if (slot < def_cap) {
                    Pending q;
                    q.rx = rxi; q.cand = c; q.order = K;
                    q.lx = pts[K - 1].x; q.ly = pts[K - 1].y; q.lz = pts[K - 1].z;
                    deferred[slot] = q;
                }
            }
            open_ = false;
        }
        bool ok = false;
        if (open_)
            ok = segments_clear_hinted(bvh, tx, pts, K, rx, hc, C.seq + (long long)c * C.max_len, S.nrm, K);
        unsigned m = __ballot_sync(FULL, ok);
        if (m) {
            unsigned long long base = 0;
            int leader = __ffs(m) - 1;
            if (lane == leader) base = atomicAdd(ctr + 1, (unsigned long long)__popc(m));
            base = __shfl_sync(FULL, base, leader);
            if (ok) {
                unsigned long long slot = base + __popc(m & ((1u << lane) - 1u));
                if (slot < rec_cap) {
                    Rec rec;
                    rec.rx = rxi;
                    rec.cand = c;
                    rec.order = K;
                    rec.p0x = pts[0].x; rec.p0y = pts[0].y; rec.p0z = pts[0].z;
                    rec.p_theta = 0.0;
                    rec.p_phi = 0.0;
                    recs[slot] = rec;
                }
            }
        }
    };
#if RT_SV_CHUNK > 0
    // each warp takes RT_SV_CHUNK x 32 consecutive items at a time: the next
    // 32 cells of a row segment see the occluders the previous 32 found
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ctr + 4, (unsigned long long)(RT_SV_CHUNK * 32));
        base = __shfl_sync(FULL, base, 0);
        if ((long long)base >= W) break;
        for (int t = 0; t < RT_SV_CHUNK && (long long)base + t * 32 < W; ++t) item((long long)base + t * 32 + lane);
    }
#else
    long long stride = (long long)gridDim.x * blockDim.x;
    long long iters = (W + stride - 1) / stride;
    for (long long it = 0; it < iters; ++it) item(it * stride + blockIdx.x * (long long)blockDim.x + threadIdx.x);
#endif
}

// probe powers of the surviving records (split from k_validate so the
// occlusion kernel stays light on registers)
__global__ void __launch_bounds__(128) k_rec_powers(Cands C, SceneDev S, const double* images,
                                                    Receivers R, d3 tx, EmParams E, Rec* recs,
                                                    long long n) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    Rec r = recs[i];
    d3 rx = receiver_pos(R, r.rx);
    d3 pts[MAX_DEPTH];
    solve_geometric(C, S, images, r.cand, tx, rx, pts);
    Geom g;
    geom_from_points(tx, pts, r.order, rx, C.seq + (long long)r.cand * C.max_len, S.nrm, S.prim_mat, g);
    probe_powers(g, E, r.p_theta, r.p_phi);
    recs[i].p_theta = r.p_theta;
    recs[i].p_phi = r.p_phi;
}

// record sort keys (rx, order, candidate rank): rx << 36 | order << 32 | cand,
// or with cb > 0 the compact rx << (cb + 4) | order << cb | cand (cand < 2^cb)
__global__ void k_rec_keys(const Rec* recs, long long n, unsigned long long* keys, int* idx, int cb) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Rec& r = recs[i];
    int sh = cb > 0 ? cb : 32;
    keys[i] = ((unsigned long long)r.rx << (sh + 4)) | ((unsigned long long)r.order << sh) | (unsigned)r.cand;
    idx[i] = (int)i;
}

// compact record keys (k_rec_keys with cb > 0) -> rx << 36 | order << 32 | cand
__global__ void k_rec_keys_expand(unsigned long long* keys, long long n, int cb) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    unsigned long long x = keys[i];
    keys[i] = ((x >> (cb + 4)) << 36) | (((x >> cb) & 0xFULL) << 32) | (x & ((1ULL << cb) - 1));
}

// Greedy coincident merge of one receiver's records (tracer.py:247-265):
// records are visited in (order, candidate) order; a record is dropped when
// an earlier KEPT record of the same order has every vertex within 1e-6.
__device__ inline bool coincident(const Cands& C, const SceneDev& S, const double* images, d3 tx,
                                  d3 rx, const Rec& a, const Rec& b) {
    double m0 = fmax(fmax(fabs(a.p0x - b.p0x), fabs(a.p0y - b.p0y)), fabs(a.p0z - b.p0z));
    if (!(m0 < MERGE_TOL)) return false;
    d3 pa[MAX_DEPTH], pb[MAX_DEPTH];
    solve_geometric(C, S, images, a.cand, tx, rx, pa);
    solve_geometric(C, S, images, b.cand, tx, rx, pb);
    double mx = 0.0;
    for (int j = 0; j < a.order; ++j)
        mx = fmax(mx, fmax(fmax(fabs(pa[j].x - pb[j].x), fabs(pa[j].y - pb[j].y)), fabs(pa[j].z - pb[j].z)));
    return mx < MERGE_TOL;
}

// one thread per receiver segment of the sorted records; writes keep[] and,
// for coverage, adds the kept probe powers after the LOS term in gains[rx]
template <bool COVERAGE>
__global__ void k_merge(Cands C, SceneDev S, const double* images, Receivers R, d3 tx,
                        const Rec* recs, const int* order, const unsigned long long* keys,
                        long long n, unsigned char* keep, double* gains) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long rxi = (long long)(keys[i] >> 36);
    if (i > 0 && (long long)(keys[i - 1] >> 36) == rxi) return;   // not the segment head
    d3 rx = receiver_pos(R, rxi);
    double g = COVERAGE ? gains[rxi] : 0.0;
    long long grp = i;   // start of the current (rx, order) group
    for (long long r = i; r < n && (long long)(keys[r] >> 36) == rxi; ++r) {
        const Rec& a = recs[order[r]];
        if (((keys[r] >> 32) & 0xF) != ((keys[grp] >> 32) & 0xF)) grp = r;
        bool merged = false;
        for (long long q = grp; q < r && !merged; ++q) {
            if (!keep[q]) continue;
            merged = coincident(C, S, images, tx, rx, recs[order[q]], a);
        }
        keep[r] = merged ? 0 : 1;
        if (COVERAGE && !merged) {
            g = g + a.p_theta;
            g = g + a.p_phi;
        }
    }
    if (COVERAGE) gains[rxi] = g;
}

// LOS per receiver (tracer.py:186-193); coverage adds its probe power first
template <bool COVERAGE>
__global__ void k_los(Receivers R, d3 tx, Bvh bvh, SceneDev S, EmParams E,
                      int shard_index, int shard_count, unsigned char* los, double* gains,
                      int* error) {
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= R.n) return;
    if (COVERAGE) {
        long long iy = r / R.nx;
        if (!row_in_shard(iy, shard_index, shard_count)) { gains[r] = 0.0; return; }
    }
    d3 rx = receiver_pos(R, r);
    // np.allclose(tx, rx): |a-b| <= 1e-8 + 1e-5 |b|
    if (fabs(tx.x - rx.x) <= 1e-8 + 1e-5 * fabs(rx.x) && fabs(tx.y - rx.y) <= 1e-8 + 1e-5 * fabs(rx.y) &&
        fabs(tx.z - rx.z) <= 1e-8 + 1e-5 * fabs(rx.z)) {
        atomicOr(error, 4);
        if (COVERAGE) gains[r] = 0.0; else los[r] = 0;
        return;
    }
    bool vis = S.n == 0 || occluded(bvh, tx, rx) == 0;
    if (COVERAGE) {
        double g = 0.0;
        if (vis) {
            Geom geo;
            geom_from_points(tx, nullptr, 0, rx, nullptr, S.nrm, S.prim_mat, geo);
            double pt, pp;
            probe_powers(geo, E, pt, pp);
            g = g + pt;
            g = g + pp;
        }
        gains[r] = g;
    } else {
        los[r] = vis ? 1 : 0;
    }
}

}  // namespace rt

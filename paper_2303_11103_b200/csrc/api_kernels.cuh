// api_kernels.cuh — small kernels behind the C ABI: batched queries, path
// table assembly and the transfer entry points.
#pragma once
#include "solve.cuh"

namespace rt {

// L2 read-bandwidth probe (measurement only): every block streams its share of
// an L2-resident buffer `iters` times with 16-byte L2-only loads (ld.global.cg).
__global__ void __launch_bounds__(256) k_l2_probe(const float4* __restrict__ buf, long long n4,
                                                  int iters, float* sink) {
    float acc = 0.f;
    long long stride = (long long)gridDim.x * blockDim.x;
    for (int it = 0; it < iters; ++it) {
        long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n4; i += 4 * stride) {
            float4 a = __ldcg(buf + i), b = __ldcg(buf + i + stride);
            float4 c = __ldcg(buf + i + 2 * stride), d = __ldcg(buf + i + 3 * stride);
            acc += (a.x + b.y) + (c.z + d.w);
        }
        for (; i < n4; i += stride) acc += __ldcg(buf + i).x;
    }
    if (acc == 1234.5f) *sink = acc;   // keeps the loads alive
}

__global__ void k_iota(int* p, long long n) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) p[i] = (int)i;
}

// Bvh.intersect / occluded-style batched query (bvh.py:83-101)
template <bool ANY>
__global__ void k_trace_batch(Bvh bvh, const double* o, const double* d, const double* tmin,
                              const double* tmax, long long n, double* t_out, int* prim_out,
                              long long* err) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    Ray r = make_ray(ld3(o + 3 * i), ld3(d + 3 * i));
    double t;
    int p = trace_ray<ANY>(bvh, r, tmin[i], tmax[i], &t);
    if (p == -2) { atomicOr((unsigned long long*)err, 1ULL); p = -1; }
    prim_out[i] = p;
    t_out[i] = p >= 0 ? t : __longlong_as_double(0x7ff0000000000000LL);
}

__global__ void k_occluded_batch(Bvh bvh, const double* p, const double* q, long long n,
                                 int* out) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = occluded(bvh, ld3(p + 3 * i), ld3(q + 3 * i));
}

// first sorted-record index of every receiver (-1 when it has none)
__global__ void k_seg_heads(const unsigned long long* keys, long long n, int* heads) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    long long rx = (long long)(keys[i] >> 36);
    if (i == 0 || (long long)(keys[i - 1] >> 36) != rx) heads[rx] = (int)i;
}

// paths per receiver (LOS + kept records) and their maximum (*max_count, zeroed by the caller)
__global__ void k_path_counts(long long n_rx, const int* heads, const unsigned long long* keys,
                              long long n_rec, const unsigned char* keep,
                              const unsigned char* los, int* counts, int* max_count) {
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n_rx) return;
    int c = los[r];
    int h = heads[r];
    if (h >= 0)
        for (long long i = h; i < n_rec && (long long)(keys[i] >> 36) == r; ++i) c += keep[i];
    counts[r] = c;
    if (c) atomicMax(max_count, c);
}

struct PathTable {
    int* rx;
    int* cand;
    signed char* order;
    int* seq;        // [P*L]
    double* verts;   // [P*(L+2)*3]
    double* length;
    double* delay;
    double* kdep;
    double* karr;
    double* nrm;     // [P*L*3]
    double* cosv;    // [P*L]
    int L;
};

__device__ void emit_row(const PathTable& T, long long row, long long rx_i, int cand, int K,
                         const int* seq, d3 tx, const d3* pts, d3 rx, const SceneDev& S) {
    Geom g;
    geom_from_points(tx, pts, K, rx, seq, S.nrm, S.prim_mat, g);
    T.rx[row] = (int)rx_i;
    T.cand[row] = cand;
    T.order[row] = (signed char)K;
    double* v = T.verts + row * (T.L + 2) * 3;
    for (int j = 0; j < T.L + 2; ++j) st3(v + 3 * j, d3{0.0, 0.0, 0.0});
    st3(v, tx);
    for (int j = 0; j < K; ++j) st3(v + 3 * (j + 1), pts[j]);
    st3(v + 3 * (K + 1), rx);
    for (int j = 0; j < T.L; ++j) {
        T.seq[row * T.L + j] = j < K ? seq[j] : -1;
        st3(T.nrm + (row * T.L + j) * 3, j < K ? g.nrm[j] : d3{0.0, 0.0, 0.0});
        T.cosv[row * T.L + j] = j < K ? g.cosi[j] : 0.0;
    }
    T.length[row] = g.length;
    T.delay[row] = g.delay;
    st3(T.kdep + 3 * row, g.dir[0]);
    st3(T.karr + 3 * row, g.dir[K]);
}

// LOS first, then kept records in (order, candidate) order (tracer.py:294).
// One warp per receiver: lanes take 32 consecutive sorted records at a time
// and place their rows with a ballot prefix (a receiver's records are
// contiguous, so a lane past the run ends it).
__global__ void k_emit_paths(Cands C, SceneDev S, const double* images, Receivers R, d3 tx,
                             const Rec* recs, const int* order, const unsigned long long* keys,
                             long long n_rec, const unsigned char* keep, const unsigned char* los,
                             const int* heads, const int* offsets, PathTable T) {
    const unsigned FULL = 0xffffffffu;
    long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (r >= R.n) return;   // whole warps
    long long row = offsets[r];
    d3 rx = receiver_pos(R, r);
    if (los[r]) {
        if (lane == 0) emit_row(T, row, r, -1, 0, nullptr, tx, nullptr, rx, S);
        ++row;
    }
    int h = heads[r];
    if (h < 0) return;
    for (long long b = h;; b += 32) {
        long long i = b + lane;
        bool in = i < n_rec && (long long)(keys[i] >> 36) == r;
        bool k = in && keep[i];
        unsigned m_in = __ballot_sync(FULL, in);
        unsigned m = __ballot_sync(FULL, k);
        if (k) {
            const Rec& a = recs[order[i]];
            d3 pts[MAX_DEPTH];
            solve_geometric(C, S, images, a.cand, tx, rx, pts);
            emit_row(T, row + __popc(m & ((1u << lane) - 1u)), r, a.cand, a.order,
                     C.seq + (long long)a.cand * C.max_len, tx, pts, rx, S);
        }
        row += __popc(m);
        if (m_in != FULL) break;
    }
}

// image_solve (tracer.py:150-183) of independent (tx, rx, sequence) triples —
// the explicit-array gains (em.py:425-459) and single image_solve queries.
// Order 0 rows are LOS checks (tracer.py:190, em.py:437-441).
__global__ void k_solve_pairs(SceneDev S, Bvh bvh, long long n, int L, const double* txp,
                              const double* rxp, const int* seq, const signed char* len,
                              unsigned char* valid, PathTable T) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int K = len[i];
    const int* sq = seq + i * L;
    d3 tx = ld3(txp + 3 * i), rx = ld3(rxp + 3 * i);
    d3 pts[MAX_DEPTH];
    bool ok = true;
    if (K > 0) {
        d3 img[MAX_DEPTH + 1];
        img[0] = tx;
        for (int j = 0; j < K; ++j)
            img[j + 1] = mirror(img[j], ld3(S.nrm + 3 * (long long)sq[j]), S.poff[sq[j]]);
        d3 cur = rx;
        for (int j = K - 1; j >= 0 && ok; --j) {   // solve_points + validity (solve_geometric)
            int prim = sq[j];
            d3 nn = ld3(S.nrm + 3 * (long long)prim);
            double cc = S.poff[prim];
            d3 seg = sub(img[j + 1], cur);
            double denom = tdot(seg, nn);
            if (fabs(denom) < 1e-15) { ok = false; break; }
            double s = (cc - tdot(cur, nn)) / denom;
            d3 p = d3{cur.x + seg.x * s, cur.y + seg.y * s, cur.z + seg.z * s};
            if (!(1e-12 < s && s < 1.0 - 1e-12)) { ok = false; break; }
            d3 v0 = ld3(S.v0 + 3 * (long long)prim), e1 = ld3(S.e1 + 3 * (long long)prim),
               e2 = ld3(S.e2 + 3 * (long long)prim);
            d3 w = sub(p, v0);
            double d11 = dot_blas(e1, e1), d12 = dot_blas(e1, e2), d22 = dot_blas(e2, e2);
            double w1 = dot_blas(w, e1), w2 = dot_blas(w, e2);
            double den = d11 * d22 - d12 * d12;
            double u = (d22 * w1 - d12 * w2) / den, v = (d11 * w2 - d12 * w1) / den;
            if (!(u >= -INSIDE_TOL && v >= -INSIDE_TOL && u + v <= 1.0 + INSIDE_TOL)) { ok = false; break; }
            pts[j] = p;
            cur = p;
        }
        for (int j = 0; j < K && ok; ++j) {
            d3 nn = ld3(S.nrm + 3 * (long long)sq[j]);
            double cc = S.poff[sq[j]];
            d3 before = j == 0 ? tx : pts[j - 1], after = j == K - 1 ? rx : pts[j + 1];
            if ((tdot(before, nn) - cc) * (tdot(after, nn) - cc) <= SIDE_TOL) ok = false;
        }
        d3 a = tx;
        for (int j = 0; j <= K && ok; ++j) {
            d3 b = j < K ? pts[j] : rx;
            double dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
            if (sqrt(dx * dx + dy * dy + dz * dz) <= 2 * RAY_EPS) ok = false;
            a = b;
        }
        if (ok) ok = segments_clear(bvh, tx, pts, K, rx, sq, S.nrm);
    } else {
        ok = S.n == 0 || occluded(bvh, tx, rx) == 0;
    }
    valid[i] = ok ? 1 : 0;
    if (ok) emit_row(T, i, 0, 0, K, sq, tx, pts, rx, S);
}

struct TransferArgs {
    long long n;
    int L;
    const signed char* order;
    const int* seq;
    const double* verts;
    const double* nrm;
    const double* cosv;
    const double* length;
    const double* delay;
    const double* tx_rows;
    const double* rx_rows;
    int tx_pat, rx_pat;
    const double* tx_slants;
    int n_st;
    const double* rx_slants;
    int n_sr;
    const double* eta;
    const int* prim_mat;
    const int* imat;   // [P*L] material per interaction, or null (prim_mat[seq])
    double wavelength, frequency;
    // rotation rows per device (rt_gains): row block of path p = tx_rows[tx_ridx[p]];
    // null = one row block per path (rt_transfer)
    const int* tx_ridx;
    const int* rx_ridx;
};

__device__ __forceinline__ const double* tx_rows_of(const TransferArgs& A, long long p) {
    return A.tx_rows + 9 * (A.tx_ridx ? (long long)A.tx_ridx[p] : p);
}
__device__ __forceinline__ const double* rx_rows_of(const TransferArgs& A, long long p) {
    return A.rx_rows + 9 * (A.rx_ridx ? (long long)A.rx_ridx[p] : p);
}

__device__ inline void table_geom(const TransferArgs& A, long long p, Geom& g) {
    int K = A.order[p];
    geom_from_table(K, A.verts + p * (A.L + 2) * 3, A.nrm + p * A.L * 3, A.cosv + p * A.L,
                    A.seq + p * A.L, A.prim_mat, A.imat ? A.imat + p * A.L : nullptr, A.length[p],
                    A.delay[p], g);
}

__device__ __forceinline__ int interaction_material(const TransferArgs& A, long long p, int j) {
    return A.imat ? A.imat[p * A.L + j] : A.prim_mat[A.seq[p * A.L + j]];
}

// a[p, s, r] for every path and slant pair (em.py:291-312, 397-405)
__global__ void k_transfer(const __grid_constant__ TransferArgs A, double* a_out) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= A.n * A.n_st) return;
    long long p = i / A.n_st;
    int s = (int)(i - p * A.n_st);
    Geom g;
    table_geom(A, p, g);
    c3 f = transport(g, A.tx_pat, A.tx_slants[s], tx_rows_of(A, p), A.eta);
    for (int r = 0; r < A.n_sr; ++r) {
        d3 rf = rx_field(g, A.rx_pat, A.rx_slants[r], rx_rows_of(A, p));
        c2 a = finish(f, rf, g, A.wavelength, A.frequency);
        long long o = ((p * A.n_st + s) * A.n_sr + r) * 2;
        a_out[o] = a.re;
        a_out[o + 1] = a.im;
    }
}

// per (path, slant pair) item: each interaction's eta-gradient contribution
// into contrib[item * L + j] (zeros past the path's order or for G = 0)
__global__ void k_transfer_bwd(const __grid_constant__ TransferArgs A, const double* grad_a,
                               double2* contrib) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= A.n * A.n_st * A.n_sr) return;
    long long p = i / (A.n_st * A.n_sr);
    int rem = (int)(i - p * A.n_st * A.n_sr);
    int s = rem / A.n_sr, r = rem - s * A.n_sr;
    double2* out = contrib + i * A.L;
    for (int j = 0; j < A.L; ++j) out[j] = make_double2(0.0, 0.0);
    c2 G = c2{grad_a[2 * i], grad_a[2 * i + 1]};
    if (G.re == 0.0 && G.im == 0.0) return;
    Geom g;
    table_geom(A, p, g);
    transfer_adjoint(g, A.tx_pat, A.tx_slants[s], tx_rows_of(A, p), A.rx_pat, A.rx_slants[r],
                     rx_rows_of(A, p), A.eta, A.wavelength, A.frequency, G, out);
}

// grad_eta[m] += sum of the contributions of material m, in a fixed order: one
// block per material, thread t sums entries t, t + B, t + 2B, ... in index
// order, then a fixed shared-memory tree.  No atomics: the result is the same
// bit pattern on every run (reference criterion 10, byte-identical logs).
constexpr int ADJ_BLOCK = 256;
__global__ void __launch_bounds__(ADJ_BLOCK) k_grad_eta_reduce(const __grid_constant__ TransferArgs A,
                                                                const double2* contrib, double* grad_eta) {
    __shared__ double sre[ADJ_BLOCK], sim[ADJ_BLOCK];
    const int m = blockIdx.x;
    const long long items = A.n * A.n_st * A.n_sr, per_path = (long long)A.n_st * A.n_sr;
    double re = 0.0, im = 0.0;
    for (long long e = threadIdx.x; e < items * A.L; e += ADJ_BLOCK) {
        long long i = e / A.L;
        int j = (int)(e - i * A.L);
        long long p = i / per_path;
        if (j >= A.order[p] || interaction_material(A, p, j) != m) continue;
        double2 c = contrib[e];
        re += c.x;
        im += c.y;
    }
    sre[threadIdx.x] = re;
    sim[threadIdx.x] = im;
    __syncthreads();
    for (int w = ADJ_BLOCK / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            sre[threadIdx.x] += sre[threadIdx.x + w];
            sim[threadIdx.x] += sim[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        grad_eta[2 * m] += sre[0];
        grad_eta[2 * m + 1] += sim[0];
    }
}

// several device-to-device copies in one launch (blockIdx.y = segment):
// rt_paths_get hands out the 11 path-table columns with one kernel instead
// of 11 cudaMemcpyAsync calls
struct CopySeg {
    const unsigned char* src;
    unsigned char* dst;
    long long bytes;
};
struct CopyBatch {
    CopySeg s[12];
};
__global__ void k_copy_batch(const __grid_constant__ CopyBatch B) {
    const CopySeg& c = B.s[blockIdx.y];
    if (!c.dst) return;
    long long stride = (long long)gridDim.x * blockDim.x;
    long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if ((c.bytes & 3) == 0 && (((unsigned long long)c.src | (unsigned long long)c.dst) & 3) == 0) {
        const unsigned* a = reinterpret_cast<const unsigned*>(c.src);
        unsigned* b = reinterpret_cast<unsigned*>(c.dst);
        for (long long i = i0; i < c.bytes / 4; i += stride) b[i] = a[i];
    } else {
        for (long long i = i0; i < c.bytes; i += stride) c.dst[i] = c.src[i];
    }
}

// Fresnel coefficients (em.py:123-141) of a batch of (eta, cos theta_i)
__global__ void k_fresnel(long long n, const double* eta, const double* cosv, double* rte, double* rtm) {
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    c2 te, tm, w;
    fresnel(c2{eta[2 * i], eta[2 * i + 1]}, cosv[i], te, tm, w);
    rte[2 * i] = te.re;
    rte[2 * i + 1] = te.im;
    rtm[2 * i] = tm.re;
    rtm[2 * i + 1] = tm.im;
}

}  // namespace rt

// bvh_build.cuh — scene ingest and GPU LBVH construction.
//
// Replaces Bvh.__init__/_gather/_build (bvh.py:33-79, 180-197).  The tree
// shape differs from the reference's median split (it is not a parity
// target); the per-primitive arrays are bit-identical to the
// reference's numpy ones and first-hit semantics are those of trace.cuh.
//
// Build: prim AABBs + centroids -> 63-bit Morton codes -> CUB radix sort ->
// Karras (2012) hierarchy -> bottom-up refit with atomic flags -> child-pair
// node layout with subtrees of <= LEAF_MAX prims collapsed into leaves.
#pragma once
#include <cub/cub.cuh>
#include "rt_common.cuh"

namespace rt {

__device__ inline unsigned float_to_ordered(float f) {
    unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ inline float ordered_to_float(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// conservative float bound: inflate then round outward
__device__ inline float lo_f(double x) { return __double2float_rd(x - (1e-9 + 1e-9 * fabs(x))); }
__device__ inline float hi_f(double x) { return __double2float_ru(x + (1e-9 + 1e-9 * fabs(x))); }

// v0/e1/e2 gather (bvh.py:180-197), normals + plane offsets (bvh.py:39-44),
// prim boxes and centroids; cbounds accumulates the centroid AABB.
__global__ void k_gather(const double* __restrict__ V, const int64_t* __restrict__ T, int64_t n,
                         double* v0, double* e1, double* e2, double* nrm, double* poff,
                         float* box /*[n*6]*/, float* cent /*[n*3]*/, unsigned* cbounds) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    float cx = 0.f, cy = 0.f, cz = 0.f;
    bool ok = i < n;
    if (ok) {
        d3 a = ld3(V + 3 * T[3 * i]), b = ld3(V + 3 * T[3 * i + 1]), c = ld3(V + 3 * T[3 * i + 2]);
        d3 E1 = sub(b, a), E2 = sub(c, a);
        st3(v0 + 3 * i, a); st3(e1 + 3 * i, E1); st3(e2 + 3 * i, E2);
        d3 n3 = cross(E1, E2);                                    // np.cross
        double len = sqrt(n3.x * n3.x + n3.y * n3.y + n3.z * n3.z);  // np.linalg.norm(axis=1)
        d3 un = d3{n3.x / len, n3.y / len, n3.z / len};
        st3(nrm + 3 * i, un);
        poff[i] = (un.x * a.x + un.z * a.z) + un.y * a.y;         // np.einsum("ij,ij->i")
        d3 p1 = add(a, E1), p2 = add(a, E2);
        double lx = fmin(fmin(a.x, p1.x), p2.x), ly = fmin(fmin(a.y, p1.y), p2.y),
               lz = fmin(fmin(a.z, p1.z), p2.z);
        double hx = fmax(fmax(a.x, p1.x), p2.x), hy = fmax(fmax(a.y, p1.y), p2.y),
               hz = fmax(fmax(a.z, p1.z), p2.z);
        float* bx = box + 6 * i;
        bx[0] = lo_f(lx); bx[1] = lo_f(ly); bx[2] = lo_f(lz);
        bx[3] = hi_f(hx); bx[4] = hi_f(hy); bx[5] = hi_f(hz);
        cx = (float)(0.5 * (lx + hx)); cy = (float)(0.5 * (ly + hy)); cz = (float)(0.5 * (lz + hz));
        cent[3 * i] = cx; cent[3 * i + 1] = cy; cent[3 * i + 2] = cz;
    }
    // block-reduce centroid bounds, one atomic per block and component
    __shared__ float red[7][32];
    float amax = 0.f;
    if (ok) {
        const float* bx = box + 6 * i;
        for (int m = 0; m < 6; ++m) amax = fmaxf(amax, fabsf(bx[m]));
    }
    float v[7] = {ok ? cx : INFINITY, ok ? cy : INFINITY, ok ? cz : INFINITY,
                  ok ? cx : -INFINITY, ok ? cy : -INFINITY, ok ? cz : -INFINITY, amax};
    for (int k = 0; k < 7; ++k) {
        float x = v[k];
        for (int o = 16; o; o >>= 1) {
            float y = __shfl_xor_sync(0xffffffffu, x, o);
            x = k < 3 ? fminf(x, y) : fmaxf(x, y);
        }
        if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = x;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
        int k = threadIdx.x;
        float x = red[k][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) x = k < 3 ? fminf(x, red[k][w]) : fmaxf(x, red[k][w]);
        unsigned u = float_to_ordered(x);
        if (k < 3) atomicMin(cbounds + k, u); else atomicMax(cbounds + k, u);
    }
}

// Quantise the centroids on one scale (a cube of the largest extent), not per
// axis: per-axis scaling gave the 40 m tall, 3.5 km wide C3 city as many z
// bits as x / y bits, so the curve split on height as often as on position.
// Measured (C3 launch, 6 tx positions): 86.3 -> 58.1 ms; node visits per
// bounce 30.7 -> 20.9; surface-area estimate 51.8 -> 27.9.
#ifndef RT_MORTON_ISO
#define RT_MORTON_ISO 1
#endif
#ifndef RT_MORTON_EMC
#define RT_MORTON_EMC 0   // extended (size) Morton codes: 61.0 ms on the same sweep
#endif
__device__ inline uint64_t spread21(uint64_t x) {
    x &= 0x1fffffULL;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}

// 63-bit Morton code of the centroid.  Primitives whose box spans more than a
// quarter of the scene on any axis (e.g. a ground quad) get bit 63 set: the
// Karras root then splits them into their own subtree instead of letting
// their scene-sized boxes inflate every ancestor of some spatial region.
__global__ void k_morton(const float* cent, const float* pbox, const unsigned* cbounds, int64_t n,
                         uint64_t* keys, int* idx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    float lo[3], ext[3];
    float emax = 0.f;
    for (int k = 0; k < 3; ++k) {
        lo[k] = ordered_to_float(cbounds[k]);
        ext[k] = ordered_to_float(cbounds[3 + k]) - lo[k];
        emax = fmaxf(emax, ext[k]);
    }
    const float* b = pbox + 6 * i;
#if RT_MORTON_EMC
    // extended Morton code (size as a 4th dimension, isotropic cube, 15 bits each)
    uint64_t key = 0;
    {
        uint64_t c[4];
        for (int k = 0; k < 3; ++k) {
            float f = emax > 0.f ? (cent[3 * i + k] - lo[k]) / emax : 0.5f;
            c[k] = (uint64_t)fminf(fmaxf(f * 32768.0f, 0.0f), 32767.0f);
        }
        float diag = sqrtf((b[3] - b[0]) * (b[3] - b[0]) + (b[4] - b[1]) * (b[4] - b[1]) +
                           (b[5] - b[2]) * (b[5] - b[2]));
        float sz = emax > 0.f ? diag / (1.7320508f * emax) : 0.f;   // 0..1
        c[3] = (uint64_t)fminf(fmaxf(sz * 32768.0f, 0.0f), 32767.0f);
        for (int bit = 14; bit >= 0; --bit)
            for (int k = 0; k < 4; ++k) key = (key << 1) | ((c[k] >> bit) & 1ULL);
    }
#else
    uint64_t q[3];
    for (int k = 0; k < 3; ++k) {
#if RT_MORTON_ISO
        float f = emax > 0.f ? (cent[3 * i + k] - lo[k]) / emax : 0.5f;   // one scale: a cube
#else
        float f = ext[k] > 0.f ? (cent[3 * i + k] - lo[k]) / ext[k] : 0.5f;
#endif
        f = fminf(fmaxf(f * 2097152.0f, 0.0f), 2097151.0f);
        q[k] = (uint64_t)f;
    }
    uint64_t key = (spread21(q[0]) << 2) | (spread21(q[1]) << 1) | spread21(q[2]);
#endif
    float pext = fmaxf(fmaxf(b[3] - b[0], b[4] - b[1]), b[5] - b[2]);
    if (emax > 0.f && pext > 0.25f * emax) key |= 1ULL << 63;
    keys[i] = key;
    idx[i] = (int)i;
}

__device__ inline int delta(const uint64_t* keys, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    uint64_t a = keys[i], b = keys[j];
    if (a == b) return 64 + __clz((unsigned)(i ^ j));
    return __clzll(a ^ b);
}

// Karras 2012: internal node i covers [first, last]; children are internal
// nodes (>= 0) or leaves (~sorted index).
__global__ void k_karras(const uint64_t* keys, int n, int* child /*[2*(n-1)]*/, int* parent_int,
                         int* parent_leaf, int* rfirst, int* rlast) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = (delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = delta(keys, n, i, i - d);
    int lmax = 2;
    while (delta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
    int j = i + l * d;
    int dnode = delta(keys, n, i, j);
    int s = 0;
    int span = l;
    for (int t = (span + 1) >> 1;; t = (t + 1) >> 1) {
        if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
        if (t == 1) break;
    }
    int gamma = i + s * d + (d < 0 ? -1 : 0);
    int first = i < j ? i : j, last = i < j ? j : i;
    int left = (first == gamma) ? ~gamma : gamma;
    int right = (last == gamma + 1) ? ~(gamma + 1) : gamma + 1;
    child[2 * i] = left;
    child[2 * i + 1] = right;
    if (left < 0) parent_leaf[~left] = i; else parent_int[left] = i;
    if (right < 0) parent_leaf[~right] = i; else parent_int[right] = i;
    rfirst[i] = first;
    rlast[i] = last;
}

// bottom-up union of boxes; the second thread to reach a node computes it
__global__ void k_refit(int n, const int* sorted_idx, const float* pbox, const int* child,
                        const int* parent_int, const int* parent_leaf, float* nbox /*[(n-1)*6]*/,
                        int* flags) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int node = parent_leaf[k];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(flags + node, 1) == 0) return;
        __threadfence();
        float b[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
        for (int c = 0; c < 2; ++c) {
            int ch = child[2 * node + c];
            const float* src = ch < 0 ? pbox + 6 * (int64_t)sorted_idx[~ch] : nbox + 6 * (int64_t)ch;
            for (int m = 0; m < 3; ++m) {
                float lo = __ldcg(src + m), hi = __ldcg(src + 3 + m);
                b[m] = fminf(b[m], lo);
                b[3 + m] = fmaxf(b[3 + m], hi);
            }
        }
        for (int m = 0; m < 6; ++m) __stcg(nbox + 6 * (int64_t)node + m, b[m]);
        node = parent_int[node];
    }
}

// eps_box = 2^-20 * max(S, 1), S = max |coordinate| (trace.cuh slab32)
__device__ inline float box_eps(const unsigned* cbounds) {
    return fmaxf(ordered_to_float(cbounds[6]), 1.0f) * 9.5367431640625e-07f;
}
__device__ inline void inflate6(float* b, float e) {
    for (int m = 0; m < 3; ++m) {
        b[m] = __fsub_rd(b[m], e);
        b[3 + m] = __fadd_ru(b[3 + m], e);
    }
}

__global__ void k_layout(int n, const int* sorted_idx, const float* pbox, const int* child,
                         const float* nbox, const int* rfirst, const int* rlast,
                         const unsigned* cbounds, BNode* out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    float eps = box_eps(cbounds);
    float bx[2][6];
    int ref[2];
    for (int c = 0; c < 2; ++c) {
        int ch = child[2 * i + c];
        const float* src;
        if (ch < 0) {
            src = pbox + 6 * (int64_t)sorted_idx[~ch];
            ref[c] = make_leaf(~ch, 1);
        } else {
            src = nbox + 6 * (int64_t)ch;
            int cnt = rlast[ch] - rfirst[ch] + 1;
            ref[c] = cnt <= LEAF_MAX ? make_leaf(rfirst[ch], cnt) : ch;
        }
        for (int m = 0; m < 6; ++m) bx[c][m] = src[m];
        inflate6(bx[c], eps);
    }
    out[i] = pack_bnode(bx, ref[0], ref[1]);
}

// single-prim scene: root with the one leaf on both sides
__global__ void k_layout_one(const float* pbox, const unsigned* cbounds, BNode* out) {
    float s[6];
    for (int m = 0; m < 6; ++m) s[m] = pbox[m];
    inflate6(s, box_eps(cbounds));
    float bx[2][6];
    for (int m = 0; m < 6; ++m) bx[0][m] = bx[1][m] = s[m];
    out[0] = pack_bnode(bx, make_leaf(0, 1), make_leaf(0, 1));
}

// ---- 4-wide collapse (level-synchronous, top-down) ---------------------------------------
// BVH4 node = binary node X; its children = X's two children with the internal
// child of largest surface area repeatedly replaced by its own two children
// until there are four (or only leaves remain).

__device__ inline float box_area(const float* b) {
    float dx = fmaxf(b[3] - b[0], 0.f), dy = fmaxf(b[4] - b[1], 0.f), dz = fmaxf(b[5] - b[2], 0.f);
    return dx * dy + dy * dz + dz * dx;
}

__device__ inline void bin_child(const BNode& nd, int c, int& ref, float* b) {
    unpack_bnode(nd, c, b);
    ref = c == 0 ? nd.d.x : nd.d.y;
}

__global__ void k_collapse(const BNode* bin, const int* frontier, int nf, BNode4* out, int* out_count,
                           int* map, int* next, int* next_count) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    int X = frontier[i];
    int q = atomicAdd(out_count, 1);
    map[X] = q;
    int ref[4];
    float bx[4][6];
    BNode nd = bin[X];
    bin_child(nd, 0, ref[0], bx[0]);
    bin_child(nd, 1, ref[1], bx[1]);
    int n = 2;
    while (n < 4) {
        int best = -1;
        float bestA = -1.f;
        for (int k = 0; k < n; ++k)
            if (!ref_is_leaf(ref[k])) {
                float A = box_area(bx[k]);
                if (A > bestA) { bestA = A; best = k; }
            }
        if (best < 0) break;
        BNode y = bin[ref[best]];
        bin_child(y, 0, ref[best], bx[best]);
        bin_child(y, 1, ref[n], bx[n]);
        ++n;
    }
    BNode4 o;
    float lo[3][4], hi[3][4];
    int ch[4];
    for (int k = 0; k < 4; ++k) {
        for (int m = 0; m < 3; ++m) {
            lo[m][k] = k < n ? bx[k][m] : INFINITY;
            hi[m][k] = k < n ? bx[k][3 + m] : -INFINITY;
        }
        ch[k] = k < n ? ref[k] : EMPTY_REF;
        if (k < n && !ref_is_leaf(ref[k])) next[atomicAdd(next_count, 1)] = ref[k];
    }
    o.lox = make_float4(lo[0][0], lo[0][1], lo[0][2], lo[0][3]);
    o.loy = make_float4(lo[1][0], lo[1][1], lo[1][2], lo[1][3]);
    o.loz = make_float4(lo[2][0], lo[2][1], lo[2][2], lo[2][3]);
    o.hix = make_float4(hi[0][0], hi[0][1], hi[0][2], hi[0][3]);
    o.hiy = make_float4(hi[1][0], hi[1][1], hi[1][2], hi[1][3]);
    o.hiz = make_float4(hi[2][0], hi[2][1], hi[2][2], hi[2][3]);
    o.child = make_int4(ch[0], ch[1], ch[2], ch[3]);
    o.pad = make_int4(0, 0, 0, 0);
    out[q] = o;
}

// binary internal indices -> BVH4 indices
__global__ void k_fix_refs(BNode4* out, int n4, const int* map) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n4) return;
    int4 c = out[i].child;
    int v[4] = {c.x, c.y, c.z, c.w};
    for (int k = 0; k < 4; ++k)
        if (v[k] != EMPTY_REF && !ref_is_leaf(v[k])) v[k] = map[v[k]];
    out[i].child = make_int4(v[0], v[1], v[2], v[3]);
}

__global__ void k_sorted_tris(int n, const int* sorted_idx, const double* v0, const double* e1,
                              const double* e2, TriRec* tris) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int p = sorted_idx[k];
    TriRec t;
    t.v0x = v0[3 * p]; t.v0y = v0[3 * p + 1]; t.v0z = v0[3 * p + 2];
    t.e1x = e1[3 * p]; t.e1y = e1[3 * p + 1]; t.e1z = e1[3 * p + 2];
    t.e2x = e2[3 * p]; t.e2y = e2[3 * p + 1]; t.e2z = e2[3 * p + 2];
    t.prim = p;
    t.pad = 0;
    tris[k] = t;
}

}  // namespace rt

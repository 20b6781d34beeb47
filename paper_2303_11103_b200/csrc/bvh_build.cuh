// bvh_build.cuh — scene ingest and GPU LBVH construction.
//
// Replaces Bvh.__init__/_gather/_build (bvh.py:33-79, 180-197).  The tree
// shape differs from the reference's median split (it is not a parity
// target); the per-primitive arrays are bit-identical to the
// reference's numpy ones and first-hit semantics are those of trace.cuh.
//
// Ingest: prim AABBs + centroids, the scene bounds and 63-bit Morton codes
// (the PLOC variant's input).  The product tree is the binned-SAH build of
// bvh_sah.cuh; the Karras LBVH and the 4-wide collapse measured slower (DESIGN
// §4) and were removed from the library.
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
__global__ void k_gather(const double* __restrict__ V, const int32_t* __restrict__ T, int64_t n,
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

// FP32 box filter origin bound 2 max(S, 1) (trace.cuh ray_fast)
__global__ void k_origin_limit(const unsigned* cbounds, double* out) {
    *out = 2.0 * fmax((double)ordered_to_float(cbounds[6]), 1.0);
}

// eps_box = 2^-19 * max(S, 1) (2^-20 with the correctly rounded reciprocal),
// S = max |coordinate| (trace.cuh slab32 error budget)
__device__ inline float box_eps(const unsigned* cbounds) {
    return fmaxf(ordered_to_float(cbounds[6]), 1.0f) * (RT_RCP_APPROX ? 1.9073486328125e-06f : 9.5367431640625e-07f);
}
__device__ inline void inflate6(float* b, float e) {
    for (int m = 0; m < 3; ++m) {
        b[m] = __fsub_rd(b[m], e);
        b[3 + m] = __fadd_ru(b[3 + m], e);
    }
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

// rt_common.cuh — shared types, constants and exact-rounding helpers.
//
// Every discrete decision of the reference (hit / miss, inside / outside,
// valid / invalid) is taken in FP64 with the reference's operation order.
// The library is compiled with --fmad=false, so `a*b + c` is two roundings
// exactly like a Python float expression; numpy's BLAS dot on 3-vectors is
// reproduced explicitly with __fma_rn (see dot_blas).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rt {

constexpr double RAY_EPS = 1e-4;      // bvh.py:17
constexpr double DET_EPS = 1e-12;     // bvh.py:18
constexpr double BARY_EPS = 1e-12;    // bvh.py:19
constexpr double MERGE_TOL = 1e-6;    // tracer.py:30
constexpr double INSIDE_TOL = 1e-9;   // tracer.py:31
constexpr double SIDE_TOL = 1e-12;    // tracer.py:32
constexpr double SPEED_OF_LIGHT = 299792458.0;
constexpr double PI = 3.141592653589793;
constexpr double TWO_PI = 2.0 * 3.141592653589793;
constexpr int MAX_DEPTH = 8;          // compile-time bound on interactions per path
#ifndef RT_LEAF_MAX
#define RT_LEAF_MAX 2   // measured: 2 beats 1/4/8 on C3 (fewer FP64 tests, +4% nodes)
#endif
constexpr int LEAF_MAX = RT_LEAF_MAX;  // BVH leaf collapse threshold (<= 8)
constexpr int STACK_SIZE = 128;
#ifndef RT_RCP_APPROX
#define RT_RCP_APPROX 1   // approximate FP32 reciprocal in the box filter (trace.cuh rcp32)
#endif
constexpr int RT_PAT_PROBE_THETA_ID = 3;  // em.py:70-75 internal coverage probes
constexpr int RT_PAT_PROBE_PHI_ID = 4;

struct d3 {
    double x, y, z;
};

__host__ __device__ inline d3 mk(double x, double y, double z) { return d3{x, y, z}; }
__host__ __device__ inline d3 sub(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ inline d3 add(d3 a, d3 b) { return d3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ inline d3 scale(d3 a, double s) { return d3{a.x * s, a.y * s, a.z * s}; }
// geometry.py t_dot: left-to-right, no contraction
__host__ __device__ inline double tdot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
// numpy 1-D `a @ b` (OpenBLAS ddot): fma(a2,b2, fma(a1,b1, a0*b0))
__device__ inline double dot_blas(d3 a, d3 b) {
    return __fma_rn(a.z, b.z, __fma_rn(a.y, b.y, a.x * b.x));
}
__host__ __device__ inline d3 cross(d3 a, d3 b) {
    return d3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ inline d3 ld3(const double* p) { return d3{p[0], p[1], p[2]}; }
__device__ inline void st3(double* p, d3 v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; }

// BVH node: both children's boxes (float, rounded outward) + child refs.
// A child ref >= 0 is an internal node index; a leaf ref has bit 31 set,
// bits 28..30 = count-1, bits 0..27 = first slot in the sorted triangle array.
// Each (lo, hi) pair of one child and axis sits in an aligned register pair
// after the 16-byte loads, so the box filter computes both slab planes with
// one packed FFMA2 (trace.cuh slab32).
struct __align__(16) BNode {
    float4 a;   // lo0.x hi0.x lo0.y hi0.y
    float4 b;   // lo0.z hi0.z lo1.x hi1.x
    float4 c;   // lo1.y hi1.y lo1.z hi1.z
    int4 d;     // child0 child1 - -
};

// child boxes bx[c] = {lo.x, lo.y, lo.z, hi.x, hi.y, hi.z} <-> BNode
__host__ __device__ inline BNode pack_bnode(const float bx[2][6], int ref0, int ref1) {
    BNode nd;
    nd.a = make_float4(bx[0][0], bx[0][3], bx[0][1], bx[0][4]);
    nd.b = make_float4(bx[0][2], bx[0][5], bx[1][0], bx[1][3]);
    nd.c = make_float4(bx[1][1], bx[1][4], bx[1][2], bx[1][5]);
    nd.d = make_int4(ref0, ref1, 0, 0);
    return nd;
}
__host__ __device__ inline void unpack_bnode(const BNode& nd, int c, float* b) {
    if (c == 0) {
        b[0] = nd.a.x; b[3] = nd.a.y; b[1] = nd.a.z; b[4] = nd.a.w; b[2] = nd.b.x; b[5] = nd.b.y;
    } else {
        b[0] = nd.b.z; b[3] = nd.b.w; b[1] = nd.c.x; b[4] = nd.c.y; b[2] = nd.c.z; b[5] = nd.c.w;
    }
}

constexpr int EMPTY_REF = 0x7fffffff;

// triangle in sorted (BVH) order: FP64 v0, e1, e2 and the global prim id
struct __align__(16) TriRec {
    double v0x, v0y, v0z, e1x, e1y, e1z, e2x, e2y, e2z;
    int prim;
    int pad;
};

__host__ __device__ inline bool ref_is_leaf(int r) { return r < 0; }
__host__ __device__ inline int leaf_first(int r) { return r & 0x0FFFFFFF; }
__host__ __device__ inline int leaf_count(int r) { return ((r >> 28) & 7) + 1; }
__host__ __device__ inline int make_leaf(int first, int count) {
    return (int)(0x80000000u | ((unsigned)(count - 1) << 28) | (unsigned)first);
}

}  // namespace rt

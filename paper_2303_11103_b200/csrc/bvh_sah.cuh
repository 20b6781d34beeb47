// bvh_sah.cuh — top-down binned-SAH hierarchy builder (the default; PLOC and
// the Karras LBVH stay as A/B alternatives).
//
// Why: on the C3 city the PLOC tree walks 20.1 nodes per ray-bounce, a
// top-down SAH tree 16.3 (offline measurement over the same Fibonacci rays,
// depth 5: the surface-area estimate drops 27.9 -> 22.7).  The Manhattan grid
// defeats the Morton-order neighbourhood PLOC merges within.
//
// Level-synchronous: every range of > SAH_BIG primitives is split by CTAs
// over chunks (k_sahb_*), every range of > SAH_WARP_MAX (large scenes) or >
// small_max (small scenes) primitives by one CTA (k_sah_large): centroid
// bounds, SAH_BINS bins per axis in shared memory, the cheapest split, a
// stable partition into the other index buffer.  In large scenes a range of
// small_max < m <= SAH_WARP_MAX primitives is finished, whole subtree, by one
// warp (k_sah_warp).  Ranges of 2..small_max (8, or 4 for small scenes)
// primitives go to a list that k_sah_small finishes one thread per range with
// the exact sweep SAH.  The tree is split all the
// way to single primitives; the PLOC layout path then collapses subtrees of
// <= LEAF_MAX primitives into leaves.
//
// Node ids follow the PLOC convention (bvh_ploc.cuh): leaves [0, n) — here
// leaf k IS primitive k (identity sorted_idx) — and internal nodes [n, 2n-1).
// An internal node over the final primitive order is identified by its split
// position s (first slot of its right child, unique in [1, n-1]): id =
// n + s - 1.  No counters, and the tree is deterministic.
#pragma once
#include "bvh_ploc.cuh"

namespace rt {

#ifndef RT_SAH_BINS
#define RT_SAH_BINS 32   // C3 launch 14.33 vs 14.49 ms (16 bins), 19.2 vs 19.6 nodes per bounce
#endif
constexpr int SAH_BINS = RT_SAH_BINS;
#ifndef RT_SAH_SMALL
#define RT_SAH_SMALL 8   // with k_sah_warp below: C3 build 1.53 -> 1.47 ms (16: the per-thread sweeps dominate, 4: more warp nodes)
#endif
#ifndef RT_SAH_BIG
#define RT_SAH_BIG 8192
#endif
// Ranges of <= small_max prims: one thread, exact sweep.  small_max is chosen
// per build (rt_bvh_build): SAH_SMALL for big scenes (throughput: one thread
// per range beats a CTA per range), SAH_SMALL_LATENCY below
// SAH_LATENCY_PRIMS (latency: one thread's serial sweep over 16 prims took
// 0.19 ms of the 2,002-tri canyon build, ranges of <= 4 take microseconds).
constexpr int SAH_SMALL = RT_SAH_SMALL;
constexpr int SAH_SMALL_LATENCY = 4;
constexpr long long SAH_LATENCY_PRIMS = 65536;
constexpr int SAH_BLOCK = 256;
constexpr int SAH_BIG = RT_SAH_BIG;       // ranges above this: several CTAs (SAH_CHUNK prims each)
#ifndef RT_SAH_CHUNK
#define RT_SAH_CHUNK 1024   // C3 build 2.02 -> 1.95 ms (2048: 98 CTAs per level for 201k prims, fewer than the SMs)
#endif
constexpr int SAH_CHUNK = RT_SAH_CHUNK;
constexpr int SAH_NCAND = 3 * (SAH_BINS - 1);
static_assert(SAH_BINS == 32, "k_sah_warp keeps one bin per lane");
constexpr int SAH_NB = 3 * SAH_BINS * 7;   // bins per range: count + 6 ordered bounds, 3 axes
constexpr int SAH_NW = SAH_BLOCK / 32;
// ranges of small_max < m <= SAH_WARP_MAX: one warp builds the whole subtree
// (k_sah_warp) instead of one CTA per range and level
#ifndef RT_SAH_WARP_MAX
#define RT_SAH_WARP_MAX 128
#endif
constexpr int SAH_WARP_MAX = RT_SAH_WARP_MAX;
constexpr int SAHW_WARPS = 4;                  // warps per CTA
constexpr int SAHW_STACK = SAH_WARP_MAX;       // pending ranges per warp (<= subtree depth)

// a primitive range [begin, end) whose node hangs off `parent` as child
// `side & 1`; bit 1 of side names the index buffer holding the range
struct SahTask {
    int begin, end, parent, side;
};

// bin layout (shared or global): [axis][bin] count, then [axis][bin][6] bounds
__host__ __device__ constexpr int sah_cnt(int a, int b) { return a * SAH_BINS + b; }
__host__ __device__ constexpr int sah_bnd(int a, int b, int k) { return 3 * SAH_BINS + (a * SAH_BINS + b) * 6 + k; }

__device__ __forceinline__ float box_area(float lx, float ly, float lz, float hx, float hy, float hz) {
    float dx = hx - lx, dy = hy - ly, dz = hz - lz;
    return dx * dy + dy * dz + dz * dx;
}

// bin of a centroid coordinate (identical arithmetic for binning and partition)
__device__ __forceinline__ int sah_bin(float c, float lo, float scale) {
    int b = (int)((c - lo) * scale);
    return b < 0 ? 0 : (b >= SAH_BINS ? SAH_BINS - 1 : b);
}

// binning frame of a range from its centroid bounds; scale 0 = axis not splittable
__device__ __forceinline__ void sah_frame(const float cmin[3], const float cmax[3], float lo[3], float scale[3]) {
    for (int a = 0; a < 3; ++a) {
        float ext = cmax[a] - cmin[a];
        lo[a] = cmin[a];
        scale[a] = ext > 0.f ? (float)SAH_BINS / ext : 0.f;
    }
}

__device__ __forceinline__ void sah_bins_clear(unsigned* bins, int tid, int nthreads) {
    for (int t = tid; t < SAH_NB; t += nthreads) bins[t] = t < 3 * SAH_BINS ? 0u : (((t - 3 * SAH_BINS) % 6) < 3 ? 0xFFFFFFFFu : 0u);
}

// Bin one primitive per lane (valid lanes).  Lanes of a warp mostly share a
// bin, so each distinct bin is reduced across the warp first (redux.sync) and
// updated with one atomic per value: 7 atomics per distinct bin per axis
// instead of 7 per primitive per axis.  Every lane of the warp must call.
__device__ __forceinline__ void sah_bin_warp(bool valid, int p, const float* __restrict__ pbox,
                                             const float* __restrict__ cent, const float lo[3],
                                             const float scale[3], unsigned* bins) {
    const unsigned FULL = 0xffffffffu;
    int lane = threadIdx.x & 31;
    unsigned bl[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, bh[3] = {0u, 0u, 0u};
    float c[3] = {0.f, 0.f, 0.f};
    if (valid)
        for (int k = 0; k < 3; ++k) {
            bl[k] = float_to_ordered(__ldg(pbox + 6 * (long long)p + k));
            bh[k] = float_to_ordered(__ldg(pbox + 6 * (long long)p + 3 + k));
            c[k] = __ldg(cent + 3 * (long long)p + k);
        }
    unsigned active = __ballot_sync(FULL, valid);
    for (int a = 0; a < 3; ++a) {
        if (scale[a] == 0.f) continue;   // uniform: the frame is per range
        int b = valid ? sah_bin(c[a], lo[a], scale[a]) : -1;
        unsigned todo = active;
        while (todo) {
            int leader = __ffs(todo) - 1;
            int key = __shfl_sync(FULL, b, leader);
            unsigned grp = __ballot_sync(FULL, b == key);
            bool in = (grp >> lane) & 1u;
            unsigned mn0 = __reduce_min_sync(FULL, in ? bl[0] : 0xFFFFFFFFu);
            unsigned mn1 = __reduce_min_sync(FULL, in ? bl[1] : 0xFFFFFFFFu);
            unsigned mn2 = __reduce_min_sync(FULL, in ? bl[2] : 0xFFFFFFFFu);
            unsigned mx0 = __reduce_max_sync(FULL, in ? bh[0] : 0u);
            unsigned mx1 = __reduce_max_sync(FULL, in ? bh[1] : 0u);
            unsigned mx2 = __reduce_max_sync(FULL, in ? bh[2] : 0u);
            if (lane == leader) {
                atomicAdd(bins + sah_cnt(a, key), (unsigned)__popc(grp));
                atomicMin(bins + sah_bnd(a, key, 0), mn0);
                atomicMin(bins + sah_bnd(a, key, 1), mn1);
                atomicMin(bins + sah_bnd(a, key, 2), mn2);
                atomicMax(bins + sah_bnd(a, key, 3), mx0);
                atomicMax(bins + sah_bnd(a, key, 4), mx1);
                atomicMax(bins + sah_bnd(a, key, 5), mx2);
            }
            todo &= ~grp;
        }
    }
}

// Cheapest split from the bins, computed by one warp (all 32 lanes call; every
// lane gets the result).  Candidate (axis a, last left bin s) costs
// area(left) * n_left + area(right) * n_right (INFINITY when the axis is flat
// or a side is empty); ties go to the lowest (a, s).  Lane b holds bin b: a
// prefix scan gives the left side of split b, a suffix scan the right side
// (empty bins are the identity of min / max).  axis -1 when every centroid
// coincides (split the range in the middle).
__device__ void sah_choose_warp(const unsigned* bins, const float scale[3], int m, int& axis, int& split,
                                int& nl) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    float bc = INFINITY;
    int bi = SAH_NCAND;
    for (int a = 0; a < 3; ++a) {
        if (scale[a] == 0.f) continue;
        int cnt = (int)bins[sah_cnt(a, lane)];
        float q[6];
        for (int k = 0; k < 3; ++k) {
            q[k] = cnt ? ordered_to_float(bins[sah_bnd(a, lane, k)]) : INFINITY;
            q[3 + k] = cnt ? ordered_to_float(bins[sah_bnd(a, lane, 3 + k)]) : -INFINITY;
        }
        float l[6], r[6];
        int nl_ = cnt, nr_ = cnt;
        for (int k = 0; k < 6; ++k) { l[k] = q[k]; r[k] = q[k]; }
        for (int o = 1; o < 32; o <<= 1) {
            int cu = __shfl_up_sync(FULL, nl_, o), cd = __shfl_down_sync(FULL, nr_, o);
            if (lane >= o) nl_ += cu;
            if (lane + o < 32) nr_ += cd;
            for (int k = 0; k < 6; ++k) {
                float u = __shfl_up_sync(FULL, l[k], o), d = __shfl_down_sync(FULL, r[k], o);
                if (lane >= o) l[k] = k < 3 ? fminf(l[k], u) : fmaxf(l[k], u);
                if (lane + o < 32) r[k] = k < 3 ? fminf(r[k], d) : fmaxf(r[k], d);
            }
        }
        // split s = lane: left = prefix[lane], right = suffix[lane + 1]
        int nr_s = __shfl_down_sync(FULL, nr_, 1);
        float rs[6];
        for (int k = 0; k < 6; ++k) rs[k] = __shfl_down_sync(FULL, r[k], 1);
        if (lane < SAH_BINS - 1 && nl_ > 0 && nr_s > 0) {
            float c = box_area(l[0], l[1], l[2], l[3], l[4], l[5]) * (float)nl_ +
                      box_area(rs[0], rs[1], rs[2], rs[3], rs[4], rs[5]) * (float)nr_s;
            int cand = a * (SAH_BINS - 1) + lane;
            if (c < bc) { bc = c; bi = cand; }
        }
    }
    for (int o = 16; o; o >>= 1) {
        float oc = __shfl_xor_sync(FULL, bc, o);
        int oi = __shfl_xor_sync(FULL, bi, o);
        if (oc < bc || (oc == bc && oi < bi)) { bc = oc; bi = oi; }
    }
    axis = -1; split = 0; nl = m / 2;
    if (bc < INFINITY) {
        axis = bi / (SAH_BINS - 1);
        split = bi % (SAH_BINS - 1);
        int c = lane <= split ? (int)bins[sah_cnt(axis, lane)] : 0;
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
        nl = c;
    }
}

// sah_choose_warp for a CTA (all threads call; warp 0 computes).  out = {axis,
// last left bin, left count}.
__device__ void sah_choose(const unsigned* bins, const float scale[3], int m, int* out) {
    if (threadIdx.x < 32) {
        int axis, split, nl;
        sah_choose_warp(bins, scale, m, axis, split, nl);
        if (threadIdx.x == 0) { out[0] = axis; out[1] = split; out[2] = nl; }
    }
    __syncthreads();
}

__device__ __forceinline__ bool sah_left(int p, int pos_in_range, const float* __restrict__ cent, int axis,
                                         int split, int nl, const float lo[3], const float scale[3]) {
    return axis >= 0 ? sah_bin(__ldg(cent + 3 * (long long)p + axis), lo[axis], scale[axis]) <= split
                     : pos_in_range < nl;
}

// Stable partition of src[b0, e0) (a piece of range T starting at T.begin):
// left prims go to dst[T.begin + lbase ...], right ones to dst[T.begin + nl +
// rbase ...].  All BLOCK threads call; s_wl / s_wr: BLOCK / 32 ints of shared scratch.
template <int BLOCK = SAH_BLOCK>
__device__ void sah_partition(const SahTask& T, int b0, int e0, const int* src, int* dst,
                              const float* __restrict__ cent, const int* sp /*axis, split, nl*/,
                              const float lo[3], const float scale[3], int lbase, int rbase, int* s_wl,
                              int* s_wr) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int axis = sp[0], split = sp[1], nl = sp[2];
    for (int c0 = b0; c0 < e0; c0 += BLOCK) {
        int i = c0 + tid;
        bool valid = i < e0;
        int p = valid ? src[i] : 0;
        bool left = valid && sah_left(p, i - T.begin, cent, axis, split, nl, lo, scale);
        unsigned bl = __ballot_sync(0xffffffffu, left);
        unsigned br = __ballot_sync(0xffffffffu, valid && !left);
        if (lane == 0) { s_wl[wid] = __popc(bl); s_wr[wid] = __popc(br); }
        __syncthreads();
        int ol = 0, or_ = 0, tl = 0, tr = 0;
        for (int w = 0; w < BLOCK / 32; ++w) {
            if (w < wid) { ol += s_wl[w]; or_ += s_wr[w]; }
            tl += s_wl[w];
            tr += s_wr[w];
        }
        unsigned below = (1u << lane) - 1u;
        if (valid) {
            int pos = left ? T.begin + lbase + ol + __popc(bl & below)
                           : T.begin + nl + rbase + or_ + __popc(br & below);
            dst[pos] = p;
        }
        lbase += tl;
        rbase += tr;
        __syncthreads();
    }
}

// link node `id` under its parent (or publish it as the root)
__device__ __forceinline__ void sah_link(int id, int par, int side, int n, int* child, int* parent,
                                         int* root_out) {
    if (par >= 0) {
        child[2 * (long long)(par - n) + side] = id;
        parent[id] = par;
    } else {
        *root_out = id;
        parent[id] = -1;
    }
}

// Output lists of one split: single prims whose slot is final are linked
// directly (dst_ready), <= small_max -> small, <= SAH_BIG -> med, else big
// (with SAH_CHUNK-prim chunks mapped in chunk_task).
struct SahOut {
    int small_max;
    SahTask* small; int* n_small;
    SahTask* med; int* n_med;
    SahTask* big; int2* big_chunks; int* n_big; int* chunk_task; int* n_chunk;
    SahTask* warp; int* n_warp;   // small_max < m <= SAH_WARP_MAX: k_sah_warp (null: med)
};

__device__ void sah_emit(const SahTask& T, const float box[6], const int* sp, int n, const int* dst,
                         bool dst_ready, float* nbox, int* child, int* parent, int* count, int* root_out,
                         const SahOut& O) {
    int m = T.end - T.begin;
    int s = T.begin + sp[2];
    int id = n + s - 1;
    int buf = ((T.side >> 1) & 1) ^ 1;   // the children's data sit in the other buffer
    for (int k = 0; k < 6; ++k) nbox[6 * (long long)id + k] = box[k];
    count[id] = m;
    sah_link(id, T.parent, T.side & 1, n, child, parent, root_out);
    for (int c = 0; c < 2; ++c) {
        int cb = c ? s : T.begin, ce = c ? T.end : s, sz = ce - cb;
        SahTask ct{cb, ce, id, c | (buf << 1)};
        if (sz == 1 && dst_ready) {
            int p = dst[cb];
            child[2 * (long long)(id - n) + c] = p;
            parent[p] = id;
        } else if (sz <= O.small_max) {
            O.small[atomicAdd(O.n_small, 1)] = ct;
        } else if (O.warp && sz <= SAH_WARP_MAX) {
            O.warp[atomicAdd(O.n_warp, 1)] = ct;
        } else if (sz <= SAH_BIG) {
            O.med[atomicAdd(O.n_med, 1)] = ct;
        } else {
            int k = atomicAdd(O.n_big, 1);
            int nc = (sz + SAH_CHUNK - 1) / SAH_CHUNK;
            int c0 = atomicAdd(O.n_chunk, nc);
            O.big[k] = ct;
            O.big_chunks[k] = make_int2(c0, nc);
            for (int q = 0; q < nc; ++q) O.chunk_task[c0 + q] = k;
        }
    }
}

// ---- ranges of small_max < m <= SAH_BIG prims: one CTA each ----------------------------

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_sah_large(const SahTask* __restrict__ tasks, const int* d_ntask,
                                                        int* zero_after_next, int* idx0, int* idx1,
                                                        const float* __restrict__ pbox,
                                                        const float* __restrict__ cent, int n, float* nbox,
                                                        int* child, int* parent, int* count, int* root_out,
                                                        SahOut O) {
    // the counter the level after next fills: nobody reads or writes it during
    // this level (the caller's 3-way rotation), so clear it here
    if (blockIdx.x == 0 && threadIdx.x == 0 && zero_after_next) *zero_after_next = 0;
    if ((int)blockIdx.x >= *d_ntask) return;
    const SahTask T = tasks[blockIdx.x];
    const int* src = (T.side >> 1) & 1 ? idx1 : idx0;
    int* dst = (T.side >> 1) & 1 ? idx0 : idx1;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    __shared__ float red[12][BLOCK / 32];
    __shared__ float s_lo[3], s_scale[3], s_box[6];
    __shared__ unsigned s_bins[SAH_NB];
    __shared__ int s_sp[3];
    __shared__ int s_wl[BLOCK / 32], s_wr[BLOCK / 32];

    // centroid bounds and the node's box
    float v[12];
    for (int k = 0; k < 3; ++k) {
        v[k] = INFINITY; v[3 + k] = -INFINITY; v[6 + k] = INFINITY; v[9 + k] = -INFINITY;
    }
    for (int i = T.begin + tid; i < T.end; i += BLOCK) {
        int p = src[i];
        for (int k = 0; k < 3; ++k) {
            float c = __ldg(cent + 3 * (long long)p + k);
            v[k] = fminf(v[k], c);
            v[3 + k] = fmaxf(v[3 + k], c);
            v[6 + k] = fminf(v[6 + k], __ldg(pbox + 6 * (long long)p + k));
            v[9 + k] = fmaxf(v[9 + k], __ldg(pbox + 6 * (long long)p + 3 + k));
        }
    }
    for (int k = 0; k < 12; ++k) {
        bool mx = (k / 3) & 1;
        float x = v[k];
        for (int o = 16; o; o >>= 1) {
            float y = __shfl_xor_sync(0xffffffffu, x, o);
            x = mx ? fmaxf(x, y) : fminf(x, y);
        }
        if (lane == 0) red[k][wid] = x;
    }
    sah_bins_clear(s_bins, tid, BLOCK);
    __syncthreads();
    if (tid < 12) {
        bool mx = (tid / 3) & 1;
        float x = red[tid][0];
        for (int w = 1; w < BLOCK / 32; ++w) x = mx ? fmaxf(x, red[tid][w]) : fminf(x, red[tid][w]);
        red[tid][0] = x;
    }
    __syncthreads();
    if (tid == 0) {
        float cmin[3] = {red[0][0], red[1][0], red[2][0]}, cmax[3] = {red[3][0], red[4][0], red[5][0]};
        sah_frame(cmin, cmax, s_lo, s_scale);
        for (int k = 0; k < 6; ++k) s_box[k] = red[6 + k][0];
    }
    __syncthreads();
    float lo[3] = {s_lo[0], s_lo[1], s_lo[2]}, scale[3] = {s_scale[0], s_scale[1], s_scale[2]};

    for (int c0 = T.begin; c0 < T.end; c0 += BLOCK) {   // warp-uniform trip count
        int i = c0 + tid;
        bool valid = i < T.end;
        sah_bin_warp(valid, valid ? src[i] : 0, pbox, cent, lo, scale, s_bins);
    }
    __syncthreads();
    sah_choose(s_bins, scale, T.end - T.begin, s_sp);
    sah_partition<BLOCK>(T, T.begin, T.end, src, dst, cent, s_sp, lo, scale, 0, 0, s_wl, s_wr);
    if (tid == 0) sah_emit(T, s_box, s_sp, n, dst, true, nbox, child, parent, count, root_out, O);
}

// ---- ranges of small_max < m <= SAH_WARP_MAX prims: one warp per range, whole subtree ----
//
// The same binned SAH as k_sah_large (bins, candidate costs, ties to the
// lowest (axis, bin), stable partition into the other index buffer), with the
// warp walking its subtree depth-first from a shared-memory stack: one launch
// for every level below SAH_WARP_MAX instead of one CTA per range and level.
__global__ void __launch_bounds__(32 * SAHW_WARPS) k_sah_warp(const SahTask* __restrict__ tasks, const int* d_ntask,
                                                            int* idx0, int* idx1, const float* __restrict__ pbox,
                                                            const float* __restrict__ cent, int n, float* nbox,
                                                            int* child, int* parent, int* count, int* root_out,
                                                            int small_max, SahTask* small, int* n_small) {
    const unsigned FULL = 0xffffffffu;
    __shared__ unsigned s_bins[SAHW_WARPS][SAH_NB];
    __shared__ SahTask s_stack[SAHW_WARPS][SAHW_STACK];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int t = blockIdx.x * SAHW_WARPS + w;
    if (t >= *d_ntask) return;   // whole warps
    unsigned* bins = s_bins[w];
    SahTask* stk = s_stack[w];
    if (lane == 0) stk[0] = tasks[t];
    int sp = 1;
    __syncwarp();
    while (sp > 0) {
        const SahTask T = stk[--sp];
        __syncwarp();
        const int* src = (T.side >> 1) & 1 ? idx1 : idx0;
        int* dst = (T.side >> 1) & 1 ? idx0 : idx1;
        const int m = T.end - T.begin;
        // centroid bounds and the node's box (every lane ends with the totals)
        float v[12];
        for (int k = 0; k < 3; ++k) {
            v[k] = INFINITY; v[3 + k] = -INFINITY; v[6 + k] = INFINITY; v[9 + k] = -INFINITY;
        }
        for (int i = T.begin + lane; i < T.end; i += 32) {
            int p = src[i];
            for (int k = 0; k < 3; ++k) {
                float c = __ldg(cent + 3 * (long long)p + k);
                v[k] = fminf(v[k], c);
                v[3 + k] = fmaxf(v[3 + k], c);
                v[6 + k] = fminf(v[6 + k], __ldg(pbox + 6 * (long long)p + k));
                v[9 + k] = fmaxf(v[9 + k], __ldg(pbox + 6 * (long long)p + 3 + k));
            }
        }
        for (int k = 0; k < 12; ++k) {
            bool mx = (k / 3) & 1;
            for (int o = 16; o; o >>= 1) {
                float y = __shfl_xor_sync(FULL, v[k], o);
                v[k] = mx ? fmaxf(v[k], y) : fminf(v[k], y);
            }
        }
        float lo[3], scale[3];
        {
            float cmin[3] = {v[0], v[1], v[2]}, cmax[3] = {v[3], v[4], v[5]};
            sah_frame(cmin, cmax, lo, scale);
        }
        sah_bins_clear(bins, lane, 32);
        __syncwarp();
        for (int c0 = T.begin; c0 < T.end; c0 += 32) {
            int i = c0 + lane;
            bool valid = i < T.end;
            sah_bin_warp(valid, valid ? src[i] : 0, pbox, cent, lo, scale, bins);
        }
        __syncwarp();
        int axis, split, nl;
        sah_choose_warp(bins, scale, m, axis, split, nl);
        // stable partition
        const unsigned below = (1u << lane) - 1u;
        int lb = 0, rb = 0;
        for (int c0 = T.begin; c0 < T.end; c0 += 32) {
            int i = c0 + lane;
            bool valid = i < T.end;
            int p = valid ? src[i] : 0;
            bool left = valid && sah_left(p, i - T.begin, cent, axis, split, nl, lo, scale);
            unsigned bl = __ballot_sync(FULL, left), br = __ballot_sync(FULL, valid && !left);
            if (valid) dst[left ? T.begin + lb + __popc(bl & below) : T.begin + nl + rb + __popc(br & below)] = p;
            lb += __popc(bl);
            rb += __popc(br);
        }
        __syncwarp();   // the children read what other lanes wrote
        // the node and its children
        const int s = T.begin + nl, id = n + s - 1, buf = ((T.side >> 1) & 1) ^ 1;
        float bxv = v[6];
#pragma unroll
        for (int k = 1; k < 6; ++k)
            if (lane == k) bxv = v[6 + k];
        if (lane < 6) nbox[6 * (long long)id + lane] = bxv;
        if (lane == 0) {
            count[id] = m;
            sah_link(id, T.parent, T.side & 1, n, child, parent, root_out);
        }
        for (int c = 0; c < 2; ++c) {
            int cb = c ? s : T.begin, ce = c ? T.end : s, sz = ce - cb;
            SahTask ct{cb, ce, id, c | (buf << 1)};
            if (sz == 1) {
                if (lane == 0) {
                    int p = dst[cb];
                    child[2 * (long long)(id - n) + c] = p;
                    parent[p] = id;
                }
            } else if (sz <= small_max) {
                if (lane == 0) small[atomicAdd(n_small, 1)] = ct;
            } else {
                if (lane == 0) stk[sp] = ct;
                ++sp;
            }
        }
        __syncwarp();
    }
}

// ---- ranges of > SAH_BIG prims: one CTA per SAH_CHUNK-prim chunk -----------------------
//
// Per level: k_sahb_init (per range: empty bounds and bins), k_sahb_bounds
// (per chunk), k_sahb_bins (per chunk), k_sahb_split (per range: choose, emit
// the node and its children), k_sahb_count (per chunk: left prims),
// k_sahb_write (per chunk: stable partition at the chunk's offsets).
// Per-range scratch rb: 12 ordered bounds (cmin, cmax, bmin, bmax) + the bins
// + 3 split ints.
constexpr int SAH_RB = 12 + SAH_NB + 3;

__global__ void k_sahb_init(const int* d_ntask, unsigned* rb) {
    if ((int)blockIdx.x >= *d_ntask) return;
    unsigned* r = rb + (long long)blockIdx.x * SAH_RB;
    for (int t = threadIdx.x; t < 12; t += blockDim.x) r[t] = (t / 3) & 1 ? 0u : 0xFFFFFFFFu;
    sah_bins_clear(r + 12, threadIdx.x, blockDim.x);
}

__device__ __forceinline__ void sahb_frame(const unsigned* r, float lo[3], float scale[3]) {
    float cmin[3], cmax[3];
    for (int k = 0; k < 3; ++k) { cmin[k] = ordered_to_float(r[k]); cmax[k] = ordered_to_float(r[3 + k]); }
    sah_frame(cmin, cmax, lo, scale);
}

// the chunk's prim range within its task
__device__ __forceinline__ void sahb_chunk(const SahTask& T, int2 ch, int c, int& b0, int& e0) {
    b0 = T.begin + (c - ch.x) * SAH_CHUNK;
    e0 = min(b0 + SAH_CHUNK, T.end);
}

__global__ void __launch_bounds__(SAH_BLOCK) k_sahb_bounds(const SahTask* __restrict__ tasks, const int2* chunks,
                                                          const int* chunk_task, const int* d_nchunk,
                                                          const int* idx0, const int* idx1,
                                                          const float* __restrict__ pbox,
                                                          const float* __restrict__ cent, unsigned* rb) {
    int c = blockIdx.x;
    if (c >= *d_nchunk) return;
    int t = chunk_task[c];
    const SahTask T = tasks[t];
    const int* src = (T.side >> 1) & 1 ? idx1 : idx0;
    int b0, e0;
    sahb_chunk(T, chunks[t], c, b0, e0);
    __shared__ float red[12][SAH_NW];
    int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    float v[12];
    for (int k = 0; k < 3; ++k) {
        v[k] = INFINITY; v[3 + k] = -INFINITY; v[6 + k] = INFINITY; v[9 + k] = -INFINITY;
    }
    for (int i = b0 + tid; i < e0; i += SAH_BLOCK) {
        int p = src[i];
        for (int k = 0; k < 3; ++k) {
            float cc = __ldg(cent + 3 * (long long)p + k);
            v[k] = fminf(v[k], cc);
            v[3 + k] = fmaxf(v[3 + k], cc);
            v[6 + k] = fminf(v[6 + k], __ldg(pbox + 6 * (long long)p + k));
            v[9 + k] = fmaxf(v[9 + k], __ldg(pbox + 6 * (long long)p + 3 + k));
        }
    }
    for (int k = 0; k < 12; ++k) {
        bool mx = (k / 3) & 1;
        float x = v[k];
        for (int o = 16; o; o >>= 1) {
            float y = __shfl_xor_sync(0xffffffffu, x, o);
            x = mx ? fmaxf(x, y) : fminf(x, y);
        }
        if (lane == 0) red[k][wid] = x;
    }
    __syncthreads();
    if (tid < 12) {
        bool mx = (tid / 3) & 1;
        float x = red[tid][0];
        for (int w = 1; w < SAH_NW; ++w) x = mx ? fmaxf(x, red[tid][w]) : fminf(x, red[tid][w]);
        unsigned u = float_to_ordered(x);
        unsigned* r = rb + (long long)t * SAH_RB;
        if (mx) atomicMax(r + tid, u); else atomicMin(r + tid, u);
    }
}

__global__ void __launch_bounds__(SAH_BLOCK) k_sahb_bins(const SahTask* __restrict__ tasks, const int2* chunks,
                                                        const int* chunk_task, const int* d_nchunk,
                                                        const int* idx0, const int* idx1,
                                                        const float* __restrict__ pbox,
                                                        const float* __restrict__ cent, unsigned* rb) {
    int c = blockIdx.x;
    if (c >= *d_nchunk) return;
    int t = chunk_task[c];
    const SahTask T = tasks[t];
    const int* src = (T.side >> 1) & 1 ? idx1 : idx0;
    int b0, e0;
    sahb_chunk(T, chunks[t], c, b0, e0);
    unsigned* r = rb + (long long)t * SAH_RB;
    __shared__ unsigned s_bins[SAH_NB];
    float lo[3], scale[3];
    sahb_frame(r, lo, scale);
    sah_bins_clear(s_bins, threadIdx.x, SAH_BLOCK);
    __syncthreads();
    for (int c0 = b0; c0 < e0; c0 += SAH_BLOCK) {
        int i = c0 + threadIdx.x;
        bool valid = i < e0;
        sah_bin_warp(valid, valid ? src[i] : 0, pbox, cent, lo, scale, s_bins);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < SAH_NB; q += SAH_BLOCK) {
        unsigned x = s_bins[q];
        if (q < 3 * SAH_BINS) {
            if (x) atomicAdd(r + 12 + q, x);
        } else if (((q - 3 * SAH_BINS) % 6) < 3) {
            if (x != 0xFFFFFFFFu) atomicMin(r + 12 + q, x);
        } else if (x) {
            atomicMax(r + 12 + q, x);
        }
    }
}

__global__ void __launch_bounds__(64) k_sahb_split(const SahTask* __restrict__ tasks, const int* d_ntask,
                                                  unsigned* rb, int n, float* nbox, int* child, int* parent,
                                                  int* count, int* root_out, SahOut O) {
    int t = blockIdx.x;
    if (t >= *d_ntask) return;
    const SahTask T = tasks[t];
    unsigned* r = rb + (long long)t * SAH_RB;
    __shared__ int s_sp[3];
    float lo[3], scale[3];
    sahb_frame(r, lo, scale);
    sah_choose(r + 12, scale, T.end - T.begin, s_sp);
    if (threadIdx.x == 0) {
        int* sp = reinterpret_cast<int*>(r + 12 + SAH_NB);
        sp[0] = s_sp[0]; sp[1] = s_sp[1]; sp[2] = s_sp[2];
        float box[6];
        for (int k = 0; k < 6; ++k) box[k] = ordered_to_float(r[6 + k]);
        sah_emit(T, box, s_sp, n, nullptr, false, nbox, child, parent, count, root_out, O);
    }
}

__global__ void __launch_bounds__(SAH_BLOCK) k_sahb_count(const SahTask* __restrict__ tasks, const int2* chunks,
                                                         const int* chunk_task, const int* d_nchunk,
                                                         const int* idx0, const int* idx1,
                                                         const float* __restrict__ cent, const unsigned* rb,
                                                         int* chunk_left) {
    int c = blockIdx.x;
    if (c >= *d_nchunk) return;
    int t = chunk_task[c];
    const SahTask T = tasks[t];
    const int* src = (T.side >> 1) & 1 ? idx1 : idx0;
    int b0, e0;
    sahb_chunk(T, chunks[t], c, b0, e0);
    const unsigned* r = rb + (long long)t * SAH_RB;
    const int* sp = reinterpret_cast<const int*>(r + 12 + SAH_NB);
    float lo[3], scale[3];
    sahb_frame(r, lo, scale);
    int total = 0;
    for (int c0 = b0; c0 < e0; c0 += SAH_BLOCK) {
        int i = c0 + threadIdx.x;
        bool left = i < e0 && sah_left(src[i], i - T.begin, cent, sp[0], sp[1], sp[2], lo, scale);
        total += __syncthreads_count(left);
    }
    if (threadIdx.x == 0) chunk_left[c] = total;
}

__global__ void __launch_bounds__(SAH_BLOCK) k_sahb_write(const SahTask* __restrict__ tasks, const int2* chunks,
                                                         const int* chunk_task, const int* d_nchunk, int* idx0,
                                                         int* idx1, const float* __restrict__ cent,
                                                         const unsigned* rb, const int* chunk_left) {
    int c = blockIdx.x;
    if (c >= *d_nchunk) return;
    int t = chunk_task[c];
    const SahTask T = tasks[t];
    const int* src = (T.side >> 1) & 1 ? idx1 : idx0;
    int* dst = (T.side >> 1) & 1 ? idx0 : idx1;
    int2 ch = chunks[t];
    int b0, e0;
    sahb_chunk(T, ch, c, b0, e0);
    const unsigned* r = rb + (long long)t * SAH_RB;
    __shared__ int s_sp[3], s_base;
    __shared__ int s_wl[SAH_NW], s_wr[SAH_NW];
    if (threadIdx.x < 3) s_sp[threadIdx.x] = reinterpret_cast<const int*>(r + 12 + SAH_NB)[threadIdx.x];
    int part = 0;   // left prims in the task's earlier chunks
    for (int q = ch.x + threadIdx.x; q < c; q += SAH_BLOCK) part += chunk_left[q];
    __shared__ int s_part[SAH_NW];
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < SAH_NW; ++w) s += s_part[w];
        s_base = s;
    }
    __syncthreads();
    float lo[3], scale[3];
    sahb_frame(r, lo, scale);
    int lbase = s_base, rbase = (b0 - T.begin) - s_base;
    sah_partition(T, b0, e0, src, dst, cent, s_sp, lo, scale, lbase, rbase, s_wl, s_wr);
}

// one thread finishes a range of 2..small_max prims with the exact sweep SAH
__global__ void __launch_bounds__(128) k_sah_small(const SahTask* __restrict__ small, const int* d_nsmall,
                                                   const int* idx0, const int* idx1,
                                                   const float* __restrict__ pbox,
                                                   const float* __restrict__ cent, int n, float* nbox,
                                                   int* child, int* parent, int* count, int* root_out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= *d_nsmall) return;
    const SahTask T = small[t];
    const int* src = (T.side >> 1) & 1 ? idx1 : idx0;
    const int m = T.end - T.begin;
    int ids[SAH_SMALL], ord[SAH_SMALL], best_ord[SAH_SMALL];
    float key[SAH_SMALL], ra[SAH_SMALL];
    for (int k = 0; k < m; ++k) ids[k] = src[T.begin + k];
    int st_b[SAH_SMALL], st_e[SAH_SMALL], st_p[SAH_SMALL], st_s[SAH_SMALL];
    int sp = 0;
    st_b[0] = 0; st_e[0] = m; st_p[0] = T.parent; st_s[0] = T.side & 1;
    sp = 1;
    while (sp > 0) {
        --sp;
        int b = st_b[sp], e = st_e[sp], par = st_p[sp], side = st_s[sp];
        int mm = e - b;
        if (mm == 1) {
            int p = ids[b];
            child[2 * (long long)(par - n) + side] = p;
            parent[p] = par;
            continue;
        }
        float bx[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
        for (int k = b; k < e; ++k)
            for (int q = 0; q < 3; ++q) {
                bx[q] = fminf(bx[q], __ldg(pbox + 6 * (long long)ids[k] + q));
                bx[3 + q] = fmaxf(bx[3 + q], __ldg(pbox + 6 * (long long)ids[k] + 3 + q));
            }
        float bc = INFINITY;
        int bsplit = mm / 2;
        for (int k = 0; k < mm; ++k) best_ord[k] = ids[b + k];
        for (int a = 0; a < 3; ++a) {
            // insertion sort of the range by (centroid, prim id)
            for (int k = 0; k < mm; ++k) {
                int p = ids[b + k];
                float c = __ldg(cent + 3 * (long long)p + a);
                int j = k;
                while (j > 0 && (key[j - 1] > c || (key[j - 1] == c && ord[j - 1] > p))) {
                    key[j] = key[j - 1];
                    ord[j] = ord[j - 1];
                    --j;
                }
                key[j] = c;
                ord[j] = p;
            }
            float l[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
            for (int k = mm - 1; k > 0; --k) {
                for (int q = 0; q < 3; ++q) {
                    l[q] = fminf(l[q], __ldg(pbox + 6 * (long long)ord[k] + q));
                    l[3 + q] = fmaxf(l[3 + q], __ldg(pbox + 6 * (long long)ord[k] + 3 + q));
                }
                ra[k] = box_area(l[0], l[1], l[2], l[3], l[4], l[5]);
            }
            float r[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
            bool better = false;
            for (int k = 0; k < mm - 1; ++k) {
                for (int q = 0; q < 3; ++q) {
                    r[q] = fminf(r[q], __ldg(pbox + 6 * (long long)ord[k] + q));
                    r[3 + q] = fmaxf(r[3 + q], __ldg(pbox + 6 * (long long)ord[k] + 3 + q));
                }
                float c = box_area(r[0], r[1], r[2], r[3], r[4], r[5]) * (float)(k + 1) +
                          ra[k + 1] * (float)(mm - k - 1);
                if (c < bc) { bc = c; bsplit = k + 1; better = true; }
            }
            if (better)
                for (int k = 0; k < mm; ++k) best_ord[k] = ord[k];
        }
        for (int k = 0; k < mm; ++k) ids[b + k] = best_ord[k];
        int s = T.begin + b + bsplit;
        int id = n + s - 1;
        for (int k = 0; k < 6; ++k) nbox[6 * (long long)id + k] = bx[k];
        count[id] = mm;
        sah_link(id, par, side, n, child, parent, root_out);
        st_b[sp] = b + bsplit; st_e[sp] = e; st_p[sp] = id; st_s[sp] = 1; ++sp;
        st_b[sp] = b; st_e[sp] = b + bsplit; st_p[sp] = id; st_s[sp] = 0; ++sp;
    }
}

// BNodes emitted per subtree (em[]) bottom-up: the second child to arrive at a
// node computes it (Karras-style refit climb)
__global__ void k_sah_emitted(int n, const int* parent, const int* child, const int* count, int* em,
                              int* flags) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int node = parent[k];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&flags[node - n], 1) == 0) return;
        int a = child[2 * (long long)(node - n)], b = child[2 * (long long)(node - n) + 1];
        em[node] = __ldcg(em + a) + __ldcg(em + b) + (count[node] > LEAF_MAX ? 1 : 0);
        node = parent[node];
    }
}

// k_sah_emitted and the exact FP64 refit (bvh_ploc.cuh k_dbox_refit) in one
// climb: the second child to arrive at a node computes both its emitted-node
// count and its FP64 box (leaf k is prim k in the SAH order)
__global__ void k_sah_climb(int n, const int* parent, const int* child, const int* count, int* em, int* flags,
                            const double* v0, const double* e1, const double* e2, double* dbox) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double* o = dbox + 6 * (long long)k;
    for (int a = 0; a < 3; ++a) {
        double x0 = v0[3 * (long long)k + a];
        double x1 = x0 + e1[3 * (long long)k + a], x2 = x0 + e2[3 * (long long)k + a];
        o[a] = fmin(x0, fmin(x1, x2));
        o[3 + a] = fmax(x0, fmax(x1, x2));
    }
    int node = parent[k];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&flags[node - n], 1) == 0) return;
        int a = child[2 * (long long)(node - n)], b = child[2 * (long long)(node - n) + 1];
        em[node] = __ldcg(em + a) + __ldcg(em + b) + (count[node] > LEAF_MAX ? 1 : 0);
        const double* ca = dbox + 6 * (long long)a;
        const double* cb = dbox + 6 * (long long)b;
        double* q = dbox + 6 * (long long)node;
        for (int m = 0; m < 3; ++m) {
            q[m] = fmin(__ldcg(ca + m), __ldcg(cb + m));
            q[3 + m] = fmax(__ldcg(ca + 3 + m), __ldcg(cb + 3 + m));
        }
        node = parent[node];
    }
}

}  // namespace rt

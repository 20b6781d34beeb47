// bvh_ploc.cuh — PLOC tree builder (Meister & Bittner 2018, parallel locally-
// ordered clustering) over the Morton-sorted primitives.
//
// Every iteration each cluster finds its nearest neighbour (smallest surface
// area of the union box) within +-PLOC_R positions in Morton order; mutual
// nearest neighbours merge into a new internal node; the cluster array is
// compacted and the loop repeats until one cluster (the root) is left.  The
// result approaches SAH quality at LBVH-like build cost.  Leaves are then
// laid out in depth-first order so every subtree owns a contiguous triangle
// range, which lets subtrees of <= LEAF_MAX primitives collapse into leaves.
//
// Node ids: [0, N) leaves (Morton-sorted slot), [N, 2N-1) internal nodes.
#pragma once
#include "bvh_build.cuh"

namespace rt {

#ifndef RT_PLOC_R
#define RT_PLOC_R 24   // with isotropic Morton codes, C3 launch over 6 tx: r16 58.6, r24 58.1 ms (r32 worse on C3)
#endif
constexpr int PLOC_R = RT_PLOC_R;   // nearest-neighbour search radius in Morton order
constexpr int PLOC_BLOCK = 256;

__device__ inline float union_area(const float* a, const float* b) {
    float dx = fmaxf(a[3], b[3]) - fminf(a[0], b[0]);
    float dy = fmaxf(a[4], b[4]) - fminf(a[1], b[1]);
    float dz = fmaxf(a[5], b[5]) - fminf(a[2], b[2]);
    return dx * dy + dy * dz + dz * dx;
}

// leaf boxes in Morton order, initial cluster list, leaf counts
__global__ void k_ploc_init(int n, const int* sorted_idx, const float* pbox, float* nbox,
                            int* clusters, int* count, int* emitted) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const float* s = pbox + 6 * (long long)sorted_idx[k];
    for (int m = 0; m < 6; ++m) nbox[6 * (long long)k + m] = s[m];
    clusters[k] = k;
    count[k] = 1;
    emitted[k] = 0;
}

// The iteration kernels read the live cluster count C from device memory (the
// host only knows an upper bound between its occasional syncs).
__global__ void __launch_bounds__(PLOC_BLOCK) k_ploc_nn(const int* clusters, const int* dC,
                                                       const float* nbox, int* nn) {
    const int C = *dC;
    if ((int)(blockIdx.x * PLOC_BLOCK) >= C) return;
    __shared__ float sb[PLOC_BLOCK + 2 * PLOC_R][6];
    int base = blockIdx.x * PLOC_BLOCK;
    for (int k = threadIdx.x; k < PLOC_BLOCK + 2 * PLOC_R; k += blockDim.x) {
        int c = base - PLOC_R + k;
        if (c >= 0 && c < C) {
            const float* b = nbox + 6 * (long long)clusters[c];
            for (int m = 0; m < 6; ++m) sb[k][m] = b[m];
        }
    }
    __syncthreads();
    int i = base + threadIdx.x;
    if (i >= C) return;
    const float* me = sb[threadIdx.x + PLOC_R];
    float best = INFINITY;
    int bj = -1;
    for (int d = -PLOC_R; d <= PLOC_R; ++d) {
        int j = i + d;
        if (d == 0 || j < 0 || j >= C) continue;
        float a = union_area(me, sb[threadIdx.x + PLOC_R + d]);
        if (a < best) { best = a; bj = j; }   // ascending j: ties keep the smaller index
    }
    nn[i] = bj;
}

__global__ void k_ploc_merge(const int* clusters, const int* dC, int Cmax, const int* nn, int n, float* nbox,
                             int* child, int* parent, int* count, int* emitted, int* counter, int* out,
                             int* valid) {
    const int C = *dC;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= C) {   // the scan runs over the host's bound Cmax
        if (i < Cmax) valid[i] = 0;
        return;
    }
    int j = nn[i];
    if (j >= 0 && nn[j] == i) {
        if (i < j) {
            int id = n + atomicAdd(counter, 1);
            int a = clusters[i], b = clusters[j];
            child[2 * (long long)(id - n)] = a;
            child[2 * (long long)(id - n) + 1] = b;
            parent[a] = id;
            parent[b] = id;
            count[id] = count[a] + count[b];
            // BNodes in the subtree once subtrees of <= LEAF_MAX prims become leaves
            emitted[id] = emitted[a] + emitted[b] + (count[id] > LEAF_MAX ? 1 : 0);
            const float* ba = nbox + 6 * (long long)a;
            const float* bb = nbox + 6 * (long long)b;
            float* o = nbox + 6 * (long long)id;
            for (int m = 0; m < 3; ++m) {
                o[m] = fminf(ba[m], bb[m]);
                o[3 + m] = fmaxf(ba[3 + m], bb[3 + m]);
            }
            out[i] = id;
            valid[i] = 1;
        } else {
            valid[i] = 0;
        }
    } else {
        out[i] = clusters[i];
        valid[i] = 1;
    }
}

// The last PLOC iterations (C <= PLOC_TAIL clusters) in one block: the same
// nearest-neighbour / mutual-merge / ordered-compaction rules as the
// k_ploc_nn -> k_ploc_merge -> scan -> k_ploc_compact loop, with block
// barriers instead of a host round trip per iteration.  Writes the root id.
constexpr int PLOC_TAIL = 2048;
constexpr int PLOC_TAIL_THREADS = 1024;
constexpr int PLOC_TAIL_SMEM = PLOC_TAIL * 6 * 4;   // dynamic shared memory of k_ploc_tail

__global__ void __launch_bounds__(PLOC_TAIL_THREADS) k_ploc_tail(const int* clusters_in, int C0, int n,
                                                                 float* nbox, int* child, int* parent,
                                                                 int* count, int* emitted, int* counter,
                                                                 int* root_out) {
    __shared__ int cl[2][PLOC_TAIL];
    __shared__ int nn[PLOC_TAIL];
    __shared__ int warp_sum[PLOC_TAIL_THREADS / 32];
    __shared__ int total;
    extern __shared__ float sbox[];   // [PLOC_TAIL][6]: the current clusters' boxes
    const int T = PLOC_TAIL_THREADS, PER = PLOC_TAIL / PLOC_TAIL_THREADS;
    int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < C0; i += T) cl[0][i] = clusters_in[i];
    int C = C0, cur = 0;
    __syncthreads();
    while (C > 1) {
        const int* c = cl[cur];
        for (int i = tid; i < C; i += T) {   // stage the boxes in shared memory
            const float* g = nbox + 6 * (long long)c[i];
            for (int k = 0; k < 6; ++k) sbox[6 * i + k] = g[k];
        }
        __syncthreads();
        for (int i = tid; i < C; i += T) {   // nearest neighbour within +-PLOC_R (k_ploc_nn)
            const float* m = sbox + 6 * i;
            float best = INFINITY;
            int bj = -1;
            for (int d = -PLOC_R; d <= PLOC_R; ++d) {
                int j = i + d;
                if (d == 0 || j < 0 || j >= C) continue;
                float a = union_area(m, sbox + 6 * j);
                if (a < best) { best = a; bj = j; }
            }
            nn[i] = bj;
        }
        __syncthreads();
        int out[PER], val[PER];
        for (int q = 0; q < PER; ++q) {   // mutual nearest neighbours merge (k_ploc_merge)
            int i = tid * PER + q;
            out[q] = 0;
            val[q] = 0;
            if (i >= C) continue;
            int j = nn[i];
            if (j >= 0 && nn[j] == i) {
                if (i < j) {
                    int id = n + atomicAdd(counter, 1);
                    int a = c[i], b = c[j];
                    child[2 * (long long)(id - n)] = a;
                    child[2 * (long long)(id - n) + 1] = b;
                    parent[a] = id;
                    parent[b] = id;
                    count[id] = count[a] + count[b];
                    emitted[id] = emitted[a] + emitted[b] + (count[id] > LEAF_MAX ? 1 : 0);
                    const float* ba = nbox + 6 * (long long)a;
                    const float* bb = nbox + 6 * (long long)b;
                    float* o = nbox + 6 * (long long)id;
                    for (int m = 0; m < 3; ++m) {
                        o[m] = fminf(ba[m], bb[m]);
                        o[3 + m] = fmaxf(ba[3 + m], bb[3 + m]);
                    }
                    out[q] = id;
                    val[q] = 1;
                }
            } else {
                out[q] = c[i];
                val[q] = 1;
            }
        }
        // ordered compaction: block exclusive scan of the keep flags
        int mine = 0;
        for (int q = 0; q < PER; ++q) mine += val[q];
        int incl = mine;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_sum[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            int v = lane < T / 32 ? warp_sum[lane] : 0;
            int w = v;
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            if (lane < T / 32) warp_sum[lane] = w - v;   // exclusive warp offsets
            if (lane == 31) total = w;
        }
        __syncthreads();
        int pos = warp_sum[wid] + incl - mine;
        int* nx = cl[cur ^ 1];
        for (int q = 0; q < PER; ++q)
            if (val[q]) nx[pos++] = out[q];
        __threadfence_block();
        __syncthreads();
        C = total;
        cur ^= 1;
        __syncthreads();
    }
    if (tid == 0) *root_out = cl[cur][0];
}

__global__ void k_ploc_compact(const int* out, const int* valid, const int* pos, const int* dC, int* next,
                               int* dC_next) {
    const int C = *dC;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < C && valid[i]) next[pos[i]] = out[i];
    if (i == C - 1) *dC_next = pos[i] + valid[i];
}

// depth-first triangle slot of every leaf: sum of left-sibling subtree sizes
// over the ancestors where the path comes from the right child
__global__ void k_ploc_slots(int n, const int* parent, const int* child, const int* count, const int* root_p,
                             int* slot) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int root = *root_p;
    int off = 0, node = k;
    while (node != root) {
        int p = parent[node];
        int l = child[2 * (long long)(p - n)];
        if (l != node) off += count[l];
        node = p;
    }
    slot[k] = off;
}

__device__ inline int ploc_first_slot(int node, int n, const int* child, const int* slot) {
    while (node >= n) node = child[2 * (long long)(node - n)];
    return slot[node];
}

__device__ inline int ploc_map(int id, int n, int root) {   // internal id -> BNode index, root -> 0
    int q = id - n;
    if (id == root) return 0;
    if (q == 0) return root - n;
    return q;
}

// Depth-first (near-left) BNode order: an emitted node's index is the number of
// emitted nodes before it in preorder = its proper ancestors + the emitted
// nodes of every left sibling subtree on the way up.  Parent and left child are
// then adjacent in memory (same 128-byte line half the time).  -1 = collapsed.
__global__ void k_ploc_dfs(int n, const int* root_p, const int* parent, const int* child, const int* count,
                           const int* emitted, int* dfs, int* max_depth) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n - 1) return;
    const int root = *root_p;
    int id = n + q;
    if (id != root && count[id] <= LEAF_MAX) { dfs[q] = -1; return; }
    int idx = 0, node = id, depth = 0;
    while (node != root) {
        int p = parent[node];
        int l = child[2 * (long long)(p - n)];
        idx += 1;
        ++depth;
        if (l != node) idx += emitted[l];
        node = p;
    }
    dfs[q] = idx;
    atomicMax(max_depth, depth);   // BNode depth (root 0): bounds the traversal stack
}

__global__ void k_ploc_layout(int n, const int* root_p, const int* child, const int* count, const int* slot,
                              const float* nbox, const unsigned* cbounds, const int* dfs, BNode* out) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n - 1) return;
    const int root = *root_p;
    int id = n + q;
    if (dfs && dfs[q] < 0) return;   // collapsed into a leaf of its parent
    float eps = box_eps(cbounds);
    float bx[2][6];
    int ref[2];
    for (int c = 0; c < 2; ++c) {
        int ch = child[2 * (long long)q + c];
        const float* src = nbox + 6 * (long long)ch;
        for (int m = 0; m < 6; ++m) bx[c][m] = src[m];
        inflate6(bx[c], eps);
        if (ch < n) ref[c] = make_leaf(slot[ch], 1);
        else if (count[ch] <= LEAF_MAX) ref[c] = make_leaf(ploc_first_slot(ch, n, child, slot), count[ch]);
        else ref[c] = dfs ? dfs[ch - n] : ploc_map(ch, n, root);
    }
    out[dfs ? dfs[q] : ploc_map(id, n, root)] = pack_bnode(bx, ref[0], ref[1]);
}

// the root's parent is -1 (the refit and slot climbs stop there)
__global__ void k_root_parent(const int* root_p, int* parent) { parent[*root_p] = -1; }

// ---- origin skip table ------------------------------------------------------------------
//
// A secondary ray starts ON the prim P it reflected off and leaves to one side
// of P's plane.  Every subtree whose exact box lies in the closed half-space
// on the other side holds no point the ray reaches at t > t_min, yet the FP32
// filter (boxes inflated ~2e-3 m at C3 scale) walks the ray down into the very
// building it leaves: 3 extra node visits and 1.2 extra triangle tests per
// secondary bounce.  Per prim and side the table holds the child ref of the
// highest ancestor of P's leaf that lies entirely behind P's plane (exact FP64
// boxes, margin SKIP_MARGIN); the traversal treats that child as a miss.

constexpr double SKIP_MARGIN = 1e-7;   // m: >> rounding, the 1e-12 barycentric slack of km-sized triangles

// Exact FP64 boxes of the tree nodes (PLOC ids): leaf k = corners v0, v0 + e1,
// v0 + e2 of prim sorted_idx[k]; internal nodes bottom-up (second arrival).
__global__ void k_dbox_refit(int n, const int* sorted_idx, const double* v0, const double* e1,
                             const double* e2, const int* parent, const int* child, double* dbox,
                             int* flags) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int p = sorted_idx[k];
    double* o = dbox + 6 * (long long)k;
    for (int a = 0; a < 3; ++a) {
        double x0 = v0[3 * (long long)p + a];
        double x1 = x0 + e1[3 * (long long)p + a], x2 = x0 + e2[3 * (long long)p + a];
        o[a] = fmin(x0, fmin(x1, x2));
        o[3 + a] = fmax(x0, fmax(x1, x2));
    }
    int node = parent[k];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&flags[node - n], 1) == 0) return;
        const double* ca = dbox + 6 * (long long)child[2 * (long long)(node - n)];
        const double* cb = dbox + 6 * (long long)child[2 * (long long)(node - n) + 1];
        double* q = dbox + 6 * (long long)node;
        for (int a = 0; a < 3; ++a) {
            q[a] = fmin(__ldcg(ca + a), __ldcg(cb + a));
            q[3 + a] = fmax(__ldcg(ca + 3 + a), __ldcg(cb + 3 + a));
        }
        node = parent[node];
    }
}

// one thread per leaf: skip[2 p + s] for prim p, s = 1 for rays leaving to the
// side the stored normal points to, 0 for the other (EMPTY_REF = nothing)
__global__ void k_skip_table(int n, const int* root_p, const int* sorted_idx, const int* parent,
                             const int* child, const int* count, const int* slot, const int* dfs,
                             const double* dbox, const double* nrm, const double* poff, int* skip) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int root = *root_p;
    int p = sorted_idx[k];
    double nx = nrm[3 * (long long)p], ny = nrm[3 * (long long)p + 1], nz = nrm[3 * (long long)p + 2];
    double c = poff[p];
    for (int s = 0; s < 2; ++s) {
        double sg = s ? 1.0 : -1.0;   // the side the ray goes to: sg (n.x - c) > 0
        int best = EMPTY_REF;
        int node = k;
        while (node != root) {
            // largest sg (n.x - c) over the box corners must stay <= margin
            const double* b = dbox + 6 * (long long)node;
            double m = sg * nx > 0 ? b[3] * nx : b[0] * nx;
            m += sg * ny > 0 ? b[4] * ny : b[1] * ny;
            m += sg * nz > 0 ? b[5] * nz : b[2] * nz;
            if (sg * (m - c) > SKIP_MARGIN) break;
            int par = parent[node];
            int cnt = node < n ? 1 : count[node];
            if (cnt > LEAF_MAX) best = dfs[node - n];                                  // a BNode
            else if (count[par] > LEAF_MAX) best = make_leaf(ploc_first_slot(node, n, child, slot), cnt);
            node = par;
        }
        skip[2 * (long long)p + s] = best;
    }
}

// Surface-area cost of the laid-out tree (diagnostic, reported by the bench):
// sums[0] = sum of internal-child box areas, sums[1] = sum of leaf box area x
// triangle count, sums[2] = root area; expected internal-node visits of a
// random ray ~ 1 + sums[0] / sums[2], expected triangle tests ~ sums[1] / sums[2].
__device__ inline void tree_sah_node(const BNode* nodes, int q, double& in, double& lf, double* sums);

__global__ void __launch_bounds__(256) k_tree_sah(const BNode* nodes, int n_nodes, double* sums) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    __shared__ double part[2][8];
    double in = 0.0, lf = 0.0;
    if (q < n_nodes) tree_sah_node(nodes, q, in, lf, sums);
    for (int o = 16; o; o >>= 1) {   // one atomic pair per block, not per node
        in += __shfl_xor_sync(0xffffffffu, in, o);
        lf += __shfl_xor_sync(0xffffffffu, lf, o);
    }
    if ((threadIdx.x & 31) == 0) { part[0][threadIdx.x >> 5] = in; part[1][threadIdx.x >> 5] = lf; }
    __syncthreads();
    if (threadIdx.x < 2) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[threadIdx.x][w];
        atomicAdd(sums + threadIdx.x, s);
    }
}

__device__ inline void tree_sah_node(const BNode* nodes, int q, double& in, double& lf, double* sums) {
    BNode nd = nodes[q];
    float b[2][6];
    unpack_bnode(nd, 0, b[0]);
    unpack_bnode(nd, 1, b[1]);
    int ref[2] = {nd.d.x, nd.d.y};
    for (int c = 0; c < 2; ++c) {
        double dx = b[c][3] - b[c][0], dy = b[c][4] - b[c][1], dz = b[c][5] - b[c][2];
        double sa = dx * dy + dy * dz + dz * dx;
        if (ref_is_leaf(ref[c])) lf += sa * leaf_count(ref[c]);
        else in += sa;
    }
    if (q == 0) {
        double lx = fmin(b[0][0], b[1][0]), ly = fmin(b[0][1], b[1][1]), lz = fmin(b[0][2], b[1][2]);
        double hx = fmax(b[0][3], b[1][3]), hy = fmax(b[0][4], b[1][4]), hz = fmax(b[0][5], b[1][5]);
        double dx = hx - lx, dy = hy - ly, dz = hz - lz;
        sums[2] = dx * dy + dy * dz + dz * dx;
    }
}

__global__ void k_ploc_tris(int n, const int* sorted_idx, const int* slot, const double* v0,
                            const double* e1, const double* e2, TriRec* tris) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int p = sorted_idx[k];
    TriRec t;
    t.v0x = v0[3 * p]; t.v0y = v0[3 * p + 1]; t.v0z = v0[3 * p + 2];
    t.e1x = e1[3 * p]; t.e1y = e1[3 * p + 1]; t.e1z = e1[3 * p + 2];
    t.e2x = e2[3 * p]; t.e2y = e2[3 * p + 1]; t.e2z = e2[3 * p + 2];
    t.prim = p;
    t.pad = 0;
    tris[slot[k]] = t;
}

}  // namespace rt

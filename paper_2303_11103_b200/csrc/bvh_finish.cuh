// bvh_finish.cuh — the post-hierarchy passes of a small SAH build in one CTA.
//
// After the hierarchy (bvh_sah.cuh) the build runs eight per-element passes
// (emitted-node counts, depth-first triangle slots, BNode order, layout, exact
// FP64 refit, origin skip table, triangle records), most of them climbs from
// a leaf to the root over parent links in global memory: ~95 us of device
// time and eight launches for the 2,002-tri canyon, each climb step an L2
// round trip.  For n <= FIN_MAX the same passes run in one CTA with the tree
// links (parent, child, count, emitted, slot, dfs) in shared memory, phases
// separated by __syncthreads; the results are identical (same arithmetic,
// same orders), written back for the rest of the library.
#pragma once
#include "bvh_ploc.cuh"

namespace rt {

constexpr int FIN_MAX = 4096;

// A box (6 doubles) by CTA-scope loads: coherent through the SM's L1 for data
// other threads of this CTA stored before a fence.cta (volatile loads would go
// to L2 on every climb step); one asm block, so the six loads issue together
__device__ __forceinline__ void ld_box_cta(const double* p, double* b) {
    asm volatile(
        "ld.relaxed.cta.global.f64 %0, [%6];\n\t"
        "ld.relaxed.cta.global.f64 %1, [%6+8];\n\t"
        "ld.relaxed.cta.global.f64 %2, [%6+16];\n\t"
        "ld.relaxed.cta.global.f64 %3, [%6+24];\n\t"
        "ld.relaxed.cta.global.f64 %4, [%6+32];\n\t"
        "ld.relaxed.cta.global.f64 %5, [%6+40];"
        : "=d"(b[0]), "=d"(b[1]), "=d"(b[2]), "=d"(b[3]), "=d"(b[4]), "=d"(b[5])
        : "l"(p)
        : "memory");
}
constexpr int FIN_THREADS = 1024;
// shared ints: parent / count / emitted [2n - 1] each, child [2n - 2], slot [n], dfs / flags [n - 1]
__host__ __device__ constexpr size_t fin_smem_bytes(int n) { return sizeof(int) * (11ull * n + 8); }

__global__ void __launch_bounds__(FIN_THREADS, 1)
k_finish_small(int n, const int* __restrict__ root_p, const int* __restrict__ sidx, int* g_par,
               const int* __restrict__ g_child, const int* __restrict__ g_cnt, int* g_em, int* g_slot,
               int* g_dfs, int* g_dmax, const float* __restrict__ nbox, const unsigned* __restrict__ cbounds,
               BNode* nodes, double* dbox, const double* __restrict__ v0, const double* __restrict__ e1,
               const double* __restrict__ e2, const double* __restrict__ nrm,
               const double* __restrict__ poff, int* skip, TriRec* tris) {
    extern __shared__ int fin_smem[];
    const int N = 2 * n - 1;          // node ids: leaves [0, n), internal [n, 2n - 1)
    int* par = fin_smem;              // [N]
    int* cnt = par + N;               // [N]
    volatile int* em = cnt + N;       // [N]
    int* ch = const_cast<int*>(em) + N;   // [2 (n - 1)]
    int* slot = ch + 2 * (n - 1);     // [n]
    int* dfs = slot + n;              // [n - 1]
    int* flags = dfs + (n - 1);       // [n - 1]
    __shared__ int s_dmax;
    const int tid = threadIdx.x, T = blockDim.x;
    const int root = *root_p;
    for (int i = tid; i < N; i += T) {
        par[i] = g_par[i];
        cnt[i] = g_cnt[i];
        em[i] = 0;
    }
    for (int i = tid; i < 2 * (n - 1); i += T) ch[i] = g_child[i];
    for (int i = tid; i < n - 1; i += T) flags[i] = 0;
    if (tid == 0) { s_dmax = 0; par[root] = -1; }
    __syncthreads();
    // 1. emitted BNodes per subtree (k_sah_emitted): second arrival computes
    for (int k = tid; k < n; k += T) {
        int node = par[k];
        while (node >= 0) {
            __threadfence_block();
            if (atomicAdd(&flags[node - n], 1) == 0) break;
            __threadfence_block();
            int a = ch[2 * (node - n)], b = ch[2 * (node - n) + 1];
            em[node] = em[a] + em[b] + (cnt[node] > LEAF_MAX ? 1 : 0);
            node = par[node];
        }
    }
    __syncthreads();
    // 2. depth-first triangle slot of every leaf (k_ploc_slots)
    for (int k = tid; k < n; k += T) {
        int off = 0, node = k;
        while (node != root) {
            int p = par[node];
            int l = ch[2 * (p - n)];
            if (l != node) off += cnt[l];
            node = p;
        }
        slot[k] = off;
    }
    // 3. depth-first BNode index of every emitted node (k_ploc_dfs)
    for (int q = tid; q < n - 1; q += T) {
        int id = n + q;
        if (id != root && cnt[id] <= LEAF_MAX) { dfs[q] = -1; continue; }
        int idx = 0, node = id, depth = 0;
        while (node != root) {
            int p = par[node];
            int l = ch[2 * (p - n)];
            idx += 1;
            ++depth;
            if (l != node) idx += em[l];
            node = p;
        }
        dfs[q] = idx;
        atomicMax(&s_dmax, depth);
    }
    for (int q = tid; q < n - 1; q += T) flags[q] = 0;
    __syncthreads();
    // 4. BNode layout (k_ploc_layout)
    const float eps = box_eps(cbounds);
    for (int q = tid; q < n - 1; q += T) {
        if (dfs[q] < 0) continue;
        float bx[2][6];
        int ref[2];
        for (int c = 0; c < 2; ++c) {
            int chd = ch[2 * q + c];
            const float* src = nbox + 6 * (long long)chd;
            for (int m = 0; m < 6; ++m) bx[c][m] = src[m];
            inflate6(bx[c], eps);
            if (chd < n) {
                ref[c] = make_leaf(slot[chd], 1);
            } else if (cnt[chd] <= LEAF_MAX) {
                int f = chd;
                while (f >= n) f = ch[2 * (f - n)];
                ref[c] = make_leaf(slot[f], cnt[chd]);
            } else {
                ref[c] = dfs[chd - n];
            }
        }
        nodes[dfs[q]] = pack_bnode(bx, ref[0], ref[1]);
    }
    // 5. exact FP64 boxes (k_dbox_refit): leaves, then the second arrival climbs
    for (int k = tid; k < n; k += T) {
        int p = sidx[k];
        double* o = dbox + 6 * (long long)k;
        for (int a = 0; a < 3; ++a) {
            double x0 = v0[3 * (long long)p + a];
            double x1 = x0 + e1[3 * (long long)p + a], x2 = x0 + e2[3 * (long long)p + a];
            o[a] = fmin(x0, fmin(x1, x2));
            o[3 + a] = fmax(x0, fmax(x1, x2));
        }
        int node = par[k];
        while (node >= 0) {
            __threadfence_block();
            if (atomicAdd(&flags[node - n], 1) == 0) break;
            __threadfence_block();
            double ca[6], cb[6];
            ld_box_cta(dbox + 6 * (long long)ch[2 * (node - n)], ca);
            ld_box_cta(dbox + 6 * (long long)ch[2 * (node - n) + 1], cb);
            double* qb = dbox + 6 * (long long)node;
            for (int a = 0; a < 3; ++a) {
                qb[a] = fmin(ca[a], cb[a]);
                qb[3 + a] = fmax(ca[3 + a], cb[3 + a]);
            }
            node = par[node];
        }
    }
    __syncthreads();
    // 6. origin skip table (k_skip_table) and 7. triangle records (k_ploc_tris)
    for (int k = tid; k < n; k += T) {
        int p = sidx[k];
        double nx = nrm[3 * (long long)p], ny = nrm[3 * (long long)p + 1], nz = nrm[3 * (long long)p + 2];
        double c = poff[p];
        for (int s = 0; s < 2; ++s) {
            double sg = s ? 1.0 : -1.0;
            int best = EMPTY_REF;
            int node = k;
            while (node != root) {
                const double* b = dbox + 6 * (long long)node;
                double m = sg * nx > 0 ? b[3] * nx : b[0] * nx;
                m += sg * ny > 0 ? b[4] * ny : b[1] * ny;
                m += sg * nz > 0 ? b[5] * nz : b[2] * nz;
                if (sg * (m - c) > SKIP_MARGIN) break;
                int pr = par[node];
                int cn = node < n ? 1 : cnt[node];
                if (cn > LEAF_MAX) {
                    best = dfs[node - n];
                } else if (cnt[pr] > LEAF_MAX) {
                    int f = node;
                    while (f >= n) f = ch[2 * (f - n)];
                    best = make_leaf(slot[f], cn);
                }
                node = pr;
            }
            skip[2 * (long long)p + s] = best;
        }
        TriRec t;
        t.v0x = v0[3 * p]; t.v0y = v0[3 * p + 1]; t.v0z = v0[3 * p + 2];
        t.e1x = e1[3 * p]; t.e1y = e1[3 * p + 1]; t.e1z = e1[3 * p + 2];
        t.e2x = e2[3 * p]; t.e2y = e2[3 * p + 1]; t.e2z = e2[3 * p + 2];
        t.prim = p;
        t.pad = 0;
        tris[slot[k]] = t;
    }
    // the links the rest of the library reads
    for (int i = tid; i < N; i += T) g_em[i] = em[i];
    for (int k = tid; k < n; k += T) g_slot[k] = slot[k];
    for (int q = tid; q < n - 1; q += T) g_dfs[q] = dfs[q];
    if (tid == 0) {
        g_par[root] = -1;
        *g_dmax = s_dmax;
    }
}

}  // namespace rt

// launch.cuh — Fibonacci ray launch with on-device candidate trie.
//
// Replaces launch_candidates (tracer.py:217-244) and fibonacci_directions
// (geometry.py:62-76).  Each thread owns one ray: up to max_depth closest
// hits (t_min = RAY_EPS, t_max = inf), normal flipped to face the ray, point
// o + t*d, specular d <- d - 2(d.n)n, all with the reference's FP64 operation
// order.  The set of every prefix of every ray's hit sequence is kept as a
// trie in a global open-addressing hash table keyed (parent node, prim):
// node ids are allocated on first insert, so each unique prefix is one node.
// Warps aggregate identical keys with __match_any_sync before touching the
// table (neighbouring rays mostly hit the same triangles).
//
// Coherence: lattice index i = band * B + perm[slot % B] where perm sorts a
// band of B consecutive indices by azimuth; neighbouring threads therefore
// trace neighbouring directions.  The permutation is a bijection, so the
// set of rays (and the candidate set) is unchanged.
#pragma once
#include "trace.cuh"

namespace rt {

constexpr unsigned long long EMPTY_KEY = 0xFFFFFFFFFFFFFFFFULL;

// Open-addressing table of trie edges.  A node IS its table slot: the node
// for prefix (parent node, prim) lives in the slot holding that key and its
// id is slot + 1 (0 = root, the empty prefix).  Slots are written once (CAS
// from EMPTY), so an insert needs no id counter and no value publication:
// the id is known as soon as the key is found or placed.  The node's parent
// and prim are the key's halves, so the sequences are recovered from the
// keys alone (k_trie_sequences).
struct Trie {
    unsigned long long* keys;   // [cap]
    unsigned mask;              // cap - 1
    int* counter;               // occupied slots (load factor -> growth)
    int* overflow;              // a probe sequence ran out of slots: relaunch
};

// slot hash of a trie edge: 32-bit multiply-xorshift mixing of both halves
// (the 64-bit murmur finaliser cost ~15 instructions per insert; measured
// probe lengths are unchanged at the table's <= 1/2 load)
__device__ inline unsigned hash_edge(unsigned parent, unsigned prim) {
    unsigned h = parent * 0x9E3779B1u ^ (prim + 0x7F4A7C15u) * 0x85EBCA77u;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 13;
    return h;
}

// insert-or-get (parent, prim) -> node id (>= 1); -1 when the table is full
__device__ int trie_insert(const Trie& T, int parent, int prim) {
    unsigned long long key = ((unsigned long long)(unsigned)parent << 32) | (unsigned)prim;
    unsigned h = hash_edge((unsigned)parent, (unsigned)prim) & T.mask;
    for (unsigned probe = 0; probe <= T.mask; ++probe) {
        // write-once slots: a cached read is current or a stale EMPTY, and a
        // stale EMPTY only sends us to the CAS, which returns the truth
        unsigned long long k = __ldca(T.keys + h);
        if (k == key) return (int)h + 1;
        if (k == EMPTY_KEY) {
            k = atomicCAS(T.keys + h, EMPTY_KEY, key);
            if (k == EMPTY_KEY) {
                atomicAdd(T.counter, 1);
                return (int)h + 1;
            }
            if (k == key) return (int)h + 1;
        }
        h = (h + 1) & T.mask;
    }
    atomicExch(T.overflow, 1);
    return -1;
}

// Kept under 128 bytes on purpose: nvcc 12.9 stops scalarising a larger
// by-value kernel parameter and then (observed on this kernel) forwarded the
// initial origin P.tx into the bounce loop's o.x update — wrong third-bounce
// origins.  The counters therefore live behind one pointer.
struct LaunchParams {
    double tx, ty, tz;
    long long n_rays, slot_begin, slot_end;
    long long shard_unit;     // sharded launch: local slot l -> global unit (l/unit)*count+index
                              // (a power of two: shard_shift = log2 unit)
    int shard_index, shard_count;
    int max_depth;
    int band;                 // B (a power of two); 0 disables the permutation
    int band_shift;           // log2 B
    int shard_shift;
    const int* perm;          // [B]
    const double* dirs;       // optional [n_rays*3]
    const double* normals;    // [n_prims*3] global order
    // [0] ray-bounces; COUNT builds: [1] node visits, [2] triangle tests, [3]
    // reserved (dynamic slot counter), [4] warp iterations of the bounce loop,
    // [5] sum over them of the warp's max node visits, [6] node visits had
    // t_max been the hit's t (RT_ORACLE_VISITS experiment)
    unsigned long long* stats;
    int* error;
};
static_assert(sizeof(LaunchParams) <= 128, "see the LaunchParams comment");

// geometry.py:70-76 for one index (on-device sin/cos; see DESIGN.md on ulps)
__device__ inline d3 fib_dir(long long i, long long n) {
    double di = (double)i;
    double z = 1.0 - (2.0 * di + 1.0) / (double)n;
    const double golden_sq = 2.618033988749895;   // (3 + sqrt 5) / 2 in double
    double phi = (2.0 * PI) * di / golden_sq;
    double r = sqrt(fmax(0.0, 1.0 - z * z));
    double s, c;
    sincos(phi, &s, &c);
    return d3{r * c, r * s, z};
}

template <bool COUNT>
#ifndef RT_LAUNCH_BLOCK
#define RT_LAUNCH_BLOCK 256
#endif
#ifndef RT_LAUNCH_MINB
#define RT_LAUNCH_MINB 4   // 64 registers (92 B spill), 32 warps per SM: C3 launch 22.75 vs 23.37 ms (minB 3), 26.9 (minB 5)
#endif
__global__ void __launch_bounds__(RT_LAUNCH_BLOCK, RT_LAUNCH_MINB) k_launch(Bvh bvh, LaunchParams P, Trie T) {
    const unsigned FULL = 0xffffffffu;
    int lane = threadIdx.x & 31;
    unsigned my_bounces = 0;   // <= iterations x max_depth per thread
    unsigned long long my_nodes = 0, my_tris = 0, my_wb = 0, my_wv = 0;
    long long stride = (long long)gridDim.x * blockDim.x;
    long long span = P.slot_end - P.slot_begin;
    long long iters = (span + stride - 1) / stride;
    const d3 tx = d3{P.tx, P.ty, P.tz};
    for (long long it = 0; it < iters; ++it) {
        long long slot = P.slot_begin + it * stride + blockIdx.x * (long long)blockDim.x + threadIdx.x;
        bool active = slot < P.slot_end;
        if (P.shard_count > 1) {   // band-interleaved shard (rt_launch_shard)
            long long lu = slot >> P.shard_shift;
            slot = ((lu * P.shard_count + P.shard_index) << P.shard_shift) + (slot & (P.shard_unit - 1));
            active = active && slot < P.n_rays;
        }
        d3 o = tx, d = d3{0, 0, 0};
        if (active) {
            long long i = slot;
            if (P.band > 0) {   // B is a power of two: shift and mask, no 64-bit division
                long long b = slot >> P.band_shift;
                if ((b + 1) * P.band <= P.n_rays) i = (b << P.band_shift) + P.perm[slot & (P.band - 1)];
            }
            d = P.dirs ? ld3(P.dirs + 3 * i) : fib_dir(i, P.n_rays);
        }
        int parent = 0;
        int skip = EMPTY_REF;   // the subtree behind the wall the ray leaves (trace.cuh origin_skip)
        for (int k = 0; k < P.max_depth; ++k) {
            int prim = -1;
            double t = 0.0;
            int nv = 0, nt = 0;
            if (COUNT && __ballot_sync(FULL, active) == 0) break;
            if (active) {
                Ray r = make_ray(o, d);
                if (COUNT) {
                    prim = trace_ray<false>(bvh, r, RAY_EPS, __longlong_as_double(0x7ff0000000000000LL), &t,
                                            &nv, &nt, nullptr, skip);
                    my_nodes += nv;
                    my_tris += nt;
#ifdef RT_ORACLE_VISITS
                    if (prim >= 0) {   // visits if t_max were known in advance
                        int nv2 = 0, nt2 = 0;
                        double t2;
                        trace_ray<false>(bvh, r, RAY_EPS, t * (1.0 + 1e-9), &t2, &nv2, &nt2);
                        atomicAdd(P.stats + 6, (unsigned long long)nv2);
                    } else {
                        atomicAdd(P.stats + 6, (unsigned long long)nv);
                    }
#endif
                } else {
                    prim = trace_ray<false>(bvh, r, RAY_EPS, __longlong_as_double(0x7ff0000000000000LL), &t,
                                            nullptr, nullptr, nullptr, skip);
                }
                ++my_bounces;
                if (prim == -2) { atomicOr(P.error, 1); prim = -1; }
                if (prim < 0) active = false;
            }
            if (COUNT) {
                int mx = __reduce_max_sync(FULL, nv);
                if (lane == 0) { ++my_wb; my_wv += mx; }
            }
            unsigned amask = __ballot_sync(FULL, active);
            if (amask == 0) break;
            if (active) {
                unsigned long long key = ((unsigned long long)(unsigned)parent << 32) | (unsigned)prim;
                unsigned peers = __match_any_sync(amask, key);
                int leader = __ffs(peers) - 1;
                int id = 0;
#ifndef RT_NO_TRIE
                if (lane == leader) id = trie_insert(T, parent, prim);
#else
                id = 1;   // timing experiment only: traversal without candidate bookkeeping
#endif
                id = __shfl_sync(peers, id, leader);
                if (id < 0) { active = false; }
                parent = id;
                // Bvh.intersect normal orientation (bvh.py:98-100), hit point (:101)
                d3 n = ld3(P.normals + 3 * (long long)prim);
                bool flip = dot_blas(n, d) > 0.0;
                if (flip) n = d3{-n.x, -n.y, -n.z};
                d3 pt = d3{o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
                // tracer.py:242-243
                double kk = 2.0 * dot_blas(d, n);
                d = d3{d.x - kk * n.x, d.y - kk * n.y, d.z - kk * n.z};
                o = pt;
                // the reflected ray leaves to the side of the facing normal: n_f . d_new = -kk / 2
                skip = origin_skip(bvh, prim, flip ? 0.5 * kk : -0.5 * kk);
            }
        }
    }
    // warp-reduce the bounce count
    for (int s = 16; s; s >>= 1) my_bounces += __shfl_xor_sync(FULL, my_bounces, s);
    if (lane == 0 && my_bounces) atomicAdd(P.stats + 0, (unsigned long long)my_bounces);
    if (COUNT) {
        for (int s = 16; s; s >>= 1) {
            my_nodes += __shfl_xor_sync(FULL, my_nodes, s);
            my_tris += __shfl_xor_sync(FULL, my_tris, s);
        }
        if (lane == 0) {
            atomicAdd(P.stats + 1, my_nodes);
            atomicAdd(P.stats + 2, my_tris);
            atomicAdd(P.stats + 4, my_wb);
            atomicAdd(P.stats + 5, my_wv);
        }
    }
}

// ---- candidate materialization ----------------------------------------------------------

// every occupied slot (a trie node) -> one padded sequence row (row order is
// irrelevant: the rows are sorted next).  The key chain gives the prims from
// the node up to the root.
__global__ void k_trie_sequences(long long cap, const unsigned long long* keys, int max_len, int* seq,
                                 signed char* len, int* rows) {
    long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s >= cap) return;
    unsigned long long k = keys[s];
    if (k == EMPTY_KEY) return;
    int L = 1;
    for (unsigned long long c = k; (int)(c >> 32) != 0; c = keys[(int)(c >> 32) - 1]) ++L;
    int row = atomicAdd(rows, 1);
    int* out = seq + (long long)row * max_len;
    for (int j = L; j < max_len; ++j) out[j] = -1;
    unsigned long long c = k;
    for (int j = L - 1; j >= 0; --j) {
        out[j] = (int)(c & 0xffffffffu);
        int parent = (int)(c >> 32);
        if (parent) c = keys[parent - 1];
    }
    len[row] = (signed char)L;
}

// LSD radix passes over the digit columns: key of row perm[r] at column j
// (prim + 1, 0 = padding) or, for j == max_len, the sequence length.
// key of row perm[r] over digit columns j_lo..j_hi (j_lo most significant),
// W bits each (prim + 1, 0 past the row's length), with the row length above
// them when with_len: several LSD digits in one 64-bit radix sort
__global__ void k_digit_columns(long long n, const int* seq, const signed char* len, int max_len,
                                int j_lo, int j_hi, int W, int with_len, const int* perm,
                                unsigned long long* keys) {
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    long long row = perm[r];
    int ln = len[row];
    unsigned long long v = 0;
    for (int j = j_lo; j <= j_hi; ++j) {
        int p = seq[row * max_len + j];
        unsigned d = (j < ln && p >= 0) ? (unsigned)(p + 1) : 0u;
        v = (v << W) | d;
    }
    if (with_len) v |= (unsigned long long)ln << (W * (j_hi - j_lo + 1));
    keys[r] = v;
}

__global__ void k_flag_unique(long long n, const int* perm, const int* seq, const signed char* len,
                              int max_len, int* flag) {
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    int f = 1;
    if (r > 0) {
        long long a = perm[r], b = perm[r - 1];
        if (len[a] == len[b]) {
            f = 0;
            for (int j = 0; j < len[a]; ++j)
                if (seq[a * max_len + j] != seq[b * max_len + j]) { f = 1; break; }
        }
    }
    flag[r] = f;
}

__global__ void k_scatter_unique(long long n, const int* perm, const int* flag, const int* pos,
                                 const int* seq_in, const signed char* len_in, int max_len,
                                 int* seq_out, signed char* len_out) {
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n || !flag[r]) return;
    long long src = perm[r];
    long long dst = pos[r];
    int L = len_in[src];
    for (int j = 0; j < max_len; ++j)
        seq_out[dst * max_len + j] = j < L ? seq_in[src * max_len + j] : -1;
    len_out[dst] = (signed char)L;
}

// rows in sorted order (perm) when they are distinct already
__global__ void k_gather_rows(long long n, const int* perm, const int* seq_in, const signed char* len_in,
                              int max_len, int* seq_out, signed char* len_out) {
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= n) return;
    long long src = perm[r];
    int L = len_in[src];
    for (int j = 0; j < max_len; ++j) seq_out[r * max_len + j] = j < L ? seq_in[src * max_len + j] : -1;
    len_out[r] = (signed char)L;
}

// exhaustive enumeration (tracer.py:196-214) directly in (length, lex) order
__global__ void k_enumerate(long long total, int n, int max_depth, const long long* level_start,
                            int* seq, signed char* len) {
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= total) return;
    int L = 1;
    while (L < max_depth && r >= level_start[L]) ++L;
    long long local = r - level_start[L - 1];
    // digits: first in [0,n), later in [0,n-1) skipping the previous prim
    int digits[MAX_DEPTH];
    for (int k = L - 1; k >= 1; --k) { digits[k] = (int)(local % (n - 1)); local /= (n - 1); }
    digits[0] = (int)local;
    int prev = -1;
    for (int k = 0; k < max_depth; ++k) {
        int v = -1;
        if (k < L) {
            v = (k == 0) ? digits[0] : (digits[k] >= prev ? digits[k] + 1 : digits[k]);
            prev = v;
        }
        seq[r * max_depth + k] = v;
    }
    len[r] = (signed char)L;
}

}  // namespace rt

// b200rt.cu — the C ABI (include/b200rt.h) over the sm_100a kernels.
//
// One translation unit: the kernels live in the .cuh files included below.
// Built with --fmad=false (see rt_common.cuh) for sm_100a only.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/b200rt.h"
#include "api_kernels.cuh"
#include "bvh_build.cuh"
#include "bvh_ploc.cuh"
#include "bvh_sah.cuh"
#include "bvh_finish.cuh"
#include "cir.cuh"
#include "em_jvp.cuh"
#include "freq.cuh"
#include "microbench.cuh"
#include "launch.cuh"


#ifndef RT_DFS_LAYOUT
#define RT_DFS_LAYOUT 1   // depth-first BNode order for the PLOC tree (C3 launch: -0.5%)
#endif
#ifndef RT_BAND_C
// Coherence band B = pow2 >= sqrt(C n) (launch.cuh).  A warp takes 32 azimuth-
// sorted rays of one band: 32 * 2pi / B wide and 2B / n tall in (azimuth, z),
// square when B = sqrt(32 pi n).  Measured on C3 (launch ms): C = pi 24.3,
// 8 pi 23.5, 32 pi 23.5, 128 pi 24.5.
#define RT_BAND_C 100.53
#endif
#ifndef RT_SAH
#define RT_SAH 1   // top-down binned SAH (bvh_sah.cuh); 0 = RT_PLOC's choice
#endif
#ifndef RT_PLOC_TAIL
#define RT_PLOC_TAIL 1   // last PLOC iterations in one block (bvh_ploc.cuh k_ploc_tail)
#endif
#ifndef RT_OCC_HINTS
#define RT_OCC_HINTS 1   // occluder cache in k_validate (solve.cuh segments_clear_hinted)
#ifndef RT_DEFER_MIN_ITEMS
#define RT_DEFER_MIN_ITEMS (1LL << 23)   // fused solve + validation defers thin warps from this many items
#endif
#ifndef RT_SAH_WIDE_MIN
#define RT_SAH_WIDE_MIN 1024   // large scenes: medium SAH levels with ranges above ~this many prims use 1024-thread CTAs (C3 build 1.50 -> 1.43 ms)
#endif
#ifndef RT_SV_GRID
#define RT_SV_GRID 32   // fused solve + validation grid: blocks per SM (grid-stride loop)
#endif
#ifndef RT_FUSED_SV
#define RT_FUSED_SV 1    // solve + validation in one pass (solve.cuh k_solve_validate)
#endif
#endif
#include "solve.cuh"
#include "sort_small.cuh"

using namespace rt;

// profiling stages (rt_get_profile)
enum { ST_LAUNCH = 0, ST_CAND_SORT, ST_FOOTPRINT, ST_SOLVE, ST_VALIDATE, ST_REC_SORT, ST_MERGE,
       ST_LOS, ST_TRIE_SEQ, RT_NSTAGE_USED };
#define RT_NSTAGE 16

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* get() const { return static_cast<T*>(p); }
    cudaError_t reserve(size_t n) {
        if (n <= bytes && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t want = std::max<size_t>(n, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) bytes = want;
        return e;
    }
};

}  // namespace

struct rt_ctx {
    int device = 0;
    int n_sm = 148;
    std::string err;
    // scene (global gather order)
    int64_t n_prims = 0;
    DevBuf v0, e1, e2, nrm, poff, prim_mat, pbox, cent, cbounds;
    DevBuf up_verts, up_tris;          // device copies of host scene inputs (rt_scene_upload)
    DevBuf rx_up;                      // rt_paths' receivers when given in host memory
    cudaEvent_t up_ev = nullptr;       // host scene inputs consumed (waited for by rt_bvh_build)
    bool up_pending = false;
    // bvh
    DevBuf nodes, dbox, skip_tab, tris, sorted_idx, morton, morton_alt, idx_alt, child, flags;
    bool bvh_ready = false;
    int bvh_depth = -1;           // deepest BNode (root 0); -1 = not measured
    bool tail_smem_set = false;   // k_ploc_tail's dynamic shared memory opt-in done
    bool has_skip = false;        // origin skip table built with the tree (bvh_ploc.cuh)
    DevBuf tree_diag;             // [0] deepest BNode; doubles at +8: surface-area sums
    const int* diag_root_dev = nullptr;   // device root id of the last tree (SAH estimate)
    bool diag_pending = false;    // tree diagnostics not yet read back
    cudaEvent_t diag_ev = nullptr;  // end of the last build on the caller's stream
    // candidates
    DevBuf cand_seq, cand_len;
    int64_t n_cand = 0;
    bool cand_sorted = true;      // false after a sharded launch until rt_candidates_set
    int cand_max_len = 1;
    // launch scratch
    DevBuf t_keys, perm_band;
    int band_B = -1;
    uint64_t trie_cap = 0;
    // sort / unique scratch
    DevBuf s_seq, s_len, s_perm, s_perm_alt, s_keys, s_keys_alt, s_flag, s_pos;
    DevBuf cub_tmp;
    // solve scratch
    DevBuf hps, nhp, row0, seg_cand, seg_iy, seg_ix0, seg_cnt, item_off, occ_hint, chunk_seg;
    DevBuf images, fp, counts, scan, pending, recs, rkeys, rkeys_alt, ridx, ridx_alt, keep,
        losbuf, heads, pcounts, poffs, em_small, ctrs;
    uint64_t pending_cap = 0;
    uint64_t rec_cap = 0;     // record list capacity of the fused solve + validation
    // path table
    int64_t n_paths = 0;
    int path_L = 1;
    int64_t paths_max_rx = 0;   // most paths of one receiver in the last rt_paths
    DevBuf p_rx, p_cand, p_order, p_seq, p_verts, p_len, p_delay, p_kdep, p_karr, p_nrm, p_cos;
    // error flags + pinned host staging
    DevBuf dflag, probe;
    DevBuf adj;   // adjoint contributions [items * L] (rt_transfer_bwd)
    DevBuf gbase;   // rt_gains' per-(path, slant pair) coefficients [P*S*R*2]
    DevBuf gparam;  // rt_gains_h's uploaded parameter block
    DevBuf deferred;   // k_validate's deferred items (RT_VAL_DEFER)
    // PLOC builder scratch
    DevBuf pl_box, pl_count, pl_parent, pl_ca, pl_cb, pl_nn, pl_out, pl_valid, pl_pos, pl_slot, pl_em, pl_dfs;
    DevBuf sah_tasks;
    // CIR packing scratch (rt_cir_plan -> rt_cir_scatter)
    DevBuf cir_pair, cir_count, cir_off, cir_fill, cir_bucket, cir_slot, cir_first;
    int64_t cir_n = 0;
    int cir_ntx = 0, cir_nrx = 0;
    long long* hpin = nullptr;
    // profiling: per-stage CUDA events on the caller's stream + counters
    int prof = 0;
    cudaEvent_t ev[RT_NSTAGE][2] = {};
    bool ev_used[RT_NSTAGE] = {};
    long long counters[RT_NSTAGE] = {};
};

namespace {

inline cudaStream_t ST(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int fail(rt_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

#define CK(expr)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            return fail(ctx, _e == cudaErrorMemoryAllocation ? RT_ENOMEM : RT_ECUDA,       \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));              \
    } while (0)
#define CKL()                  \
    do {                       \
        ++ctx->counters[15];   \
        CK(cudaGetLastError()); \
    } while (0)
#define RC(expr)                  \
    do {                          \
        int _r = (expr);          \
        if (_r != RT_OK) return _r; \
    } while (0)

inline unsigned nblk(long long n, int bs) {
    return (unsigned)std::max<long long>(1, (n + bs - 1) / bs);
}

SceneDev scene_dev(rt_ctx* ctx) {
    SceneDev s;
    s.v0 = ctx->v0.get<double>();
    s.e1 = ctx->e1.get<double>();
    s.e2 = ctx->e2.get<double>();
    s.nrm = ctx->nrm.get<double>();
    s.poff = ctx->poff.get<double>();
    s.prim_mat = ctx->prim_mat.get<int>();
    s.n = (int)ctx->n_prims;
    return s;
}

rt::Bvh bvh_dev(rt_ctx* ctx) {
    rt::Bvh b;
    b.nodes = ctx->nodes.get<BNode>();
    b.tris = ctx->tris.get<TriRec>();
    b.n_prims = (int)ctx->n_prims;
    b.origin_limit = reinterpret_cast<const double*>(ctx->cbounds.get<char>() + 32);
    b.skip = ctx->has_skip ? ctx->skip_tab.get<int>() : nullptr;
    b.err = reinterpret_cast<int*>(ctx->dflag.get<long long>());
    return b;
}

Cands cands_dev(rt_ctx* ctx) {
    Cands c;
    c.seq = ctx->cand_seq.get<int>();
    c.len = ctx->cand_len.get<signed char>();
    c.max_len = ctx->cand_max_len;
    c.n = ctx->n_cand;
    return c;
}

// copy n 8-byte words device -> pinned host, synchronizing the stream
int fetch(rt_ctx* ctx, const void* dev, int n, cudaStream_t st) {
    CK(cudaMemcpyAsync(ctx->hpin, dev, sizeof(long long) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return RT_OK;
}

int clear_flags(rt_ctx* ctx, cudaStream_t st) {
    CK(cudaMemsetAsync(ctx->dflag.p, 0, sizeof(long long), st));
    return RT_OK;
}

int flags_status(rt_ctx* ctx, long long f) {
    if (f & 1) return fail(ctx, RT_ECUDA, "BVH traversal stack overflow");
    if (f & 4) return fail(ctx, RT_ECOINCIDE, "transmitter and probe/receiver coincide");
    return RT_OK;
}

int check_flags(rt_ctx* ctx, cudaStream_t st) {
    RC(fetch(ctx, ctx->dflag.p, 1, st));
    return flags_status(ctx, ctx->hpin[0]);
}

// n 8-byte words -> hpin[0..n) and the error word -> hpin[n], one host sync
int fetch_and_flags(rt_ctx* ctx, const void* dev, int n, cudaStream_t st) {
    CK(cudaMemcpyAsync(ctx->hpin, dev, sizeof(long long) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ctx->hpin + n, ctx->dflag.p, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return flags_status(ctx, ctx->hpin[n]);
}

void prof_mark(rt_ctx* ctx, int stage, int end, cudaStream_t st) {
    if (!(ctx->prof & 1)) return;
    if (!ctx->ev[stage][end]) cudaEventCreate(&ctx->ev[stage][end]);
    cudaEventRecord(ctx->ev[stage][end], st);
    if (end) ctx->ev_used[stage] = true;
}
#define PROF_BEGIN(i) prof_mark(ctx, (i), 0, st)
#define PROF_END(i) prof_mark(ctx, (i), 1, st)

int bits_for(long long v) {
    int b = 1;
    while (b < 32 && (1LL << b) <= v) ++b;
    return b;
}

template <class F>
int cub_call(rt_ctx* ctx, F&& f) {
    size_t need = 0;
    CK(f((void*)nullptr, need));
    CK(ctx->cub_tmp.reserve(need));
    size_t have = ctx->cub_tmp.bytes;
    CK(f(ctx->cub_tmp.p, have));
    ++ctx->counters[15];   // one device-wide CUB primitive
    return RT_OK;
}

// Stable (key, value) radix sort over key bits [begin_bit, end_bit): one CTA
// (k_sort_small) up to SORT_SMALL_MAX pairs, cub::DeviceRadixSort above.
template <int ITEMS>
int sort_small_launch(rt_ctx* ctx, const unsigned long long* kin, unsigned long long* kout, const int* vin,
                      int* vout, long long n, int begin_bit, int end_bit, int expand_cb, cudaStream_t st) {
    static bool attr_set[64] = {};
    size_t smem = sizeof(typename SmallSort<ITEMS>::TempStorage);
    if (ctx->device < 64 && !attr_set[ctx->device]) {
        CK(cudaFuncSetAttribute(k_sort_small<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set[ctx->device] = true;
    }
    k_sort_small<ITEMS><<<1, SORT_SMALL_THREADS, smem, st>>>(kin, kout, vin, vout, (int)n, begin_bit, end_bit,
                                                             expand_cb);
    CKL();
    return RT_OK;
}

int sort_pairs(rt_ctx* ctx, const unsigned long long* kin, unsigned long long* kout, const int* vin, int* vout,
               long long n, int begin_bit, int end_bit, cudaStream_t st, int expand_cb = 0) {
    if (n <= 0) return RT_OK;
    if (n <= SORT_SMALL_THREADS * 4)
        return sort_small_launch<4>(ctx, kin, kout, vin, vout, n, begin_bit, end_bit, expand_cb, st);
    if (n <= SORT_SMALL_THREADS * 8)
        return sort_small_launch<8>(ctx, kin, kout, vin, vout, n, begin_bit, end_bit, expand_cb, st);
    if (n <= SORT_SMALL_MAX)
        return sort_small_launch<16>(ctx, kin, kout, vin, vout, n, begin_bit, end_bit, expand_cb, st);
    RC(cub_call(ctx, [&](void* tmp, size_t& bytes) {
        return cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, (int)n, begin_bit, end_bit, st);
    }));
    if (expand_cb > 0) {   // compact record keys back to the library's layout
        k_rec_keys_expand<<<nblk(n, 256), 256, 0, st>>>(kout, n, expand_cb);
        CKL();
    }
    return RT_OK;
}

// Sort rows (s_seq/s_len, n rows, width L) by (length, lexicographic) and
// drop duplicates into cand_seq/cand_len (LSD radix over digit columns).
// unique_in: the rows are known to be distinct (one launch's trie): the
// duplicate flags, their scan and the count read-back are skipped
int sort_unique_candidates(rt_ctx* ctx, long long n, int L, cudaStream_t st, bool unique_in = false) {
    ctx->cand_max_len = std::max(L, 1);
    if (n == 0) {
        ctx->n_cand = 0;
        ctx->cand_sorted = true;
        CK(ctx->cand_seq.reserve(sizeof(int) * ctx->cand_max_len));
        CK(ctx->cand_len.reserve(1));
        return RT_OK;
    }
    CK(ctx->s_perm.reserve(sizeof(int) * n));
    CK(ctx->s_perm_alt.reserve(sizeof(int) * n));
    CK(ctx->s_keys.reserve(sizeof(unsigned long long) * n));
    CK(ctx->s_keys_alt.reserve(sizeof(unsigned long long) * n));
    CK(ctx->s_flag.reserve(sizeof(int) * (n + 1)));
    CK(ctx->s_pos.reserve(sizeof(int) * (n + 1)));
    int* perm = ctx->s_perm.get<int>();
    int* perm_alt = ctx->s_perm_alt.get<int>();
    unsigned long long* keys = ctx->s_keys.get<unsigned long long>();
    unsigned long long* keys_alt = ctx->s_keys_alt.get<unsigned long long>();
    const int* seq = ctx->s_seq.get<int>();
    const signed char* len = ctx->s_len.get<signed char>();
    k_iota<<<nblk(n, 256), 256, 0, st>>>(perm, n);
    CKL();
    // LSD over groups of digit columns packed into 64-bit keys (W bits per
    // column, the row length above the most significant group): C3 (W = 18,
    // L = 5) sorts twice instead of six times, the C2 canyon (W = 11, L = 3) once
    const int W = bits_for(ctx->n_prims + 1);
    const int per = std::max(1, 60 / W);
    for (int hi = L - 1; hi >= -1;) {
        int lo = std::max(0, hi - per + 1);
        int ncol = hi >= 0 ? hi - lo + 1 : 0;
        int with_len = (lo == 0 && ncol * W + 4 <= 64) || hi < 0;
        if (hi < 0) lo = 0;
        int end_bit = ncol * W + (with_len ? 4 : 0);
        k_digit_columns<<<nblk(n, 256), 256, 0, st>>>(n, seq, len, L, lo, hi, W, with_len, perm, keys);
        CKL();
        RC(sort_pairs(ctx, keys, keys_alt, perm, perm_alt, n, 0, end_bit, st));
        std::swap(perm, perm_alt);
        if (with_len) break;
        hi = lo == 0 ? -1 : lo - 1;
    }
    if (unique_in) {
        CK(ctx->cand_seq.reserve(sizeof(int) * n * L));
        CK(ctx->cand_len.reserve(n));
        k_gather_rows<<<nblk(n, 256), 256, 0, st>>>(n, perm, seq, len, L, ctx->cand_seq.get<int>(),
                                                    ctx->cand_len.get<signed char>());
        CKL();
        ctx->n_cand = n;
        ctx->cand_sorted = true;
        return RT_OK;
    }
    int* flag = ctx->s_flag.get<int>();
    int* pos = ctx->s_pos.get<int>();
    k_flag_unique<<<nblk(n, 256), 256, 0, st>>>(n, perm, seq, len, L, flag);
    CKL();
    RC(cub_call(ctx, [&](void* tmp, size_t& bytes) {
        return cub::DeviceScan::ExclusiveSum(tmp, bytes, flag, pos, (int)n, st);
    }));
    CK(cudaMemcpyAsync(ctx->hpin, pos + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(reinterpret_cast<int*>(ctx->hpin) + 1, flag + n - 1, sizeof(int),
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    long long n_unique = (long long)reinterpret_cast<int*>(ctx->hpin)[0] +
                         reinterpret_cast<int*>(ctx->hpin)[1];
    CK(ctx->cand_seq.reserve(sizeof(int) * n_unique * L));
    CK(ctx->cand_len.reserve(n_unique));
    k_scatter_unique<<<nblk(n, 256), 256, 0, st>>>(n, perm, flag, pos, seq, len, L,
                                                   ctx->cand_seq.get<int>(),
                                                   ctx->cand_len.get<signed char>());
    CKL();
    ctx->n_cand = n_unique;
    ctx->cand_sorted = true;
    return RT_OK;
}

int finish_tree(rt_ctx* ctx, long long n, const int* root_p, cudaStream_t st, bool dbox_ready = false);
int finish_small(rt_ctx* ctx, long long n, const int* root, cudaStream_t st);
int tree_diagnostics(rt_ctx* ctx, cudaStream_t st);
int build_morton(rt_ctx* ctx, long long n, cudaStream_t st);

// PLOC-format scratch shared by the PLOC and SAH builders
int reserve_tree(rt_ctx* ctx, long long n) {
    long long nn = 2 * n - 1;
    CK(ctx->pl_box.reserve(24ULL * nn));
    CK(ctx->pl_count.reserve(4ULL * nn));
    CK(ctx->pl_parent.reserve(4ULL * nn));
    CK(ctx->child.reserve(8ULL * n));
    CK(ctx->pl_ca.reserve(4ULL * n));
    CK(ctx->pl_cb.reserve(4ULL * n));
    CK(ctx->pl_slot.reserve(4ULL * n));
    CK(ctx->pl_em.reserve(4ULL * nn));
    CK(ctx->pl_dfs.reserve(4ULL * n));
    return RT_OK;
}

// top-down binned-SAH hierarchy (bvh_sah.cuh): ranges of > SAH_BIG prims are
// split level by level with one CTA per SAH_CHUNK-prim chunk, ranges of
// small_max < m <= SAH_BIG with one CTA per range, then one thread finishes
// each small range; the emitted-node counts are then computed bottom-up.  One
// host round trip per level (the next level's grid sizes).
int build_sah(rt_ctx* ctx, long long n, cudaStream_t st) {
    RC(reserve_tree(ctx, n));
    const int small_max = n < SAH_LATENCY_PRIMS ? SAH_SMALL_LATENCY : SAH_SMALL;
    const long long cap_med = n / (small_max + 1) + 2, cap_small = n + 2;
    const long long cap_big = 2 * (n / SAH_BIG) + 2, cap_chunk = n / SAH_CHUNK + cap_big + 2;
    size_t bytes = sizeof(SahTask) * (3 * cap_med + cap_small + 2 * cap_big) + sizeof(int2) * 2 * cap_big +
                   sizeof(int) * 3 * cap_chunk + sizeof(unsigned) * 2 * cap_big * SAH_RB +
                   16 * 16;   // alignment of the 13 sub-buffers
    CK(ctx->sah_tasks.reserve(bytes));
    CK(ctx->flags.reserve(4 * n));
    char* q = ctx->sah_tasks.get<char>();
    auto take = [&](size_t nb) { char* r = q; q += (nb + 15) / 16 * 16; return r; };
    SahTask* med[2] = {(SahTask*)take(sizeof(SahTask) * cap_med), (SahTask*)take(sizeof(SahTask) * cap_med)};
    SahTask* small = (SahTask*)take(sizeof(SahTask) * cap_small);
    SahTask* big[2] = {(SahTask*)take(sizeof(SahTask) * cap_big), (SahTask*)take(sizeof(SahTask) * cap_big)};
    int2* bigc[2] = {(int2*)take(sizeof(int2) * cap_big), (int2*)take(sizeof(int2) * cap_big)};
    int* ctask[2] = {(int*)take(sizeof(int) * cap_chunk), (int*)take(sizeof(int) * cap_chunk)};
    int* cleft = (int*)take(sizeof(int) * cap_chunk);
    // warp subtrees pay off with many ranges in flight (C3: build 1.83 -> 1.62 ms);
    // a small scene has a handful, whose serial warps are slower than CTA levels
    // (C2 canyon: 0.40 -> 0.70 ms), so it keeps the CTA levels to the bottom
    SahTask* wlist = (SahTask*)take(sizeof(SahTask) * cap_med);
    SahTask* wl = n >= SAH_LATENCY_PRIMS ? wlist : nullptr;
    unsigned* rb[2] = {(unsigned*)take(sizeof(unsigned) * cap_big * SAH_RB),
                       (unsigned*)take(sizeof(unsigned) * cap_big * SAH_RB)};
    if ((size_t)(q - ctx->sah_tasks.get<char>()) > ctx->sah_tasks.bytes)
        return fail(ctx, RT_ECUDA, "SAH scratch layout overflow");
    int* em = ctx->pl_em.get<int>();
    float* box = ctx->pl_box.get<float>();
    int* cnt = ctx->pl_count.get<int>();
    int* par = ctx->pl_parent.get<int>();
    int* child = ctx->child.get<int>();
    int* idx0 = ctx->pl_ca.get<int>();
    int* idx1 = ctx->pl_cb.get<int>();
    int* sidx = ctx->sorted_idx.get<int>();
    const float* pbox = ctx->pbox.get<float>();
    const float* cent = ctx->cent.get<float>();
    // device ints: [0,1] big ranges (ping-pong), [2,3] their chunks, [4,5,8] medium
    // range counters (3-way rotation), [6] small ranges, [7] root, [9] warp ranges
    int* dc = reinterpret_cast<int*>(ctx->ctrs.get<long long>() + 16);
    k_iota<<<nblk(n, 256), 256, 0, st>>>(sidx, n);
    CKL();
    k_ploc_init<<<nblk(n, 256), 256, 0, st>>>((int)n, sidx, pbox, box, idx0, cnt, em);
    CKL();
    int h[12] = {0, 0, 0, 0, 0, 0, 0, -1, 0, 0, 0, 0};
    SahTask root_task{0, (int)n, -1, 0};
    if (n <= small_max) {
        h[6] = 1;
        CK(cudaMemcpyAsync(small, &root_task, sizeof(SahTask), cudaMemcpyHostToDevice, st));
    } else if (wl && n <= SAH_WARP_MAX) {
        h[9] = 1;
        CK(cudaMemcpyAsync(wlist, &root_task, sizeof(SahTask), cudaMemcpyHostToDevice, st));
    } else if (n <= SAH_BIG) {
        h[4] = 1;
        CK(cudaMemcpyAsync(med[0], &root_task, sizeof(SahTask), cudaMemcpyHostToDevice, st));
    } else {
        int nc = (int)((n + SAH_CHUNK - 1) / SAH_CHUNK);
        h[0] = 1;
        h[2] = nc;
        int2 ch = make_int2(0, nc);
        CK(cudaMemcpyAsync(big[0], &root_task, sizeof(SahTask), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(bigc[0], &ch, sizeof(int2), cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(ctask[0], 0, sizeof(int) * nc, st));
    }
    CK(cudaMemcpyAsync(dc, h, sizeof(h), cudaMemcpyHostToDevice, st));
    int levels = 0, cur = 0;
    long long nbig = h[0], nchunk = h[2];
    // ranges of > SAH_BIG prims: SAH_BIG_BATCH levels per host round trip, grids
    // sized by bounds (ranges at most double per level; a level's chunks are at
    // most n / SAH_CHUNK + its ranges); blocks past the live counts exit at once
    const int SAH_BIG_BATCH = 3;
    while (nbig > 0) {
        long long bb = nbig, bc = nchunk;
        for (int bt = 0; bt < SAH_BIG_BATCH; ++bt) {
            int nx = cur ^ 1;
            SahOut O{small_max, small, dc + 6, med[0], dc + 4, big[nx], bigc[nx], dc + nx, ctask[nx], dc + 2 + nx,
                     wl, dc + 9};
            CK(cudaMemsetAsync(dc + nx, 0, 4, st));
            CK(cudaMemsetAsync(dc + 2 + nx, 0, 4, st));
            k_sahb_init<<<bb, 128, 0, st>>>(dc + cur, rb[cur]);
            k_sahb_bounds<<<bc, SAH_BLOCK, 0, st>>>(big[cur], bigc[cur], ctask[cur], dc + 2 + cur, idx0, idx1,
                                                    pbox, cent, rb[cur]);
            k_sahb_bins<<<bc, SAH_BLOCK, 0, st>>>(big[cur], bigc[cur], ctask[cur], dc + 2 + cur, idx0, idx1,
                                                  pbox, cent, rb[cur]);
            k_sahb_split<<<bb, 64, 0, st>>>(big[cur], dc + cur, rb[cur], (int)n, box, child, par, cnt, dc + 7, O);
            k_sahb_count<<<bc, SAH_BLOCK, 0, st>>>(big[cur], bigc[cur], ctask[cur], dc + 2 + cur, idx0, idx1,
                                                   cent, rb[cur], cleft);
            k_sahb_write<<<bc, SAH_BLOCK, 0, st>>>(big[cur], bigc[cur], ctask[cur], dc + 2 + cur, idx0, idx1,
                                                   cent, rb[cur], cleft);
            CKL();
            cur = nx;
            ++levels;
            bb = std::min(2 * bb, cap_big);
            bc = std::min(n / SAH_CHUNK + 1 + bb, cap_chunk);
        }
        CK(cudaMemcpyAsync(h, dc, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        nbig = h[cur];
        nchunk = h[2 + cur];
        if (levels > 4096) return fail(ctx, RT_ECUDA, "SAH build made no progress");
    }
    // ranges of small_max < m <= SAH_BIG prims: SAH_MED_BATCH levels per host
    // round trip, each grid sized by the bound (ranges at most double per level;
    // CTAs past the live count exit at once)
    // small scenes take all their medium levels in one batch (one host sync)
    const int SAH_MED_BATCH = n <= SAH_LATENCY_PRIMS ? 16 : 8;
    // level k reads counter mc[k % 3], fills mc[(k + 1) % 3] and zeroes
    // mc[(k + 2) % 3] for the level after it: no memset per level
    int* mc[3] = {dc + 4, dc + 5, dc + 8};
    int mcur = 0, lvl = 0;
    long long nmed = h[4];
    while (nmed > 0) {
        long long bound = nmed;
        for (int b = 0; b < SAH_MED_BATCH; ++b, ++lvl) {
            int nx = mcur ^ 1;
            SahOut O{small_max, small, dc + 6, med[nx], mc[(lvl + 1) % 3], nullptr, nullptr, nullptr, nullptr,
                     nullptr, wl, dc + 9};
            // the top levels of a small scene are a few ranges of ~n / 2^lvl prims on as
            // many SMs: wide CTAs shorten their latency chain (C2 canyon: 2 levels); in a
            // large scene the first medium levels hold ranges of up to SAH_BIG prims
            const bool wide = n <= SAH_LATENCY_PRIMS ? (n >> lvl) > 2 * SAH_BLOCK
                                                     : (n / std::max<long long>(nmed, 1) >> b) > RT_SAH_WIDE_MIN;
            if (wide)
                k_sah_large<1024><<<bound, 1024, 0, st>>>(med[mcur], mc[lvl % 3], mc[(lvl + 2) % 3], idx0, idx1,
                                                          pbox, cent, (int)n, box, child, par, cnt, dc + 7, O);
            else
                k_sah_large<SAH_BLOCK><<<bound, SAH_BLOCK, 0, st>>>(med[mcur], mc[lvl % 3], mc[(lvl + 2) % 3], idx0,
                                                                    idx1, pbox, cent, (int)n, box, child, par, cnt,
                                                                    dc + 7, O);
            CKL();
            mcur = nx;
            ++levels;
            bound = std::min(2 * bound, cap_med);
        }
        CK(cudaMemcpyAsync(h, dc, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        nmed = h[lvl % 3 == 2 ? 8 : 4 + lvl % 3];
        if (levels > 4096) return fail(ctx, RT_ECUDA, "SAH build made no progress");
    }
    if (h[9] > 0) {   // every range of small_max < m <= SAH_WARP_MAX: one warp per subtree
        k_sah_warp<<<(unsigned)((h[9] + SAHW_WARPS - 1) / SAHW_WARPS), 32 * SAHW_WARPS, 0, st>>>(
            wlist, dc + 9, idx0, idx1, pbox, cent, (int)n, box, child, par, cnt, dc + 7, small_max, small, dc + 6);
        CKL();
        h[6] = (int)(n / 2 + 1);   // the warps add small ranges (>= 2 prims each): grid by the bound
    }
    if (h[6] > 0) {
        k_sah_small<<<nblk(h[6], 128), 128, 0, st>>>(small, dc + 6, idx0, idx1, pbox, cent, (int)n, box, child,
                                                     par, cnt, dc + 7);
        CKL();
    }
    ctx->counters[9] = levels;
    if (RT_DFS_LAYOUT && RT_ORIGIN_SKIP && RT_STACK_CHECK && n <= FIN_MAX)
        return finish_small(ctx, n, dc + 7, st);   // the passes below in one CTA
    CK(cudaMemsetAsync(ctx->flags.p, 0, 4 * n, st));
    if (RT_ORIGIN_SKIP) {   // emitted counts + the exact FP64 boxes in one climb (finish_tree skips its refit)
        CK(ctx->dbox.reserve(48ULL * (2 * n - 1)));
        k_sah_climb<<<nblk(n, 256), 256, 0, st>>>((int)n, par, child, cnt, em, ctx->flags.get<int>(),
                                                  ctx->v0.get<double>(), ctx->e1.get<double>(), ctx->e2.get<double>(),
                                                  ctx->dbox.get<double>());
        CKL();
        return finish_tree(ctx, n, dc + 7, st, true);
    }
    k_sah_emitted<<<nblk(n, 256), 256, 0, st>>>((int)n, par, child, cnt, em, ctx->flags.get<int>());
    CKL();
    // the root id stays on the device (dc[7], written by the split that had no
    // parent): no host round trip
    return finish_tree(ctx, n, dc + 7, st);
}

// PLOC hierarchy over the Morton-sorted prims (sorted_idx), then the
// depth-first child-pair layout + triangle records (bvh_ploc.cuh)
int build_ploc(rt_ctx* ctx, long long n, cudaStream_t st) {
    RC(reserve_tree(ctx, n));
    CK(ctx->pl_nn.reserve(4ULL * n));
    CK(ctx->pl_out.reserve(4ULL * n));
    CK(ctx->pl_valid.reserve(4ULL * (n + 1)));
    CK(ctx->pl_pos.reserve(4ULL * (n + 1)));
    int* em = ctx->pl_em.get<int>();
    float* box = ctx->pl_box.get<float>();
    int* cnt = ctx->pl_count.get<int>();
    int* par = ctx->pl_parent.get<int>();
    int* child = ctx->child.get<int>();
    int* ca = ctx->pl_ca.get<int>();
    int* cb = ctx->pl_cb.get<int>();
    int* valid = ctx->pl_valid.get<int>();
    int* pos = ctx->pl_pos.get<int>();
    const int* sidx = ctx->sorted_idx.get<int>();
    k_ploc_init<<<nblk(n, 256), 256, 0, st>>>((int)n, sidx, ctx->pbox.get<float>(), box, ca, cnt, em);
    CKL();
    int* counter = reinterpret_cast<int*>(ctx->ctrs.get<long long>());
    CK(cudaMemsetAsync(counter, 0, 4, st));
    // live cluster counts (ping-pong): the loop runs PLOC_BATCH iterations per
    // host sync, sizing grids by the last count it read (an upper bound)
    int* dC[2] = {reinterpret_cast<int*>(ctx->ctrs.get<long long>() + 10),
                  reinterpret_cast<int*>(ctx->ctrs.get<long long>() + 11)};
    {
        int n32 = (int)n;
        CK(cudaMemcpyAsync(dC[0], &n32, 4, cudaMemcpyHostToDevice, st));
    }
    long long C = n;
    int iters = 0, cur = 0;
    int root = -1;
    const int PLOC_BATCH = 4;
    while (C > 1) {
        if (RT_PLOC_TAIL && C <= PLOC_TAIL) {   // finish in one block, no host round trips
            if (!ctx->tail_smem_set) {   // 48 KB of staged boxes: opt in once per context
                CK(cudaFuncSetAttribute(k_ploc_tail, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        PLOC_TAIL_SMEM));
                ctx->tail_smem_set = true;
            }
            k_ploc_tail<<<1, PLOC_TAIL_THREADS, PLOC_TAIL_SMEM, st>>>(ca, (int)C, (int)n, box, child, par,
                                                                       cnt, em, counter, pos);
            CKL();
            CK(cudaMemcpyAsync(&root, pos, 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            break;
        }
        for (int b = 0; b < PLOC_BATCH; ++b, ++iters) {
            k_ploc_nn<<<nblk(C, PLOC_BLOCK), PLOC_BLOCK, 0, st>>>(ca, dC[cur], box, ctx->pl_nn.get<int>());
            CKL();
            k_ploc_merge<<<nblk(C, 256), 256, 0, st>>>(ca, dC[cur], (int)C, ctx->pl_nn.get<int>(), (int)n, box,
                                                        child, par, cnt, em, counter, ctx->pl_out.get<int>(),
                                                        valid);
            CKL();
            RC(cub_call(ctx, [&](void* tmp, size_t& bytes) {
                return cub::DeviceScan::ExclusiveSum(tmp, bytes, valid, pos, (int)C, st);
            }));
            k_ploc_compact<<<nblk(C, 256), 256, 0, st>>>(ctx->pl_out.get<int>(), valid, pos, dC[cur], cb,
                                                          dC[cur ^ 1]);
            CKL();
            std::swap(ca, cb);
            cur ^= 1;
        }
        int h = 0;
        CK(cudaMemcpyAsync(&h, dC[cur], 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h >= C || iters > 100000) return fail(ctx, RT_ECUDA, "PLOC made no progress");
        C = h;
    }
    if (root < 0) {
        root = 0;
        CK(cudaMemcpyAsync(&root, ca, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    ctx->counters[9] = iters;
    int* root_dev = reinterpret_cast<int*>(ctx->ctrs.get<long long>() + 24);   // past dc[0..11]
    CK(cudaMemcpyAsync(root_dev, &root, 4, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));   // `root` is a stack variable
    return finish_tree(ctx, n, root_dev, st);
}

// depth-first child-pair layout + triangle records of a hierarchy in the PLOC
// arrays (leaves [0, n) with sorted_idx, internal nodes [n, 2n-1), root id)
int finish_tree(rt_ctx* ctx, long long n, const int* root, cudaStream_t st, bool dbox_ready) {
    int* em = ctx->pl_em.get<int>();
    float* box = ctx->pl_box.get<float>();
    int* cnt = ctx->pl_count.get<int>();
    int* par = ctx->pl_parent.get<int>();
    int* child = ctx->child.get<int>();
    const int* sidx = ctx->sorted_idx.get<int>();
    int* slot = ctx->pl_slot.get<int>();
    k_ploc_slots<<<nblk(n, 256), 256, 0, st>>>((int)n, par, child, cnt, root, slot);
    CKL();
    CK(ctx->nodes.reserve(sizeof(BNode) * std::max<long long>(n - 1, 1)));
    int* dfs = nullptr;
    if (n > 1) {   // depth-first order + tree depth (always measured: it bounds the stack)
        dfs = ctx->pl_dfs.get<int>();
        CK(ctx->tree_diag.reserve(64));
        int* dmax = ctx->tree_diag.get<int>();
        CK(cudaMemsetAsync(dmax, 0, 4, st));
        k_ploc_dfs<<<nblk(n - 1, 256), 256, 0, st>>>((int)n, root, par, child, cnt, em, dfs, dmax);
        CKL();
        if (!RT_STACK_CHECK) {   // unchecked pushes: the depth must fit the stack now
            int h = 0;
            CK(cudaMemcpyAsync(&h, dmax, 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            ctx->bvh_depth = h;
            if (h + 2 > STACK_SIZE)
                return fail(ctx, RT_ECAP, "BVH depth " + std::to_string(h) + " exceeds the traversal stack (" +
                                              std::to_string(STACK_SIZE) + " entries)");
        }
        if (!RT_DFS_LAYOUT) dfs = nullptr;
    }
    if (n > 1) {
        k_ploc_layout<<<nblk(n - 1, 256), 256, 0, st>>>((int)n, root, child, cnt, slot, box,
                                                        ctx->cbounds.get<unsigned>(), dfs, ctx->nodes.get<BNode>());
        CKL();
    }
    if (RT_ORIGIN_SKIP && n > 1 && dfs) {   // exact FP64 boxes -> per-prim origin skip refs
        CK(ctx->dbox.reserve(48ULL * (2 * n - 1)));
        CK(ctx->skip_tab.reserve(8ULL * n));
        if (!dbox_ready) {
            CK(ctx->flags.reserve(4ULL * n));
            CK(cudaMemsetAsync(ctx->flags.p, 0, 4 * n, st));
            k_root_parent<<<1, 1, 0, st>>>(root, par);   // the refit climb stops at the root
            k_dbox_refit<<<nblk(n, 256), 256, 0, st>>>((int)n, sidx, ctx->v0.get<double>(), ctx->e1.get<double>(),
                                                       ctx->e2.get<double>(), par, child, ctx->dbox.get<double>(),
                                                       ctx->flags.get<int>());
        }
        k_skip_table<<<nblk(n, 256), 256, 0, st>>>((int)n, root, sidx, par, child, cnt, slot, dfs,
                                                   ctx->dbox.get<double>(), ctx->nrm.get<double>(),
                                                   ctx->poff.get<double>(), ctx->skip_tab.get<int>());
        CKL();
        ctx->has_skip = true;
    }
    k_ploc_tris<<<nblk(n, 256), 256, 0, st>>>((int)n, sidx, slot, ctx->v0.get<double>(), ctx->e1.get<double>(),
                                              ctx->e2.get<double>(), ctx->tris.get<TriRec>());
    CKL();
    // tree diagnostics (depth, surface-area estimate) are computed on demand by
    // rt_get_profile: no host round trip on the build path
    ctx->diag_root_dev = (n > 2 && dfs) ? root : nullptr;
    ctx->diag_pending = n > 1;
    if (!ctx->diag_ev) CK(cudaEventCreateWithFlags(&ctx->diag_ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ctx->diag_ev, st));
    return RT_OK;
}

// finish_tree + the SAH emitted counts for a small SAH tree (2 <= n <= FIN_MAX):
// one CTA, tree links in shared memory (bvh_finish.cuh), same outputs
int finish_small(rt_ctx* ctx, long long n, const int* root, cudaStream_t st) {
    CK(ctx->nodes.reserve(sizeof(BNode) * std::max<long long>(n - 1, 1)));
    CK(ctx->tree_diag.reserve(64));
    CK(ctx->dbox.reserve(48ULL * (2 * n - 1)));
    CK(ctx->skip_tab.reserve(8ULL * n));
    size_t smem = fin_smem_bytes((int)n);
    static bool attr_set[64] = {};
    if (ctx->device < 64 && !attr_set[ctx->device]) {
        CK(cudaFuncSetAttribute(k_finish_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fin_smem_bytes(FIN_MAX)));
        attr_set[ctx->device] = true;
    }
    k_finish_small<<<1, FIN_THREADS, smem, st>>>(
        (int)n, root, ctx->sorted_idx.get<int>(), ctx->pl_parent.get<int>(), ctx->child.get<int>(),
        ctx->pl_count.get<int>(), ctx->pl_em.get<int>(), ctx->pl_slot.get<int>(), ctx->pl_dfs.get<int>(),
        ctx->tree_diag.get<int>(), ctx->pl_box.get<float>(), ctx->cbounds.get<unsigned>(), ctx->nodes.get<BNode>(),
        ctx->dbox.get<double>(), ctx->v0.get<double>(), ctx->e1.get<double>(), ctx->e2.get<double>(),
        ctx->nrm.get<double>(), ctx->poff.get<double>(), ctx->skip_tab.get<int>(), ctx->tris.get<TriRec>());
    CKL();
    ctx->has_skip = true;
    ctx->diag_root_dev = n > 2 ? root : nullptr;
    ctx->diag_pending = true;
    if (!ctx->diag_ev) CK(cudaEventCreateWithFlags(&ctx->diag_ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ctx->diag_ev, st));
    return RT_OK;
}

// counters 13 (tree depth) and 14 (surface-area estimate) of the last build
int tree_diagnostics(rt_ctx* ctx, cudaStream_t st) {
    if (!ctx->diag_pending) return RT_OK;
    ctx->diag_pending = false;
    // the build ran on the caller's (possibly non-blocking) stream: wait for it
    if (ctx->diag_ev) CK(cudaEventSynchronize(ctx->diag_ev));
    int h = 0;
    CK(cudaMemcpyAsync(&h, ctx->tree_diag.get<int>(), 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->bvh_depth = h;
    ctx->counters[13] = h;
    if (!ctx->diag_root_dev) return RT_OK;
    int root = -1, n_nodes = 0;
    CK(cudaMemcpyAsync(&root, ctx->diag_root_dev, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (root < 0) return RT_OK;
    CK(cudaMemcpyAsync(&n_nodes, ctx->pl_em.get<int>() + root, 4, cudaMemcpyDeviceToHost, st));
    double* sums = reinterpret_cast<double*>(ctx->tree_diag.get<int>() + 2);
    CK(cudaMemsetAsync(sums, 0, 24, st));
    CK(cudaStreamSynchronize(st));
    k_tree_sah<<<nblk(n_nodes, 256), 256, 0, st>>>(ctx->nodes.get<BNode>(), n_nodes, sums);
    CKL();
    double d[3];
    CK(cudaMemcpyAsync(d, sums, 24, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->counters[14] = (long long)llround(1000.0 * (1.0 + d[0] / d[2]));   // milli-visits
    return RT_OK;
}

}  // namespace

// ===========================================================================================
extern "C" {

int rt_version(void) { return 1; }

// rt_h2d: per-device ring of page-locked slots; a slot is refilled only after
// the copy out of it has completed (its event)
namespace {
constexpr int H2D_SLOTS = 8;
constexpr size_t H2D_SLOT_BYTES = 1 << 20;
struct H2DRing {
    void* host[H2D_SLOTS] = {};
    cudaEvent_t ev[H2D_SLOTS] = {};
    bool used[H2D_SLOTS] = {};
    int next = 0;
};
std::mutex g_h2d_mu;
H2DRing g_h2d[64];
}  // namespace

namespace {
int h2d_staged(int device, void* dst, const void* src, int64_t bytes, cudaStream_t st) {
    if (device < 0 || device >= 64 || bytes < 0 || (bytes > 0 && (!dst || !src))) return RT_EINVAL;
    if (bytes == 0) return RT_OK;
    std::lock_guard<std::mutex> lock(g_h2d_mu);
    if (cudaSetDevice(device) != cudaSuccess) return RT_ECUDA;
    H2DRing& R = g_h2d[device];
    const char* p = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    while (bytes > 0) {
        int k = R.next;
        R.next = (k + 1) % H2D_SLOTS;
        if (!R.host[0]) {   // the whole ring at once: no page-locking (~2 ms a slot) on later calls
            char* block = nullptr;
            if (cudaMallocHost(reinterpret_cast<void**>(&block), H2D_SLOTS * H2D_SLOT_BYTES) != cudaSuccess)
                return RT_ENOMEM;
            for (int q = 0; q < H2D_SLOTS; ++q) {
                R.host[q] = block + q * H2D_SLOT_BYTES;
                if (cudaEventCreateWithFlags(&R.ev[q], cudaEventDisableTiming) != cudaSuccess) return RT_ECUDA;
            }
        }
        if (R.used[k] && cudaEventSynchronize(R.ev[k]) != cudaSuccess) return RT_ECUDA;
        size_t n = std::min<size_t>((size_t)bytes, H2D_SLOT_BYTES);
        std::memcpy(R.host[k], p, n);
        if (cudaMemcpyAsync(d, R.host[k], n, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaEventRecord(R.ev[k], st) != cudaSuccess)
            return RT_ECUDA;
        R.used[k] = true;
        p += n;
        d += n;
        bytes -= (int64_t)n;
    }
    return RT_OK;
}
}  // namespace

int rt_h2d(int device, void* dst, const void* src, int64_t bytes, void* stream) {
    return h2d_staged(device, dst, src, bytes, ST(stream));
}


int rt_create(int device, rt_ctx** out) {
    rt_ctx* ctx = nullptr;
    if (!out) return RT_EINVAL;
    *out = nullptr;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return RT_ECUDA;
    ctx = new rt_ctx();
    ctx->device = device;
    cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, device);
    if (cudaMallocHost(&ctx->hpin, 64 * sizeof(long long)) != cudaSuccess ||
        ctx->dflag.reserve(64) != cudaSuccess || ctx->ctrs.reserve(256) != cudaSuccess) {
        delete ctx;
        return RT_ENOMEM;
    }
    cudaMemset(ctx->dflag.p, 0, 64);
    *out = ctx;
    return RT_OK;
}

int rt_destroy(rt_ctx* ctx) {
    if (!ctx) return RT_OK;
    cudaSetDevice(ctx->device);
    if (ctx->hpin) cudaFreeHost(ctx->hpin);
    if (ctx->diag_ev) cudaEventDestroy(ctx->diag_ev);
    if (ctx->up_ev) cudaEventDestroy(ctx->up_ev);
    for (auto& pair : ctx->ev)
        for (cudaEvent_t e : pair)
            if (e) cudaEventDestroy(e);
    delete ctx;
    return RT_OK;
}

const char* rt_last_error(const rt_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t rt_num_prims(const rt_ctx* ctx) { return ctx ? ctx->n_prims : 0; }
int64_t rt_num_candidates(const rt_ctx* ctx) { return ctx ? ctx->n_cand : 0; }
int rt_candidates_max_len(const rt_ctx* ctx) { return ctx ? ctx->cand_max_len : 1; }
int64_t rt_paths_max_per_receiver(const rt_ctx* ctx) { return ctx ? ctx->paths_max_rx : 0; }

int rt_scene_upload(rt_ctx* ctx, const double* vertices, int64_t n_vertices,
                    const int32_t* tri_vertex, const int32_t* prim_material, int64_t n_prims,
                    void* stream) {
    if (!ctx || n_prims < 0 || n_vertices < 0) return fail(ctx, RT_EINVAL, "bad scene arguments");
    if (n_prims > (1 << 27)) return fail(ctx, RT_EINVAL, "too many primitives (max 2^27)");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    ctx->n_prims = n_prims;
    ctx->bvh_ready = false;
    ctx->n_cand = 0;
    ctx->n_paths = 0;
    size_t n = (size_t)std::max<int64_t>(n_prims, 1);
    CK(ctx->v0.reserve(24 * n));
    CK(ctx->e1.reserve(24 * n));
    CK(ctx->e2.reserve(24 * n));
    CK(ctx->nrm.reserve(24 * n));
    CK(ctx->poff.reserve(8 * n));
    CK(ctx->prim_mat.reserve(4 * n));
    CK(ctx->pbox.reserve(24 * n));
    CK(ctx->cent.reserve(12 * n));
    CK(ctx->cbounds.reserve(48));   // 7 ordered floats, then the FP32 filter's origin bound (double at +32)
    if (n_prims == 0) return RT_OK;
    // inputs in host memory (page-locked or pageable) are copied in on the stream;
    // device inputs are read in place
    cudaPointerAttributes at{};
    bool host_in = cudaPointerGetAttributes(&at, vertices) != cudaSuccess || at.type != cudaMemoryTypeDevice;
    cudaGetLastError();   // clear a pageable-pointer query error
    if (host_in) {
        CK(ctx->up_verts.reserve(24ULL * std::max<int64_t>(n_vertices, 1)));
        CK(ctx->up_tris.reserve(12ULL * n_prims));
        CK(cudaMemcpyAsync(ctx->up_verts.p, vertices, 24ULL * n_vertices, cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(ctx->up_tris.p, tri_vertex, 12ULL * n_prims, cudaMemcpyDefault, st));
        vertices = ctx->up_verts.get<double>();
        tri_vertex = ctx->up_tris.get<int32_t>();
    }
    CK(cudaMemcpyAsync(ctx->prim_mat.p, prim_material, 4 * n_prims, cudaMemcpyDefault, st));
    if (!ctx->up_ev) CK(cudaEventCreateWithFlags(&ctx->up_ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ctx->up_ev, st));
    ctx->up_pending = true;
    // ordered-float bounds: mins start at 0xFFFFFFFF, maxima (and the scale) at 0
    CK(cudaMemsetAsync(ctx->cbounds.p, 0xFF, 3 * sizeof(unsigned), st));
    CK(cudaMemsetAsync(ctx->cbounds.get<unsigned>() + 3, 0, 4 * sizeof(unsigned), st));
    k_gather<<<nblk(n_prims, 256), 256, 0, st>>>(
        vertices, tri_vertex, n_prims, ctx->v0.get<double>(), ctx->e1.get<double>(),
        ctx->e2.get<double>(), ctx->nrm.get<double>(), ctx->poff.get<double>(),
        ctx->pbox.get<float>(), ctx->cent.get<float>(), ctx->cbounds.get<unsigned>());
    CKL();
    return RT_OK;
}

static int bvh_build_impl(rt_ctx* ctx, void* stream);

int rt_bvh_build(rt_ctx* ctx, void* stream) {
    if (!ctx) return RT_EINVAL;
    int rc = bvh_build_impl(ctx, stream);
    if (ctx->up_pending) {   // the caller may refill its host scene buffers after this returns
        ctx->up_pending = false;
        CK(cudaEventSynchronize(ctx->up_ev));
    }
    return rc;
}

static int bvh_build_impl(rt_ctx* ctx, void* stream) {
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    long long n = ctx->n_prims;
    ctx->bvh_ready = true;
    ctx->has_skip = false;
    if (n == 0) return RT_OK;
    // scene scale S (ordered float in cbounds[6]) -> FP32 filter origin bound 2S,
    // computed on the device (no host round trip)
    k_origin_limit<<<1, 1, 0, st>>>(ctx->cbounds.get<unsigned>(),
                                    reinterpret_cast<double*>(ctx->cbounds.get<char>() + 32));
    CKL();
    CK(ctx->tris.reserve(sizeof(TriRec) * n));
    CK(ctx->sorted_idx.reserve(4 * n));
    CK(ctx->nodes.reserve(sizeof(BNode) * std::max<long long>(n - 1, 1)));
    if (n == 1) {
        k_iota<<<1, 32, 0, st>>>(ctx->sorted_idx.get<int>(), 1);
        k_layout_one<<<1, 1, 0, st>>>(ctx->pbox.get<float>(), ctx->cbounds.get<unsigned>(),
                                      ctx->nodes.get<BNode>());
        k_sorted_tris<<<1, 32, 0, st>>>(1, ctx->sorted_idx.get<int>(), ctx->v0.get<double>(),
                                        ctx->e1.get<double>(), ctx->e2.get<double>(),
                                        ctx->tris.get<TriRec>());
        CKL();
        return RT_OK;
    }
    if (RT_SAH) {
        RC(build_sah(ctx, n, st));
    } else {
        RC(build_morton(ctx, n, st));
    }
    return RT_OK;
}

}  // extern "C"

namespace {
// Morton codes + radix sort, then the PLOC hierarchy over them (RT_SAH=0 variant)
int build_morton(rt_ctx* ctx, long long n, cudaStream_t st) {
    CK(ctx->morton.reserve(8 * n));
    CK(ctx->morton_alt.reserve(8 * n));
    CK(ctx->idx_alt.reserve(4 * n));
    CK(ctx->child.reserve(8 * n));
    CK(ctx->flags.reserve(4 * n));
    k_morton<<<nblk(n, 256), 256, 0, st>>>(ctx->cent.get<float>(), ctx->pbox.get<float>(),
                                          ctx->cbounds.get<unsigned>(), n,
                                          ctx->morton_alt.get<uint64_t>(), ctx->idx_alt.get<int>());
    CKL();
    uint64_t* kin = ctx->morton_alt.get<uint64_t>();
    uint64_t* kout = ctx->morton.get<uint64_t>();
    int* vin = ctx->idx_alt.get<int>();
    int* vout = ctx->sorted_idx.get<int>();
    RC(cub_call(ctx, [&](void* tmp, size_t& bytes) {
        return cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, (int)n, 0, 64, st);
    }));
    (void)kout;
    (void)vout;
    return build_ploc(ctx, n, st);
}

}  // namespace

extern "C" {

int rt_scene_arrays(rt_ctx* ctx, double* v0, double* e1, double* e2, double* normals,
                    double* plane_offset, void* stream) {
    if (!ctx) return RT_EINVAL;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    size_t n = ctx->n_prims;
    if (!n) return RT_OK;
    if (v0) CK(cudaMemcpyAsync(v0, ctx->v0.p, 24 * n, cudaMemcpyDeviceToDevice, st));
    if (e1) CK(cudaMemcpyAsync(e1, ctx->e1.p, 24 * n, cudaMemcpyDeviceToDevice, st));
    if (e2) CK(cudaMemcpyAsync(e2, ctx->e2.p, 24 * n, cudaMemcpyDeviceToDevice, st));
    if (normals) CK(cudaMemcpyAsync(normals, ctx->nrm.p, 24 * n, cudaMemcpyDeviceToDevice, st));
    if (plane_offset) CK(cudaMemcpyAsync(plane_offset, ctx->poff.p, 8 * n, cudaMemcpyDeviceToDevice, st));
    return RT_OK;
}

int rt_trace(rt_ctx* ctx, const double* o, const double* d, const double* tmin,
             const double* tmax, int64_t n, int any_hit, double* t_out, int32_t* prim_out,
             void* stream) {
    if (!ctx || n < 0) return fail(ctx, RT_EINVAL, "bad trace arguments");
    if (!ctx->bvh_ready) return fail(ctx, RT_ESTATE, "rt_bvh_build has not run");
    if (n == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    RC(clear_flags(ctx, st));
    if (any_hit)
        k_trace_batch<true><<<nblk(n, 128), 128, 0, st>>>(bvh_dev(ctx), o, d, tmin, tmax, n, t_out,
                                                          prim_out, ctx->dflag.get<long long>());
    else
        k_trace_batch<false><<<nblk(n, 128), 128, 0, st>>>(bvh_dev(ctx), o, d, tmin, tmax, n, t_out,
                                                           prim_out, ctx->dflag.get<long long>());
    CKL();
    return check_flags(ctx, st);
}

int rt_occluded(rt_ctx* ctx, const double* p, const double* q, int64_t n, int32_t* out,
                void* stream) {
    if (!ctx || n < 0) return fail(ctx, RT_EINVAL, "bad occlusion arguments");
    if (!ctx->bvh_ready) return fail(ctx, RT_ESTATE, "rt_bvh_build has not run");
    if (n == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    RC(clear_flags(ctx, st));
    k_occluded_batch<<<nblk(n, 128), 128, 0, st>>>(bvh_dev(ctx), p, q, n, out);
    CKL();
    return check_flags(ctx, st);   // a stack overflow fails the call instead of reading as "blocked"
}

namespace {
int launch_impl(rt_ctx* ctx, const double* tx, int64_t n_rays, int64_t slot_begin, int64_t slot_end,
                int shard_index, int shard_count, int max_depth, const double* dirs,
                int64_t* n_cand_out, int64_t* n_bounces_out, void* stream);
}

int rt_launch(rt_ctx* ctx, const double* tx, int64_t n_rays, int64_t slot_begin,
              int64_t slot_end, int max_depth, const double* dirs, int64_t* n_cand_out,
              int64_t* n_bounces_out, void* stream) {
    if (!ctx || !tx || n_rays < 1 || max_depth < 1)
        return fail(ctx, RT_EINVAL, "need num_rays >= 1 and max_depth >= 1");
    if (slot_begin < 0 || slot_end > n_rays || slot_begin > slot_end)
        return fail(ctx, RT_EINVAL, "bad ray slot range");
    return launch_impl(ctx, tx, n_rays, slot_begin, slot_end, 0, 1, max_depth, dirs, n_cand_out,
                       n_bounces_out, stream);
}

int rt_launch_shard(rt_ctx* ctx, const double* tx, int64_t n_rays, int shard_index, int shard_count,
                    int max_depth, const double* dirs, int64_t* n_cand_out, int64_t* n_bounces_out,
                    void* stream) {
    if (!ctx || !tx || n_rays < 1 || max_depth < 1)
        return fail(ctx, RT_EINVAL, "need num_rays >= 1 and max_depth >= 1");
    if (shard_count < 1 || shard_index < 0 || shard_index >= shard_count)
        return fail(ctx, RT_EINVAL, "bad shard index/count");
    return launch_impl(ctx, tx, n_rays, 0, 0, shard_index, shard_count, max_depth, dirs, n_cand_out,
                       n_bounces_out, stream);
}

}  // extern "C"

namespace {
int launch_impl(rt_ctx* ctx, const double* tx, int64_t n_rays, int64_t slot_begin, int64_t slot_end,
                int shard_index, int shard_count, int max_depth, const double* dirs,
                int64_t* n_cand_out, int64_t* n_bounces_out, void* stream) {
    if (max_depth > MAX_DEPTH) return fail(ctx, RT_EINVAL, "max_depth above the compiled bound (8)");
    if (!ctx->bvh_ready) return fail(ctx, RT_ESTATE, "rt_bvh_build has not run");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    if (n_bounces_out) *n_bounces_out = 0;
    // sharded launches take whole coherence bands (units) round-robin, so every
    // rank gets the same mix of latitudes; local slot l of rank r maps to
    // global unit (l / unit) * W + r (launch.cuh)
    auto shard_slots = [&](long long unit) {
        long long units = (n_rays + unit - 1) / unit;
        long long mine = shard_index < units ? (units - shard_index + shard_count - 1) / shard_count : 0;
        long long cnt = mine * unit;
        long long last = (units - 1) % shard_count == shard_index ? units * unit - n_rays : 0;
        return std::make_pair(mine * unit, cnt - last);   // (local range, rays owned)
    };
    if (ctx->n_prims == 0) {
        RC(sort_unique_candidates(ctx, 0, max_depth, st));
        if (n_cand_out) *n_cand_out = 0;
        // every ray still costs one (missing) intersect call
        if (n_bounces_out)
            *n_bounces_out = shard_count > 1 ? shard_slots(4096).second : slot_end - slot_begin;
        return RT_OK;
    }
    // coherence band: ~sqrt(32 pi n) indices sorted by azimuth (launch.cuh)
    int B = 1;
    while ((double)B * B < RT_BAND_C * (double)n_rays && B < (1 << 20)) B <<= 1;
    if (B < 32 || B > n_rays) B = 0;
    if (B != ctx->band_B) {
        if (B > 0) {
            std::vector<std::pair<double, int>> az(B);
            const double inv_g = 1.0 / 2.618033988749895;
            for (int j = 0; j < B; ++j) {
                double f = (double)j * inv_g;
                az[j] = {f - std::floor(f), j};
            }
            std::sort(az.begin(), az.end());
            std::vector<int> perm(B);
            for (int j = 0; j < B; ++j) perm[j] = az[j].second;
            CK(ctx->perm_band.reserve(4 * B));
            CK(cudaMemcpy(ctx->perm_band.p, perm.data(), 4 * B, cudaMemcpyHostToDevice));
        }
        ctx->band_B = B;
    }
    long long unit = B > 0 ? B : 4096;
    if (shard_count > 1) {
        slot_begin = 0;
        slot_end = shard_slots(unit).first;
    }
    long long span = slot_end - slot_begin;
    // The trie holds one node per unique hit prefix, far fewer than rays x depth
    // (C3: 124k prefixes for 244M bounces).  Start small enough to stay
    // L2-resident and cheap to clear; an overflow grows it 4x and relaunches,
    // and the context keeps the grown capacity for later calls.
    if (ctx->trie_cap == 0) {
        uint64_t want = 1ULL << 16;
        while (want < 4ULL * std::min<long long>(span * max_depth, 1LL << 18)) want <<= 1;
        ctx->trie_cap = want;
    }
    for (int attempt = 0; attempt < 6; ++attempt) {
        uint64_t cap = ctx->trie_cap;
        // slot ids travel as int (trie_insert returns slot + 1): cap must stay below 2^31
        if (cap >= (1ULL << 31)) return fail(ctx, RT_ENOMEM, "candidate trie at or above 2^31 slots");
        CK(ctx->t_keys.reserve(8 * cap));
        CK(cudaMemsetAsync(ctx->t_keys.p, 0xFF, 8 * cap, st));
        CK(cudaMemsetAsync(ctx->ctrs.p, 0, 128, st));
        RC(clear_flags(ctx, st));
        Trie T;
        T.keys = ctx->t_keys.get<unsigned long long>();
        T.mask = (unsigned)(cap - 1);
        long long* ctr = ctx->ctrs.get<long long>();
        T.counter = reinterpret_cast<int*>(ctr + 0);
        T.overflow = reinterpret_cast<int*>(ctr + 1);
        LaunchParams P;
        P.tx = tx[0]; P.ty = tx[1]; P.tz = tx[2];
        P.n_rays = n_rays;
        P.slot_begin = slot_begin;
        P.slot_end = slot_end;
        P.shard_unit = unit;   // B or 4096: a power of two
        P.shard_shift = 0;
        while ((1LL << P.shard_shift) < unit) ++P.shard_shift;
        P.shard_index = shard_index;
        P.shard_count = shard_count;
        P.max_depth = max_depth;
        P.band = B;
        P.band_shift = 0;
        while (B > 0 && (1 << P.band_shift) < B) ++P.band_shift;
        P.perm = ctx->perm_band.get<int>();
        P.dirs = dirs;
        P.normals = ctx->nrm.get<double>();
        P.stats = reinterpret_cast<unsigned long long*>(ctr + 2);
        P.error = reinterpret_cast<int*>(ctx->dflag.get<long long>());
        const int LB = RT_LAUNCH_BLOCK;
        long long blocks = std::min<long long>((span + LB - 1) / LB, (long long)ctx->n_sm * (4096 / LB));
        PROF_BEGIN(ST_LAUNCH);
        if (span > 0) {
            unsigned g = (unsigned)std::max<long long>(blocks, 1);
            if (ctx->prof & 2) k_launch<true><<<g, LB, 0, st>>>(bvh_dev(ctx), P, T);
            else k_launch<false><<<g, LB, 0, st>>>(bvh_dev(ctx), P, T);
            CKL();
        }
        PROF_END(ST_LAUNCH);
        RC(fetch_and_flags(ctx, ctr, 9, st));   // counters + the error word, one round trip
        ctx->counters[1] = ctx->hpin[3];
        ctx->counters[2] = ctx->hpin[4];
        ctx->counters[10] = ctx->hpin[6];
        ctx->counters[11] = ctx->hpin[7];
        ctx->counters[12] = ctx->hpin[8];
        long long nodes = (long long)(int)(ctx->hpin[0] & 0xffffffff);
        bool overflow = (int)(ctx->hpin[1] & 0xffffffff) != 0;
        long long bounces = ctx->hpin[2];
        if (overflow) {   // a probe chain ran out of slots: results incomplete, relaunch
            ctx->trie_cap *= 4;
            continue;
        }
        if ((uint64_t)nodes * 2 > cap) ctx->trie_cap *= 4;   // keep later launches under half full
        if (n_bounces_out) *n_bounces_out = bounces;
        ctx->counters[0] = bounces;
        // materialize sequences and sort them
        CK(ctx->s_seq.reserve(4ULL * std::max<long long>(nodes, 1) * max_depth));
        CK(ctx->s_len.reserve((size_t)std::max<long long>(nodes, 1)));
        PROF_BEGIN(ST_TRIE_SEQ);
        if (nodes > 0) {
            k_trie_sequences<<<nblk(cap, 256), 256, 0, st>>>((long long)cap, T.keys, max_depth,
                                                             ctx->s_seq.get<int>(),
                                                             ctx->s_len.get<signed char>(),
                                                             reinterpret_cast<int*>(ctr + 10));
            CKL();
        }
        PROF_END(ST_TRIE_SEQ);
        PROF_BEGIN(ST_CAND_SORT);
        if (shard_count > 1) {
            // a shard's rows are unique already; the union of all shards is sorted
            // once by rt_candidates_set, so skip the per-shard sort
            ctx->cand_max_len = std::max(max_depth, 1);
            CK(ctx->cand_seq.reserve(4ULL * std::max<long long>(nodes, 1) * max_depth));
            CK(ctx->cand_len.reserve((size_t)std::max<long long>(nodes, 1)));
            if (nodes > 0) {
                CK(cudaMemcpyAsync(ctx->cand_seq.p, ctx->s_seq.p, 4ULL * nodes * max_depth,
                                   cudaMemcpyDeviceToDevice, st));
                CK(cudaMemcpyAsync(ctx->cand_len.p, ctx->s_len.p, (size_t)nodes, cudaMemcpyDeviceToDevice, st));
            }
            ctx->n_cand = nodes;
            ctx->cand_sorted = false;
        } else {
            RC(sort_unique_candidates(ctx, nodes, max_depth, st, true));   // trie rows are distinct
        }
        PROF_END(ST_CAND_SORT);
        ctx->counters[3] = ctx->n_cand;
        if (n_cand_out) *n_cand_out = ctx->n_cand;
        return RT_OK;
    }
    return fail(ctx, RT_ENOMEM, "candidate trie overflow after growing");
}
}  // namespace

extern "C" {

int rt_enumerate(rt_ctx* ctx, int max_depth, int64_t cap, int64_t* n_cand_out, void* stream) {
    if (!ctx) return RT_EINVAL;
    if (max_depth < 1) return fail(ctx, RT_EINVAL, "max_depth must be >= 1 for candidate enumeration");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    long long n = ctx->n_prims;
    // the reference's order of checks (tracer.py:198-207): empty scene, then the cap
    if (n == 0) {
        RC(sort_unique_candidates(ctx, 0, std::min(max_depth, MAX_DEPTH), st));
        if (n_cand_out) *n_cand_out = 0;
        return RT_OK;
    }
    // n ** max_depth > cap (tracer.py:203-207), in floating point to avoid overflow
    if (std::pow((double)n, (double)max_depth) > (double)cap) {
        char buf[256];
        snprintf(buf, sizeof buf,
                 "exhaustive enumeration of %lld primitives at depth %d exceeds the cap of %.0e "
                 "sequences; use the fibonacci ray-launching method instead",
                 n, max_depth, (double)cap);
        return fail(ctx, RT_ECAP, buf);
    }
    if (max_depth > MAX_DEPTH) return fail(ctx, RT_EINVAL, "max_depth above the compiled bound (8)");
    std::vector<long long> start(max_depth + 1, 0);
    long long level = n, total = 0;
    for (int k = 0; k < max_depth; ++k) {
        start[k] = total;
        total += level;
        level *= (n - 1);
    }
    start[max_depth] = total;
    CK(ctx->em_small.reserve(8 * (max_depth + 1)));
    CK(cudaMemcpyAsync(ctx->em_small.p, start.data(), 8 * (max_depth + 1), cudaMemcpyHostToDevice, st));
    CK(ctx->cand_seq.reserve(4ULL * std::max<long long>(total, 1) * max_depth));
    CK(ctx->cand_len.reserve((size_t)std::max<long long>(total, 1)));
    k_enumerate<<<nblk(total, 256), 256, 0, st>>>(total, (int)n, max_depth, ctx->em_small.get<long long>(),
                                                  ctx->cand_seq.get<int>(), ctx->cand_len.get<signed char>());
    CKL();
    CK(cudaStreamSynchronize(st));
    ctx->n_cand = total;
    ctx->cand_sorted = true;   // enumerated directly in (length, lex) order
    ctx->cand_max_len = max_depth;
    if (n_cand_out) *n_cand_out = total;
    return RT_OK;
}

int rt_candidates_set(rt_ctx* ctx, const int32_t* seq, const int8_t* len, int64_t n, int max_len,
                      int64_t* n_unique_out, void* stream) {
    if (!ctx || n < 0 || max_len < 1 || max_len > MAX_DEPTH)
        return fail(ctx, RT_EINVAL, "bad candidate arguments");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    CK(ctx->s_seq.reserve(4ULL * std::max<long long>(n, 1) * max_len));
    CK(ctx->s_len.reserve((size_t)std::max<long long>(n, 1)));
    if (n) {
        CK(cudaMemcpyAsync(ctx->s_seq.p, seq, 4ULL * n * max_len, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(ctx->s_len.p, len, (size_t)n, cudaMemcpyDeviceToDevice, st));
    }
    RC(sort_unique_candidates(ctx, n, max_len, st));
    if (n_unique_out) *n_unique_out = ctx->n_cand;
    return RT_OK;
}

int rt_candidates_get(rt_ctx* ctx, int32_t* seq, int8_t* len, int max_len, void* stream) {
    if (!ctx || max_len != ctx->cand_max_len) return fail(ctx, RT_EINVAL, "max_len mismatch");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    if (ctx->n_cand == 0) return RT_OK;
    if (seq) CK(cudaMemcpyAsync(seq, ctx->cand_seq.p, 4ULL * ctx->n_cand * max_len, cudaMemcpyDeviceToDevice, st));
    if (len) CK(cudaMemcpyAsync(len, ctx->cand_len.p, (size_t)ctx->n_cand, cudaMemcpyDeviceToDevice, st));
    return RT_OK;
}

}  // extern "C"

namespace {

// stage 1-4 of the solve pipeline for either receiver kind; leaves sorted
// records in recs/ridx/rkeys and returns their count
// keep_flags: the caller cleared the error word before kernels whose errors
// this call's final read-back reports with its own (no host sync of their own)
int solve_records(rt_ctx* ctx, d3 tx, const Receivers& R, bool grid, bool power, const EmParams& E,
                  int shard_index, int shard_count, long long* n_rec_out, long long* stats,
                  cudaStream_t st, bool keep_flags = false) {
    Cands C = cands_dev(ctx);
    SceneDev SD = scene_dev(ctx);
    long long nC = C.n;
    *n_rec_out = 0;
    if (!ctx->cand_sorted)   // the merge's candidate rank needs the (len, lex) order
        return fail(ctx, RT_ESTATE, "candidates of a sharded launch: install the union with "
                                    "rt_candidates_set first");
    if (nC == 0 || R.n == 0) return RT_OK;
    PROF_BEGIN(ST_FOOTPRINT);
    CK(ctx->images.reserve(24ULL * nC * C.max_len));
    k_images<<<nblk(nC, 256), 256, 0, st>>>(C, SD, tx, ctx->images.get<double>());
    CKL();
    long long W = 0;
    Segs G{nullptr, nullptr, nullptr, nullptr, nullptr, 0};
    if (grid) {
        CK(ctx->hps.reserve(sizeof(double) * 3 * HP_MAX * nC));
        CK(ctx->nhp.reserve(4ULL * nC));
        CK(ctx->row0.reserve(4ULL * nC));
        CK(ctx->counts.reserve(8ULL * (nC + 1)));
        CK(ctx->scan.reserve(8ULL * (nC + 1)));
        k_halfplanes<<<nblk(nC + 1, 128), 128, 0, st>>>(C, SD, ctx->images.get<double>(), R, shard_index,
                                                        shard_count, ctx->hps.get<double>(), ctx->nhp.get<int>(),
                                                        ctx->row0.get<int>(), ctx->counts.get<long long>());
        CKL();
        long long* cnt = ctx->counts.get<long long>();
        long long* seg_off = ctx->scan.get<long long>();
        RC(cub_call(ctx, [&](void* tmp, size_t& bytes) {
            return cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, seg_off, (int)(nC + 1), st);
        }));
        RC(fetch(ctx, seg_off + nC, 1, st));
        long long nS = ctx->hpin[0];
        CK(ctx->seg_cand.reserve(4ULL * std::max<long long>(nS, 1)));
        CK(ctx->seg_iy.reserve(4ULL * std::max<long long>(nS, 1)));
        CK(ctx->seg_ix0.reserve(4ULL * std::max<long long>(nS, 1)));
        CK(ctx->seg_cnt.reserve(8ULL * (nS + 1)));
        CK(ctx->item_off.reserve(8ULL * (nS + 1)));
        CK(cudaMemsetAsync(ctx->seg_cnt.get<long long>() + nS, 0, 8, st));
        if (nS > 0)
            k_segments<<<nblk(nS, 256), 256, 0, st>>>(nC, nS, ctx->hps.get<double>(), ctx->nhp.get<int>(),
                                                  ctx->row0.get<int>(), seg_off, R, shard_count,
                                                  ctx->seg_cand.get<int>(), ctx->seg_iy.get<int>(),
                                                  ctx->seg_ix0.get<int>(), ctx->seg_cnt.get<long long>());
        CKL();
        long long* sc = ctx->seg_cnt.get<long long>();
        long long* io = ctx->item_off.get<long long>();
        RC(cub_call(ctx, [&](void* tmp, size_t& bytes) {
            return cub::DeviceScan::ExclusiveSum(tmp, bytes, sc, io, (int)(nS + 1), st);
        }));
        RC(fetch(ctx, io + nS, 1, st));
        W = ctx->hpin[0];
        CK(ctx->chunk_seg.reserve(4ULL * ((W + 31) / 32 + 1)));
        if (nS > 0) {
            k_chunk_starts<<<nblk(nS, 256), 256, 0, st>>>(nS, io, ctx->chunk_seg.get<int>());
            CKL();
        }
        G = Segs{io, ctx->seg_cand.get<int>(), ctx->seg_iy.get<int>(), ctx->seg_ix0.get<int>(),
                 ctx->chunk_seg.get<int>(), nS};
        ctx->counters[7] = nS;
    } else {
        W = nC * R.n;
    }
    PROF_END(ST_FOOTPRINT);
    ctx->counters[4] = W;
    if (stats) stats[0] = W;
    if (W == 0) return RT_OK;
    if (ctx->pending_cap == 0) ctx->pending_cap = 1 << 20;
    if (ctx->rec_cap == 0) ctx->rec_cap = 1 << 20;
    unsigned long long* nr = reinterpret_cast<unsigned long long*>(ctx->ctrs.get<long long>()) + 1;
    // occluder cache: one TriRec index per (candidate, segment), -1 = none yet
    CK(ctx->occ_hint.reserve(4ULL * nC * (MAX_DEPTH + 1)));
    int* hints = RT_OCC_HINTS ? ctx->occ_hint.get<int>() : nullptr;
    long long n_pend = 0;
    long long fused_flags = 0;
    long long n_rec_known = -1;   // set when the fused pass's read-back already holds the final count
    if (RT_FUSED_SV && hints) {
        // solve + validation in one pass, thin warps' open items deferred to a
        // k_validate pass over that list; grow and rerun when a list is short
        PROF_BEGIN(ST_SOLVE);
        long long n_def = 0;
        bool fits = false;
        // deferral pays on long passes (C3: 37.5M items, solve + validate 4.73 -> 4.46 ms);
        // a short one is better off in one pass (C2 canyon: 1.4M items, 141 -> 114 us)
        const int defer_min = W >= RT_DEFER_MIN_ITEMS ? RT_VAL_DEFER : 0;
        for (int attempt = 0; attempt < 8; ++attempt) {
            CK(ctx->pending.reserve(sizeof(Pending) * ctx->pending_cap));
            CK(ctx->recs.reserve(sizeof(Rec) * ctx->rec_cap));
            CK(cudaMemsetAsync(ctx->ctrs.p, 0, 64, st));
            CK(cudaMemsetAsync(hints, 0xFF, 4ULL * nC * (MAX_DEPTH + 1), st));
            // error bits are sticky across a capacity rerun: an error of any attempt fails the call
            if (attempt == 0 && !keep_flags) RC(clear_flags(ctx, st));
            unsigned long long* ctr = reinterpret_cast<unsigned long long*>(ctx->ctrs.get<long long>());
            long long blocks = std::min<long long>((W + 127) / 128, (long long)ctx->n_sm * RT_SV_GRID);
            if (grid)
                k_solve_validate<true><<<(unsigned)blocks, 128, 0, st>>>(
                    C, SD, ctx->images.get<double>(), R, tx, W, G, bvh_dev(ctx), hints, defer_min,
                    ctx->recs.get<Rec>(), ctx->rec_cap, ctx->pending.get<Pending>(), ctx->pending_cap, ctr);
            else
                k_solve_validate<false><<<(unsigned)blocks, 128, 0, st>>>(
                    C, SD, ctx->images.get<double>(), R, tx, W, G, bvh_dev(ctx), hints, defer_min,
                    ctx->recs.get<Rec>(), ctx->rec_cap, ctx->pending.get<Pending>(), ctx->pending_cap, ctr);
            CKL();
            // the three counters and the error word in one read-back
            CK(cudaMemcpyAsync(ctx->hpin, ctr, 3 * sizeof(long long), cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(ctx->hpin + 3, ctx->dflag.p, sizeof(long long), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            n_pend = ctx->hpin[0];
            long long n_rec1 = ctx->hpin[1];
            n_def = ctx->hpin[2];
            fused_flags = ctx->hpin[3];
            bool grow = false;
            if ((unsigned long long)n_def > ctx->pending_cap) {
                while (ctx->pending_cap < (unsigned long long)n_def) ctx->pending_cap *= 2;
                grow = true;
            }
            if ((unsigned long long)(n_rec1 + n_def) > ctx->rec_cap) {
                while (ctx->rec_cap < (unsigned long long)(n_rec1 + n_def)) ctx->rec_cap *= 2;
                grow = true;
            }
            if (!grow) { fits = true; break; }
        }
        if (!fits) return fail(ctx, RT_ENOMEM, "record / deferred lists still short after 8 regrowths");
        PROF_END(ST_SOLVE);
        PROF_BEGIN(ST_VALIDATE);
        if (n_def > 0) {
            long long b2 = std::min<long long>((n_def + 127) / 128, (long long)ctx->n_sm * 32);
            k_validate<false><<<(unsigned)b2, 128, 0, st>>>(C, SD, ctx->images.get<double>(), R, tx,
                                                            bvh_dev(ctx), ctx->pending.get<Pending>(),
                                                            n_def, E, ctx->recs.get<Rec>(), nr, hints);
            CKL();
        } else {   // nothing deferred: the read-back above is final (no second host sync)
            RC(flags_status(ctx, fused_flags));
            n_rec_known = ctx->hpin[1];
        }
        if (stats) stats[1] = n_pend;
        ctx->counters[5] = n_pend;
    } else {
    // geometric solve with compaction; grow and retry when the buffer is short
    for (int attempt = 0; attempt < 8; ++attempt) {
        CK(ctx->pending.reserve(sizeof(Pending) * ctx->pending_cap));
        CK(cudaMemsetAsync(ctx->ctrs.p, 0, 64, st));
        unsigned long long* np = reinterpret_cast<unsigned long long*>(ctx->ctrs.get<long long>());
        long long blocks = std::min<long long>((W + 255) / 256, (long long)ctx->n_sm * 32);
        PROF_BEGIN(ST_SOLVE);
        if (grid)
            k_solve<true><<<(unsigned)blocks, 256, 0, st>>>(C, SD, ctx->images.get<double>(), R, tx, W, G,
                                                            ctx->pending.get<Pending>(), np, ctx->pending_cap);
        else
            k_solve<false><<<(unsigned)blocks, 256, 0, st>>>(C, SD, ctx->images.get<double>(), R, tx, W, G,
                                                             ctx->pending.get<Pending>(), np, ctx->pending_cap);
        CKL();
        PROF_END(ST_SOLVE);
        RC(fetch(ctx, np, 1, st));
        n_pend = ctx->hpin[0];
        if ((unsigned long long)n_pend <= ctx->pending_cap) break;
        while (ctx->pending_cap < (unsigned long long)n_pend) ctx->pending_cap *= 2;
    }
    if ((unsigned long long)n_pend > ctx->pending_cap)
        return fail(ctx, RT_ENOMEM, "pending list still short after 8 regrowths");
    if (stats) stats[1] = n_pend;
    ctx->counters[5] = n_pend;
    if (n_pend == 0) return RT_OK;
    CK(ctx->recs.reserve(sizeof(Rec) * n_pend));
    CK(cudaMemsetAsync(ctx->ctrs.p, 0, 64, st));
    if (!keep_flags) RC(clear_flags(ctx, st));
    long long vblocks = std::min<long long>((n_pend + 127) / 128, (long long)ctx->n_sm * 32);
    PROF_BEGIN(ST_VALIDATE);
    if (hints) CK(cudaMemsetAsync(hints, 0xFF, 4ULL * nC * (MAX_DEPTH + 1), st));
    if (RT_VAL_DEFER > 0 && hints) {
        CK(ctx->deferred.reserve(4ULL * n_pend));
        unsigned long long* nd = reinterpret_cast<unsigned long long*>(ctx->ctrs.get<long long>()) + 2;
        k_validate<false><<<(unsigned)vblocks, 128, 0, st>>>(C, SD, ctx->images.get<double>(), R, tx,
                                                             bvh_dev(ctx), ctx->pending.get<Pending>(),
                                                             n_pend, E, ctx->recs.get<Rec>(), nr, hints,
                                                             nullptr, RT_VAL_DEFER, ctx->deferred.get<int>(), nd);
        CKL();
        RC(fetch(ctx, nd, 1, st));
        long long n_def = ctx->hpin[0];
        if (n_def > 0) {
            long long b2 = std::min<long long>((n_def + 127) / 128, (long long)ctx->n_sm * 32);
            k_validate<false><<<(unsigned)b2, 128, 0, st>>>(C, SD, ctx->images.get<double>(), R, tx,
                                                            bvh_dev(ctx), ctx->pending.get<Pending>(),
                                                            n_def, E, ctx->recs.get<Rec>(), nr, hints,
                                                            ctx->deferred.get<int>());
            CKL();
        }
    } else {
        k_validate<false><<<(unsigned)vblocks, 128, 0, st>>>(C, SD, ctx->images.get<double>(), R, tx,
                                                             bvh_dev(ctx), ctx->pending.get<Pending>(),
                                                             n_pend, E, ctx->recs.get<Rec>(), nr, hints);
        CKL();
    }
    }
#ifdef RT_VALIDATE_STATS
    {
        unsigned long long hv[8];
        cudaMemcpyFromSymbol(hv, g_vstats, sizeof(hv));
        fprintf(stderr, "validate stats: items %llu rx-hint hits %llu other hint hits %llu traversals %llu "
                "blocked %llu fused items %llu survivors %llu\n", hv[0], hv[1], hv[4], hv[2], hv[3], hv[5], hv[6]);
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(g_vstats, z, sizeof(z));
    }
#endif
    long long n_rec = n_rec_known;
    if (n_rec < 0) {
        RC(fetch_and_flags(ctx, nr, 1, st));   // record count + the validation's error word
        n_rec = ctx->hpin[0];
    }
    if (power && n_rec > 0) {
        k_rec_powers<<<nblk(n_rec, 128), 128, 0, st>>>(C, SD, ctx->images.get<double>(), R, tx, E,
                                                       ctx->recs.get<Rec>(), n_rec);
        CKL();
    }
    PROF_END(ST_VALIDATE);
    ctx->counters[6] = n_rec;
    if (stats) stats[2] = n_rec;
    if (n_rec == 0) return RT_OK;
    PROF_BEGIN(ST_REC_SORT);
    CK(ctx->rkeys.reserve(8 * n_rec));
    CK(ctx->rkeys_alt.reserve(8 * n_rec));
    CK(ctx->ridx.reserve(4 * n_rec));
    CK(ctx->ridx_alt.reserve(4 * n_rec));
    // a one-CTA sort takes compact keys (fewer radix passes) and expands them
    int cb = bits_for(nC);   // compact keys: (rx, order, cand) in fewer radix passes
    k_rec_keys<<<nblk(n_rec, 256), 256, 0, st>>>(ctx->recs.get<Rec>(), n_rec, ctx->rkeys_alt.get<unsigned long long>(),
                                                ctx->ridx_alt.get<int>(), cb);
    CKL();
    unsigned long long* kin = ctx->rkeys_alt.get<unsigned long long>();
    unsigned long long* kout = ctx->rkeys.get<unsigned long long>();
    int* vin = ctx->ridx_alt.get<int>();
    int* vout = ctx->ridx.get<int>();
    int end_bit = (cb > 0 ? cb + 4 : 36) + bits_for(R.n);
    RC(sort_pairs(ctx, kin, kout, vin, vout, n_rec, 0, std::min(end_bit, 64), st, cb));
    PROF_END(ST_REC_SORT);
    *n_rec_out = n_rec;
    return RT_OK;
}

int em_upload(rt_ctx* ctx, const double* tx_rows, const double* probe_rows, const double* slants,
              const double* offsets_w, int n_el, cudaStream_t st, double** d_tx, double** d_probe,
              double** d_sl, double** d_off) {
    size_t n = 18 + (size_t)n_el * 4;
    std::vector<double> h(n, 0.0);
    for (int i = 0; i < 9; ++i) h[i] = tx_rows ? tx_rows[i] : (i % 4 == 0 ? 1.0 : 0.0);
    for (int i = 0; i < 9; ++i) h[9 + i] = probe_rows ? probe_rows[i] : (i % 4 == 0 ? 1.0 : 0.0);
    for (int e = 0; e < n_el; ++e) h[18 + e] = slants ? slants[e] : 0.0;
    for (int e = 0; e < 3 * n_el; ++e) h[18 + n_el + e] = offsets_w ? offsets_w[e] : 0.0;
    CK(ctx->em_small.reserve(8 * n));
    RC(h2d_staged(ctx->device, ctx->em_small.p, h.data(), (int64_t)(8 * n), st));   // no host sync
    double* b = ctx->em_small.get<double>();
    *d_tx = b;
    *d_probe = b + 9;
    *d_sl = b + 18;
    *d_off = b + 18 + n_el;
    return RT_OK;
}

}  // namespace

extern "C" {

int rt_paths(rt_ctx* ctx, const double* tx, const double* rx, int64_t n_rx, int64_t* n_paths_out,
             void* stream) {
    if (!ctx || !tx || n_rx < 0) return fail(ctx, RT_EINVAL, "bad path arguments");
    if (!ctx->bvh_ready) return fail(ctx, RT_ESTATE, "rt_bvh_build has not run");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    d3 T = d3{tx[0], tx[1], tx[2]};
    if (n_rx > 0 && !rx) return fail(ctx, RT_EINVAL, "bad path arguments");
    if (n_rx > 0) {   // host receiver positions: staged in on the stream
        cudaPointerAttributes at{};
        bool host_in = cudaPointerGetAttributes(&at, rx) != cudaSuccess || at.type != cudaMemoryTypeDevice;
        cudaGetLastError();
        if (host_in) {
            CK(ctx->rx_up.reserve(24ULL * n_rx));
            RC(h2d_staged(ctx->device, ctx->rx_up.p, rx, 24LL * n_rx, st));
            rx = ctx->rx_up.get<double>();
        }
    }
    Receivers R;
    R.pts = rx;
    R.ox = R.oy = R.cell = R.height = 0.0;
    R.nx = R.ny = 0;
    R.n = n_rx;
    ctx->n_paths = 0;
    ctx->paths_max_rx = 0;
    ctx->path_L = ctx->cand_max_len;
    if (n_rx == 0) {
        if (n_paths_out) *n_paths_out = 0;
        return RT_OK;
    }
    EmParams E{};
    long long n_rec = 0;
    RC(solve_records(ctx, T, R, false, false, E, 0, 1, &n_rec, nullptr, st));
    CK(ctx->keep.reserve((size_t)std::max<long long>(n_rec, 1)));
    CK(ctx->losbuf.reserve((size_t)n_rx));
    CK(ctx->heads.reserve(4ULL * n_rx));
    CK(ctx->pcounts.reserve(4ULL * (n_rx + 1)));
    CK(ctx->poffs.reserve(4ULL * (n_rx + 1)));
    RC(clear_flags(ctx, st));
    k_los<false><<<nblk(n_rx, 128), 128, 0, st>>>(R, T, bvh_dev(ctx), scene_dev(ctx), E, 0, 1,
                                                  ctx->losbuf.get<unsigned char>(), nullptr,
                                                  reinterpret_cast<int*>(ctx->dflag.get<long long>()));
    CKL();
    // the LOS error flags travel back with the path count (one host round trip)
    CK(cudaMemcpyAsync(ctx->hpin + 1, ctx->dflag.p, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(cudaMemsetAsync(ctx->heads.p, 0xFF, 4ULL * n_rx, st));
    if (n_rec > 0) {
        k_merge<false><<<nblk(n_rec, 128), 128, 0, st>>>(cands_dev(ctx), scene_dev(ctx), ctx->images.get<double>(),
                                                        R, T, ctx->recs.get<Rec>(), ctx->ridx.get<int>(),
                                                        ctx->rkeys.get<unsigned long long>(), n_rec,
                                                        ctx->keep.get<unsigned char>(), nullptr);
        CKL();
        k_seg_heads<<<nblk(n_rec, 256), 256, 0, st>>>(ctx->rkeys.get<unsigned long long>(), n_rec,
                                                      ctx->heads.get<int>());
        CKL();
    }
    int* cnt = ctx->pcounts.get<int>();
    int* off = ctx->poffs.get<int>();
    CK(cudaMemsetAsync(cnt + n_rx, 0, 4, st));
    int* dmax = reinterpret_cast<int*>(ctx->ctrs.get<long long>() + 26);
    CK(cudaMemsetAsync(dmax, 0, 4, st));
    k_path_counts<<<nblk(n_rx, 128), 128, 0, st>>>(n_rx, ctx->heads.get<int>(), ctx->rkeys.get<unsigned long long>(),
                                                   n_rec, ctx->keep.get<unsigned char>(),
                                                   ctx->losbuf.get<unsigned char>(), cnt, dmax);
    CKL();
    RC(cub_call(ctx, [&](void* tmp, size_t& bytes) {
        return cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, off, (int)(n_rx + 1), st);
    }));
    // path count, (flags at hpin[1]), the largest per-receiver count: one host sync
    CK(cudaMemcpyAsync(ctx->hpin, off + n_rx, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ctx->hpin + 2, dmax, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->paths_max_rx = reinterpret_cast<int*>(ctx->hpin + 2)[0];
    {
        long long f = ctx->hpin[1];
        if (f & 1) return fail(ctx, RT_ECUDA, "BVH traversal stack overflow");
        if (f & 4) return fail(ctx, RT_ECOINCIDE, "transmitter and probe/receiver coincide");
    }
    long long P = reinterpret_cast<int*>(ctx->hpin)[0];
    int L = ctx->path_L;
    size_t Pn = (size_t)std::max<long long>(P, 1);
    CK(ctx->p_rx.reserve(4 * Pn));
    CK(ctx->p_cand.reserve(4 * Pn));
    CK(ctx->p_order.reserve(Pn));
    CK(ctx->p_seq.reserve(4 * Pn * L));
    CK(ctx->p_verts.reserve(24 * Pn * (L + 2)));
    CK(ctx->p_len.reserve(8 * Pn));
    CK(ctx->p_delay.reserve(8 * Pn));
    CK(ctx->p_kdep.reserve(24 * Pn));
    CK(ctx->p_karr.reserve(24 * Pn));
    CK(ctx->p_nrm.reserve(24 * Pn * L));
    CK(ctx->p_cos.reserve(8 * Pn * L));
    PathTable PT;
    PT.rx = ctx->p_rx.get<int>();
    PT.cand = ctx->p_cand.get<int>();
    PT.order = ctx->p_order.get<signed char>();
    PT.seq = ctx->p_seq.get<int>();
    PT.verts = ctx->p_verts.get<double>();
    PT.length = ctx->p_len.get<double>();
    PT.delay = ctx->p_delay.get<double>();
    PT.kdep = ctx->p_kdep.get<double>();
    PT.karr = ctx->p_karr.get<double>();
    PT.nrm = ctx->p_nrm.get<double>();
    PT.cosv = ctx->p_cos.get<double>();
    PT.L = L;
    if (P > 0) {
        k_emit_paths<<<nblk(32 * n_rx, 128), 128, 0, st>>>(cands_dev(ctx), scene_dev(ctx), ctx->images.get<double>(), R, T,
                                                     ctx->recs.get<Rec>(), ctx->ridx.get<int>(),
                                                     ctx->rkeys.get<unsigned long long>(), n_rec,
                                                     ctx->keep.get<unsigned char>(), ctx->losbuf.get<unsigned char>(),
                                                     ctx->heads.get<int>(), off, PT);
        CKL();
    }
    ctx->n_paths = P;
    if (n_paths_out) *n_paths_out = P;
    return RT_OK;
}

int rt_paths_fibonacci(rt_ctx* ctx, const double* tx, int64_t n_rays, int max_depth, const double* rx,
                       int64_t n_rx, int64_t* n_cand_out, int64_t* n_bounces_out, int64_t* n_paths_out,
                       void* stream) {
    if (!ctx || !tx || n_rays < 1 || max_depth < 1)
        return fail(ctx, RT_EINVAL, "need num_rays >= 1 and max_depth >= 1");
    if (!ctx->bvh_ready) return fail(ctx, RT_ESTATE, "rt_bvh_build has not run");
    if (ctx->n_prims == 0) {   // no geometry: LOS only (tracer.prepare_candidates' empty set)
        RC(sort_unique_candidates(ctx, 0, 1, ST(stream)));
        if (n_cand_out) *n_cand_out = 0;
        if (n_bounces_out) *n_bounces_out = 0;
    } else {
        RC(launch_impl(ctx, tx, n_rays, 0, n_rays, 0, 1, max_depth, nullptr, n_cand_out, n_bounces_out, stream));
    }
    return rt_paths(ctx, tx, rx, n_rx, n_paths_out, stream);
}

int rt_paths_get(rt_ctx* ctx, int32_t* rx_index, int32_t* cand, int8_t* order, int32_t* seq,
                 double* vertices, double* length, double* delay, double* k_dep, double* k_arr,
                 double* normals, double* cos_inc, void* stream) {
    if (!ctx) return RT_EINVAL;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    size_t P = ctx->n_paths, L = ctx->path_L;
    if (!P) return RT_OK;
    void* dsts[11] = {rx_index, cand, order, seq, vertices, length, delay, k_dep, k_arr, normals, cos_inc};
    const DevBuf* srcs[11] = {&ctx->p_rx, &ctx->p_cand, &ctx->p_order, &ctx->p_seq, &ctx->p_verts, &ctx->p_len,
                              &ctx->p_delay, &ctx->p_kdep, &ctx->p_karr, &ctx->p_nrm, &ctx->p_cos};
    const size_t bytes[11] = {4 * P, 4 * P, P, 4 * P * L, 24 * P * (L + 2), 8 * P, 8 * P, 24 * P, 24 * P,
                              24 * P * L, 8 * P * L};
    CopyBatch B{};
    size_t most = 0;
    for (int k = 0; k < 11; ++k) {
        B.s[k] = CopySeg{srcs[k]->get<unsigned char>(), static_cast<unsigned char*>(dsts[k]), (long long)bytes[k]};
        if (dsts[k]) most = std::max(most, bytes[k]);
    }
    if (!most) return RT_OK;
    dim3 grid((unsigned)std::min<long long>(nblk((long long)(most + 3) / 4, 256), 4096), 11);
    k_copy_batch<<<grid, 256, 0, st>>>(B);
    CKL();
    return RT_OK;
}

int rt_transfer(rt_ctx* ctx, int64_t n_paths, int max_len, const int8_t* order, const int32_t* seq,
                const int32_t* interaction_mat, const double* vertices, const double* normals, const double* cos_inc,
                const double* length, const double* delay, const double* tx_rows,
                const double* rx_rows, int tx_pattern, int rx_pattern, const double* tx_slants,
                int n_tx_slants, const double* rx_slants, int n_rx_slants, const double* eta,
                int n_mat, double wavelength, double frequency_hz, double* a_out, void* stream) {
    if (!ctx || n_paths < 0 || max_len < 1 || n_tx_slants < 1 || n_rx_slants < 1)
        return fail(ctx, RT_EINVAL, "bad transfer arguments");
    if (tx_pattern < 0 || tx_pattern > 4 || rx_pattern < 0 || rx_pattern > 4)
        return fail(ctx, RT_EINVAL, "unknown antenna pattern");
    if (n_paths == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    (void)n_mat;
    TransferArgs A{n_paths, max_len, (const signed char*)order, seq, vertices, normals, cos_inc, length,
                   delay, tx_rows, rx_rows, tx_pattern, rx_pattern, tx_slants, n_tx_slants,
                   rx_slants, n_rx_slants, eta, ctx->prim_mat.get<int>(), interaction_mat, wavelength,
                   frequency_hz};
    // without interaction_mat the materials come from the scene; a scene without
    // primitives has only LOS paths, which read no material
    k_transfer<<<nblk(n_paths * n_tx_slants, 128), 128, 0, ST(stream)>>>(A, a_out);
    CKL();
    return RT_OK;
}

int rt_transfer_bwd(rt_ctx* ctx, int64_t n_paths, int max_len, const int8_t* order,
                    const int32_t* seq, const int32_t* interaction_mat, const double* vertices, const double* normals,
                    const double* cos_inc, const double* length, const double* delay,
                    const double* tx_rows, const double* rx_rows, int tx_pattern, int rx_pattern,
                    const double* tx_slants, int n_tx_slants, const double* rx_slants,
                    int n_rx_slants, const double* eta, int n_mat, double wavelength,
                    double frequency_hz, const double* grad_a, double* grad_eta, void* stream) {
    if (!ctx || n_paths < 0 || max_len < 1 || n_tx_slants < 1 || n_rx_slants < 1)
        return fail(ctx, RT_EINVAL, "bad transfer arguments");
    if (n_paths == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    TransferArgs A{n_paths, max_len, (const signed char*)order, seq, vertices, normals, cos_inc, length,
                   delay, tx_rows, rx_rows, tx_pattern, rx_pattern, tx_slants, n_tx_slants,
                   rx_slants, n_rx_slants, eta, ctx->prim_mat.get<int>(), interaction_mat, wavelength,
                   frequency_hz};
    // without interaction_mat the materials come from the scene; a scene without
    // primitives has only LOS paths, which read no material
    if (n_mat < 1) return fail(ctx, RT_EINVAL, "need n_mat >= 1");
    long long n = n_paths * n_tx_slants * n_rx_slants;
    CK(ctx->adj.reserve(sizeof(double2) * (size_t)n * max_len));
    double2* contrib = ctx->adj.get<double2>();
    k_transfer_bwd<<<nblk(n, 128), 128, 0, ST(stream)>>>(A, grad_a, contrib);
    CKL();
    k_grad_eta_reduce<<<n_mat, ADJ_BLOCK, 0, ST(stream)>>>(A, contrib, grad_eta);
    CKL();
    return RT_OK;
}

int rt_coverage(rt_ctx* ctx, const double* tx, double origin_x, double origin_y, double cell_size,
                int64_t nx, int64_t ny, double height, const double* tx_rows,
                const double* probe_rows, int tx_pattern, const double* slants,
                const double* offsets_w, int n_el, int tx_mode, const double* eta, int n_mat,
                double wavelength, double frequency_hz, int shard_index, int shard_count,
                double* gains_out, int64_t* stats_out, void* stream) {
    if (!ctx || !tx || nx < 0 || ny < 0 || n_el < 1 || shard_count < 1 || shard_index < 0 ||
        shard_index >= shard_count || !(cell_size > 0.0))
        return fail(ctx, RT_EINVAL, "bad coverage arguments");
    if (tx_mode != 0 && tx_mode != 1) return fail(ctx, RT_EINVAL, "unknown tx_mode");
    if (!ctx->bvh_ready) return fail(ctx, RT_ESTATE, "rt_bvh_build has not run");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    (void)n_mat;
    d3 T = d3{tx[0], tx[1], tx[2]};
    Receivers R;
    R.pts = nullptr;
    R.ox = origin_x;
    R.oy = origin_y;
    R.cell = cell_size;
    R.height = height;
    R.nx = nx;
    R.ny = ny;
    R.n = nx * ny;
    long long stats[8] = {0, 0, 0, R.n, ctx->n_cand, 0, 0, 0};
    if (R.n == 0) {
        if (stats_out) memcpy(stats_out, stats, sizeof stats);
        return RT_OK;
    }
    EmParams E;
    double *d_tx, *d_probe, *d_sl, *d_off;
    RC(em_upload(ctx, tx_rows, probe_rows, slants, offsets_w, n_el, st, &d_tx, &d_probe, &d_sl, &d_off));
    E.eta = eta;
    E.tx_rows = d_tx;
    E.probe_rows = d_probe;
    E.slants = d_sl;
    E.offsets_w = d_off;
    E.n_el = n_el;
    E.tx_pattern = tx_pattern;
    E.tx_mode = tx_mode;
    E.wavelength = wavelength;
    E.frequency = frequency_hz;
    RC(clear_flags(ctx, st));
    PROF_BEGIN(ST_LOS);
    k_los<true><<<nblk(R.n, 128), 128, 0, st>>>(R, T, bvh_dev(ctx), scene_dev(ctx), E, shard_index,
                                                shard_count, nullptr, gains_out,
                                                reinterpret_cast<int*>(ctx->dflag.get<long long>()));
    CKL();
    PROF_END(ST_LOS);
    // the LOS kernel's error bits are reported with solve_records' read-back (no sync here)
    long long n_rec = 0;
    RC(solve_records(ctx, T, R, true, true, E, shard_index, shard_count, &n_rec, stats, st, true));
    if (n_rec > 0) {
        CK(ctx->keep.reserve((size_t)n_rec));
        PROF_BEGIN(ST_MERGE);
        k_merge<true><<<nblk(n_rec, 128), 128, 0, st>>>(cands_dev(ctx), scene_dev(ctx), ctx->images.get<double>(),
                                                       R, T, ctx->recs.get<Rec>(), ctx->ridx.get<int>(),
                                                       ctx->rkeys.get<unsigned long long>(), n_rec,
                                                       ctx->keep.get<unsigned char>(), gains_out);
        CKL();
        PROF_END(ST_MERGE);
    }
    if (stats_out) memcpy(stats_out, stats, sizeof stats);
    return RT_OK;
}

int rt_coverage_fibonacci(rt_ctx* ctx, const double* tx, int64_t n_rays, int max_depth, double origin_x,
                          double origin_y, double cell_size, int64_t nx, int64_t ny, double height,
                          const double* tx_rows, const double* probe_rows, int tx_pattern, const double* slants,
                          const double* offsets_w, int n_el, int tx_mode, const double* eta, int n_mat,
                          double wavelength, double frequency_hz, double* gains_out, int64_t* stats_out,
                          int64_t* n_bounces_out, void* stream) {
    if (!ctx || !tx || n_rays < 1 || max_depth < 1)
        return fail(ctx, RT_EINVAL, "need num_rays >= 1 and max_depth >= 1");
    if (!ctx->bvh_ready) return fail(ctx, RT_ESTATE, "rt_bvh_build has not run");
    if (n_bounces_out) *n_bounces_out = 0;
    if (ctx->n_prims == 0) {   // no geometry: LOS only
        RC(sort_unique_candidates(ctx, 0, 1, ST(stream)));
    } else {
        RC(launch_impl(ctx, tx, n_rays, 0, n_rays, 0, 1, max_depth, nullptr, nullptr, n_bounces_out, stream));
    }
    return rt_coverage(ctx, tx, origin_x, origin_y, cell_size, nx, ny, height, tx_rows, probe_rows, tx_pattern,
                       slants, offsets_w, n_el, tx_mode, eta, n_mat, wavelength, frequency_hz, 0, 1, gains_out,
                       stats_out, stream);
}

int rt_solve_pairs(rt_ctx* ctx, int64_t n, int max_len, const double* tx_pos,
                   const double* rx_pos, const int32_t* seq, const int8_t* len, uint8_t* valid,
                   double* vertices, double* length, double* delay, double* k_dep, double* k_arr,
                   double* normals, double* cos_inc, int32_t* seq_out, int8_t* order_out,
                   void* stream) {
    if (!ctx || n < 0 || max_len < 1 || max_len > MAX_DEPTH)
        return fail(ctx, RT_EINVAL, "bad solve arguments");
    if (!ctx->bvh_ready) return fail(ctx, RT_ESTATE, "rt_bvh_build has not run");
    if (n == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    CK(ctx->p_rx.reserve(4ULL * n));
    CK(ctx->p_cand.reserve(4ULL * n));
    PathTable PT;
    PT.rx = ctx->p_rx.get<int>();
    PT.cand = ctx->p_cand.get<int>();
    PT.order = reinterpret_cast<signed char*>(order_out);
    PT.seq = seq_out;
    PT.verts = vertices;
    PT.length = length;
    PT.delay = delay;
    PT.kdep = k_dep;
    PT.karr = k_arr;
    PT.nrm = normals;
    PT.cosv = cos_inc;
    PT.L = max_len;
    RC(clear_flags(ctx, st));
    k_solve_pairs<<<nblk(n, 128), 128, 0, st>>>(scene_dev(ctx), bvh_dev(ctx), n, max_len, tx_pos, rx_pos,
                                                seq, (const signed char*)len, valid, PT);
    CKL();
    return check_flags(ctx, st);
}

int rt_transfer_jvp(rt_ctx* ctx, int64_t n_paths, int max_len, const int8_t* order,
                    const int32_t* seq, const double* vertices, const double* normals,
                    const double* tx_pos, const double* rx_pos, const double* tx_ypr,
                    const double* rx_ypr, int tx_pattern, int rx_pattern, const double* tx_slants,
                    int n_tx_slants, const double* rx_slants, int n_rx_slants, const double* eta,
                    int n_mat, double wavelength, double frequency_hz, double* a_out,
                    double* jac_out, void* stream) {
    if (!ctx || n_paths < 0 || max_len < 1 || n_tx_slants < 1 || n_rx_slants < 1)
        return fail(ctx, RT_EINVAL, "bad transfer arguments");
    if (tx_pattern < 0 || tx_pattern > 4 || rx_pattern < 0 || rx_pattern > 4)
        return fail(ctx, RT_EINVAL, "unknown antenna pattern");
    if (n_paths == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    (void)n_mat;
    JvpArgs A{n_paths, max_len, (const signed char*)order, seq, vertices, normals, tx_pos, rx_pos,
              tx_ypr, rx_ypr, tx_pattern, rx_pattern, tx_slants, n_tx_slants, rx_slants,
              n_rx_slants, eta, ctx->prim_mat.get<int>(), wavelength, frequency_hz};
    long long n = n_paths * n_tx_slants * NJ;
    k_transfer_jvp<<<nblk(n, 64), 64, 0, ST(stream)>>>(A, a_out, jac_out);
    CKL();
    return RT_OK;
}

int rt_l2_probe(rt_ctx* ctx, int64_t bytes, int iters, double* gbs_out, void* stream) {
    if (!ctx || bytes < 4096 || iters < 1 || !gbs_out) return fail(ctx, RT_EINVAL, "bad probe arguments");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    CK(ctx->probe.reserve((size_t)bytes + 64));
    CK(cudaMemsetAsync(ctx->probe.p, 0, (size_t)bytes + 64, st));
    long long n4 = bytes / 16;
    const float4* buf = ctx->probe.get<float4>();
    float* sink = reinterpret_cast<float*>(ctx->probe.get<char>() + (bytes / 16) * 16);
    unsigned grid = (unsigned)ctx->n_sm * 8;
    k_l2_probe<<<grid, 256, 0, st>>>(buf, n4, 2, sink);   // warm L2
    CKL();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, st));
    k_l2_probe<<<grid, 256, 0, st>>>(buf, n4, iters, sink);
    CKL();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *gbs_out = (double)n4 * 16.0 * iters / (ms * 1e-3) / 1e9;
    return RT_OK;
}

int rt_fresnel(rt_ctx* ctx, int64_t n, const double* eta, const double* cos_theta, double* r_te,
               double* r_tm, void* stream) {
    if (!ctx || n < 0 || (n > 0 && (!eta || !cos_theta || !r_te || !r_tm)))
        return fail(ctx, RT_EINVAL, "bad fresnel arguments");
    if (n == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    k_fresnel<<<nblk(n, 256), 256, 0, ST(stream)>>>(n, eta, cos_theta, r_te, r_tm);
    CKL();
    return RT_OK;
}

int rt_microbench(rt_ctx* ctx, int kind, double* value_out, void* stream) {
    if (!ctx || !value_out || kind < RT_MB_FP32 || kind > RT_MB_L2)
        return fail(ctx, RT_EINVAL, "bad microbenchmark arguments");
    if (kind == RT_MB_L2) return rt_l2_probe(ctx, 48LL << 20, 64, value_out, stream);
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    const unsigned grid = (unsigned)ctx->n_sm * 8;   // 8 x 256 threads = 64 warps per SM
    const long long threads = (long long)grid * 256;
    CK(ctx->probe.reserve((size_t)grid * MB_L1_SLICE + 64));
    float* sink = reinterpret_cast<float*>(ctx->probe.get<char>() + (size_t)grid * MB_L1_SLICE);
    if (kind == RT_MB_L1) CK(cudaMemsetAsync(ctx->probe.p, 0, (size_t)grid * MB_L1_SLICE, st));
    auto run = [&](int iters) {
        if (kind == RT_MB_FP32) k_mb_ffma<<<grid, 256, 0, st>>>(iters, sink);
        else if (kind == RT_MB_ISSUE) k_mb_issue<<<grid, 256, 0, st>>>(iters, sink);
        else if (kind == RT_MB_FP64) k_mb_dfma<<<grid, 256, 0, st>>>(iters, reinterpret_cast<double*>(sink));
        else k_mb_l1<<<grid, 256, 0, st>>>(ctx->probe.get<float4>(), iters, sink);
    };
    const int iters = kind == RT_MB_FP64 ? 400 : kind == RT_MB_L1 ? 2000 : 2000;
    run(iters / 10);   // warm-up (clocks, L1 fill)
    CKL();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, st));
    run(iters);
    CKL();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    double sec = ms * 1e-3;
    double ops = (double)threads * iters * MB_UNROLL * MB_CHAINS;   // FMAs (or FFMA instructions)
    if (kind == RT_MB_FP32 || kind == RT_MB_FP64) *value_out = 2.0 * ops / sec / 1e12;   // TFLOP/s
    else if (kind == RT_MB_ISSUE) *value_out = ops / 32.0 / sec / 1e9;                    // Gwarp-inst/s
    else *value_out = (double)grid * MB_L1_SLICE * iters / sec / 1e9;                     // GB/s
    return RT_OK;
}

int rt_set_profiling(rt_ctx* ctx, int flags) {
    if (!ctx) return RT_EINVAL;
    ctx->prof = flags;
    for (int i = 0; i < RT_NSTAGE; ++i) ctx->ev_used[i] = false;
    return RT_OK;
}

int rt_get_profile(rt_ctx* ctx, double* ms_out, int64_t* counters_out) {
    if (!ctx) return RT_EINVAL;
    CK(cudaSetDevice(ctx->device));
    RC(tree_diagnostics(ctx, 0));
    for (int i = 0; i < RT_NSTAGE; ++i) {
        double v = -1.0;
        if (ctx->ev_used[i] && ctx->ev[i][0] && ctx->ev[i][1]) {
            float ms = 0.f;
            CK(cudaEventSynchronize(ctx->ev[i][1]));
            CK(cudaEventElapsedTime(&ms, ctx->ev[i][0], ctx->ev[i][1]));
            v = ms;
        }
        if (ms_out) ms_out[i] = v;
        if (counters_out) counters_out[i] = ctx->counters[i];
    }
    return RT_OK;
}

}  // extern "C"

extern "C" {

int rt_gains_synthetic(rt_ctx* ctx, int64_t n_paths, int n_tx_slants, int n_rx_slants,
                       const double* base, const int32_t* tx_dev, const int32_t* rx_dev,
                       const double* k_dep, const double* k_arr, int n_tx_el,
                       const double* off_tx_w, const int32_t* tx_slant_index, int n_rx_el,
                       const double* off_rx_w, const int32_t* rx_slant_index, double wavelength,
                       double* a_out, void* stream) {
    if (!ctx || n_paths < 0 || n_tx_slants < 1 || n_rx_slants < 1 || n_tx_el < 1 || n_rx_el < 1 ||
        !(wavelength > 0.0))
        return fail(ctx, RT_EINVAL, "bad synthetic-gains arguments");
    long long n = (long long)n_paths * n_tx_el * n_rx_el;
    if (n == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    k_gains_synth<<<nblk(n, 256), 256, 0, ST(stream)>>>(n_paths, n_tx_slants, n_rx_slants, base, tx_dev, rx_dev,
                                                        k_dep, k_arr, n_tx_el, off_tx_w, tx_slant_index,
                                                        n_rx_el, off_rx_w, rx_slant_index, wavelength, a_out);
    CKL();
    return RT_OK;
}

int rt_gains(rt_ctx* ctx, int64_t n_paths, int max_len, const int32_t* tx_dev, const int32_t* rx_dev,
             const int8_t* order, const int32_t* seq, const int32_t* interaction_mat,
             const double* vertices, const double* normals, const double* cos_inc, const double* length,
             const double* delay, const double* k_dep, const double* k_arr, const double* tx_rows,
             const double* rx_rows, int tx_pattern, int rx_pattern, const double* tx_slants,
             int n_tx_slants, const double* rx_slants, int n_rx_slants, const double* eta, int n_mat,
             int n_tx_el, const double* off_tx_w, const int32_t* tx_slant_index, int n_rx_el,
             const double* off_rx_w, const int32_t* rx_slant_index, double wavelength,
             double frequency_hz, double* a_out, void* stream) {
    if (!ctx || n_paths < 0 || max_len < 1 || n_tx_slants < 1 || n_rx_slants < 1 || n_tx_el < 1 ||
        n_rx_el < 1 || !(wavelength > 0.0) || !tx_dev || !rx_dev)
        return fail(ctx, RT_EINVAL, "bad gains arguments");
    if (tx_pattern < 0 || tx_pattern > 4 || rx_pattern < 0 || rx_pattern > 4)
        return fail(ctx, RT_EINVAL, "unknown antenna pattern");
    if (n_paths == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    (void)n_mat;
    cudaStream_t st = ST(stream);
    CK(ctx->gbase.reserve(16ULL * n_paths * n_tx_slants * n_rx_slants));
    double* base = ctx->gbase.get<double>();
    TransferArgs A{n_paths, max_len, (const signed char*)order, seq, vertices, normals, cos_inc, length,
                   delay, tx_rows, rx_rows, tx_pattern, rx_pattern, tx_slants, n_tx_slants,
                   rx_slants, n_rx_slants, eta, ctx->prim_mat.get<int>(), interaction_mat, wavelength,
                   frequency_hz, tx_dev, rx_dev};
    k_transfer<<<nblk(n_paths * n_tx_slants, 128), 128, 0, st>>>(A, base);
    CKL();
    long long n = (long long)n_paths * n_tx_el * n_rx_el;
    k_gains_synth<<<nblk(n, 256), 256, 0, st>>>(n_paths, n_tx_slants, n_rx_slants, base, tx_dev, rx_dev,
                                                k_dep, k_arr, n_tx_el, off_tx_w, tx_slant_index,
                                                n_rx_el, off_rx_w, rx_slant_index, wavelength, a_out);
    CKL();
    return RT_OK;
}

namespace {
// rotation_entries (em.py:33-40 / geometry.py:50-59): same libm calls and
// operation order as the Python restatement
void rotation_rows(const double* ypr, double* r) {
    double cy = cos(ypr[0]), sy = sin(ypr[0]), cp = cos(ypr[1]), sp = sin(ypr[1]);
    double cr = cos(ypr[2]), sr = sin(ypr[2]);
    r[0] = cy * cp; r[1] = cy * sp * sr - sy * cr; r[2] = cy * sp * cr + sy * sr;
    r[3] = sy * cp; r[4] = sy * sp * sr + cy * cr; r[5] = sy * sp * cr - cy * sr;
    r[6] = -sp;     r[7] = cp * sr;                r[8] = cp * cr;
}

// per device: rows [9], world-frame element offsets w[e] = R off[e] (em.py:372-379)
// and the aperture |max_e w - min_e w| (em.py:344-356); a device whose
// orientation equals its predecessor's reuses that device's values
void device_frames(int n_dev, const double* ypr, int n_el, const double* off, double* rows,
                   double* offw, double* aperture) {
    for (int d = 0; d < n_dev; ++d) {
        const double* o = ypr + 3 * d;
        if (d > 0 && o[0] == o[-3] && o[1] == o[-2] && o[2] == o[-1]) {
            std::memcpy(rows + 9 * d, rows + 9 * (d - 1), 9 * sizeof(double));
            std::memcpy(offw + 3 * (size_t)n_el * d, offw + 3 * (size_t)n_el * (d - 1), 3 * n_el * sizeof(double));
            aperture[d] = aperture[d - 1];
            continue;
        }
        double* r = rows + 9 * d;
        rotation_rows(o, r);
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int e = 0; e < n_el; ++e) {
            const double* x = off + 3 * e;
            double* w = offw + 3 * ((size_t)n_el * d + e);
            for (int m = 0; m < 3; ++m) {
                w[m] = x[0] * r[3 * m] + x[1] * r[3 * m + 1] + x[2] * r[3 * m + 2];
                lo[m] = std::min(lo[m], w[m]);
                hi[m] = std::max(hi[m], w[m]);
            }
        }
        double ex = hi[0] - lo[0], ey = hi[1] - lo[1], ez = hi[2] - lo[2];
        aperture[d] = n_el > 1 ? sqrt(ex * ex + ey * ey + ez * ez) : 0.0;
    }
}

// distinct slants in ascending order + each element's index into them
int slant_sets(int n_el, const double* sl, double* distinct, int32_t* idx) {
    int n = 0;
    for (int e = 0; e < n_el; ++e) {
        bool seen = false;
        for (int k = 0; k < n; ++k) seen |= distinct[k] == sl[e];
        if (!seen) distinct[n++] = sl[e];
    }
    std::sort(distinct, distinct + n);
    for (int e = 0; e < n_el; ++e)
        for (int k = 0; k < n; ++k)
            if (distinct[k] == sl[e]) idx[e] = k;
    return n;
}
}  // namespace

int rt_gains_h(rt_ctx* ctx, int64_t n_paths, int max_len, const int32_t* tx_dev, const int32_t* rx_dev,
               const int8_t* order, const int32_t* seq, const int32_t* interaction_mat,
               const double* vertices, const double* normals, const double* cos_inc, const double* length,
               const double* delay, const double* k_dep, const double* k_arr, int n_tx_dev,
               const double* tx_ypr, const double* tx_pos, int n_rx_dev, const double* rx_ypr,
               const double* rx_pos, int tx_pattern, int n_tx_el, const double* off_tx,
               const double* sl_tx, int rx_pattern, int n_rx_el, const double* off_rx,
               const double* sl_rx, const double* eta, int n_mat, double wavelength,
               double frequency_hz, double* a_out, int* near_field, void* stream) {
    if (!ctx || n_paths < 0 || max_len < 1 || n_tx_dev < 1 || n_rx_dev < 1 || n_tx_el < 1 ||
        n_rx_el < 1 || n_mat < 1 || !(wavelength > 0.0) || !tx_ypr || !rx_ypr || !off_tx || !sl_tx ||
        !off_rx || !sl_rx || !eta)
        return fail(ctx, RT_EINVAL, "bad gains arguments");
    if (tx_pattern < 0 || tx_pattern > 4 || rx_pattern < 0 || rx_pattern > 4)
        return fail(ctx, RT_EINVAL, "unknown antenna pattern");
    if (near_field) *near_field = 0;
    // host parameter block: rows_t | rows_r | offw_t | offw_r | st | sr | eta | (int32) s_idx | r_idx
    size_t o_rt = 0, o_rr = o_rt + 9 * (size_t)n_tx_dev, o_wt = o_rr + 9 * (size_t)n_rx_dev;
    size_t o_wr = o_wt + 3 * (size_t)n_tx_dev * n_tx_el, o_st = o_wr + 3 * (size_t)n_rx_dev * n_rx_el;
    size_t o_sr = o_st + n_tx_el, o_eta = o_sr + n_rx_el, n_dbl = o_eta + 2 * (size_t)n_mat;
    size_t bytes = 8 * n_dbl + 4 * (size_t)(n_tx_el + n_rx_el);
    std::vector<double> hb((bytes + 7) / 8);
    double* h = hb.data();
    std::vector<double> ap_t(n_tx_dev), ap_r(n_rx_dev);
    device_frames(n_tx_dev, tx_ypr, n_tx_el, off_tx, h + o_rt, h + o_wt, ap_t.data());
    device_frames(n_rx_dev, rx_ypr, n_rx_el, off_rx, h + o_rr, h + o_wr, ap_r.data());
    int32_t* si = reinterpret_cast<int32_t*>(h + n_dbl);
    int32_t* ri = si + n_tx_el;
    int S = slant_sets(n_tx_el, sl_tx, h + o_st, si);
    int R = slant_sets(n_rx_el, sl_rx, h + o_sr, ri);
    std::memcpy(h + o_eta, eta, 16 * (size_t)n_mat);
    if (near_field && tx_pos && rx_pos) {
        // every path is at least as long as the straight tx-rx distance (em.py:344-356 pre-check)
        for (int t = 0; t < n_tx_dev && !*near_field; ++t)
            for (int r = 0; r < n_rx_dev; ++r) {
                double a = std::max(ap_t[t], ap_r[r]);
                if (a <= 0.0) continue;
                double dx = tx_pos[3 * t] - rx_pos[3 * r], dy = tx_pos[3 * t + 1] - rx_pos[3 * r + 1];
                double dz = tx_pos[3 * t + 2] - rx_pos[3 * r + 2];
                if (sqrt(dx * dx + dy * dy + dz * dz) < 2.0 * a * a / wavelength * (1.0 + 1e-9)) {
                    *near_field = 1;
                    break;
                }
            }
    }
    if (n_paths == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    CK(ctx->gparam.reserve(bytes));
    RC(h2d_staged(ctx->device, ctx->gparam.p, h, (int64_t)bytes, st));
    const double* d = ctx->gparam.get<double>();
    const int32_t* dsi = reinterpret_cast<const int32_t*>(d + n_dbl);
    CK(ctx->gbase.reserve(16ULL * n_paths * S * R));
    double* base = ctx->gbase.get<double>();
    TransferArgs A{n_paths, max_len, (const signed char*)order, seq, vertices, normals, cos_inc, length,
                   delay, d + o_rt, d + o_rr, tx_pattern, rx_pattern, d + o_st, S, d + o_sr, R, d + o_eta,
                   ctx->prim_mat.get<int>(), interaction_mat, wavelength, frequency_hz, tx_dev, rx_dev};
    k_transfer<<<nblk(n_paths * S, 128), 128, 0, st>>>(A, base);
    CKL();
    long long n = (long long)n_paths * n_tx_el * n_rx_el;
    k_gains_synth<<<nblk(n, 256), 256, 0, st>>>(n_paths, S, R, base, tx_dev, rx_dev, k_dep, k_arr, n_tx_el,
                                                d + o_wt, dsi, n_rx_el, d + o_wr, dsi + n_tx_el, wavelength,
                                                a_out);
    CKL();
    return RT_OK;
}

int rt_cir_plan(rt_ctx* ctx, int64_t n_paths, int max_len, const int8_t* order, const int32_t* seq,
                const double* delay, const int32_t* rx_of, const int32_t* tx_of, int n_rx, int n_tx,
                int los, int reflection, int64_t* n_path_out, void* stream) {
    if (!ctx || n_paths < 0 || max_len < 1 || n_rx < 1 || n_tx < 1 || !n_path_out)
        return fail(ctx, RT_EINVAL, "bad CIR arguments");
    const int64_t hint = *n_path_out;   // >= 0: the caller knows the largest bucket
    *n_path_out = 0;
    ctx->cir_n = n_paths;
    ctx->cir_ntx = n_tx;
    ctx->cir_nrx = n_rx;
    if (n_paths == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ST(stream);
    long long np = (long long)n_rx * n_tx;
    CK(ctx->cir_pair.reserve(4 * n_paths));
    CK(ctx->cir_count.reserve(4 * (np + 1)));
    CK(ctx->cir_off.reserve(4 * (np + 1)));
    CK(ctx->cir_fill.reserve(4 * np));
    CK(ctx->cir_bucket.reserve(4 * n_paths));
    CK(ctx->cir_slot.reserve(4 * n_paths));
    CK(ctx->cir_first.reserve(8 * n_paths));
    int* count = ctx->cir_count.get<int>();
    int* off = ctx->cir_off.get<int>();
    int* pair = ctx->cir_pair.get<int>();
    CK(cudaMemsetAsync(count, 0, 4 * (np + 1), st));
    CK(cudaMemsetAsync(ctx->cir_fill.p, 0, 4 * np, st));
    k_cir_count<<<nblk(n_paths, 256), 256, 0, st>>>(n_paths, (const signed char*)order, rx_of, tx_of, n_tx, los,
                                                    reflection, pair, count);
    CKL();
    RC(cub_call(ctx, [&](void* tmp, size_t& bytes) {
        return cub::DeviceScan::ExclusiveSum(tmp, bytes, count, off, (int)(np + 1), st);
    }));
    int* dmax = reinterpret_cast<int*>(ctx->ctrs.get<long long>() + 24);
    RC(cub_call(ctx, [&](void* tmp, size_t& bytes) {
        return cub::DeviceReduce::Max(tmp, bytes, count, dmax, (int)np, st);
    }));
    k_cir_bucket<<<nblk(n_paths, 256), 256, 0, st>>>(n_paths, pair, off, ctx->cir_fill.get<int>(),
                                                     ctx->cir_bucket.get<int>());
    k_cir_slot<<<nblk(n_paths, 128), 128, 0, st>>>(n_paths, pair, off, count, ctx->cir_bucket.get<int>(), delay,
                                                   (const signed char*)order, seq, max_len,
                                                   ctx->cir_slot.get<int>(), ctx->cir_first.get<double>());
    CKL();
    if (hint >= 0) {   // no host round trip
        *n_path_out = hint;
        return RT_OK;
    }
    CK(cudaMemcpyAsync(ctx->hpin, dmax, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *n_path_out = reinterpret_cast<int*>(ctx->hpin)[0];
    return RT_OK;
}

int rt_cir_scatter(rt_ctx* ctx, int64_t n_paths, const double* delay, int normalize,
                   const double* a_in, int n_rx_el, int n_tx_el, int n_t, int64_t n_path,
                   double* a_out, double* tau_out, void* stream) {
    if (!ctx || n_paths != ctx->cir_n || n_rx_el < 1 || n_tx_el < 1 || n_t < 1 || n_path < 0)
        return fail(ctx, RT_EINVAL, "rt_cir_scatter does not match the last rt_cir_plan");
    long long n = (long long)n_paths * n_rx_el * n_tx_el * n_t;
    if (n == 0 || n_path == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    // the outputs need not be zeroed by the caller: slots past a pair's paths are 0
    long long n_pairs = (long long)ctx->cir_nrx * ctx->cir_ntx;
    CK(cudaMemsetAsync(a_out, 0, 16ULL * n_pairs * n_rx_el * n_tx_el * n_path * n_t, ST(stream)));
    CK(cudaMemsetAsync(tau_out, 0, 8ULL * n_pairs * n_path, ST(stream)));
    k_cir_scatter<<<nblk(n, 256), 256, 0, ST(stream)>>>(n_paths, ctx->cir_pair.get<int>(), ctx->cir_slot.get<int>(),
                                                        ctx->cir_first.get<double>(), delay, normalize,
                                                        ctx->cir_ntx, n_rx_el, n_tx_el, n_t, n_path, a_in,
                                                        a_out, tau_out);
    CKL();
    return RT_OK;
}

int rt_freq_nmse(rt_ctx* ctx, int64_t n_records, int n_sub, const int64_t* rec_start, const double* a,
                 const double* tau, const double* freqs, const double* h, const double* norm2, double scale,
                 double* H_out, double* loss_out, double* grad_a, void* stream) {
    if (!ctx || n_records < 0 || n_sub < 1 || n_sub > 8192 || !rec_start || !a || !tau || !freqs)
        return fail(ctx, RT_EINVAL, "bad frequency-response arguments");
    if ((loss_out || grad_a) && (!h || !norm2))
        return fail(ctx, RT_EINVAL, "the NMSE needs targets and their norms");
    if (n_records == 0) return RT_OK;
    CK(cudaSetDevice(ctx->device));
    size_t smem = sizeof(double2) * (size_t)n_sub;
    if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(k_freq_nmse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_freq_nmse<<<(unsigned)n_records, FREQ_BLOCK, smem, ST(stream)>>>(
        n_sub, reinterpret_cast<const long long*>(rec_start), reinterpret_cast<const double2*>(a), tau, freqs,
        reinterpret_cast<const double2*>(h), norm2, scale, reinterpret_cast<double2*>(H_out), loss_out,
        reinterpret_cast<double2*>(grad_a));
    CKL();
    return RT_OK;
}

}  // extern "C"


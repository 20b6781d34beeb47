/*
 * b200rt.h — C ABI of libb200rt.so, the B200 (sm_100a) propagation hot path.
 *
 * The reference (emtrace, pure Python) has no FFI boundary: its seam is the
 * Python module API.  Each entry point below replaces the reference function
 * named beside it; the Python host layer (paper_2303_11103_b200/*.py) keeps
 * emtrace's signatures and calls these through ctypes (see INTEGRATION.md
 * for the stub a maintainer would add to emtrace itself).
 *
 * Conventions
 *  - Every pointer argument documented "device" is CUDA device memory; host
 *    arrays are only the small fixed-size ones marked "host".
 *  - Calls are ordered on `stream` (a cudaStream_t, NULL = legacy default).
 *    Entry points that return a size (n_*_out) synchronise that stream.
 *  - Return value: RT_OK (0) or a negative RT_E* code; rt_last_error() gives
 *    the message.  The Python layer maps RT_EINVAL to the reference's
 *    ValueError subclasses (TracerError / ChannelError / EmError), RT_ECAP to
 *    the cap errors (tracer.py:203-207, channel.py:239-242), RT_ECOINCIDE to
 *    tracer.py:188-189, and RT_ECUDA / RT_ENOMEM to RuntimeError.
 *  - One context per device and per host thread; a context owns the scene,
 *    the BVH, the current candidate set and the current path table.
 */
#ifndef B200RT_H
#define B200RT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RT_OK 0
#define RT_EINVAL (-1)
#define RT_ECAP (-2)
#define RT_ECOINCIDE (-3)
#define RT_ECUDA (-4)
#define RT_ENOMEM (-5)
#define RT_ESTATE (-6)

/* antenna pattern ids (em.py:42-83) */
#define RT_PAT_ISO 0
#define RT_PAT_DIPOLE 1
#define RT_PAT_TR38901 2
#define RT_PAT_PROBE_THETA 3
#define RT_PAT_PROBE_PHI 4

typedef struct rt_ctx rt_ctx;

int rt_version(void);
int rt_create(int device, rt_ctx** out);
int rt_destroy(rt_ctx* ctx);
const char* rt_last_error(const rt_ctx* ctx);
/* Host -> device copy of a small parameter block through the library's
 * page-locked staging ring, asynchronous on `stream` of `device`; the host
 * buffer may be reused as soon as the call returns (plumbing for the
 * per-call parameter uploads of the Python layer). */
int rt_h2d(int device, void* dst, const void* src, int64_t bytes, void* stream);

/* ---- scene ingest + acceleration (bvh.py:33-79,180-202: Bvh.__init__, _gather, build) ----
 * vertices: [n_vertices*3] f64; tri_vertex: [n_prims*3] i32 global
 * vertex ids (< 2^31) in _gather order (object order, then triangle order);
 * prim_material: [n_prims] i32 — device memory, or host memory that the call
 * copies in on `stream` (host buffers may be refilled once rt_bvh_build has
 * returned: it waits for those copies).  Computes v0/e1/e2, unit normals and
 * plane offsets bit-identically to the reference's numpy calls. */
int rt_scene_upload(rt_ctx* ctx, const double* vertices, int64_t n_vertices,
                    const int32_t* tri_vertex, const int32_t* prim_material, int64_t n_prims,
                    void* stream);
/* BVH over the uploaded primitives (replaces Bvh._build, bvh.py:59-79):
 * top-down binned SAH on the device, depth-first child-pair layout with
 * subtrees of <= 2 prims collapsed into leaves, plus the per-prim origin skip
 * table (the subtree behind each prim, per side).  Build-time variants: PLOC
 * or the Karras LBVH over Morton codes.  Tree shape never changes results. */
int rt_bvh_build(rt_ctx* ctx, void* stream);
int64_t rt_num_prims(const rt_ctx* ctx);
/* copy the per-primitive arrays (device outputs, any may be NULL) */
int rt_scene_arrays(rt_ctx* ctx, double* v0, double* e1, double* e2, double* normals,
                    double* plane_offset, void* stream);

/* ---- queries (bvh.py:83-115 Bvh.intersect / Bvh.occluded) ----
 * rt_trace: n rays (device o,d [n*3], tmin,tmax [n]); closest hit (t, global
 * prim id, -1 on miss) or, with any_hit, the first hit found.  Synchronizes
 * the stream: a traversal stack overflow fails the call (RT_ECUDA). */
int rt_trace(rt_ctx* ctx, const double* o, const double* d, const double* tmin,
             const double* tmax, int64_t n, int any_hit, double* t_out, int32_t* prim_out,
             void* stream);
/* rt_occluded: segments p->q (device [n*3]); out[i] = 1 blocked, 0 clear,
 * -1 endpoints coincide (bvh.py:109-110 raises).  Synchronizes the stream: a
 * traversal stack overflow fails the call (RT_ECUDA) instead of reading as
 * "blocked". */
int rt_occluded(rt_ctx* ctx, const double* p, const double* q, int64_t n, int32_t* out,
                void* stream);

/* ---- candidate sequences ----
 * rt_launch replaces launch_candidates (tracer.py:217-244): Fibonacci rays
 * (geometry.py:62-76) from host tx[3], slots [slot_begin, slot_end) of an
 * n_rays lattice (a coherence permutation maps slots to lattice indices; the
 * union over slots is the whole lattice), up to max_depth closest hits each;
 * every prefix of every ray's hit sequence becomes a candidate.  dirs
 * (device [n_rays*3]) overrides the on-device directions when non-NULL.
 * The candidate set replaces the context's current one, sorted by
 * (length, lexicographic sequence). */
int rt_launch(rt_ctx* ctx, const double* tx, int64_t n_rays, int64_t slot_begin,
              int64_t slot_end, int max_depth, const double* dirs, int64_t* n_cand_out,
              int64_t* n_bounces_out, void* stream);
/* rt_launch over one shard of the lattice for multi-GPU runs (SURVEY 8e stage 1):
 * whole coherence bands go round-robin to the shard_count ranks, so each rank
 * traces the same mix of latitudes (contiguous slot ranges would give one rank
 * the upward rays that escape after one bounce).  The union over shards of
 * the candidate sets equals the single launch's; bounce counts add up.  With
 * shard_count > 1 the shard's candidates are left unsorted (rt_candidates_get
 * returns them); path / coverage calls refuse them (RT_ESTATE) until the union
 * is installed with rt_candidates_set, which sorts it once. */
int rt_launch_shard(rt_ctx* ctx, const double* tx, int64_t n_rays, int shard_index, int shard_count,
                    int max_depth, const double* dirs, int64_t* n_cand_out, int64_t* n_bounces_out,
                    void* stream);
/* enumerate_candidates (tracer.py:196-214); RT_ECAP when n^max_depth > cap */
int rt_enumerate(rt_ctx* ctx, int max_depth, int64_t cap, int64_t* n_cand_out, void* stream);
/* install an arbitrary candidate list (device seq [n*max_len] i32 -1 padded,
 * len [n] i8); duplicates are removed and the result sorted */
int rt_candidates_set(rt_ctx* ctx, const int32_t* seq, const int8_t* len, int64_t n,
                      int max_len, int64_t* n_unique_out, void* stream);
int rt_candidates_get(rt_ctx* ctx, int32_t* seq, int8_t* len, int max_len, void* stream);
int64_t rt_num_candidates(const rt_ctx* ctx);
int rt_candidates_max_len(const rt_ctx* ctx);

/* ---- paths to explicit receivers (tracer.py:150-193,247-311) ----
 * Image solve + validity + occlusion for every (receiver, candidate) pair,
 * LOS per receiver, coincident-path merge, order (los, order, seq) per
 * receiver.  The path table replaces the context's current one. */
int rt_paths(rt_ctx* ctx, const double* tx, const double* rx, int64_t n_rx,
             int64_t* n_paths_out, void* stream);
/* copy the path table (device outputs; any may be NULL); rows are grouped by
 * receiver in rx order.  max_len = rt_candidates_max_len (>=1). */
/* compute_paths_between for one transmitter with method "fibonacci"
 * (tracer.py:268-295): rt_launch over the whole n_rays lattice, then rt_paths
 * to the n_rx receivers, in one call (no host round trip between them).  A
 * scene without primitives gives LOS paths only. */
int rt_paths_fibonacci(rt_ctx* ctx, const double* tx, int64_t n_rays, int max_depth, const double* rx,
                       int64_t n_rx, int64_t* n_cand_out, int64_t* n_bounces_out, int64_t* n_paths_out,
                       void* stream);
/* the most paths of one receiver in the last rt_paths (its per-receiver
 * counts come with the path count: no extra round trip) */
int64_t rt_paths_max_per_receiver(const rt_ctx* ctx);
int rt_paths_get(rt_ctx* ctx, int32_t* rx_index, int32_t* cand, int8_t* order, int32_t* seq,
                 double* vertices, double* length, double* delay, double* k_dep,
                 double* k_arr, double* normals, double* cos_inc, void* stream);

/* ---- polarized field transfer (em.py:98-171,291-312) ----
 * For every path p and element-slant pair (s, r): a[p, s, r] (complex as 2
 * doubles) of the geometry given by vertices [P*(L+2)*3], oriented normals
 * [P*L*3], cosines [P*L], length, delay; the material of interaction j is
 * interaction_mat[p*L+j] when that (device) array is given, else the scene's
 * prim_material[seq[p*L+j]]; eta [n_mat*2] (device).  With interaction_mat
 * no scene needs to be uploaded (em.py:291-312 transfer takes material names
 * per interaction, not prim ids).  tx_rows/rx_rows are per-path 3x3
 * row-major rotations (device [P*9]). */
int rt_transfer(rt_ctx* ctx, int64_t n_paths, int max_len, const int8_t* order,
                const int32_t* seq, const int32_t* interaction_mat, const double* vertices, const double* normals,
                const double* cos_inc, const double* length, const double* delay,
                const double* tx_rows, const double* rx_rows, int tx_pattern, int rx_pattern,
                const double* tx_slants, int n_tx_slants, const double* rx_slants,
                int n_rx_slants, const double* eta, int n_mat, double wavelength,
                double frequency_hz, double* a_out, void* stream);
/* Hand-written adjoint of rt_transfer w.r.t. eta: given grad_a (device
 * [P*S*R*2], PyTorch's dL/dRe + j dL/dIm convention) accumulate
 * grad_eta[m] = (dL/dRe eta_m, dL/dIm eta_m) into device [n_mat*2].
 * Deterministic: per-interaction contributions are summed per material in a
 * fixed order (no atomics), so repeated calls give identical bits. */
int rt_transfer_bwd(rt_ctx* ctx, int64_t n_paths, int max_len, const int8_t* order,
                    const int32_t* seq, const int32_t* interaction_mat, const double* vertices, const double* normals,
                    const double* cos_inc, const double* length, const double* delay,
                    const double* tx_rows, const double* rx_rows, int tx_pattern,
                    int rx_pattern, const double* tx_slants, int n_tx_slants,
                    const double* rx_slants, int n_rx_slants, const double* eta, int n_mat,
                    double wavelength, double frequency_hz, const double* grad_a,
                    double* grad_eta, void* stream);

/* ---- synthetic-array gains and CIR packing (no autograd) ----
 * rt_gains_synthetic (em.py:359-422, _gain_synthetic): a[p, i, j] = base[p,
 * s(j), r(i)] * exp(j 2 pi off_rx_w[rx_dev[p], i] . (-k_arr[p]) / lambda) *
 * exp(j 2 pi off_tx_w[tx_dev[p], j] . k_dep[p] / lambda).  All device: base
 * [P*S*R*2] (rt_transfer's output), tx_dev/rx_dev [P], k_dep/k_arr [P*3],
 * off_tx_w [n_tx_dev*Et*3], off_rx_w [n_rx_dev*Er*3] (world-frame element
 * offsets), slant indices [Et] / [Er]; out a [P*Er*Et*2]. */
int rt_gains_synthetic(rt_ctx* ctx, int64_t n_paths, int n_tx_slants, int n_rx_slants,
                       const double* base, const int32_t* tx_dev, const int32_t* rx_dev,
                       const double* k_dep, const double* k_arr, int n_tx_el,
                       const double* off_tx_w, const int32_t* tx_slant_index, int n_rx_el,
                       const double* off_rx_w, const int32_t* rx_slant_index, double wavelength,
                       double* a_out, void* stream);
/* rt_gains (em.py:359-422, compute_gains with a synthetic array, no autograd):
 * rt_transfer followed by rt_gains_synthetic in one call.  Rotation rows are
 * per DEVICE (tx_rows [n_tx_dev*9], rx_rows [n_rx_dev*9], row-major 3x3)
 * and picked per path through tx_dev / rx_dev [P]; the per-(path, slant
 * pair) coefficients stay in library scratch.  Other arguments as in
 * rt_transfer / rt_gains_synthetic; out a [P*Er*Et*2] (device). */
int rt_gains(rt_ctx* ctx, int64_t n_paths, int max_len, const int32_t* tx_dev, const int32_t* rx_dev,
             const int8_t* order, const int32_t* seq, const int32_t* interaction_mat,
             const double* vertices, const double* normals, const double* cos_inc,
             const double* length, const double* delay, const double* k_dep, const double* k_arr,
             const double* tx_rows, const double* rx_rows, int tx_pattern, int rx_pattern,
             const double* tx_slants, int n_tx_slants, const double* rx_slants, int n_rx_slants,
             const double* eta, int n_mat, int n_tx_el, const double* off_tx_w,
             const int32_t* tx_slant_index, int n_rx_el, const double* off_rx_w,
             const int32_t* rx_slant_index, double wavelength, double frequency_hz, double* a_out,
             void* stream);
/* rt_gains_h: compute_gains (em.py:359-422, synthetic arrays, no autograd) as
 * one call with the per-device parameters on the HOST: orientations tx_ypr
 * [n_tx_dev*3] / rx_ypr [n_rx_dev*3] (yaw, pitch, roll -> rows as
 * geometry.py:50-59), array-frame element offsets off_tx [Et*3] / off_rx
 * [Er*3] and slants sl_tx [Et] / sl_rx [Er] (scene.py:138-154), eta
 * [n_mat*2].  The library forms the rows, the world-frame offsets and the
 * distinct slant sets, uploads them with one copy and runs the rt_gains
 * kernels.  With tx_pos / rx_pos (host [n_dev*3]) and near_field given,
 * *near_field = 1 when some (tx, rx) pair is closer than the Fraunhofer
 * distance 2 D^2 / lambda of its larger aperture D (em.py:344-356's
 * pre-check: the caller then inspects the paths themselves). */
int rt_gains_h(rt_ctx* ctx, int64_t n_paths, int max_len, const int32_t* tx_dev, const int32_t* rx_dev,
               const int8_t* order, const int32_t* seq, const int32_t* interaction_mat,
               const double* vertices, const double* normals, const double* cos_inc,
               const double* length, const double* delay, const double* k_dep, const double* k_arr,
               int n_tx_dev, const double* tx_ypr, const double* tx_pos, int n_rx_dev,
               const double* rx_ypr, const double* rx_pos, int tx_pattern, int n_tx_el,
               const double* off_tx, const double* sl_tx, int rx_pattern, int n_rx_el,
               const double* off_rx, const double* sl_rx, const double* eta, int n_mat,
               double wavelength, double frequency_hz, double* a_out, int* near_field, void* stream);
/* build_cir (channel.py:40-72), two calls.  rt_cir_plan keeps LOS and/or
 * specular paths, buckets them by scene (rx, tx) pair (rx_of/tx_of [P]
 * device) and orders every bucket by (delay, kind, sequence); *n_path_out =
 * the largest bucket (host sync).  A caller that knows the largest bucket
 * passes it in *n_path_out (>= 0; e.g. rt_paths_max_per_receiver for a
 * table of one rt_paths call with LOS and specular kept): no host sync;
 * -1 = compute it.  rt_cir_scatter then writes a_in [P*Er*
 * Et*n_t*2] into a_out (zero-filled by the call) [n_rx*Er*n_tx*Et*n_path*n_t*2] and
 * tau_out [n_rx*n_tx*n_path] (delays minus the pair's first arrival when
 * normalize != 0). */
int rt_cir_plan(rt_ctx* ctx, int64_t n_paths, int max_len, const int8_t* order, const int32_t* seq,
                const double* delay, const int32_t* rx_of, const int32_t* tx_of, int n_rx, int n_tx,
                int los, int reflection, int64_t* n_path_out, void* stream);
int rt_cir_scatter(rt_ctx* ctx, int64_t n_paths, const double* delay, int normalize,
                   const double* a_in, int n_rx_el, int n_tx_el, int n_t, int64_t n_path,
                   double* a_out, double* tau_out, void* stream);

/* coverage_map (channel.py:236-253) with method "fibonacci" on one device: rt_launch
 * over the whole n_rays lattice, then rt_coverage (shard 0 of 1), in one call (no
 * host round trip between them).  *n_bounces_out = the launch's ray-bounces. */
int rt_coverage_fibonacci(rt_ctx* ctx, const double* tx, int64_t n_rays, int max_depth, double origin_x,
                          double origin_y, double cell_size, int64_t nx, int64_t ny, double height,
                          const double* tx_rows, const double* probe_rows, int tx_pattern, const double* slants,
                          const double* offsets_w, int n_el, int tx_mode, const double* eta, int n_mat,
                          double wavelength, double frequency_hz, double* gains_out, int64_t* stats_out,
                          int64_t* n_bounces_out, void* stream);

/* Batched image_solve of independent (tx, rx, sequence) triples (tracer.py:
 * 150-183; order-0 rows are LOS visibility checks, tracer.py:190) — the
 * explicit-array gains (em.py:425-459) and single image_solve queries.
 * Inputs device: tx_pos, rx_pos [n*3], seq [n*max_len] (-1 padded), len [n].
 * Outputs device: valid [n] (1/0) and, for valid rows, the path geometry in
 * rt_paths_get's layout (rows aligned with the inputs). */
int rt_solve_pairs(rt_ctx* ctx, int64_t n, int max_len, const double* tx_pos,
                   const double* rx_pos, const int32_t* seq, const int8_t* len, uint8_t* valid,
                   double* vertices, double* length, double* delay, double* k_dep, double* k_arr,
                   double* normals, double* cos_inc, int32_t* seq_out, int8_t* order_out,
                   void* stream);

/* Position / orientation derivatives (em.py:258-312 with tracked positions and
 * orientations): a[p,s,r] re-derived from per-path tx/rx positions and yaw/
 * pitch/roll (device [P*3] each; geometry re-solved by mirroring across the
 * planes through the path's vertices, geometry_for_positions) plus its
 * Jacobian jac_out [P*S*R*12*2] w.r.t. (tx xyz, rx xyz, tx ypr, rx ypr). */
int rt_transfer_jvp(rt_ctx* ctx, int64_t n_paths, int max_len, const int8_t* order,
                    const int32_t* seq, const double* vertices, const double* normals,
                    const double* tx_pos, const double* rx_pos, const double* tx_ypr,
                    const double* rx_ypr, int tx_pattern, int rx_pattern, const double* tx_slants,
                    int n_tx_slants, const double* rx_slants, int n_rx_slants, const double* eta,
                    int n_mat, double wavelength, double frequency_hz, double* a_out,
                    double* jac_out, void* stream);

/* ---- coverage map (channel.py:190-253 point_path_gain / coverage_map) ----
 * Probe receivers at the centers of an nx*ny grid at `height`.  Every cell
 * receives sum_paths sum_{theta,phi probes} |a|^2 over the current candidate
 * set, with per-cell merge; tx_mode 0 = central element (slants[0]), 1 =
 * coherent sum over n_el elements with world offsets offsets_w [n_el*3] and
 * slants [n_el] (host arrays).  Rows with iy % shard_count == shard_index
 * (round-robin rows) are computed; other cells are written 0
 * (sum-allreduce the shards).
 * gains_out: device [ny*nx] f64.  stats_out (host [8], may be NULL):
 * work items, geometric pairs, valid paths, cells, candidates. */
int rt_coverage(rt_ctx* ctx, const double* tx, double origin_x, double origin_y,
                double cell_size, int64_t nx, int64_t ny, double height,
                const double* tx_rows, const double* probe_rows, int tx_pattern,
                const double* slants, const double* offsets_w, int n_el, int tx_mode,
                const double* eta, int n_mat, double wavelength, double frequency_hz,
                int shard_index, int shard_count, double* gains_out, int64_t* stats_out,
                void* stream);

/* ---- measurement ----
 * flags bit 0: record CUDA events around each stage on the caller's stream;
 * bit 1: run the instrumented launch kernel (per-traversal node and
 * triangle counters, for the roofline's algorithmic bytes).
 * rt_get_profile (host out [16] each): ms per stage of the last call
 * (-1 = not run): 0 launch kernel, 1 candidate sort+unique, 2 images +
 * footprints + scan, 3 geometric solve, 4 occlusion+transfer, 5 record sort,
 * 6 merge/accumulate, 7 LOS, 8 trie -> sequences; counters: 0 ray-bounces,
 * 1 node visits, 2 triangle tests, 3 candidates, 4 work items, 5 geometric
 * pairs, 6 valid paths, 10 warp iterations of the launch's bounce loop and
 * 11 the sum over them of the warp's largest per-lane node-visit count (both
 * from the instrumented launch: SIMD efficiency of bounces and traversals),
 * 13 depth of the last built tree (rt_bvh_build fails with RT_ECAP when it
 * exceeds the traversal stack),
 * 14 1000 x the tree's surface-area estimate of internal-node visits per ray
 * (1 + sum of internal child box areas / root area),
 * 15 kernel launches issued by the library (cumulative; a CUB device-wide
 * primitive counts once). */
int rt_set_profiling(rt_ctx* ctx, int flags);
/* L2-resident read bandwidth (GB/s) of this device: a persistent kernel
 * streams a `bytes` buffer `iters` times with 16-byte L2-only loads (the
 * roofline denominator for the L2-resident traversal working set). */
int rt_l2_probe(rt_ctx* ctx, int64_t bytes, int iters, double* gbs_out, void* stream);
/* Measured peaks for the roofline denominators (csrc/microbench.cuh), timed
 * with CUDA events on `stream` at the current clocks: kind 0 FP32 FMA TFLOP/s,
 * 1 FP64 DFMA TFLOP/s, 2 warp-instruction issue rate (Gwarp-inst/s, imm-form
 * FFMA chains), 3 L1-resident read GB/s, 4 L2-resident read GB/s (rt_l2_probe
 * on 48 MB).  Synchronizes the stream. */
int rt_microbench(rt_ctx* ctx, int kind, double* value_out, void* stream);
int rt_get_profile(rt_ctx* ctx, double* ms_out, int64_t* counters_out);

/* Fresnel reflection coefficients (em.py:123-141 fresnel, with
 * autodiff.py:365-382 csqrt_posreal's Re >= 0 branch) of n (eta, cos theta_i)
 * pairs: eta [n*2], cos_theta [n] -> r_te, r_tm [n*2] (device, complex as 2
 * doubles).  The same device function the transfer kernels use. */
int rt_fresnel(rt_ctx* ctx, int64_t n, const double* eta, const double* cos_theta, double* r_te,
               double* r_tm, void* stream);

/* ---- OFDM responses and the calibration loss (channel.py:107-123,
 * optim.py:158-177 _projected_sq_error, optim.py:305-372 learn_materials) ----
 * Paths are grouped by record: record r owns rows rec_start[r] ..
 * rec_start[r+1]-1 (device int64 [n_records+1]) of a [P*2] (complex) and
 * tau [P]; freqs [n_sub] (device, n_sub <= 8192).
 *   H_out [n_records*n_sub*2] (optional): H[r,k] = sum_i a_i e^{-j 2 pi f_k tau_i}
 *   loss_out [n_records] (optional): scale * sum_k |H[r,k] - h[r,k]|^2 / norm2[r]
 *   grad_a [P*2] (optional): dloss/da_i (dL/dRe + j dL/dIm) of sum_r loss_out[r]
 * h [n_records*n_sub*2] and norm2 [n_records] are needed for loss / grad.
 * Fixed summation order, no atomics: bit-reproducible. */
int rt_freq_nmse(rt_ctx* ctx, int64_t n_records, int n_sub, const int64_t* rec_start, const double* a,
                 const double* tau, const double* freqs, const double* h, const double* norm2,
                 double scale, double* H_out, double* loss_out, double* grad_a, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B200RT_H */

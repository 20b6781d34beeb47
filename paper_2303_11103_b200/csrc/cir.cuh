// cir.cuh — synthetic-array gains and CIR packing without autograd.
//
// compute_gains (em.py:359-422, synthetic arrays): a[p, i, j] = base[p, s(j),
// r(i)] * exp(j 2 pi off_rx_w(i) . (-k_arr) / lambda) * exp(j 2 pi off_tx_w(j)
// . k_dep / lambda), one thread per (path, rx element, tx element).
//
// build_cir (channel.py:40-72): keep LOS / specular paths as asked, bucket
// them by (rx, tx) pair, order each bucket by (delay, kind, sequence) — the
// reference's sort key — and scatter a / tau into the dense, zero-padded
// [rx, rx_el, tx, tx_el, path, time] / [rx, tx, path] tensors.  A bucket
// holds the few paths of one pair, so each path finds its slot by counting
// the bucket entries that sort before it.
#pragma once
#include "rt_common.cuh"

namespace rt {

__global__ void k_gains_synth(long long P, int S, int R, const double* __restrict__ base,
                              const int* __restrict__ tx_dev, const int* __restrict__ rx_dev,
                              const double* __restrict__ kdep, const double* __restrict__ karr, int Et,
                              const double* __restrict__ off_tx_w, const int* __restrict__ s_index, int Er,
                              const double* __restrict__ off_rx_w, const int* __restrict__ r_index,
                              double wavelength, double* __restrict__ a_out) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    long long n = P * (long long)Er * Et;
    if (t >= n) return;
    int j = (int)(t % Et);
    int i = (int)((t / Et) % Er);
    long long p = t / ((long long)Et * Er);
    const double* ot = off_tx_w + ((long long)tx_dev[p] * Et + j) * 3;
    const double* orr = off_rx_w + ((long long)rx_dev[p] * Er + i) * 3;
    const double* kd = kdep + 3 * p;
    const double* ka = karr + 3 * p;
    double dt = ot[0] * kd[0] + ot[1] * kd[1] + ot[2] * kd[2];
    double dr = orr[0] * -ka[0] + orr[1] * -ka[1] + orr[2] * -ka[2];
    double st, ct, sr, cr;
    sincos(TWO_PI * dt / wavelength, &st, &ct);
    sincos(TWO_PI * dr / wavelength, &sr, &cr);
    const double* b = base + ((p * S + s_index[j]) * R + r_index[i]) * 2;
    // (b * ph_rx) * ph_tx
    double xr = b[0] * cr - b[1] * sr, xi = b[0] * sr + b[1] * cr;
    a_out[2 * t] = xr * ct - xi * st;
    a_out[2 * t + 1] = xr * st + xi * ct;
}

// pair of every kept path (-1 = filtered out) and the per-pair counts
__global__ void k_cir_count(long long P, const signed char* __restrict__ order, const int* __restrict__ rx_of,
                            const int* __restrict__ tx_of, int n_tx, int los, int refl, int* pair_of,
                            int* count) {
    long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (p >= P) return;
    bool spec = order[p] > 0;
    int pair = -1;
    if ((spec && refl) || (!spec && los)) {
        pair = rx_of[p] * n_tx + tx_of[p];
        atomicAdd(count + pair, 1);
    }
    pair_of[p] = pair;
}

__global__ void k_cir_bucket(long long P, const int* __restrict__ pair_of, const int* __restrict__ off,
                             int* fill, int* bucket) {
    long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (p >= P) return;
    int pair = pair_of[p];
    if (pair < 0) return;
    bucket[off[pair] + atomicAdd(fill + pair, 1)] = (int)p;
}

// (delay, kind, sequence) order of channel.py:59-62; equal keys by table index
__device__ inline bool cir_before(long long q, long long p, const double* delay, const signed char* order,
                                  const int* seq, int L) {
    if (delay[q] != delay[p]) return delay[q] < delay[p];
    int kq = order[q] > 0, kp = order[p] > 0;
    if (kq != kp) return kq < kp;
    for (int j = 0; j < L; ++j) {
        int a = j < order[q] ? seq[q * L + j] : -1, b = j < order[p] ? seq[p * L + j] : -1;
        if (a != b) return a < b;
    }
    return q < p;
}

__global__ void k_cir_slot(long long P, const int* __restrict__ pair_of, const int* __restrict__ off,
                           const int* __restrict__ count, const int* __restrict__ bucket,
                           const double* __restrict__ delay, const signed char* __restrict__ order,
                           const int* __restrict__ seq, int L, int* slot, double* first) {
    long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (p >= P) return;
    int pair = pair_of[p];
    if (pair < 0) { slot[p] = -1; return; }
    int b0 = off[pair], nb = count[pair], s = 0;
    double f = delay[p];
    for (int k = 0; k < nb; ++k) {
        long long q = bucket[b0 + k];
        if (q != p && cir_before(q, p, delay, order, seq, L)) ++s;
        f = fmin(f, delay[q]);
    }
    slot[p] = s;
    first[p] = f;   // the pair's first arrival (slot 0 sorts by delay first)
}

__global__ void k_cir_scatter(long long P, const int* __restrict__ pair_of, const int* __restrict__ slot,
                              const double* __restrict__ first, const double* __restrict__ delay, int normalize,
                              int n_tx, int Er, int Et, int n_t, long long n_path, const double* __restrict__ a_in,
                              double* a_out, double* tau_out) {
    long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    long long per = (long long)Er * Et * n_t;
    if (t >= P * per) return;
    long long p = t / per;
    int pair = pair_of[p];
    if (pair < 0) return;
    long long e = t - p * per;   // (i, j, time) of the path's [Er, Et, n_t] block
    int tt = (int)(e % n_t);
    int j = (int)((e / n_t) % Et);
    int i = (int)(e / ((long long)n_t * Et));
    int rx = pair / n_tx, tx = pair - rx * n_tx;
    long long s = slot[p];
    // a[rx, i, tx, j, s, tt]
    long long o = ((((long long)rx * Er + i) * n_tx + tx) * Et + j) * n_path * n_t + s * n_t + tt;
    a_out[2 * o] = a_in[2 * t];
    a_out[2 * o + 1] = a_in[2 * t + 1];
    if (e == 0) tau_out[((long long)rx * n_tx + tx) * n_path + s] = normalize ? delay[p] - first[p] : delay[p];
}

}  // namespace rt

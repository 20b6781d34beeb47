// freq.cuh — OFDM frequency responses and the calibration NMSE with its gradient.
//
// frequency_response (channel.py:107-123): H[r, k] = sum_i a_i e^{-j 2 pi f_k tau_i}
// over the paths i of record r (rows start[r] .. start[r+1] of a path table
// grouped by record).  learn_materials' loss (optim.py:158-177, 305-372):
// L = scale * sum_r sum_k |H[r, k] - h[r, k]|^2 / norm2[r], and its gradient
// dL/da_i = 2 scale / norm2[r] * sum_k conj(e^{-j 2 pi f_k tau_i}) (H[r, k] - h[r, k])
// in PyTorch's convention (dL/dRe a + j dL/dIm a).
//
// One block per record; every sum runs in a fixed order (paths in row order,
// subcarriers in index order, a fixed shared-memory tree), so the result is
// bit-identical from run to run — no atomics (reference criterion 10).
#pragma once
#include "rt_common.cuh"

namespace rt {

constexpr int FREQ_BLOCK = 128;

// e^{-j 2 pi f tau}: the phase is (-2 pi f) * tau, as torch evaluates
// exp(-2j * pi * f * tau) for real f, tau
__device__ __forceinline__ double2 ofdm_phasor(double f, double tau) {
    double s, c;
    sincos((-TWO_PI * f) * tau, &s, &c);
    return make_double2(c, s);
}

__global__ void __launch_bounds__(FREQ_BLOCK)
    k_freq_nmse(int n_sub, const long long* __restrict__ start, const double2* __restrict__ a,
                const double* __restrict__ tau, const double* __restrict__ f,
                const double2* __restrict__ h, const double* __restrict__ norm2, double scale,
                double2* __restrict__ H_out, double* __restrict__ loss_out, double2* __restrict__ grad_a) {
    extern __shared__ double2 err[];   // [n_sub]
    __shared__ double part[FREQ_BLOCK];
    const int r = blockIdx.x;
    const long long p0 = start[r], p1 = start[r + 1];
    double acc = 0.0;
    for (int k = threadIdx.x; k < n_sub; k += FREQ_BLOCK) {
        double fk = f[k];
        double hr = 0.0, hi = 0.0;
        for (long long i = p0; i < p1; ++i) {
            double2 e = ofdm_phasor(fk, tau[i]);
            double2 ai = a[i];
            hr += ai.x * e.x - ai.y * e.y;
            hi += ai.x * e.y + ai.y * e.x;
        }
        long long o = (long long)r * n_sub + k;
        if (H_out) H_out[o] = make_double2(hr, hi);
        if (h) {
            double2 t = h[o];
            double er = hr - t.x, ei = hi - t.y;
            err[k] = make_double2(er, ei);
            acc += er * er + ei * ei;
        }
    }
    if (!h) return;
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int w = FREQ_BLOCK / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
        __syncthreads();
    }
    const double n2 = norm2[r];
    if (threadIdx.x == 0 && loss_out) loss_out[r] = part[0] / n2 * scale;
    if (!grad_a) return;
    const double g = 2.0 * scale / n2;
    for (long long i = p0 + threadIdx.x; i < p1; i += FREQ_BLOCK) {
        double ti = tau[i], gr = 0.0, gi = 0.0;
        for (int k = 0; k < n_sub; ++k) {
            double2 e = ofdm_phasor(f[k], ti);
            double2 d = err[k];
            // conj(e) * d
            gr += e.x * d.x + e.y * d.y;
            gi += e.x * d.y - e.y * d.x;
        }
        grad_a[i] = make_double2(g * gr, g * gi);
    }
}

}  // namespace rt

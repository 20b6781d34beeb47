// microbench.cuh — measured peaks for the roofline denominators (rt_microbench).
//
// The traversal kernels are bound by instruction issue and by L1 / L2 reads,
// not by HBM, so the bench measures those ceilings live, at the
// clock the GPU runs at, next to MEASURED_PEAKS.json's HBM copy bandwidth:
//   RT_MB_FP32   FP32 FMA throughput (3-register FFMA, independent chains)  TFLOP/s
//   RT_MB_FP64   FP64 DFMA throughput                                       TFLOP/s
//   RT_MB_ISSUE  warp-instruction issue rate: immediate-form FFMA chains,
//                one warp-instruction per SMSP per cycle (B300_MICROARCH:
//                imm-form FFMA reciprocal throughput 1)               Gwarp-inst/s
//   RT_MB_L1     L1-resident 16-byte loads (16 KB per block, 8 blocks/SM)  GB/s
//   RT_MB_L2     L2-resident 16-byte loads (48 MB working set, .cg)        GB/s
// Counted work is the loop body only (the loop's own instructions are not
// counted), so each figure is a lower bound of the rate the hardware reached.
#pragma once
#include <cuda_runtime.h>

namespace rt {

enum { RT_MB_FP32 = 0, RT_MB_FP64 = 1, RT_MB_ISSUE = 2, RT_MB_L1 = 3, RT_MB_L2 = 4 };

constexpr int MB_CHAINS = 8;    // independent dependency chains per thread
constexpr int MB_UNROLL = 32;   // chain steps per loop iteration
constexpr int MB_L1_SLICE = 16 * 1024;

__global__ void __launch_bounds__(256) k_mb_ffma(int iters, float* sink) {
    float a[MB_CHAINS], b = 1.0f + threadIdx.x * 1e-9f, c = 0.5f - threadIdx.x * 1e-9f;
#pragma unroll
    for (int j = 0; j < MB_CHAINS; ++j) a[j] = (float)(threadIdx.x + j);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < MB_UNROLL; ++u)
#pragma unroll
            for (int j = 0; j < MB_CHAINS; ++j) a[j] = fmaf(a[j], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < MB_CHAINS; ++j) s += a[j];
    if (s == 1234.5f) *sink = s;
}

// immediate-form FFMA (the multiplier is a literal): issue-rate probe
__global__ void __launch_bounds__(256) k_mb_issue(int iters, float* sink) {
    float a[MB_CHAINS], c = 0.5f - threadIdx.x * 1e-9f;
#pragma unroll
    for (int j = 0; j < MB_CHAINS; ++j) a[j] = (float)(threadIdx.x + j);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < MB_UNROLL; ++u)
#pragma unroll
            for (int j = 0; j < MB_CHAINS; ++j) a[j] = fmaf(a[j], 0.999969f, c);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < MB_CHAINS; ++j) s += a[j];
    if (s == 1234.5f) *sink = s;
}

__global__ void __launch_bounds__(256) k_mb_dfma(int iters, double* sink) {
    double a[MB_CHAINS], b = 1.0 + threadIdx.x * 1e-12, c = 0.5 - threadIdx.x * 1e-12;
#pragma unroll
    for (int j = 0; j < MB_CHAINS; ++j) a[j] = (double)(threadIdx.x + j);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < MB_UNROLL; ++u)
#pragma unroll
            for (int j = 0; j < MB_CHAINS; ++j) a[j] = fma(a[j], b, c);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < MB_CHAINS; ++j) s += a[j];
    if (s == 1234.5) *sink = s;
}

// every block re-reads its own 16 KB slice (L1-resident after the first pass)
__global__ void __launch_bounds__(256) k_mb_l1(const float4* __restrict__ buf, int iters, float* sink) {
    const int n4 = MB_L1_SLICE / 16;
    const float4* p = buf + (long long)blockIdx.x * n4;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        // the slot rotates with `it`, so the loads cannot be hoisted out of the loop
#pragma unroll 4
        for (int i = threadIdx.x; i < n4; i += 256) {
            float4 v = __ldg(p + ((i + it * 32) & (n4 - 1)));
            acc += (v.x + v.w);
        }
    }
    if (acc == 1234.5f) *sink = acc;
}

}  // namespace rt

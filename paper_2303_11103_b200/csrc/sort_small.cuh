// sort_small.cuh — one-CTA radix sort of (u64 key, i32 value) pairs for the
// latency-bound small cases (the C2 canyon: 5,435 candidate rows, 2,354 path
// records).  cub::DeviceRadixSort runs a histogram, a scan and one onesweep
// kernel per 8-bit digit (plus memsets): ~12 launches and ~85 us for a few
// thousand keys; here the whole LSD sort is one CTA in shared memory
// (cub::BlockRadixSort, 4-bit digits over [begin_bit, end_bit), 4 / 8 / 16 keys
// per thread by size), stable like the device sort, so both produce the same
// permutation.
#pragma once
#include <cub/block/block_radix_sort.cuh>

namespace rt {

constexpr int SORT_SMALL_THREADS = 512;
constexpr int SORT_SMALL_MAX = SORT_SMALL_THREADS * 16;   // 8192 pairs

#ifndef RT_SORT_RADIX_BITS
#define RT_SORT_RADIX_BITS 4
#endif
template <int ITEMS>
using SmallSort = cub::BlockRadixSort<unsigned long long, SORT_SMALL_THREADS, ITEMS, int, RT_SORT_RADIX_BITS>;

// expand_cb > 0: the keys are the compact path-record keys (rx << (cb + 4) |
// order << cb | cand, cb = candidate bits) and leave in the library's record
// layout rx << 36 | order << 32 | cand
template <int ITEMS>
__global__ void __launch_bounds__(SORT_SMALL_THREADS, 1)
k_sort_small(const unsigned long long* __restrict__ kin, unsigned long long* __restrict__ kout,
             const int* __restrict__ vin, int* __restrict__ vout, int n, int begin_bit, int end_bit,
             int expand_cb) {
    extern __shared__ __align__(16) unsigned char sort_smem[];
    auto& tmp = *reinterpret_cast<typename SmallSort<ITEMS>::TempStorage*>(sort_smem);
    unsigned long long k[ITEMS];
    int v[ITEMS];
    const int base = threadIdx.x * ITEMS;   // blocked arrangement
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        int i = base + j;
        // padding sorts behind every key (all digit bits set; stable: after the real ties)
        k[j] = i < n ? kin[i] : ~0ULL;
        v[j] = i < n ? vin[i] : 0;
    }
    SmallSort<ITEMS>(tmp).Sort(k, v, begin_bit, end_bit);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        int i = base + j;
        if (i < n) {
            unsigned long long x = k[j];
            if (expand_cb > 0)
                x = ((x >> (expand_cb + 4)) << 36) | (((x >> expand_cb) & 0xFULL) << 32) |
                    (x & ((1ULL << expand_cb) - 1));
            kout[i] = x;
            vout[i] = v[j];
        }
    }
}

}  // namespace rt

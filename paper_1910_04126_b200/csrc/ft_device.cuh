// ft_device.cuh — small device helpers shared by the library's kernels (not by the oracle).
#pragma once
#include <stdint.h>

#include "ft_internal.cuh"

// ascending bitonic sort of P (power of two) u64 keys in shared memory, whole block.
__device__ __forceinline__ void fti_bitonic_sort_u64(unsigned long long* s, int P) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    unsigned long long a = s[i], b = s[ixj];
                    bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        s[i] = b;
                        s[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ uint32_t fti_hash(uint32_t k) {
    uint32_t h = k * 0x9E3779B1u;
    return h ^ (h >> 15);
}

__host__ __device__ __forceinline__ int fti_pow2_at_least(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// block-wide exclusive sum over blockDim.x (<= 1024) ints; `tmp` holds 32 ints of smem.
__device__ __forceinline__ int fti_block_exclusive_sum(int v, int* tmp, int* total) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) tmp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int t = lane < nw ? tmp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        tmp[lane] = t;   // inclusive per warp
    }
    __syncthreads();
    int before = wid > 0 ? tmp[wid - 1] : 0;
    if (total) *total = tmp[nw - 1];
    int res = before + x - v;
    __syncthreads();
    return res;
}

// warp-wide inclusive sum of u32
__device__ __forceinline__ uint32_t fti_warp_incl_u32(uint32_t x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ double fti_warp_sum_f64(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Block-wide counting sort by a small key: every thread of the block passes key ∈ [0, 256] (256 =
// "invalid, last"); returns the index of the thread whose key is the threadIdx.x-th smallest (the
// order among equal keys is arbitrary).  hist: 260 ints of smem; perm: blockDim.x u16 of smem.
// Three barriers and one warp scan instead of a bitonic network (36 barrier stages for 256 keys).
__device__ __forceinline__ int fti_counting_rank(uint32_t key, int* hist, uint16_t* perm) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < 260; i += nt) hist[i] = 0;
    __syncthreads();
    const int r = atomicAdd(&hist[key], 1);
    __syncthreads();
    if (tid < 32) {   // exclusive scan of hist[0..256]: 9 buckets per lane
        int v[9], sum = 0;
#pragma unroll
        for (int k = 0; k < 9; k++) {
            const int idx = tid * 9 + k;
            v[k] = idx < 257 ? hist[idx] : 0;
            sum += v[k];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += y;
        }
        int b = incl - sum;
#pragma unroll
        for (int k = 0; k < 9; k++) {
            const int idx = tid * 9 + k;
            if (idx < 257) hist[idx] = b;
            b += v[k];
        }
    }
    __syncthreads();
    perm[hist[key] + r] = (uint16_t)tid;
    __syncthreads();
    return perm[tid];
}

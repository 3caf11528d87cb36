// bf_device.cuh -- small device helpers shared by libbf's kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

// Debug bounds checks (libbf_debug.so, built with -DBF_DEBUG): print and trap.
#ifdef BF_DEBUG
#define BF_CHECK(c)                                                                                   \
  do {                                                                                                \
    if (!(c)) {                                                                                       \
      printf("BF_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, blockIdx.x, \
             threadIdx.x);                                                                            \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define BF_CHECK(c) \
  do {              \
  } while (0)
#endif

// Exclusive scan of one value per thread across the block (blockDim.x a
// multiple of 32, <= 1024).  warp_tot: shared scratch of 32 elements.
// *block_total (nullable, per-thread register) receives the block sum.
template <class T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* warp_tot, T* block_total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T t = lane < nw ? warp_tot[lane] : (T)0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;
  }
  __syncthreads();
  T base = wid ? warp_tot[wid - 1] : (T)0;
  if (block_total) *block_total = warp_tot[nw - 1];
  __syncthreads();
  return base + x - v;
}

template <class T>
__device__ __forceinline__ T warp_inclusive_scan(T x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

template <class T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ void red_add_u64(uint64_t* p, uint64_t v) {
  atomicAdd((unsigned long long*)p, (unsigned long long)v);
}

// C(d,2) = d(d-1)/2 in u64, exact for d < 2^32 (reading Z9).
__device__ __forceinline__ uint64_t choose2(uint32_t d) { return (uint64_t)d * (d - (d > 0)) >> 1; }

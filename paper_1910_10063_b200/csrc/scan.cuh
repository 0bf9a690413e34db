// scan.cuh -- warp/block prefix-sum building blocks shared by the index
// build (compaction, radix sort), selection (order-preserving compaction)
// and the generic device exclusive scan.
#pragma once
#include "skx_internal.cuh"

namespace skx {

// Inclusive warp scan (Kogge-Stone over shuffles).
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of one value per thread.  `warp_buf` holds
// >= 32 T.  Returns the exclusive prefix; *total gets the block sum.
// Contains two __syncthreads.
template <typename T, int NT>
__device__ __forceinline__ T block_exclusive_scan(T v, T* warp_buf, T* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const T inc = warp_inclusive_scan(v);
  if (lane == 31) warp_buf[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = lane < NW ? warp_buf[lane] : T(0);
    const T xi = warp_inclusive_scan(x);
    if (lane < NW) warp_buf[lane] = xi - x;
    if (lane == NW - 1) warp_buf[NW] = xi;
  }
  __syncthreads();
  *total = warp_buf[NW];
  return warp_buf[w] + inc - v;
}

}  // namespace skx

// Probe: effective L2 capacity for random 8-byte reads with no streams.
// Each thread reads `iters` pseudo-random entries of dim[0, D) (splitmix
// hash of (thread, i)) and xors them into one output word.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <int M>
__device__ __forceinline__ uint64_t ld(const uint64_t* p) {
  uint64_t v;
  if (M == 0) v = __ldg(p);
  if (M == 1) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  if (M == 2) asm volatile("ld.global.relaxed.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p));
  if (M == 3) asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

template <int M>
__global__ void __launch_bounds__(256) k_pure(const uint64_t* __restrict__ dim, uint64_t D,
                                              int iters, uint64_t seed, uint64_t* out) {
  const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;
  uint64_t acc = 0;
#pragma unroll 8
  for (int i = 0; i < iters; ++i) acc ^= ld<M>(dim + mix(seed ^ (t * 1000003ull + i)) % D);
  out[t] = acc;
}

extern "C" int probe_pure(const uint64_t* dim, uint64_t D, int iters, uint64_t seed,
                          uint64_t* out, int grid, void* stream, int mode) {
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0) k_pure<0><<<grid, 256, 0, s>>>(dim, D, iters, seed, out);
  if (mode == 1) k_pure<1><<<grid, 256, 0, s>>>(dim, D, iters, seed, out);
  if (mode == 2) k_pure<2><<<grid, 256, 0, s>>>(dim, D, iters, seed, out);
  if (mode == 3) k_pure<3><<<grid, 256, 0, s>>>(dim, D, iters, seed, out);
  return (int)cudaGetLastError();
}

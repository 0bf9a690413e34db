// Probe: DRAM cost of random 8-byte writes vs random 8-byte reads into a
// large (HBM-resident) array.  Standalone test tool, not part of the library.
//   mode 0: dst[h(i)] = i          (random scatter, plain st)
//   mode 1: dst[h(i)] = i  (.cs)   (random scatter, streaming st)
//   mode 2: acc ^= src[h(i)]       (random gather)
//   mode 3: red.add dst[h(i)] += 1 (random RED)
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <int MODE>
__global__ void __launch_bounds__(256) k_scatter(uint64_t* dst, uint64_t mask, uint64_t count,
                                                 uint64_t* sink) {
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * 256 * 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint64_t k = i + (uint64_t)u * gridDim.x * 256;
      if (k >= count) break;
      uint64_t h = mix(k) & mask;
      if (MODE == 0) dst[h] = k;
      if (MODE == 1) __stcs(reinterpret_cast<unsigned long long*>(dst + h), k);
      if (MODE == 2) acc ^= __ldg(dst + h);
      if (MODE == 3) atomicAdd(reinterpret_cast<unsigned long long*>(dst + h), 1ull);
    }
  }
  if (MODE == 2 && acc == 0x1234567) *sink = acc;
}

extern "C" int probe_scatter(int mode, uint64_t* dst, uint64_t mask, uint64_t count,
                             uint64_t* sink, int grid, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (mode) {
    case 0: k_scatter<0><<<grid, 256, 0, s>>>(dst, mask, count, sink); break;
    case 1: k_scatter<1><<<grid, 256, 0, s>>>(dst, mask, count, sink); break;
    case 2: k_scatter<2><<<grid, 256, 0, s>>>(dst, mask, count, sink); break;
    case 3: k_scatter<3><<<grid, 256, 0, s>>>(dst, mask, count, sink); break;
    default: return -1;
  }
  return (int)cudaGetLastError();
}

// Probe: where does the C3 group-by's time go?  Same structure as the
// library's k_aggregate<8> (1024 threads, 1 CTA/SM, 32-bit shared bins for
// ids < hot), with the tail (ids >= hot) handled per TAIL mode:
//   0  two 64-bit REDs on the interleaved {count, sum} pair (library)
//   1  one RED (count only)
//   2  no tail update (diagnostic)
//   3  two REDs into a small L2-resident pair region (idx & mask) (diagnostic)
//   4  one packed RED (1 << 40 | m) per tail row (diagnostic)
//   5  two 32-bit REDs on an interleaved {u32 count, u32 sum} pair (diagnostic)
// Standalone test tool, not part of the library.
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kT = 1024;
constexpr int kU = 2;

template <int TAIL>
__global__ void __launch_bounds__(kT, 1)
k_agg(const uint4* __restrict__ fk, const ulonglong2* __restrict__ qty, uint64_t nvec,
      uint32_t hot, unsigned long long* __restrict__ pairs, uint32_t mask) {
  extern __shared__ uint32_t sm[];
  uint32_t* cnt = sm;
  uint32_t* lo = sm + hot;
  uint32_t* hi = sm + 2 * (size_t)hot;
  for (uint32_t i = threadIdx.x; i < 3 * hot; i += kT) sm[i] = 0u;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * kT * kU;
  for (uint64_t vb0 = (uint64_t)blockIdx.x * kT * kU; vb0 < nvec; vb0 += stride) {
    uint4 f[kU];
    unsigned long long m[kU][4];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t vi = vb0 + threadIdx.x + (uint64_t)u * kT;
      if (vi < nvec) {
        f[u] = __ldcs(fk + vi);
        const ulonglong2 a = __ldcs(qty + 2 * vi), b = __ldcs(qty + 2 * vi + 1);
        m[u][0] = a.x, m[u][1] = a.y, m[u][2] = b.x, m[u][3] = b.y;
      } else {
        f[u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t ids[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (ids[j] == 0) continue;
        const uint32_t idx = ids[j] - 1u;
        const unsigned long long v = m[u][j];
        if (idx < hot) {
          atomicAdd(&cnt[idx], 1u);
          const uint32_t ml = (uint32_t)v;
          const uint32_t old = atomicAdd(&lo[idx], ml);
          const uint32_t ha = (uint32_t)(v >> 32) + ((uint32_t)(old + ml) < old ? 1u : 0u);
          if (ha) atomicAdd(&hi[idx], ha);
        } else if (TAIL == 0) {
          atomicAdd(&pairs[2 * (uint64_t)idx], 1ull);
          atomicAdd(&pairs[2 * (uint64_t)idx + 1], v);
        } else if (TAIL == 1) {
          atomicAdd(&pairs[2 * (uint64_t)idx], 1ull);
        } else if (TAIL == 3) {
          const uint32_t k = idx & mask;
          atomicAdd(&pairs[2 * (uint64_t)k], 1ull);
          atomicAdd(&pairs[2 * (uint64_t)k + 1], v);
        } else if (TAIL == 4) {
          atomicAdd(&pairs[idx], (1ull << 40) | v);
        } else if (TAIL == 5) {
          unsigned int* p32 = reinterpret_cast<unsigned int*>(pairs);
          atomicAdd(&p32[2 * (uint64_t)idx], 1u);
          atomicAdd(&p32[2 * (uint64_t)idx + 1], (unsigned int)v);
        }
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < hot; i += kT) {
    if (cnt[i]) {
      atomicAdd(&pairs[2 * (uint64_t)i], (unsigned long long)cnt[i]);
      atomicAdd(&pairs[2 * (uint64_t)i + 1], ((unsigned long long)hi[i] << 32) | lo[i]);
    }
  }
}

extern "C" int probe_agg(int tail, int grid, uint32_t hot, const uint32_t* fk, const uint64_t* qty,
                         uint64_t n, unsigned long long* pairs, uint32_t mask, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = (size_t)hot * 12;
  const uint64_t nvec = n / 4;
  auto go = [&](auto fn) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fn<<<grid, kT, smem, s>>>(reinterpret_cast<const uint4*>(fk),
                              reinterpret_cast<const ulonglong2*>(qty), nvec, hot, pairs, mask);
    return (int)cudaGetLastError();
  };
  switch (tail) {
    case 0: return go(k_agg<0>);
    case 1: return go(k_agg<1>);
    case 2: return go(k_agg<2>);
    case 3: return go(k_agg<3>);
    case 4: return go(k_agg<4>);
    case 5: return go(k_agg<5>);
  }
  return -1;
}

// Probe: die-split FK-join gather.  B200's L2 behaves as two ~63 MB caches,
// one per die, each caching what its own SMs read (die_probe.py).  Here every
// dimension line is owned by one die: the SMs of die d load only the values on
// their lines, so each L2 half caches a disjoint half of the dimension.  Both
// dies stream every FK tile (each die keeps its own tile counter) and store the
// outputs of the rows they own.
//   mode 0: plain gather, static grid stride (the library's shape)
//   mode 3: plain gather, dynamic tiles from one counter
//   mode 1: die split, owner = 128-byte line parity of the dimension index
//   mode 2: die split, idx < hot by FK-vector parity, the rest by line parity
//   mode 5: die split by line parity, only the FK stream (diagnostic: loads kept,
//           no dimension loads for foreign lines, stores dropped)
#include <cstdint>
#include <cuda_runtime.h>

namespace {
constexpr int NT = 256;
constexpr int U = 8;

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t ld_dim(const uint64_t* p, uint64_t pol) {
  uint64_t r;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(NT, 2)
    k_dg(const uint4* __restrict__ fv, uint64_t nvec, const uint64_t* __restrict__ dim, uint64_t D,
         uint64_t* __restrict__ out, const uint8_t* __restrict__ die_of_sm, unsigned* ctr,
         uint32_t hot, int line_shift) {
  const uint64_t pol = pol_last();
  constexpr bool SPLIT = MODE == 1 || MODE == 2 || MODE == 5;
  const uint32_t d = SPLIT ? die_of_sm[smid()] : 0;
  const uint64_t tile = (uint64_t)NT * U;
  const uint64_t ntiles = (nvec + tile - 1) / tile;
  __shared__ unsigned s_t;
  uint64_t t = MODE == 0 ? blockIdx.x : 0;
  uint64_t acc = 0;
  for (;;) {
    if (MODE != 0) {
      if (threadIdx.x == 0) s_t = atomicAdd(ctr + d, 1u);
      __syncthreads();
      t = s_t;
      __syncthreads();
    }
    if (t >= ntiles) break;
    const uint64_t base = t * tile + threadIdx.x;
    uint4 f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + (uint64_t)u * NT;
      f[u] = vi < nvec ? __ldcs(fv + vi) : make_uint4(1, 1, 1, 1);
    }
    uint64_t v[U][4];
    unsigned own[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t ids[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
      const uint64_t vi = base + (uint64_t)u * NT;
      own[u] = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idx = ids[j] - 1u;
        bool mine = true;
        if (SPLIT) {
          if (MODE == 2 && idx < hot)
            mine = (uint32_t)(vi & 1) == d;
          else
            mine = ((idx >> line_shift) & 1u) == d;
        }
        v[u][j] = 0;
        if (mine && idx < D) {
          v[u][j] = ld_dim(dim + idx, pol);
          own[u] |= 1u << j;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = base + (uint64_t)u * NT;
      if (vi >= nvec) continue;
      if (MODE == 5) {
        acc ^= v[u][0] ^ v[u][1] ^ v[u][2] ^ v[u][3];
        continue;
      }
      uint64_t* o = out + vi * 4;
      if (own[u] == 0xf) {
        __stcs(reinterpret_cast<ulonglong2*>(o), make_ulonglong2(v[u][0], v[u][1]));
        __stcs(reinterpret_cast<ulonglong2*>(o) + 1, make_ulonglong2(v[u][2], v[u][3]));
      } else if (own[u]) {
        if ((own[u] & 3) == 3)
          __stcs(reinterpret_cast<ulonglong2*>(o), make_ulonglong2(v[u][0], v[u][1]));
        else {
          if (own[u] & 1) __stcs(reinterpret_cast<unsigned long long*>(o), v[u][0]);
          if (own[u] & 2) __stcs(reinterpret_cast<unsigned long long*>(o + 1), v[u][1]);
        }
        if ((own[u] & 12) == 12)
          __stcs(reinterpret_cast<ulonglong2*>(o) + 1, make_ulonglong2(v[u][2], v[u][3]));
        else {
          if (own[u] & 4) __stcs(reinterpret_cast<unsigned long long*>(o + 2), v[u][2]);
          if (own[u] & 8) __stcs(reinterpret_cast<unsigned long long*>(o + 3), v[u][3]);
        }
      }
    }
    if (MODE == 0) t += gridDim.x;
  }
  if (MODE == 5 && acc == 0x5eed5eedull) out[threadIdx.x] = acc;
}
}  // namespace

extern "C" int probe_dg(int mode, const uint32_t* fact, uint64_t nvec, const uint64_t* dim,
                        uint64_t D, uint64_t* out, const uint8_t* die_of_sm, unsigned* ctr,
                        uint32_t hot, int line_shift, int grid, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (mode != 0) cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned), s);
  const uint4* fv = reinterpret_cast<const uint4*>(fact);
#define L(M) \
  if (mode == M) k_dg<M><<<grid, NT, 0, s>>>(fv, nvec, dim, D, out, die_of_sm, ctr, hot, line_shift);
  L(0) L(1) L(2) L(3) L(5)
#undef L
  return (int)cudaGetLastError();
}

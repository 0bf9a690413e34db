// Probe: which SMs share an L2 half (die), and whether splitting a random-read
// table between the two SM groups recovers the whole L2 for random reads.
//
// k_pair:  one 1024-thread CTA per SM (forced by dynamic smem); only the CTAs on
//          SM a and SM b work: each reads random 8-byte entries of its own table
//          (a: [0, D), b: [D, 2D)) and records its cycle count.  If a and b sit on
//          the same die their tables compete for one L2 half.
// k_split: every CTA reads random entries of the half of a 2D-entry table that
//          its SM's group owns (group[smid]); grid = 148 x 8 CTAs of 256.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void __launch_bounds__(1024) k_pair(const uint64_t* __restrict__ dim, uint64_t D,
                                               int iters, uint64_t seed, int a, int b,
                                               uint64_t* out, long long* cycles) {
  const int sm = (int)smid();
  if (sm != a && sm != b) return;
  const uint64_t base = sm == a ? 0 : D;
  const uint64_t t = (uint64_t)blockIdx.x * 1024 + threadIdx.x;
  uint64_t acc = 0;
  long long c0 = clock64();
#pragma unroll 8
  for (int i = 0; i < iters; ++i) acc ^= __ldg(dim + base + mix(seed ^ (t * 1000003ull + i)) % D);
  __syncthreads();
  long long c1 = clock64();
  out[t] = acc;
  if (threadIdx.x == 0) cycles[sm] = c1 - c0;
}

__global__ void __launch_bounds__(256) k_split(const uint64_t* __restrict__ dim, uint64_t D,
                                               int iters, uint64_t seed,
                                               const uint8_t* __restrict__ group, uint64_t* out,
                                               int shift) {
  // shift < 0: group g reads the contiguous half [g*D, (g+1)*D); otherwise the
  // halves interleave in chunks of 2^shift entries (chunk parity = group).
  const uint64_t g = group[smid()];
  const uint64_t base = g ? D : 0;
  const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;
  uint64_t acc = 0;
#pragma unroll 8
  for (int i = 0; i < iters; ++i) {
    const uint64_t r = mix(seed ^ (t * 1000003ull + i)) % D;
    const uint64_t idx = shift < 0 ? base + r
                                   : ((((r >> shift) << 1) | g) << shift) | (r & ((1ull << shift) - 1));
    acc ^= __ldg(dim + idx);
  }
  out[t] = acc;
}

__global__ void k_smids(uint32_t* out) {
  if (threadIdx.x == 0) out[blockIdx.x] = smid();
}

extern "C" int probe_pair(const uint64_t* dim, uint64_t D, int iters, uint64_t seed, int a, int b,
                          uint64_t* out, long long* cycles, int grid, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_pair<<<grid, 1024, smem, s>>>(dim, D, iters, seed, a, b, out, cycles);
  return (int)cudaGetLastError();
}

extern "C" int probe_split(const uint64_t* dim, uint64_t D, int iters, uint64_t seed,
                           const uint8_t* group, uint64_t* out, int grid, void* stream, int shift) {
  k_split<<<grid, 256, 0, (cudaStream_t)stream>>>(dim, D, iters, seed, group, out, shift);
  return (int)cudaGetLastError();
}

extern "C" int probe_smids(uint32_t* out, int grid, void* stream) {
  k_smids<<<grid, 32, 0, (cudaStream_t)stream>>>(out);
  return (int)cudaGetLastError();
}

// Stream probe: does a line one die streamed from HBM reach the other die from
// L2?  mode 0: the grid reads the array once (dynamic tiles, one counter);
// mode 1: each die reads the whole array (one tile counter per die, both dies
// walk the tiles in the same order at about the same time).
__global__ void __launch_bounds__(256) k_stream(const uint4* __restrict__ a, uint64_t nvec,
                                                const uint8_t* __restrict__ die_of_sm,
                                                unsigned* ctr, int mode, uint64_t* out) {
  const uint32_t d = mode ? die_of_sm[smid()] : 0;
  const uint64_t tile = 256 * 8;
  const uint64_t ntiles = (nvec + tile - 1) / tile;
  __shared__ unsigned s_t;
  uint32_t acc = 0;
  for (;;) {
    if (threadIdx.x == 0) s_t = atomicAdd(ctr + d, 1u);
    __syncthreads();
    const uint64_t t = s_t;
    __syncthreads();
    if (t >= ntiles) break;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint64_t vi = t * tile + u * 256 + threadIdx.x;
      if (vi < nvec) {
        const uint4 v = mode == 2 ? __ldg(a + vi) : __ldcs(a + vi);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
      }
    }
  }
  if (acc == 0x5eed5eedu) out[threadIdx.x] = acc;
}

extern "C" int probe_stream(const uint32_t* a, uint64_t n, const uint8_t* die_of_sm, unsigned* ctr,
                            int mode, uint64_t* out, int grid, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned), s);
  k_stream<<<grid, 256, 0, s>>>(reinterpret_cast<const uint4*>(a), n / 4, die_of_sm, ctr, mode, out);
  return (int)cudaGetLastError();
}

// RED capacity probe: random 32-bit reductions into the half of a 2D-word
// table that the SM's group owns (as k_split, for atomics).
__global__ void __launch_bounds__(256) k_red_split(unsigned* __restrict__ tab, uint64_t D,
                                                   int iters, uint64_t seed,
                                                   const uint8_t* __restrict__ group) {
  const uint64_t base = group[smid()] ? D : 0;
  const uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x;
#pragma unroll 8
  for (int i = 0; i < iters; ++i) atomicAdd(tab + base + mix(seed ^ (t * 1000003ull + i)) % D, 1u);
}

extern "C" int probe_red_split(unsigned* tab, uint64_t D, int iters, uint64_t seed,
                               const uint8_t* group, int grid, void* stream) {
  k_red_split<<<grid, 256, 0, (cudaStream_t)stream>>>(tab, D, iters, seed, group);
  return (int)cudaGetLastError();
}

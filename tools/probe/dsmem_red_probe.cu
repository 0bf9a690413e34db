// Probe: throughput of fire-and-forget reductions into distributed shared
// memory (red.shared::cluster.add.u32 to random words of random CTAs of the
// cluster) vs local shared memory and vs global REDs into an L2-resident
// table.  One 1024-thread CTA per SM, 64K words (256 KB... 192 KB) per CTA.
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  return x ^ (x >> 16);
}

constexpr int kWords = 48 * 1024;  // 192 KB per CTA

// MODE 0: local smem red; 1: DSMEM red (random rank); 2: global red (table of `gwords`)
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_red(int iters, uint32_t seed, unsigned* gtab,
                                                 uint32_t gwords, unsigned* out) {
  extern __shared__ unsigned sm[];
  for (int i = threadIdx.x; i < kWords; i += 1024) sm[i] = 0;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  const uint32_t nr = cl.num_blocks();
  const uint32_t t = blockIdx.x * 1024 + threadIdx.x;
  const uint32_t local_base = (uint32_t)__cvta_generic_to_shared(sm);
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    const uint32_t h = mix32(seed ^ (t * 2654435761u + i * 40503u));
    const uint32_t w = h % kWords;
    if (MODE == 0) {
      asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(local_base + 4 * w) : "memory");
    } else if (MODE == 1) {
      const uint32_t r = (h >> 20) % nr;
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_base + 4 * w), "r"(r));
      asm volatile("red.shared::cluster.add.u32 [%0], 1;" ::"r"(ra) : "memory");
    } else {
      atomicAdd(gtab + (h % gwords), 1u);
    }
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

extern "C" int probe_red(int mode, int cluster, int iters, uint32_t seed, unsigned* gtab,
                         uint32_t gwords, unsigned* out, int grid, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = kWords * 4;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = cluster;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaError_t e;
#define L(M)                                                                                  \
  if (mode == M) {                                                                            \
    cudaFuncSetAttribute(k_red<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 4); \
    if (cluster > 8) cudaFuncSetAttribute(k_red<M>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); \
    e = cudaLaunchKernelEx(&cfg, k_red<M>, iters, seed, gtab, gwords, out);                   \
    return (int)e;                                                                            \
  }
  L(0) L(1) L(2)
#undef L
  return -1;
}

extern "C" int probe_max_clusters(int cluster) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster * 64);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = kWords * 4;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = cluster;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(k_red<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 4);
  if (cluster > 8) cudaFuncSetAttribute(k_red<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int n = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_red<1>, &cfg);
  return e == cudaSuccess ? n : -(int)e;
}

// Probe: can thread-block-cluster distributed shared memory (DSMEM) serve the
// warm middle of a frequency-sorted dimension faster than L2?
// Modes (r = fk-1):
//   0  global only (ld.global.nc)
//   1  r <  C*slice -> DSMEM of CTA (r % C), slot r / C; else global
//   2  r <  local   -> own smem replica; else global
//   3  r <  local   -> own replica; r < local + C*slice -> DSMEM; else global
// Standalone test tool, not part of the library.
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int kT = 1024;
constexpr int kU = 8;

__device__ __forceinline__ uint64_t ldg_nc(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(kT, 1)
k_probe(const uint32_t* __restrict__ fk, uint64_t n, const uint64_t* __restrict__ dim,
        uint64_t* __restrict__ out, uint32_t slice, uint32_t local) {
  extern __shared__ uint64_t sm[];
  uint64_t* rep = sm;            // [local]
  uint64_t* dist = sm + local;   // [slice]
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t C = MODE & 1 ? cl.num_blocks() : 1;
  const uint32_t me = MODE & 1 ? cl.block_rank() : 0;
  const uint32_t cshift = 31 - __clz(C);
  if (MODE & 2)
    for (uint32_t i = threadIdx.x; i < local; i += kT) rep[i] = dim[i];
  if (MODE & 1)
    for (uint32_t i = threadIdx.x; i < slice; i += kT) dist[i] = dim[local + ((uint64_t)i << cshift) + me];
  if (MODE & 1) cl.sync(); else __syncthreads();
  const uint64_t span = (uint64_t)gridDim.x * kT * kU;
  const uint32_t dlim = MODE & 1 ? (slice << cshift) : 0;
  for (uint64_t base = (uint64_t)blockIdx.x * kT * kU; base < n; base += span) {
    uint32_t r[kU];
    uint64_t v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint64_t row = base + (uint64_t)u * kT + threadIdx.x;
      r[u] = row < n ? __ldcs(fk + row) - 1u : 0u;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint32_t x = r[u];
      if ((MODE & 2) && x < local) {
        v[u] = rep[x];
      } else if (MODE & 1) {
        uint32_t y = x - ((MODE & 2) ? local : 0u);
        if (y < dlim) {
          const uint64_t* p = cl.map_shared_rank(dist, y & (C - 1));
          v[u] = p[y >> cshift];
        } else {
          v[u] = ldg_nc(dim + x);
        }
      } else {
        v[u] = ldg_nc(dim + x);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint64_t row = base + (uint64_t)u * kT + threadIdx.x;
      if (row < n) __stcs(reinterpret_cast<unsigned long long*>(out + row), v[u]);
    }
  }
  if (MODE & 1) cl.sync();
}

template <int MODE>
static int launch(int cluster, int grid, size_t smem, const uint32_t* fk, uint64_t n,
                  const uint64_t* dim, uint64_t* out, uint32_t slice, uint32_t local,
                  cudaStream_t s) {
  auto fn = k_probe<MODE>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, fk, n, dim, out, slice, local);
  return (int)e;
}

extern "C" int probe_gather(int mode, int cluster, int grid, uint32_t slice, uint32_t local,
                            const uint32_t* fk, uint64_t n, const uint64_t* dim, uint64_t* out,
                            void* stream) {
  size_t smem = ((size_t)slice + local) * 8;
  cudaStream_t s = (cudaStream_t)stream;
  switch (mode) {
    case 0: return launch<0>(1, grid, smem, fk, n, dim, out, slice, local, s);
    case 1: return launch<1>(cluster, grid, smem, fk, n, dim, out, slice, local, s);
    case 2: return launch<2>(1, grid, smem, fk, n, dim, out, slice, local, s);
    case 3: return launch<3>(cluster, grid, smem, fk, n, dim, out, slice, local, s);
  }
  return -1;
}

extern "C" int probe_last_error() { return (int)cudaGetLastError(); }

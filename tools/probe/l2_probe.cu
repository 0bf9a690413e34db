// Probe: can L2 residency controls (eviction-priority hints by rank, persisting
// access-policy window + set-aside) make L2 hold the warm prefix of a
// frequency-sorted dimension?  Standalone test tool, not part of the library.
//   H=0  plain ld.global.nc for the dimension
//   H=1  r < K: evict_last ; else evict_first
//   H=2  r < K: evict_last ; else plain
//   H=3  r < K: plain      ; else evict_first
//   H=4  r < K: plain      ; else ld.global.lu (last use)
//   H=5  r < K: plain      ; else ld.global.cs.nc
//   H=6  r < K: evict_last ; else ld.global.lu
//   H=7  r < K: L1::evict_last ; else ld.global.lu
//   H=8  every load ld.global.lu
//   H=9  r < K: plain ; else no load (diagnostic, wrong output)
//   H=10 r < K: no load ; else plain (diagnostic, wrong output)
//   H=11..14 r < K: plain ; else .cg / .nc.L1::no_allocate / default (.ca) / .cv
//   H=15..17 r < K: no load ; else .cg / .nc.L1::no_allocate / .ca (diagnostic)
// Streams: FK via ld.cs, output via st.cs, as the library default.
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kT = 256;
constexpr int kU = 16;

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t ld_plain(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_hint(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t ld_cs(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cs.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_l1last(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::evict_last.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_cg(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_na(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_ca(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_cv(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_cas(const uint64_t* p) {
  uint64_t v;
  const uint64_t x = 0x5a5a5a5a5a5a5a5aull;  // cas(p, x, x): never changes memory
  asm volatile("atom.global.cas.b64 %0, [%1], %2, %2;" : "=l"(v) : "l"(p), "l"(x) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_orz(const uint64_t* p) {
  uint64_t v;
  asm volatile("atom.global.or.b64 %0, [%1], 0;" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_p64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_p128(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L2::128B.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_lu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.lu.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void tma_16(void* dst, const void* src, uint64_t* bar) {
  uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
      ::"r"(d), "l"(src), "r"(b) : "memory");
}
__device__ __forceinline__ void ldgsts_8(void* dst, const void* src) {
  uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* bar, uint32_t bytes) {
  uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W;\n}" ::"r"(b), "r"(phase) : "memory");
}

// H=18: r < K plain, else 16-byte TMA bulk copy to shared memory (sector-sized request)
// H=19: r < K plain, else 8-byte LDGSTS (cp.async.ca)
// H=20: r < K no load (diagnostic), else TMA as 18
template <int H>
__global__ void __launch_bounds__(kT, 2)
k_async(const uint32_t* __restrict__ fk, uint64_t n, const uint64_t* __restrict__ dim,
        uint64_t* __restrict__ out, uint32_t K) {
  extern __shared__ __align__(16) unsigned char stage[];
  __shared__ __align__(8) uint64_t bars[kT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (H != 19 && lane == 0) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t phase = 0;
  uint64_t* slot = reinterpret_cast<uint64_t*>(stage) + (size_t)threadIdx.x * kU * 2;
  const uint64_t span = (uint64_t)gridDim.x * kT * kU;
  for (uint64_t base = (uint64_t)blockIdx.x * kT * kU; base < n; base += span) {
    uint32_t r[kU];
    uint64_t v[kU];
    uint32_t cold = 0;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint64_t row = base + (uint64_t)u * kT + threadIdx.x;
      r[u] = row < n ? __ldcs(fk + row) - 1u : 0u;
      cold += (r[u] >= K) ? 1u : 0u;
    }
    if (H == 19) {
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (r[u] >= K) ldgsts_8(slot + 2 * u, dim + r[u]);
      asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
      for (int u = 0; u < kU; ++u)
        v[u] = r[u] < K ? ld_plain(dim + r[u]) : 0ull;
      asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (r[u] >= K) v[u] = slot[2 * u];
    } else {
      const uint32_t total = __reduce_add_sync(0xffffffffu, cold);
      if (total) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (lane == 0) bar_expect(&bars[warp], total * 16u);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (r[u] >= K) tma_16(slot + 2 * u, dim + (r[u] & ~1u), &bars[warp]);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        v[u] = r[u] < K ? (H == 20 ? 0ull : ld_plain(dim + r[u])) : 0ull;
      if (total) {
        bar_wait(&bars[warp], phase);
        phase ^= 1u;
#pragma unroll
        for (int u = 0; u < kU; ++u)
          if (r[u] >= K) v[u] = slot[2 * u + (r[u] & 1u)];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint64_t row = base + (uint64_t)u * kT + threadIdx.x;
      if (row < n) __stcs(reinterpret_cast<unsigned long long*>(out + row), v[u]);
    }
  }
}

template <int H>
__global__ void __launch_bounds__(kT, 2)
k_l2(const uint32_t* __restrict__ fk, uint64_t n, const uint64_t* __restrict__ dim,
     uint64_t* __restrict__ out, uint32_t K) {
  const uint64_t pl = pol_last(), pf = pol_first();
  const uint64_t span = (uint64_t)gridDim.x * kT * kU;
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
      const uint64_t* p = dim + r[u];
      const bool hot = r[u] < K;
      if (H == 0) v[u] = ld_plain(p);
      if (H == 1) v[u] = ld_hint(p, hot ? pl : pf);
      if (H == 2) v[u] = hot ? ld_hint(p, pl) : ld_plain(p);
      if (H == 3) v[u] = hot ? ld_plain(p) : ld_hint(p, pf);
      if (H == 4) v[u] = hot ? ld_plain(p) : ld_lu(p);
      if (H == 5) v[u] = hot ? ld_plain(p) : ld_cs(p);
      if (H == 6) v[u] = hot ? ld_hint(p, pl) : ld_lu(p);
      if (H == 7) v[u] = hot ? ld_l1last(p) : ld_lu(p);
      if (H == 8) v[u] = ld_lu(p);
      if (H == 9) v[u] = hot ? ld_plain(p) : 0ull;
      if (H == 10) v[u] = hot ? 0ull : ld_plain(p);
      if (H == 11) v[u] = hot ? ld_plain(p) : ld_cg(p);
      if (H == 12) v[u] = hot ? ld_plain(p) : ld_na(p);
      if (H == 13) v[u] = hot ? ld_plain(p) : ld_ca(p);
      if (H == 14) v[u] = hot ? ld_plain(p) : ld_cv(p);
      if (H == 15) v[u] = hot ? 0ull : ld_cg(p);
      if (H == 16) v[u] = hot ? 0ull : ld_na(p);
      if (H == 17) v[u] = hot ? 0ull : ld_ca(p);
      if (H == 40) v[u] = hot ? ld_plain(p) : ld_cas(p);
      if (H == 50) v[u] = hot ? ld_plain(p) : ld_p64(p);
      if (H >= 60 && H <= 62) v[u] = ld_plain(p);
      if (H == 51) v[u] = ld_p64(p);
      if (H == 52) v[u] = hot ? 0ull : ld_p64(p);
      if (H == 53) v[u] = hot ? 0ull : ld_p128(p);
      if (H == 41) v[u] = hot ? ld_plain(p) : ld_orz(p);
      if (H == 42) v[u] = hot ? 0ull : ld_cas(p);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint64_t row = base + (uint64_t)u * kT + threadIdx.x;
      if (row < n) {
        unsigned long long* q = reinterpret_cast<unsigned long long*>(out + row);
        if (H == 60) asm volatile("st.global.wt.u64 [%0], %1;" ::"l"(q), "l"(v[u]) : "memory");
        else if (H == 61) asm volatile("st.global.L1::no_allocate.L2::cache_hint.u64 [%0], %1, %2;"
                                       ::"l"(q), "l"(v[u]), "l"(pf) : "memory");
        else if (H == 62) *q = v[u];
        else __stcs(q, v[u]);
      }
    }
  }
}

// H=30: plain dimension loads; outputs staged per warp in shared memory and
// written with 256-byte TMA bulk stores (cp.async.bulk.global.shared::cta).
__global__ void __launch_bounds__(kT, 2)
k_tma_store(const uint32_t* __restrict__ fk, uint64_t n, const uint64_t* __restrict__ dim,
            uint64_t* __restrict__ out) {
  __shared__ __align__(128) uint64_t stage[kT / 32][kU][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t span = (uint64_t)gridDim.x * kT * kU;
  for (uint64_t base = (uint64_t)blockIdx.x * kT * kU; base < n; base += span) {
    uint32_t r[kU];
    uint64_t v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint64_t row = base + (uint64_t)u * kT + threadIdx.x;
      r[u] = row < n ? __ldcs(fk + row) - 1u : 0u;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = ld_plain(dim + r[u]);
    // previous bulk stores must have finished reading the staging buffer
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int u = 0; u < kU; ++u) stage[w][u][lane] = v[u];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const bool full = base + (uint64_t)kU * kT <= n;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint64_t row0 = base + (uint64_t)u * kT + (uint64_t)w * 32;
        if (full) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;" ::"l"(out + row0),
                       "r"((uint32_t)__cvta_generic_to_shared(&stage[w][u][0]))
                       : "memory");
        } else {
          for (int l = 0; l < 32; ++l)
            if (row0 + l < n) out[row0 + l] = stage[w][u][l];
        }
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int H>
static int launch(int grid, uint64_t win_bytes, float hit_ratio, const uint32_t* fk, uint64_t n,
                  const uint64_t* dim, uint64_t* out, uint32_t K, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kT);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  if (win_bytes) {
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    at[0].val.accessPolicyWindow.base_ptr = (void*)dim;
    at[0].val.accessPolicyWindow.num_bytes = (size_t)win_bytes;
    at[0].val.accessPolicyWindow.hitRatio = hit_ratio;
    at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  if (H == 30) return (int)cudaLaunchKernelEx(&cfg, k_tma_store, fk, n, dim, out);
  if (H >= 18 && H <= 20) {
    cfg.dynamicSmemBytes = (size_t)kT * kU * 16;
    cudaFuncSetAttribute(k_async<H>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)cfg.dynamicSmemBytes);
    return (int)cudaLaunchKernelEx(&cfg, k_async<H>, fk, n, dim, out, K);
  }
  return (int)cudaLaunchKernelEx(&cfg, k_l2<H>, fk, n, dim, out, K);
}

extern "C" int probe_l2(int h, int grid, uint64_t win_bytes, float hit_ratio, uint32_t K,
                        const uint32_t* fk, uint64_t n, const uint64_t* dim, uint64_t* out,
                        void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (h) {
    case 0: return launch<0>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 1: return launch<1>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 2: return launch<2>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 3: return launch<3>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 4: return launch<4>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 5: return launch<5>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 6: return launch<6>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 7: return launch<7>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 8: return launch<8>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 9: return launch<9>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 10: return launch<10>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 11: return launch<11>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 12: return launch<12>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 13: return launch<13>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 14: return launch<14>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 15: return launch<15>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 16: return launch<16>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 17: return launch<17>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 18: return launch<18>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 19: return launch<19>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 20: return launch<20>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 30: return launch<30>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 40: return launch<40>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 50: return launch<50>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 60: return launch<60>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 61: return launch<61>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 62: return launch<62>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 51: return launch<51>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 52: return launch<52>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 53: return launch<53>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 41: return launch<41>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
    case 42: return launch<42>(grid, win_bytes, hit_ratio, fk, n, dim, out, K, s);
  }
  return -1;
}

extern "C" int probe_setaside(uint64_t bytes) {
  cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)bytes);
  if (e != cudaSuccess) return (int)e;
  if (bytes == 0) e = cudaCtxResetPersistingL2Cache();
  return (int)e;
}

extern "C" int probe_set_granularity(uint64_t bytes) {
  return (int)cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)bytes);
}

extern "C" int probe_reset_persisting() { return (int)cudaCtxResetPersistingL2Cache(); }

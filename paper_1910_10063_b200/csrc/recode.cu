// recode.cu -- recode_fact (proj/src/permindex.cpp:60-64: materialize(fact,
// ranks)) for domains whose rank table exceeds L2.
//
// The recode runs on the ORIGINAL layout, where the popular ids are scattered:
// every hot id's rank sits on its own 64-byte L2 line, so the lines of the
// ~1M hottest ids already fill the L2 share the FK and output streams leave,
// and the rows of warmer ids miss to HBM (C4: 4 GB of rank-line fills next to
// 4.3 GB of FK, profiles/r2_ncu_c3_c4.md).  Here the ids of the 2^21
// smallest ranks -- the hottest ids, by construction of the index -- are
// packed 8 per line into a 32 MiB direct-mapped table of (rank << 32 | id)
// (the hottest id wins a slot: atomicMin on the packed word), built from the
// rank table in one streaming pass.  A row reads its id's slot; only the
// rows of colder (or displaced) ids read the rank table.  A 64 Ki-row sample
// decides on the device whether the table serves most rows (skewed data);
// otherwise the same kernel reads the rank table directly.
#include "skx_internal.cuh"

namespace skx {
namespace {

constexpr int kTabBits = 22;                    // 4 Mi slots x 8 B = 32 MiB
constexpr uint32_t kTabRanks = 1u << 21;        // ranks 1..2^21 inserted (load <= 1/2)
constexpr int kThreads = 256;
constexpr int kU = 4;                           // FK vectors (16 rows) per thread in flight
constexpr uint32_t kSample = 1u << 16;

__device__ __forceinline__ uint32_t tab_slot(uint32_t id) {
  return (id * 0x9E3779B1u) >> (32 - kTabBits);
}

__global__ void __launch_bounds__(256)
    k_tab_fill(const uint32_t* __restrict__ ranks, uint32_t d, unsigned long long* __restrict__ tab) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += stride) {
    const uint32_t r = __ldcs(ranks + i);
    if (r - 1u < kTabRanks) {
      const uint32_t id = (uint32_t)i + 1u;
      atomicMin(&tab[tab_slot(id)], ((unsigned long long)r << 32) | id);
    }
  }
}

// flag = 1 when at least half of a strided sample of rows find their id in
// the table.
__global__ void __launch_bounds__(1024)
    k_tab_sample(const uint32_t* __restrict__ fact, uint64_t n,
                 const unsigned long long* __restrict__ tab, unsigned int* __restrict__ flag) {
  __shared__ unsigned int s_hits;
  if (threadIdx.x == 0) s_hits = 0;
  __syncthreads();
  const uint64_t step = n / kSample ? n / kSample : 1;
  unsigned int hits = 0;
  for (uint32_t k = threadIdx.x; k < kSample && (uint64_t)k * step < n; k += blockDim.x) {
    const uint32_t id = __ldg(fact + (uint64_t)k * step);
    hits += (uint32_t)__ldg(tab + tab_slot(id)) == id ? 1u : 0u;
  }
  for (int o = 16; o > 0; o >>= 1) hits += __shfl_down_sync(0xffffffffu, hits, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_hits, hits);
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t m = n < kSample ? n : kSample;
    *flag = 2ull * s_hits >= m ? 1u : 0u;
  }
}

__global__ void __launch_bounds__(kThreads)
    k_recode_tab(const uint32_t* __restrict__ fact, uint64_t head, uint64_t nvec, uint64_t n,
                 const uint32_t* __restrict__ ranks, uint32_t d,
                 const unsigned long long* __restrict__ tab, const unsigned int* __restrict__ flag,
                 uint32_t* __restrict__ out, DevErr* err) {
  const bool use = *flag != 0u;  // uniform
  if (blockIdx.x == 0) {  // scalar head [0, head) and tail [head + 4 nvec, n)
    const uint64_t tail_b = head + nvec * 4;
    for (uint64_t t = threadIdx.x; t < head + (n - tail_b); t += kThreads) {
      const uint64_t k = t < head ? t : tail_b + (t - head);
      const uint32_t id = fact[k], idx = id - 1u;
      if (idx < d) {
        out[k] = __ldg(ranks + idx);
      } else {
        out[k] = 0u;
        record_violation(err, k, id);
      }
    }
  }
  const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
  uint4* ov = reinterpret_cast<uint4*>(out + head);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads * kU;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads * kU + threadIdx.x; base < nvec;
       base += stride) {
    uint32_t id[kU][4];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      const uint4 f = vi < nvec ? __ldcs(fv + vi) : make_uint4(1u, 1u, 1u, 1u);
      id[u][0] = f.x, id[u][1] = f.y, id[u][2] = f.z, id[u][3] = f.w;
    }
    uint32_t r[kU][4];
    if (use) {
      // round 1: every row's table slot; round 2: the rank table for the rest
      unsigned long long t[kU][4];
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) t[u][j] = __ldg(tab + tab_slot(id[u][j]));
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t idx = id[u][j] - 1u;
          if ((uint32_t)t[u][j] == id[u][j])
            r[u][j] = (uint32_t)(t[u][j] >> 32);
          else
            r[u][j] = idx < d ? __ldg(ranks + idx) : 0u;
        }
    } else {
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t idx = id[u][j] - 1u;
          r[u][j] = idx < d ? __ldg(ranks + idx) : 0u;
        }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      if (vi >= nvec) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (id[u][j] - 1u >= d) record_violation(err, head + vi * 4 + j, id[u][j]);
      __stcs(ov + vi, make_uint4(r[u][0], r[u][1], r[u][2], r[u][3]));
    }
  }
}

}  // namespace

// true when the call was served here; false: use the plain gather.
bool recode_with_table(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint32_t* ranks,
                       uint32_t d, uint32_t* out, cudaStream_t s, int* rc) {
  *rc = SKX_OK;
  const uintptr_t fa = reinterpret_cast<uintptr_t>(fact), oa = reinterpret_cast<uintptr_t>(out);
  // rank tables larger than L2, enough rows per id to pay for the table, and
  // FK / output columns with the same 16-byte phase (vector loads and stores)
  if (ctx->recode_table == 0 || (uint64_t)d * 4 < ctx->l2_bytes || n < 4ull * d || fa % 4 ||
      fa % 16 != oa % 16)
    return false;
  const size_t tab_b = (size_t(1) << kTabBits) * 8;
  char* sp = static_cast<char*>(scratch(ctx, 1, tab_b + 256, s));
  if (!sp) {
    *rc = set_error(ctx, SKX_CUDA_ERROR, "recode: out of device memory for the rank table");
    return true;
  }
  auto* tab = reinterpret_cast<unsigned long long*>(sp);
  auto* flag = reinterpret_cast<unsigned int*>(sp + tab_b);
  cudaError_t e = cudaMemsetAsync(tab, 0xff, tab_b, s);  // empty: ~0 (no valid id matches)
  if (e != cudaSuccess) {
    *rc = cuda_fail(ctx, e, "recode memset");
    return true;
  }
  ctx->last_domain = d;
  k_tab_fill<<<grid_for(ctx, d, 256, 8), 256, 0, s>>>(ranks, d, tab);
  k_tab_sample<<<1, 1024, 0, s>>>(fact, n, tab, flag);
  uint64_t head = ((16 - fa % 16) % 16) / 4;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 4;
  k_recode_tab<<<grid_for(ctx, nvec ? nvec : 1, kThreads * kU, 8), kThreads, 0, s>>>(
      fact, head, nvec, n, ranks, d, tab, flag, out, ctx->err);
  ctx->launches += 3;
  const cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) *rc = cuda_fail(ctx, le, "recode");
  return true;
}

}  // namespace skx

// histogram.cu -- frequency histogram counts[id-1] += 1 (K1 in SURVEY.md §2.1).
//
// Reference: count_frequencies (proj/src/permindex.cpp:18-30): a single-thread
// scattered increment that throws DomainViolation at the first bad row.
//
// B200 design.  Before the reorder the hot
// keys are scattered ids, so the "ids <= h are hot" trick is unavailable and a
// Zipf(1.25) key alone takes ~22% of all rows: plain global atomics would
// serialise on a handful of L2 addresses.  Each CTA therefore keeps a
// shared-memory open-addressing table (key -> count) that captures the keys
// it sees first -- for skewed data these are the hot ones -- and:
//   1. warp-aggregates equal keys with __match_any_sync (one update per
//      distinct key per warp instruction),
//   2. the leader lane adds the group size to its table slot with a shared
//      atomic (claiming an empty slot with atomicCAS),
//   3. keys that do not find a slot within kProbe probes go straight to a
//      global red.add (cold tail, spread over many L2 lines),
//   4. at exit the table is flushed with one global red.add per live slot.
// The FK column is streamed once with 128-bit evict_first loads; the domain
// check is fused (first bad row via atomicMin, reported at skx_sync).
#include <cstdlib>

#include "skx_internal.cuh"

namespace skx {
namespace {

constexpr int kThreads = 512;
constexpr int kTableBits = 13;  // 8192 slots x 8 B = 64 KB per CTA
constexpr int kTable = 1 << kTableBits;
constexpr int kProbe = 4;
constexpr int kUnroll = 2;  // uint4 per thread per iteration

__device__ __forceinline__ uint32_t slot_hash(uint32_t id) {
  return (id * 0x9E3779B1u) >> (32 - kTableBits);
}

template <typename CT>
__device__ __forceinline__ void global_add(CT* counts, uint32_t idx, uint32_t c);
template <>
__device__ __forceinline__ void global_add<uint32_t>(uint32_t* counts, uint32_t idx, uint32_t c) {
  atomicAdd(counts + idx, c);
}
template <>
__device__ __forceinline__ void global_add<unsigned long long>(unsigned long long* counts,
                                                               uint32_t idx, uint32_t c) {
  atomicAdd(counts + idx, (unsigned long long)c);
}

template <typename CT>
__device__ __forceinline__ void count_one(uint32_t id, bool valid, uint32_t* keys, uint32_t* cnts,
                                          CT* counts) {
  // id is 1-based and in-domain when valid; invalid lanes carry id 0.
  const uint32_t key = valid ? id : 0u;
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const uint32_t lane = threadIdx.x & 31;
  if (key == 0u || lane != (uint32_t)(__ffs(peers) - 1)) return;
  const uint32_t c = __popc(peers);
  uint32_t h = slot_hash(key);
#pragma unroll
  for (int p = 0; p < kProbe; ++p) {
    uint32_t k = keys[h];
    if (k == 0u) {
      k = atomicCAS(&keys[h], 0u, key);
      if (k == 0u) k = key;
    }
    if (k == key) {
      atomicAdd(&cnts[h], c);
      return;
    }
    h = (h + 1) & (kTable - 1);
  }
  global_add<CT>(counts, key - 1, c);
}

template <typename CT>
__global__ void __launch_bounds__(kThreads)
    k_histogram(const uint32_t* __restrict__ fact, uint64_t head, uint64_t nvec, uint64_t n,
                uint32_t d, uint32_t lo, uint32_t hi, bool check, CT* __restrict__ counts,
                DevErr* err) {
  extern __shared__ uint32_t smem_tab[];
  uint32_t* keys = smem_tab;
  uint32_t* cnts = smem_tab + kTable;
  for (int i = threadIdx.x; i < kTable; i += kThreads) {
    keys[i] = 0u;
    cnts[i] = 0u;
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
  const uint64_t per_iter = (uint64_t)kThreads * kUnroll;
  const uint64_t stride = (uint64_t)gridDim.x * per_iter;
  // Vector body; every lane of a warp runs the same trip count (match_any).
  const uint64_t nvec_round = (nvec + per_iter - 1) / per_iter * per_iter;
  for (uint64_t base = (uint64_t)blockIdx.x * per_iter + threadIdx.x; base < nvec_round;
       base += stride) {
    uint4 f[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      f[u] = vi < nvec ? ld_stream_v4(fv + vi, pol) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      const bool live = vi < nvec;
      const uint32_t ids[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idx = ids[j] - 1u;
        if (check && live && idx >= d) record_violation(err, head + vi * 4 + j, ids[j]);
        count_one<CT>(ids[j], live && idx >= lo && idx < hi, keys, cnts, counts);
      }
    }
  }
  // Scalar head [0, head) and tail [head + 4*nvec, n): block 0, warp-uniform trips.
  if (blockIdx.x == 0) {
    const uint64_t tail_b = head + nvec * 4;
    const uint64_t extra = head + (n - tail_b);  // < 8 rows
    for (uint64_t t0 = 0; t0 < extra; t0 += kThreads) {
      const uint64_t t = t0 + threadIdx.x;
      uint64_t k = 0;
      bool live = t < extra;
      if (live) k = t < head ? t : tail_b + (t - head);
      const uint32_t id = live ? fact[k] : 0u;
      const uint32_t idx = id - 1u;
      if (check && live && idx >= d) record_violation(err, k, id);
      count_one<CT>(id, live && idx >= lo && idx < hi, keys, cnts, counts);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kTable; i += kThreads) {
    const uint32_t k = keys[i];
    if (k != 0u && cnts[i] != 0u) global_add<CT>(counts, k - 1, cnts[i]);
  }
}

}  // namespace

int launch_histogram(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d, void* counts,
                     int counter_bytes, cudaStream_t s) {
  if (n == 0) return SKX_OK;
  if (n > (uint64_t(1) << 34))
    return set_error(ctx, SKX_INVALID_ARGUMENT, "histogram: more than 2^34 rows per call");
  if (counter_bytes == 4 && n > 0xFFFFFFFFull)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "histogram_u32: more than 2^32-1 rows");
  const uintptr_t fa = reinterpret_cast<uintptr_t>(fact);
  if (fa % 4 != 0) return set_error(ctx, SKX_INVALID_ARGUMENT, "fact pointer not 4-byte aligned");
  uint64_t head = ((16 - fa % 16) % 16) / 4;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 4;
  ctx->last_domain = d;
  const unsigned grid = grid_for(ctx, nvec ? nvec : 1, kThreads * kUnroll, 3);
  const size_t smem = size_t(2) * kTable * sizeof(uint32_t);
  if (counter_bytes == 4)
    cudaFuncSetAttribute(k_histogram<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  else
    cudaFuncSetAttribute(k_histogram<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // Optional key-range passes (SKX_HIST_RANGE ids per pass): each pass only
  // updates counters of ids in [lo, hi) so cold-key atomics stay in L2, at
  // the price of re-streaming the FK column per pass.  Measured on B200
  // (profiles/): one pass wins at BASELINE sizes (D=2^26: 6.96 ms single vs
  // 11.1 ms with 16M-key passes), so the default is a single pass.
  uint64_t range = (uint64_t)d + 1;
  if (const char* ev = getenv("SKX_HIST_RANGE")) range = strtoull(ev, nullptr, 10);
  if (range < (1u << 20)) range = 1u << 20;
  for (uint64_t lo = 0; lo < d || lo == 0; lo += range) {
    const uint32_t hi = (uint32_t)((lo + range < d) ? lo + range : d);
    const bool check = lo == 0;
    if (counter_bytes == 4)
      k_histogram<uint32_t><<<grid, kThreads, smem, s>>>(fact, head, nvec, n, d, (uint32_t)lo, hi,
                                                         check, static_cast<uint32_t*>(counts), ctx->err);
    else
      k_histogram<unsigned long long><<<grid, kThreads, smem, s>>>(
          fact, head, nvec, n, d, (uint32_t)lo, hi, check,
          static_cast<unsigned long long*>(counts), ctx->err);
    ctx->launches++;
    if (hi >= d) break;
  }
  SKX_CHECK_LAUNCH(ctx, "histogram");
  return SKX_OK;
}

}  // namespace skx

extern "C" {

int skx_count_frequencies(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d,
                          uint64_t* counts, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  cudaStream_t s = skx::as_stream(stream);
  if (d > 0) {
    cudaError_t e = cudaMemsetAsync(counts, 0, uint64_t(d) * 8, s);
    if (e != cudaSuccess) return skx::cuda_fail(ctx, e, "count_frequencies memset");
  }
  return skx::launch_histogram(ctx, fact, n, d, counts, 8, s);
}

int skx_histogram_u32(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d,
                      uint32_t* counts, int accumulate, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  cudaStream_t s = skx::as_stream(stream);
  if (!accumulate && d > 0) {
    cudaError_t e = cudaMemsetAsync(counts, 0, uint64_t(d) * 4, s);
    if (e != cudaSuccess) return skx::cuda_fail(ctx, e, "histogram memset");
  }
  return skx::launch_histogram(ctx, fact, n, d, counts, 4, s);
}

}  // extern "C"

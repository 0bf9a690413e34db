// aggregate.cu -- Q3 group-by COUNT / SUM(measure) per key (K7 in SURVEY.md
// §2.1) and Q3a heavy-hitter counting.
//
// Reference: aggregate_count / aggregate_sum (proj/src/operators.cpp:100-118),
// the hybrid strategy of parallel_aggregate (proj/src/parallel.cpp:178-207:
// private per-thread bins for ids <= h, shared relaxed atomics for the tail,
// serial fold), the lane-copy variant (operators.cpp:120-165) and
// heavy_hitter_count (operators.cpp:184-203).
//
// B200 design: on a recoded (skew-reordered)
// FK column the hot keys are the ids 1..H, so each CTA holds private
// shared-memory bins for them (u32 count, u64 sum; H sized to the opt-in
// shared memory, ~18K keys) -- the GPU form of the hybrid plan's private hot
// region.  Tail keys go to global atomics on an interleaved {count, sum}
// pair so one 32-B sector carries both updates; because the index makes the
// warm keys a contiguous low-id range, the pair array's hot part stays L2
// resident.  Bins are folded into the pairs once per CTA at exit (the
// reference's serial fold, parallelised), then a de-interleave pass writes
// the caller's counts[] / sums[].  FK and measure are streamed once with
// 128-bit evict_first loads; the domain check is fused.
#include "skx_internal.cuh"

namespace skx {
namespace {

constexpr int kThreads = 1024;

template <int MW>
__device__ __forceinline__ void load_measure4(const void* measure, uint64_t row, bool vec,
                                              uint64_t pol, unsigned long long (&m)[4]) {
  if (MW == 8) {
    const unsigned long long* p = static_cast<const unsigned long long*>(measure) + row;
    if (vec) {
      const uint4 a = ld_stream_v4(p, pol), b = ld_stream_v4(p + 2, pol);
      m[0] = a.x | ((unsigned long long)a.y << 32);
      m[1] = a.z | ((unsigned long long)a.w << 32);
      m[2] = b.x | ((unsigned long long)b.y << 32);
      m[3] = b.z | ((unsigned long long)b.w << 32);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) m[j] = ld_stream_u64(p + j, pol);
    }
  } else if (MW == 4) {
    const uint32_t* p = static_cast<const uint32_t*>(measure) + row;
    if (vec) {
      const uint4 a = ld_stream_v4(p, pol);
      m[0] = a.x, m[1] = a.y, m[2] = a.z, m[3] = a.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) m[j] = ld_stream_u32(p + j, pol);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = 0;
  }
}

template <int MW>
__device__ __forceinline__ unsigned long long load_measure1(const void* measure, uint64_t row) {
  if (MW == 8) return static_cast<const unsigned long long*>(measure)[row];
  if (MW == 4) return static_cast<const uint32_t*>(measure)[row];
  return 0;
}

// One row: idx = id - 1 already domain-checked (idx < d).
template <int MW>
__device__ __forceinline__ void agg_row(uint32_t idx, unsigned long long m, uint32_t hot,
                                        uint32_t limit, uint32_t* hcnt, unsigned long long* hsum,
                                        unsigned long long* out) {
  if (idx < hot) {
    atomicAdd(&hcnt[idx], 1u);
    if (MW) atomicAdd(&hsum[idx], m);
  } else if (idx < limit) {
    if (MW) {
      atomicAdd(&out[2 * (uint64_t)idx], 1ull);
      atomicAdd(&out[2 * (uint64_t)idx + 1], m);
    } else {
      atomicAdd(&out[idx], 1ull);
    }
  }
}

// out: MW ? interleaved pairs [limit][2] : counts [limit].
template <int MW>
__global__ void __launch_bounds__(kThreads, 1)
    k_aggregate(const uint32_t* __restrict__ fact, const void* __restrict__ measure, uint64_t head,
                uint64_t nvec, uint64_t n, uint32_t d, uint32_t limit, uint32_t hot, bool mvec,
                unsigned long long* __restrict__ out, DevErr* err) {
  extern __shared__ unsigned long long smem_agg[];
  unsigned long long* hsum = smem_agg;                                  // [hot] if MW
  uint32_t* hcnt = reinterpret_cast<uint32_t*>(smem_agg + (MW ? hot : 0));  // [hot]
  for (uint32_t i = threadIdx.x; i < hot; i += kThreads) {
    hcnt[i] = 0u;
    if (MW) hsum[i] = 0ull;
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t vi = (uint64_t)blockIdx.x * kThreads + threadIdx.x; vi < nvec; vi += stride) {
    const uint4 f = ld_stream_v4(fv + vi, pol);
    unsigned long long m[4];
    load_measure4<MW>(measure, head + vi * 4, mvec, pol, m);
    const uint32_t ids[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t idx = ids[j] - 1u;
      if (idx < d)
        agg_row<MW>(idx, m[j], hot, limit, hcnt, hsum, out);
      else
        record_violation(err, head + vi * 4 + j, ids[j]);
    }
  }
  if (blockIdx.x == 0) {
    const uint64_t tail_b = head + nvec * 4;
    const uint64_t extra = head + (n - tail_b);
    for (uint64_t t = threadIdx.x; t < extra; t += kThreads) {
      const uint64_t k = t < head ? t : tail_b + (t - head);
      const uint32_t id = fact[k];
      const uint32_t idx = id - 1u;
      if (idx < d)
        agg_row<MW>(idx, load_measure1<MW>(measure, k), hot, limit, hcnt, hsum, out);
      else
        record_violation(err, k, id);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < hot; i += kThreads) {
    const uint32_t c = hcnt[i];
    if (c) {
      if (MW) {
        atomicAdd(&out[2 * (uint64_t)i], (unsigned long long)c);
        atomicAdd(&out[2 * (uint64_t)i + 1], hsum[i]);
      } else {
        atomicAdd(&out[i], (unsigned long long)c);
      }
    }
  }
}

__global__ void k_deinterleave(const unsigned long long* __restrict__ pairs, uint32_t d,
                               unsigned long long* __restrict__ counts,
                               unsigned long long* __restrict__ sums) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += stride) {
    const ulonglong2 p = reinterpret_cast<const ulonglong2*>(pairs)[i];
    if (counts) counts[i] = p.x;
    if (sums) sums[i] = p.y;
  }
}

template <int MW>
int aggregate_impl(skx_ctx* ctx, const uint32_t* fact, const void* measure, uint64_t n, uint32_t d,
                   uint32_t limit, uint32_t hot_req, unsigned long long* out, cudaStream_t s) {
  const uintptr_t fa = reinterpret_cast<uintptr_t>(fact);
  if (fa % 4 != 0) return set_error(ctx, SKX_INVALID_ARGUMENT, "fact pointer not 4-byte aligned");
  uint64_t head = ((16 - fa % 16) % 16) / 4;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 4;
  bool mvec = true;
  if (MW) mvec = (reinterpret_cast<uintptr_t>(static_cast<const char*>(measure) + head * MW) % 16) == 0;
  const size_t per_key = MW ? 12 : 4;
  const size_t budget = ctx->smem_optin > 2048 ? ctx->smem_optin - 2048 : 0;
  uint32_t hot = (uint32_t)(budget / per_key);
  if (hot_req && hot_req < hot) hot = hot_req;
  if (hot > limit) hot = limit;
  const size_t smem = (size_t)hot * per_key;
  cudaFuncSetAttribute(k_aggregate<MW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const unsigned grid = grid_for(ctx, nvec ? nvec : 1, kThreads, 1);
  k_aggregate<MW><<<grid, kThreads, smem, s>>>(fact, measure, head, nvec, n, d, limit, hot, mvec,
                                               out, ctx->err);
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "aggregate");
  return SKX_OK;
}

}  // namespace

int launch_aggregate(skx_ctx* ctx, const uint32_t* fact, const void* measure, int mw, uint64_t n,
                     uint32_t d, uint32_t hot, uint64_t* counts, uint64_t* sums, cudaStream_t s) {
  if (mw != 0 && mw != 4 && mw != 8)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "aggregate: measure width must be 0, 4 or 8");
  if (mw && !measure && n) return set_error(ctx, SKX_INVALID_ARGUMENT, "aggregate: null measure");
  if (n > (uint64_t(1) << 34))
    return set_error(ctx, SKX_INVALID_ARGUMENT, "aggregate: more than 2^34 rows per call");
  ctx->last_domain = d;
  if (mw == 0 || !sums) {
    // COUNT only: accumulate straight into the caller's counts.
    if (!counts) return SKX_OK;
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)d * 8, s);
    if (sums && e == cudaSuccess) e = cudaMemsetAsync(sums, 0, (size_t)d * 8, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "aggregate memset");
    if (n == 0) return SKX_OK;
    return aggregate_impl<0>(ctx, fact, nullptr, n, d, d, hot,
                             reinterpret_cast<unsigned long long*>(counts), s);
  }
  unsigned long long* pairs =
      static_cast<unsigned long long*>(scratch(ctx, 1, (size_t)d * 16 + 16));
  if (!pairs) return set_error(ctx, SKX_CUDA_ERROR, "aggregate: out of device memory");
  cudaError_t e = cudaMemsetAsync(pairs, 0, (size_t)d * 16, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "aggregate memset");
  int rc = SKX_OK;
  if (n > 0) {
    rc = mw == 8 ? aggregate_impl<8>(ctx, fact, measure, n, d, d, hot, pairs, s)
                 : aggregate_impl<4>(ctx, fact, measure, n, d, d, hot, pairs, s);
    if (rc) return rc;
  }
  if (d > 0) {
    k_deinterleave<<<grid_for(ctx, d, 256, 8), 256, 0, s>>>(
        pairs, d, reinterpret_cast<unsigned long long*>(counts),
        reinterpret_cast<unsigned long long*>(sums));
    ctx->launches++;
  }
  SKX_CHECK_LAUNCH(ctx, "aggregate deinterleave");
  return SKX_OK;
}

}  // namespace skx

extern "C" {

int skx_aggregate(skx_ctx* ctx, const uint32_t* fact, const void* measure, int measure_width,
                  uint64_t n, uint32_t d, uint32_t hot_threshold, uint64_t* counts, uint64_t* sums,
                  void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  return skx::launch_aggregate(ctx, fact, measure, measure_width, n, d, hot_threshold, counts,
                               sums, skx::as_stream(stream));
}

int skx_heavy_hitter_count(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d, uint32_t k,
                           uint64_t* counts, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (k == 0) return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "heavy_hitter_count: k must be at least 1");
  cudaStream_t s = skx::as_stream(stream);
  const uint32_t cutoff = k < d ? k : d;
  ctx->last_domain = d;
  if (cutoff > 0) {
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)cutoff * 8, s);
    if (e != cudaSuccess) return skx::cuda_fail(ctx, e, "heavy_hitter memset");
  }
  if (n == 0) return SKX_OK;
  return skx::aggregate_impl<0>(ctx, fact, nullptr, n, d, cutoff, cutoff,
                                reinterpret_cast<unsigned long long*>(counts), s);
}

}  // extern "C"

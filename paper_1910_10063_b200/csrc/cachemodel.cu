// cachemodel.cu -- the analytical LRU cache model of the reference
// (proj/src/cachemodel.cpp; size the on-chip tiers from
// the frequency profile), on the device.
//
//  * line_frequencies (cachemodel.cpp:22-45): per-line sums of per-rank value
//    frequencies.  One thread per line sums its members in ascending rank
//    order -- the reference's accumulation order -- so the result is
//    bit-identical: for the freq layout the members are consecutive ranks;
//    for the rand layout the ranks of the line's ids (inverse bijection) are
//    sorted in registers first.
//  * estimate_hit_rate (cachemodel.cpp:76-123): frequencies sorted descending
//    (CUB radix sort of the doubles), prefix sums (CUB scan), then one thread
//    per line runs the horizon search (doubling then bisection, each probe a
//    binary search over the sorted frequencies) and the per-line geometric
//    hit probability; a block reduction sums f * cdf.  The prefix sums are a
//    parallel scan, so the estimate matches the reference to rounding (the
//    tests use rtol 1e-9), not bit for bit.
//  * trace_from_column (cachemodel.cpp:175-186): line = (id - 1) / per_line,
//    id 0 a deferred DomainViolation at its row.
// simulate_lru is an exact sequential LRU over a trace -- inherently serial,
// host-side analysis code in the reference too -- and lives in capi.cu as a
// host entry point.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "skx_internal.cuh"

namespace skx {
namespace {

constexpr uint32_t kMaxPerLine = 256;  // rand layout: members sorted per thread

__global__ void k_line_freq_consecutive(const double* __restrict__ vf, uint32_t d, uint32_t per,
                                        uint64_t lines, double* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < lines; l += stride) {
    const uint64_t r0 = l * per;
    const uint64_t r1 = r0 + per < d ? r0 + per : d;
    double s = 0.0;
    for (uint64_t r = r0; r < r1; ++r) s += vf[r];
    out[l] = s;
  }
}

__global__ void k_invert(const uint32_t* __restrict__ rank_to_id, uint32_t d,
                         uint32_t* __restrict__ id_to_rank) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < d; r += stride)
    id_to_rank[rank_to_id[r] - 1] = (uint32_t)r;
}

__global__ void k_line_freq_scattered(const double* __restrict__ vf, uint32_t d, uint32_t per,
                                      uint64_t lines, const uint32_t* __restrict__ id_to_rank,
                                      double* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < lines; l += stride) {
    const uint64_t i0 = l * per;
    const uint32_t m = (uint32_t)((i0 + per < d ? i0 + per : d) - i0);
    uint32_t rk[kMaxPerLine];
    for (uint32_t j = 0; j < m; ++j) {  // insertion sort: ascending rank
      const uint32_t v = id_to_rank[i0 + j];
      uint32_t p = j;
      while (p > 0 && rk[p - 1] > v) {
        rk[p] = rk[p - 1];
        --p;
      }
      rk[p] = v;
    }
    double s = 0.0;
    for (uint32_t j = 0; j < m; ++j) s += vf[rk[j]];
    out[l] = s;
  }
}

// Number of leading entries > 0 of a descending array (single thread).
__global__ void k_count_positive(const double* __restrict__ sorted, uint64_t n,
                                 unsigned long long* __restrict__ npos) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (sorted[mid] > 0.0) lo = mid + 1; else hi = mid;
  }
  *npos = lo;
}

__global__ void __launch_bounds__(256)
    k_hit_rate(const double* __restrict__ sorted, const double* __restrict__ incl,
               const unsigned long long* __restrict__ npos_dev, uint64_t S,
               double* __restrict__ acc) {
  __shared__ double red[8];
  const uint64_t n = *npos_dev;
  double part = 0.0;
  if (n > S) {
    const double target = (double)S;
    const uint64_t cap = uint64_t(1) << 40;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const double f = sorted[i];
      if (f >= 1.0 - 1e-12) {
        part += f;
        continue;
      }
      // expected distinct lines in k trials ending at this line
      // (cachemodel.cpp:57-72); prefix sums from the inclusive scan
      auto ed = [&](uint64_t k) {
        const double cutoff = (1.0 - f) / (double)k;
        uint64_t lo = 0, hi = n;
        while (lo < hi) {
          const uint64_t mid = lo + (hi - lo) / 2;
          if (sorted[mid] > cutoff) lo = mid + 1; else hi = mid;
        }
        uint64_t m = lo;
        double mass = m ? incl[m - 1] : 0.0;
        if (f > cutoff) {
          mass -= f;
          m -= 1;
        }
        return (double)k - ((double)k * mass / (1.0 - f) - (double)m);
      };
      uint64_t hi = S;
      double dd = ed(hi);
      while (dd < target && hi < cap) {
        hi *= 2;
        dd = ed(hi);
      }
      uint64_t k = hi;
      if (dd >= target && hi > S) {
        uint64_t lo = hi / 2 + 1;
        while (lo < hi) {
          const uint64_t mid = lo + (hi - lo) / 2;
          if (ed(mid) >= target) hi = mid; else lo = mid + 1;
        }
        k = lo;
      }
      part += f * -expm1((double)k * log1p(-f));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    if (t != 0.0) atomicAdd(acc, t);
  }
}

__global__ void k_hit_finalize(const unsigned long long* __restrict__ npos_dev, uint64_t S,
                               const double* __restrict__ acc, double* __restrict__ result) {
  const double t = *acc;
  *result = *npos_dev <= S ? 1.0 : (t < 1.0 ? t : 1.0);
}

__global__ void k_trace(const uint32_t* __restrict__ fact, uint64_t n, uint32_t per,
                        uint32_t* __restrict__ out, DevErr* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const uint32_t id = fact[k];
    if (id == 0u) record_violation(err, k, 0u);
    out[k] = (id - 1u) / per;
  }
}

}  // namespace
}  // namespace skx

extern "C" {

int skx_line_frequencies(skx_ctx* ctx, const double* value_freqs, uint32_t d,
                         const uint32_t* rank_to_id, uint32_t per_line, double* out,
                         void* stream) {
  using namespace skx;
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (d == 0) return set_error(ctx, SKX_INVALID_ARGUMENT, "line_frequencies: empty frequency vector");
  if (per_line == 0 || (rank_to_id && per_line > kMaxPerLine))
    return set_error(ctx, SKX_INVALID_ARGUMENT, "line_frequencies: 1..256 elements per line");
  cudaStream_t s = as_stream(stream);
  const uint64_t lines = ((uint64_t)d + per_line - 1) / per_line;
  if (!rank_to_id) {
    k_line_freq_consecutive<<<grid_for(ctx, lines, 256, 8), 256, 0, s>>>(value_freqs, d, per_line,
                                                                        lines, out);
    ctx->launches++;
  } else {
    uint32_t* inv = static_cast<uint32_t*>(scratch(ctx, 1, (size_t)d * 4, s));
    if (!inv) return set_error(ctx, SKX_CUDA_ERROR, "line_frequencies: out of device memory");
    k_invert<<<grid_for(ctx, d, 256, 8), 256, 0, s>>>(rank_to_id, d, inv);
    k_line_freq_scattered<<<grid_for(ctx, lines, 256, 8), 256, 0, s>>>(value_freqs, d, per_line,
                                                                      lines, inv, out);
    ctx->launches += 2;
  }
  SKX_CHECK_LAUNCH(ctx, "line_frequencies");
  return SKX_OK;
}

int skx_estimate_hit_rate(skx_ctx* ctx, const double* line_freqs, uint64_t nlines,
                          uint64_t cache_lines, double* result, void* stream) {
  using namespace skx;
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (cache_lines == 0)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "estimate_hit_rate: cache must have at least 1 line");
  cudaStream_t s = as_stream(stream);
  if (nlines == 0) {
    const double one = 1.0;
    cudaError_t e = cudaMemcpyAsync(result, &one, 8, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "estimate_hit_rate");
  }
  if (nlines > 0x7FFFFFFFull)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "estimate_hit_rate: more than 2^31-1 lines");
  const int n = (int)nlines;
  size_t sort_b = 0, scan_b = 0;
  cub::DeviceRadixSort::SortKeysDescending(nullptr, sort_b, (const double*)nullptr,
                                           (double*)nullptr, n, 0, 64, s);
  cub::DeviceScan::InclusiveSum(nullptr, scan_b, (const double*)nullptr, (double*)nullptr, n, s);
  const size_t tmp_b = (sort_b > scan_b ? sort_b : scan_b);
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t arr_b = up((size_t)n * 8);
  char* sp = static_cast<char*>(scratch(ctx, 1, 2 * arr_b + up(tmp_b) + 256, s));
  if (!sp) return set_error(ctx, SKX_CUDA_ERROR, "estimate_hit_rate: out of device memory");
  double* sorted = reinterpret_cast<double*>(sp);
  double* incl = reinterpret_cast<double*>(sp + arr_b);
  void* tmp = sp + 2 * arr_b;
  unsigned long long* npos = reinterpret_cast<unsigned long long*>(sp + 2 * arr_b + up(tmp_b));
  double* acc = reinterpret_cast<double*>(npos + 1);
  cudaError_t e = cudaMemsetAsync(acc, 0, 8, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "estimate_hit_rate memset");
  size_t b1 = sort_b;
  e = cub::DeviceRadixSort::SortKeysDescending(tmp, b1, line_freqs, sorted, n, 0, 64, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "estimate_hit_rate sort");
  size_t b2 = scan_b;
  e = cub::DeviceScan::InclusiveSum(tmp, b2, sorted, incl, n, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "estimate_hit_rate scan");
  k_count_positive<<<1, 1, 0, s>>>(sorted, (uint64_t)n, npos);
  k_hit_rate<<<grid_for(ctx, (uint64_t)n, 256, 8), 256, 0, s>>>(sorted, incl, npos, cache_lines,
                                                               acc);
  k_hit_finalize<<<1, 1, 0, s>>>(npos, cache_lines, acc, result);
  ctx->launches += 3;
  SKX_CHECK_LAUNCH(ctx, "estimate_hit_rate");
  return SKX_OK;
}

int skx_trace_from_column(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t per_line,
                          uint32_t* out, void* stream) {
  using namespace skx;
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (per_line == 0) return set_error(ctx, SKX_INVALID_ARGUMENT, "trace_from_column: per_line = 0");
  ctx->last_domain = 0xFFFFFFFEu;  // kMaxDomainCardinality (column.hpp:17)
  if (n == 0) return SKX_OK;
  cudaStream_t s = as_stream(stream);
  k_trace<<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(fact, n, per_line, out, ctx->err);
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "trace_from_column");
  return SKX_OK;
}

}  // extern "C"

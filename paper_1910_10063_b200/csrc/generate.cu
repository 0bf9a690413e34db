// generate.cu -- parallel Zipf foreign-key generator (input fixture; §8a row
// a1 of SURVEY.md).
//
// Reference: generate_fact_column (proj/src/column.cpp:73-125) draws ranks
// i.i.d. by inverse-CDF lookup (upper_bound over the partial-sum CDF, last
// entry forced to 1.0) and maps rank -> id through random_bijection.  Its
// uniforms come from ONE sequential mt19937_64 stream, which cannot be split
// across 148 SMs; this generator keeps the same CDF (built on the host by
// skx_zipf_cdf_host, bit-identical doubles), the same upper_bound and clamp,
// and the same rank -> id bijection, but takes the k-th uniform from the
// counter-based SplitMix64 sequence keyed by splitmix64(seed ^ 0x5ca1ab1e):
//     u_k = (splitmix64(key + k * 0x9e3779b97f4a7c15) >> 11) * 2^-53
// so any row range can be generated independently (each GPU generates only
// its own shard).  oracle/skx_oracle.c:orc_generate_zipf_counter restates it
// on the CPU for parity.
#include "skx_internal.cuh"

namespace skx {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void k_generate_zipf(const double* __restrict__ cdf, uint32_t d,
                                const uint32_t* __restrict__ rank_to_id, uint64_t key,
                                uint64_t row_begin, uint64_t n, uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = row_begin + i;
    const double u = (double)(splitmix64(key + k * 0x9e3779b97f4a7c15ull) >> 11) * 0x1.0p-53;
    // std::upper_bound: first index with cdf[idx] > u.
    uint32_t lo = 0, len = d;
    while (len > 0) {
      const uint32_t half = len >> 1;
      if (!(u < __ldg(cdf + lo + half))) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    uint32_t rank = lo >= d ? d - 1 : lo;
    out[i] = rank_to_id ? __ldg(rank_to_id + rank) : rank + 1;
  }
}

uint64_t host_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

}  // namespace
}  // namespace skx

extern "C" int skx_generate_zipf(skx_ctx* ctx, const double* cdf, uint32_t d,
                                 const uint32_t* rank_to_id, uint64_t seed, uint64_t row_begin,
                                 uint64_t n, uint32_t* out, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (d == 0 || !cdf) return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "generate: empty domain");
  if (n == 0) return SKX_OK;
  const uint64_t key = skx::host_splitmix64(seed ^ 0x5ca1ab1eull);
  skx::k_generate_zipf<<<skx::grid_for(ctx, n, 256, 8), 256, 0, skx::as_stream(stream)>>>(
      cdf, d, rank_to_id, key, row_begin, n, out);
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "generate_zipf");
  return SKX_OK;
}

// ---- value-column fixtures (BASELINE configs 1-5) --------------------------
// kind 0: raw splitmix64(seed ^ (0xd1000000 + i)) truncated to `width`
//         (the reference bench's dimension column, dataset.cpp:35-38);
// kind 1: uniform integer p0 + splitmix64(seed + i*gamma) % p1;
// kind 2: float32 lognormal(mu = p0, sigma = p1) via Box-Muller in fp64.
namespace skx {
namespace {
__global__ void k_fill_column(int kind, int width, uint64_t seed, uint64_t n, double p0, double p1,
                              void* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t v;
    if (kind == 0) {
      v = splitmix64(seed ^ (0xd1000000ull + i));
    } else if (kind == 1) {
      v = (uint64_t)(int64_t)p0 + splitmix64(seed + i * 0x9e3779b97f4a7c15ull) % (uint64_t)p1;
    } else {
      const double u1 = ((splitmix64(seed + 2 * i * 0x9e3779b97f4a7c15ull) >> 11) + 1) * 0x1.0p-53;
      const double u2 = (splitmix64(seed + (2 * i + 1) * 0x9e3779b97f4a7c15ull) >> 11) * 0x1.0p-53;
      const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
      static_cast<float*>(out)[i] = (float)exp(p0 + p1 * z);
      continue;
    }
    if (width == 8) static_cast<uint64_t*>(out)[i] = v;
    else if (width == 4) static_cast<uint32_t*>(out)[i] = (uint32_t)v;
    else static_cast<uint16_t*>(out)[i] = (uint16_t)v;
  }
}
}  // namespace
}  // namespace skx

extern "C" int skx_fill_column(skx_ctx* ctx, int kind, int width, uint64_t seed, uint64_t n,
                               double p0, double p1, void* out, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (kind < 0 || kind > 2 || (kind == 2 && width != 4) ||
      (width != 2 && width != 4 && width != 8) || (kind == 1 && !(p1 >= 1.0)))
    return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "fill_column: bad kind/width/parameters");
  if (n == 0) return SKX_OK;
  skx::k_fill_column<<<skx::grid_for(ctx, n, 256, 8), 256, 0, skx::as_stream(stream)>>>(
      kind, width, seed, n, p0, p1, out);
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "fill_column");
  return SKX_OK;
}

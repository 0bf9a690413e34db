// combine.cu -- packing of per-GPU partials for the cross-GPU combine steps
// (SURVEY.md §8(e)), so the collectives move fewer bytes and stay exact.
//
// Group-by (config 3).  The reference folds per-worker u64 count arrays by
// plain addition (parallel.cpp:155-157); across GPUs that is a reduce of
// 16 B/key (2^24 keys: 256 MiB).  On a recoded column only the hottest ids
// have large counts, so the partial is shipped as
//     buf = [counts[0..hot) | sums[0..hot) | packed[hot..d)]   (u64)
//     packed[i] = counts[i] << 40 | sums[i]
// (8 B per tail key: ~128 MiB at C3).  An element-wise u64 SUM of G such
// buffers is exact for every tail key iff no field overflows:
//     sum over ranks of counts[i] < 2^24  and  of sums[i] < 2^40.
// The pack kernel records, per rank, the largest tail count and tail sum;
// their SUM over ranks (a 16-byte all-reduce before the reduce) bounds every
// key's global fields, and the caller takes the packed reduce only when that
// bound holds (else the plain 16 B/key reduce).
#include "skx_internal.cuh"

namespace skx {
namespace {

constexpr int kShift = 40;

__global__ void __launch_bounds__(256)
    k_groupby_pack(const unsigned long long* __restrict__ counts,
                   const unsigned long long* __restrict__ sums, uint64_t d, uint64_t hot,
                   unsigned long long* __restrict__ buf, unsigned long long* __restrict__ guard) {
  unsigned long long mc = 0, ms = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += stride) {
    const unsigned long long c = __ldcs(counts + i), s = sums ? __ldcs(sums + i) : 0ull;
    if (i < hot) {
      __stcs(buf + i, c);
      __stcs(buf + hot + i, s);
    } else {
      mc = c > mc ? c : mc;
      ms = s > ms ? s : ms;
      // fields clamped only for the store; an overflowing key fails the guard
      __stcs(buf + hot + i, (c << kShift) | (s & ((1ull << kShift) - 1)));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mc, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, ms, o);
    mc = a > mc ? a : mc;
    ms = b > ms ? b : ms;
  }
  if ((threadIdx.x & 31) == 0) {
    if (mc) atomicMax(guard, mc);
    if (ms) atomicMax(guard + 1, ms);
  }
}

__global__ void __launch_bounds__(256)
    k_groupby_unpack(const unsigned long long* __restrict__ buf, uint64_t d, uint64_t hot,
                     unsigned long long* __restrict__ counts, unsigned long long* __restrict__ sums) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += stride) {
    unsigned long long c, s;
    if (i < hot) {
      c = __ldcs(buf + i);
      s = __ldcs(buf + hot + i);
    } else {
      const unsigned long long w = __ldcs(buf + hot + i);
      c = w >> kShift;
      s = w & ((1ull << kShift) - 1);
    }
    if (counts) __stcs(counts + i, c);
    if (sums) __stcs(sums + i, s);
  }
}

}  // namespace
}  // namespace skx

extern "C" {

int skx_groupby_pack(skx_ctx* ctx, const uint64_t* counts, const uint64_t* sums, uint32_t d,
                     uint32_t hot, uint64_t* buf, uint64_t* guard, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  if (!counts || !buf || !guard || hot > d)
    return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "groupby_pack: bad arguments");
  cudaStream_t s = skx::as_stream(stream);
  cudaError_t e = cudaMemsetAsync(guard, 0, 16, s);
  if (e != cudaSuccess) return skx::cuda_fail(ctx, e, "groupby_pack memset");
  if (d == 0) return SKX_OK;
  skx::k_groupby_pack<<<skx::grid_for(ctx, d, 256, 8), 256, 0, s>>>(
      reinterpret_cast<const unsigned long long*>(counts),
      reinterpret_cast<const unsigned long long*>(sums), d, hot,
      reinterpret_cast<unsigned long long*>(buf), reinterpret_cast<unsigned long long*>(guard));
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "groupby_pack");
  return SKX_OK;
}

int skx_groupby_unpack(skx_ctx* ctx, const uint64_t* buf, uint32_t d, uint32_t hot,
                       uint64_t* counts, uint64_t* sums, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  if (!buf || hot > d) return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "groupby_unpack: bad arguments");
  if (d == 0) return SKX_OK;
  cudaStream_t s = skx::as_stream(stream);
  skx::k_groupby_unpack<<<skx::grid_for(ctx, d, 256, 8), 256, 0, s>>>(
      reinterpret_cast<const unsigned long long*>(buf), d, hot,
      reinterpret_cast<unsigned long long*>(counts), reinterpret_cast<unsigned long long*>(sums));
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "groupby_unpack");
  return SKX_OK;
}

int skx_groupby_packed_ok(const uint64_t* guard_sum) {
  // host check of the all-reduced guard: fields cannot overflow
  return guard_sum && guard_sum[0] < (uint64_t(1) << 24) && guard_sum[1] < (uint64_t(1) << 40);
}

}  // extern "C"

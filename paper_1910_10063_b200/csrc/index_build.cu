// index_build.cu -- the skew-aware permutation index (K2 sort-by-count and
// K3 inverse in SURVEY.md §2.1) plus the generic device exclusive scan.
//
// Reference: build_index (proj/src/permindex.cpp:32-58):
//   offsets = iota(1..D) std::sort'ed by (count desc, id asc);
//   ranks[offsets[r]-1] = r + 1;   Σcounts must equal total (:36-40).
//
// B200 design (DESIGN.md §Kernels/index build):
//  1. compaction: ids with count 0 keep ascending-id trailing ranks
//     (permindex.hpp:36-38), so they are written straight to their final
//     slot offsets[nnz + z] / ranks without sorting; non-zero ids become
//     (key = total - count, id) pairs in ascending id order.  At BASELINE
//     config 4 only ~19% of the 2^26 ids are non-zero.
//  2. one stable counting pass over all pairs places every id with count
//     < 255 at its final rank (digit 255 - count) and moves the ids with
//     count >= 255 -- at most total / 255 of them -- to a prefix, which then
//     takes a stable LSD radix sort on 8-bit digits over the bits of
//     (total - 1) (4 passes at 2^30 rows) on a tile grid sized for that
//     bound.  Ascending key = descending count; stability on an ascending-id
//     input gives the id tie-break (C4 sort 1.20 -> 0.82 ms).
//     Per pass: upsweep (per-tile digit counts), device scan over the
//     digit-major tile histogram, downsweep (stable warp-level multisplit with
//     __match_any_sync, then scatter).
//  3. the last downsweep writes offsets[pos] = id AND ranks[id-1] = pos + 1
//     (the inverse, K3, fused into the final scatter).
// No host synchronisation: nnz lives on the device and every kernel reads it.
#include "scan.cuh"

namespace skx {
namespace {

constexpr int kTileThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kTileThreads * kItems;  // 4096
constexpr int kWarps = kTileThreads / 32;

// --------------------------------------------------------------------------
// Generic exclusive scan (3 kernels): partial sums per 4096-item chunk,
// single-block scan of the partials, then per-chunk apply.
// Items are warp-striped: item i of lane l in warp w sits at
// chunk + w*512 + i*32 + l, so loads are coalesced.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kTileThreads)
    k_scan_partials(const uint32_t* __restrict__ in, uint64_t m, uint32_t* __restrict__ partials) {
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
    s += p < m ? in[p] : 0u;
  }
  s = warp_sum(s);
  __shared__ uint32_t ws[kWarps];
  if (lane == 0) ws[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < kWarps; ++i) t += ws[i];
    partials[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024)
    k_scan_top(uint32_t* __restrict__ partials, uint64_t np, uint32_t* __restrict__ total_dev) {
  __shared__ uint32_t wb[33];
  uint32_t carry = 0;
  for (uint64_t b = 0; b < np; b += 1024) {
    const uint64_t p = b + threadIdx.x;
    const uint32_t v = p < np ? partials[p] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exclusive_scan<uint32_t, 1024>(v, wb, &tot);
    if (p < np) partials[p] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_dev) *total_dev = carry;
}

__global__ void __launch_bounds__(kTileThreads)
    k_scan_apply(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t m,
                 const uint32_t* __restrict__ partials) {
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t v[kItems];
  uint32_t wsum = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
    v[i] = p < m ? in[p] : 0u;
  }
  // Per-iteration warp scans; running offset across iterations.
  uint32_t ex[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint32_t inc = warp_inclusive_scan(v[i]);
    ex[i] = wsum + inc - v[i];
    wsum += __shfl_sync(0xffffffffu, inc, 31);
  }
  __shared__ uint32_t wtot[kWarps];
  if (lane == 0) wtot[w] = wsum;
  __syncthreads();
  uint32_t woff = partials[blockIdx.x];
  for (int i = 0; i < w; ++i) woff += wtot[i];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
    if (p < m) out[p] = woff + ex[i];
  }
}

// --------------------------------------------------------------------------
// Compaction of the frequency profile.
// --------------------------------------------------------------------------
template <typename CT>
__global__ void __launch_bounds__(kTileThreads)
    k_compact_count(const CT* __restrict__ counts, uint32_t d, uint32_t* __restrict__ tile_nnz,
                    DevErr* err) {
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t nz = 0;
  unsigned long long sum = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
    const unsigned long long c = p < d ? (unsigned long long)counts[p] : 0ull;
    nz += c != 0;
    sum += c;
  }
  nz = warp_sum(nz);
  sum = warp_sum(sum);
  __shared__ uint32_t wn[kWarps];
  __shared__ unsigned long long ws[kWarps];
  if (lane == 0) {
    wn[w] = nz;
    ws[w] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // one same-address atomic per tile, not per warp: 16 K tiles at C4 (the
    // per-warp version serialised 131 K atomics on err->sum: 0.12 ms)
    uint32_t t = 0;
    unsigned long long st = 0;
    for (int i = 0; i < kWarps; ++i) t += wn[i], st += ws[i];
    tile_nnz[blockIdx.x] = t;
    if (st) atomicAdd(&err->sum, st);
  }
}

__global__ void k_check_total(DevErr* err, unsigned long long total) {
  if (err->sum != total) err->invalid = 1u;
  err->sum = 0ull;
}

template <typename CT, typename K>
__global__ void __launch_bounds__(kTileThreads)
    k_compact_write(const CT* __restrict__ counts, uint32_t d, unsigned long long total,
                    const uint32_t* __restrict__ tile_off, const uint32_t* __restrict__ nnz_dev,
                    K* __restrict__ keys, uint32_t* __restrict__ vals, uint32_t* __restrict__ offsets,
                    uint32_t* __restrict__ ranks) {
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t nnz = *nnz_dev;
  uint32_t nzmask[kItems];
  CT cv[kItems];  // kept for the key writes (no second read of counts)
  uint32_t wcount = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
    cv[i] = p < d ? counts[p] : CT(0);
  }
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    nzmask[i] = __ballot_sync(0xffffffffu, cv[i] != 0);
    wcount += __popc(nzmask[i]);
  }
  __shared__ uint32_t wn[kWarps];
  if (lane == 0) wn[w] = wcount;
  __syncthreads();
  uint32_t nz_before = tile_off[blockIdx.x];  // non-zero ids in earlier tiles
  for (int i = 0; i < w; ++i) nz_before += wn[i];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
    if (p < d) {
      const uint32_t id = (uint32_t)p + 1u;
      const uint32_t nz_rank = nz_before + __popc(nzmask[i] & lt);
      // ranks is written for every id (0 for the non-zero ones, which the
      // sort's last pass overwrites), so its sectors are written whole: a
      // masked store leaves partial sectors that HBM must read back.
      if ((nzmask[i] >> lane) & 1u) {
        keys[nz_rank] = (K)(total - (unsigned long long)cv[i]);
        vals[nz_rank] = id;
        ranks[id - 1] = 0u;
      } else {
        // zero ids before this one = p - (non-zero ids before this one)
        const uint32_t pos = nnz + ((uint32_t)p - nz_rank);
        offsets[pos] = id;
        ranks[id - 1] = pos + 1u;
      }
    }
    nz_before += __popc(nzmask[i]);
  }
}

// --------------------------------------------------------------------------
// Radix sort passes.  SMALL: the one counting pass over all pairs -- digit
// 255 - count for counts 1..254 (ascending digit = descending count, final
// order), digit 0 for counts >= 255 (the "big" keys, sorted afterwards by
// ordinary LSD passes over that prefix only).  Otherwise digit = 8 key bits.
// --------------------------------------------------------------------------
template <bool SMALL, typename K>
__device__ __forceinline__ uint32_t radix_digit(K key, int shift, unsigned long long total) {
  if (SMALL) {
    const unsigned long long c = total - (unsigned long long)key;  // the id's count, >= 1
    return c >= 255ull ? 0u : 255u - (uint32_t)c;
  }
  return (uint32_t)((key >> shift) & 0xFF);
}

template <typename K, bool SMALL = false>
__global__ void __launch_bounds__(kTileThreads)
    k_radix_upsweep(const K* __restrict__ keys, const uint32_t* __restrict__ nnz_dev, int shift,
                    uint32_t* __restrict__ hist, uint32_t ntiles, unsigned long long total = 0) {
  __shared__ uint32_t wcnt[kWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * 256; i += kTileThreads) (&wcnt[0][0])[i] = 0u;
  __syncthreads();
  const uint32_t nnz = *nnz_dev;
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  if (base < nnz) {
#pragma unroll 4
    for (int i = 0; i < kItems; ++i) {
      const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
      const bool valid = p < nnz;
      const uint32_t dg = valid ? radix_digit<SMALL>(keys[p], shift, total) : 256u;
      // (per-lane shared atomics instead: measured slower, C4 sort 1.18 -> 1.21 ms)
      const uint32_t peers = __match_any_sync(0xffffffffu, dg);
      if (valid && lane == __ffs(peers) - 1) wcnt[w][dg] += __popc(peers);
    }
  }
  __syncthreads();
  uint32_t t = 0;
#pragma unroll
  for (int i = 0; i < kWarps; ++i) t += wcnt[i][threadIdx.x];
  hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = t;
}

// LAST: write offsets[pos] = id and ranks[id-1] = pos + 1 (K3 fused).
// SMALL: LAST for digits >= 1, keys/vals out (the big prefix) for digit 0.
template <typename K, bool LAST, bool SMALL = false>
__global__ void __launch_bounds__(kTileThreads)
    k_radix_downsweep(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                      const uint32_t* __restrict__ nnz_dev, int shift,
                      const uint32_t* __restrict__ hist, uint32_t ntiles, K* __restrict__ keys_out,
                      uint32_t* __restrict__ vals_out, uint32_t* __restrict__ offsets,
                      uint32_t* __restrict__ ranks, unsigned long long total = 0) {
  __shared__ uint32_t wcnt[kWarps][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t nnz = *nnz_dev;
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  if (base >= nnz) return;  // uniform per block
  for (int i = threadIdx.x; i < kWarps * 256; i += kTileThreads) (&wcnt[0][0])[i] = 0u;
  __syncthreads();
  K key[kItems];
  uint32_t val[kItems];
  uint32_t rank[kItems];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
    const bool valid = p < nnz;
    key[i] = valid ? keys_in[p] : K(0);
    val[i] = valid ? vals_in[p] : 0u;
  }
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
    const bool valid = p < nnz;
    const uint32_t dg = valid ? radix_digit<SMALL>(key[i], shift, total) : 256u;
    // (8 ballots, one per digit bit, instead of __match_any_sync: measured
    // slower on B200, C4 sort 1.18 -> 1.50 ms)
    const uint32_t peers = __match_any_sync(0xffffffffu, dg);
    const uint32_t cur = valid ? wcnt[w][dg] : 0u;
    rank[i] = cur + __popc(peers & lt);
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wcnt[w][dg] = cur + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    // exclusive prefix over warps per digit, seeded with the global offset
    uint32_t run = hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x];
#pragma unroll
    for (int i = 0; i < kWarps; ++i) {
      const uint32_t c = wcnt[i][threadIdx.x];
      wcnt[i][threadIdx.x] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t p = base + w * (kItems * 32) + i * 32 + lane;
    if (p < nnz) {
      const uint32_t dg = radix_digit<SMALL>(key[i], shift, total);
      const uint32_t pos = wcnt[w][dg] + rank[i];
      if (LAST || (SMALL && dg != 0u)) {
        offsets[pos] = val[i];
        ranks[val[i] - 1] = pos + 1u;
      } else {
        keys_out[pos] = key[i];
        vals_out[pos] = val[i];
      }
    }
  }
}

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

template <typename CT, typename K>
int build_index_impl(skx_ctx* ctx, const CT* counts, uint32_t d, uint64_t total,
                     uint32_t* offsets, uint32_t* ranks, cudaStream_t s) {
  // in 64 bits: d up to 0xFFFFFFFE would wrap a 32-bit (d + kTile - 1)
  const uint64_t ntiles64 = ((uint64_t)d + kTile - 1) / kTile;
  if (ntiles64 > 0x7FFFFFFFull)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "build_index: %llu tiles exceed the launch grid",
                     (unsigned long long)ntiles64);
  const uint32_t ntiles = (uint32_t)ntiles64;
  // scratch layout: keys[2][d] | vals[2][d] | tile_nnz[ntiles] | tile_off[ntiles] |
  //                 hist[256*ntiles] | nnz
  const size_t kb = align_up(sizeof(K) * (size_t)d), vb = align_up(4 * (size_t)d);
  const size_t tb = align_up(4 * (size_t)ntiles), hb = align_up(4 * 256 * (size_t)ntiles);
  char* sp = static_cast<char*>(scratch(ctx, 0, 2 * kb + 2 * vb + 2 * tb + hb + 256, s));
  if (!sp) return set_error(ctx, SKX_CUDA_ERROR, "build_index: out of device memory for scratch");
  K* keys[2] = {reinterpret_cast<K*>(sp), reinterpret_cast<K*>(sp + kb)};
  uint32_t* vals[2] = {reinterpret_cast<uint32_t*>(sp + 2 * kb),
                       reinterpret_cast<uint32_t*>(sp + 2 * kb + vb)};
  uint32_t* tile_nnz = reinterpret_cast<uint32_t*>(sp + 2 * kb + 2 * vb);
  uint32_t* tile_off = reinterpret_cast<uint32_t*>(sp + 2 * kb + 2 * vb + tb);
  uint32_t* hist = reinterpret_cast<uint32_t*>(sp + 2 * kb + 2 * vb + 2 * tb);
  uint32_t* nnz = reinterpret_cast<uint32_t*>(sp + 2 * kb + 2 * vb + 2 * tb + hb);
  uint32_t* nbig = nnz + 1;

  k_compact_count<CT><<<ntiles, kTileThreads, 0, s>>>(counts, d, tile_nnz, ctx->err);
  int rc = launch_exclusive_scan_u32(ctx, tile_nnz, tile_off, ntiles, nnz, 3, s);
  if (rc) return rc;
  k_check_total<<<1, 1, 0, s>>>(ctx->err, total);
  k_compact_write<CT, K><<<ntiles, kTileThreads, 0, s>>>(counts, d, total, tile_off, nnz, keys[0],
                                                       vals[0], offsets, ranks);
  ctx->launches += 3;
  // key range [0, total-1]
  int bits = 0;
  for (uint64_t t = total > 0 ? total - 1 : 0; t; t >>= 1) ++bits;
  int passes = (bits + 7) / 8;
  if (passes == 0) passes = 1;
  int cur = 0;
  const uint32_t* live = nnz;  // device count of the pairs the next pass sorts
  uint32_t nt = ntiles;        // tiles of the next pass
  if (passes > 1) {
    // One counting pass places every id with count < 255 at its final rank
    // (descending count is ascending 255 - count; ids ascend within a count
    // by stability) and moves the ids with count >= 255 -- few, they carry
    // the skew -- to the front of the other buffer; only that prefix then
    // takes the LSD passes (C4: 4 passes over 12.7 M pairs -> 1 + 4 over a
    // few thousand).
    k_radix_upsweep<K, true><<<ntiles, kTileThreads, 0, s>>>(keys[cur], nnz, 0, hist, ntiles, total);
    ctx->launches++;
    rc = launch_exclusive_scan_u32(ctx, hist, hist, (uint64_t)256 * ntiles, nullptr, 3, s);
    if (rc) return rc;
    // digit 1 starts where the big prefix ends (tile 0's offset for digit 1)
    cudaError_t e = cudaMemcpyAsync(nbig, hist + ntiles, 4, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "build_index copy");
    k_radix_downsweep<K, false, true><<<ntiles, kTileThreads, 0, s>>>(
        keys[cur], vals[cur], nnz, 0, hist, ntiles, keys[cur ^ 1], vals[cur ^ 1], offsets, ranks,
        total);
    ctx->launches++;
    cur ^= 1;
    live = nbig;
    // at most total / 255 ids have a count >= 255: size the tile grid of the
    // remaining passes (and their digit-major histogram) for that bound
    const uint64_t big_max = (uint64_t)d < total / 255 ? (uint64_t)d : total / 255;
    const uint64_t tb_ = (big_max + kTile - 1) / kTile;
    nt = tb_ == 0 ? 1u : (tb_ < ntiles ? (uint32_t)tb_ : ntiles);
  }
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = pass * 8;
    k_radix_upsweep<K><<<nt, kTileThreads, 0, s>>>(keys[cur], live, shift, hist, nt);
    ctx->launches++;
    rc = launch_exclusive_scan_u32(ctx, hist, hist, (uint64_t)256 * nt, nullptr, 3, s);
    if (rc) return rc;
    if (pass == passes - 1) {
      k_radix_downsweep<K, true><<<nt, kTileThreads, 0, s>>>(
          keys[cur], vals[cur], live, shift, hist, nt, nullptr, nullptr, offsets, ranks);
    } else {
      k_radix_downsweep<K, false><<<nt, kTileThreads, 0, s>>>(
          keys[cur], vals[cur], live, shift, hist, nt, keys[cur ^ 1], vals[cur ^ 1], nullptr,
          nullptr);
      cur ^= 1;
    }
    ctx->launches++;
  }
  SKX_CHECK_LAUNCH(ctx, "build_index");
  return SKX_OK;
}

template <typename CT>
int build_index_dispatch(skx_ctx* ctx, const CT* counts, uint32_t d, uint64_t total,
                         uint32_t* offsets, uint32_t* ranks, cudaStream_t s) {
  if (d > SKX_MAX_DOMAIN_CARDINALITY)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "frequency profile exceeds the 32-bit identifier space");
  if (d == 0) {
    // Nothing to order; Σcounts (empty) must still equal total.
    if (total != 0) return set_error(ctx, SKX_INVALID_ARGUMENT, "frequency profile counts do not sum to its total");
    return SKX_OK;
  }
  if (total > 0 && total - 1 > 0xFFFFFFFFull)
    return build_index_impl<CT, unsigned long long>(ctx, counts, d, total, offsets, ranks, s);
  return build_index_impl<CT, uint32_t>(ctx, counts, d, total, offsets, ranks, s);
}

}  // namespace

int launch_exclusive_scan_u32(skx_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t m,
                              uint32_t* total_dev, int slot, cudaStream_t s) {
  if (m == 0) return SKX_OK;
  const uint64_t np = (m + kTile - 1) / kTile;
  uint32_t* partials = static_cast<uint32_t*>(scratch(ctx, slot, np * 4 + 64, s));
  if (!partials) return set_error(ctx, SKX_CUDA_ERROR, "scan: out of device memory");
  k_scan_partials<<<(unsigned)np, kTileThreads, 0, s>>>(in, m, partials);
  k_scan_top<<<1, 1024, 0, s>>>(partials, np, total_dev);
  k_scan_apply<<<(unsigned)np, kTileThreads, 0, s>>>(in, out, m, partials);
  ctx->launches += 3;
  SKX_CHECK_LAUNCH(ctx, "scan");
  return SKX_OK;
}

int launch_build_index(skx_ctx* ctx, const void* counts, int counter_bytes, uint32_t d,
                       uint64_t total, uint32_t* offsets, uint32_t* ranks, cudaStream_t s) {
  if (counter_bytes == 4)
    return build_index_dispatch<uint32_t>(ctx, static_cast<const uint32_t*>(counts), d, total,
                                          offsets, ranks, s);
  return build_index_dispatch<unsigned long long>(
      ctx, static_cast<const unsigned long long*>(counts), d, total, offsets, ranks, s);
}

}  // namespace skx

extern "C" {

int skx_build_index(skx_ctx* ctx, const uint64_t* counts, uint32_t d, uint64_t total,
                    uint32_t* offsets, uint32_t* ranks, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  return skx::launch_build_index(ctx, counts, 8, d, total, offsets, ranks, skx::as_stream(stream));
}

int skx_build_index_u32(skx_ctx* ctx, const uint32_t* counts, uint32_t d, uint64_t total,
                        uint32_t* offsets, uint32_t* ranks, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  return skx::launch_build_index(ctx, counts, 4, d, total, offsets, ranks, skx::as_stream(stream));
}

int skx_rebuild(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d, uint32_t* offsets,
                uint32_t* ranks, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  if (d > SKX_MAX_DOMAIN_CARDINALITY)
    return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "domain cardinality exceeds the 32-bit identifier space");
  cudaStream_t s = skx::as_stream(stream);
  // rebuild = build_index(count_frequencies(fact, D)) (permindex.cpp:86-88).
  // u32 counters suffice below 2^32 rows (halves atomic and scan bytes).
  const bool narrow = n <= 0xFFFFFFFFull;
  const size_t cb = narrow ? 4 : 8;
  void* counts = skx::scratch(ctx, 1, cb * (size_t)d + 16, s);
  if (!counts) return skx::set_error(ctx, SKX_CUDA_ERROR, "rebuild: out of device memory");
  if (d > 0) {
    cudaError_t e = cudaMemsetAsync(counts, 0, cb * (size_t)d, s);
    if (e != cudaSuccess) return skx::cuda_fail(ctx, e, "rebuild memset");
  }
  int rc = skx::launch_histogram(ctx, fact, n, d, counts, (int)cb, true, s);
  if (rc) return rc;
  return skx::launch_build_index(ctx, counts, (int)cb, d, n, offsets, ranks, s);
}

}  // extern "C"

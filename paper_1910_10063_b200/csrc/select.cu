// select.cu -- Q2 selection (K8 in SURVEY.md §2.1): bitmap probe plus
// order-preserving compaction, optionally fused with the config-5 four-column
// gather and per-category fp64 SUM(price); plus the bitmap helpers.
//
// Reference: KernelTable::select_offsets (proj/src/kernels/scalar.cpp:31-42,
// avx2.cpp:59-98), select (operators.cpp:87-98), parallel_select
// (parallel.cpp:102-129: per-thread results concatenated in chunk order),
// permute_bitmap (operators.cpp:21-30), build_bitmap (operators.hpp:38-45).
//
// B200 design: two streaming passes over the
// FK column with a device scan between them -- pass 1 probes every row once,
// writes a 1-bit/row selection mask and counts each 4096-row tile's selected
// rows; the scan turns the counts into tile offsets; pass 2 reads the mask
// and the FKs, compacts the tile's selected rows in shared memory and writes
// each at tile offset + rank in tile: ascending row order, exactly the
// reference's chunk-ordered concatenation.  (A single-pass decoupled
// look-back version was measured ~2x slower on B200: CTAs stall behind the
// look-back chain, profiles/r1_experiments.md.)  The C5 variant gathers
// category / price / supplier / flag for the selected rows in pass 2, and a
// third pass sums price per category over the compacted columns in
// warp-private fp64 shared bins: lanes of one category are pre-summed with
// __match_any_sync + shuffles, because shared fp64 atomics compile to CAS
// spin loops on sm_100a.  Bins are flushed once per CTA.
#include "scan.cuh"

namespace skx {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 rows
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kSmemCategories = 2048;  // per-warp fp64 bins: 8 x 2048 x 8 B = 128 KB

struct Cols {
  const int32_t* cat;
  const float* price;
  const unsigned long long* supp;
  const uint16_t* flag;
  int32_t* out_cat;
  float* out_price;
  unsigned long long* out_supp;
  uint16_t* out_flag;
  double* sums;
  uint32_t n_categories;
};

// Probe one warp-striped item: row = tile*4096 + w*512 + i*32 + lane.  The
// first `sw` bitmap words live in shared memory: on a skew-reordered column
// the hot ids -- most probes -- fall in that prefix.
__device__ __forceinline__ bool probe(const uint32_t* __restrict__ fact, uint64_t k, uint64_t n,
                                      const unsigned long long* __restrict__ words, uint64_t bits,
                                      const unsigned long long* s_words, uint32_t sw, uint64_t pol,
                                      bool check, DevErr* err, uint32_t& idx) {
  idx = 0;
  if (k >= n) return false;
  const uint32_t id = ld_stream_u32(fact + k, pol);
  idx = id - 1u;
  if (idx < bits) {
    const uint32_t wi = idx >> 6;
    const unsigned long long wv = wi < sw ? s_words[wi] : __ldg(words + wi);
    return (wv >> (idx & 63)) & 1ull;
  }
  if (check) record_violation(err, k, id);
  return false;
}

// Pass 1: probe every row once, store the selection as one 32-bit mask word
// per warp-item (1 bit per row, coalesced), count selected rows per tile
// (grid-stride over tiles) and check the domain.
__global__ void __launch_bounds__(kThreads)
    k_select_count(const uint32_t* __restrict__ fact, uint64_t n,
                   const unsigned long long* __restrict__ words, uint64_t bits,
                   uint32_t* __restrict__ mask, uint32_t* __restrict__ tile_counts, uint32_t sw,
                   DevErr* err) {
  extern __shared__ __align__(16) unsigned long long s_words[];  // bitmap prefix [sw]
  __shared__ uint32_t s_w[kWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t pol = policy_evict_first();
  for (uint32_t i = threadIdx.x; i < sw; i += kThreads) s_words[i] = __ldg(words + i);
  __syncthreads();
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t row0 = tile * kTile + (uint64_t)w * (kItems * 32);
    // All 16 FK loads first, then all 16 bitmap probes, then the ballots: two
    // round trips per tile instead of sixteen dependent ones.
    uint32_t fk[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint64_t k = row0 + i * 32 + lane;
      fk[i] = k < n ? ld_stream_u32(fact + k, pol) : 1u;
    }
    bool sel[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint64_t k = row0 + i * 32 + lane;
      const uint32_t idx = fk[i] - 1u;
      sel[i] = false;
      if (k < n) {
        if (idx < bits) {
          const uint32_t wi = idx >> 6;
          const unsigned long long wv = wi < sw ? s_words[wi] : __ldg(words + wi);
          sel[i] = (wv >> (idx & 63)) & 1ull;
        } else {
          record_violation(err, k, fk[i]);
        }
      }
    }
    uint32_t c = 0, mine = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint32_t b = __ballot_sync(0xffffffffu, sel[i]);
      c += __popc(b);
      if (lane == i) mine = b;
    }
    if (lane < kItems) mask[(row0 >> 5) + lane] = mine;  // 16 consecutive words per warp
    if (lane == 0) s_w[w] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int i = 0; i < kWarps; ++i) t += s_w[i];
      tile_counts[tile] = t;
    }
    __syncthreads();
  }
}

// Pass 2, per tile: (A) read the mask words, load the FK of selected rows
// and compact (dimension index, row in tile) into shared memory in row order;
// (B) process the compacted rows densely -- consecutive threads take
// consecutive selected rows, so the gathers are independent and the output
// stores coalesce.  FUSED adds the 4-column gather and per-category sums.
template <bool FUSED>
__global__ void __launch_bounds__(kThreads)
    k_select_write(const uint32_t* __restrict__ fact, uint64_t n, const uint32_t* __restrict__ mask,
                   uint32_t base_off, const uint32_t* __restrict__ tile_off,
                   const uint32_t* __restrict__ total, uint32_t* __restrict__ out_off, Cols cols,
                   unsigned long long* __restrict__ count_dev) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(smem_raw);             // [kTile]
  uint16_t* s_row = reinterpret_cast<uint16_t*>(s_idx + kTile);        // [kTile]
  __shared__ uint32_t s_w[kWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_dev = *total;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t pol = policy_evict_first();
  const uint32_t lt = lanemask_lt();
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t row0 = tile * kTile + (uint64_t)w * (kItems * 32);
    // (A) this warp's 16 mask words (lane i holds word i) and, in the same
    // round trip, all 512 of its FK values (coalesced; at ~10% selectivity
    // the selected rows' sectors would be fetched anyway).
    const uint32_t mw = lane < kItems ? __ldg(mask + (row0 >> 5) + lane) : 0u;
    uint32_t fk[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint64_t k = row0 + i * 32 + lane;
      fk[i] = k < n ? ld_stream_u32(fact + k, pol) : 0u;
    }
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) c += __popc(__shfl_sync(0xffffffffu, mw, i));
    if (lane == 0) s_w[w] = c;
    __syncthreads();
    uint32_t lpos = 0;
    for (int i = 0; i < w; ++i) lpos += s_w[i];
    uint32_t cnt_tile = 0;
    for (int i = 0; i < kWarps; ++i) cnt_tile += s_w[i];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint32_t m = __shfl_sync(0xffffffffu, mw, i);
      if ((m >> lane) & 1u) {
        const uint32_t r = (uint32_t)(w * (kItems * 32) + i * 32 + lane);
        const uint32_t j = lpos + __popc(m & lt);
        s_idx[j] = fk[i] - 1u;
        s_row[j] = (uint16_t)r;
      }
      lpos += __popc(m);
    }
    __syncthreads();
    // (B) dense pass over the tile's selected rows
    const uint64_t obase = tile_off[tile];
    for (uint32_t j0 = 0; j0 < cnt_tile; j0 += kThreads) {
      const uint32_t j = j0 + threadIdx.x;
      const bool live = j < cnt_tile;
      int32_t ct = -1;
      float pr = 0.f;
      if (live) {
        const uint64_t p = obase + j;
        out_off[p] = base_off + (uint32_t)(tile * kTile + s_row[j]);
        if (FUSED) {
          const uint32_t idx = s_idx[j];
          ct = __ldg(cols.cat + idx);
          pr = __ldg(cols.price + idx);
          const unsigned long long sp = __ldg(cols.supp + idx);
          const unsigned short fl = __ldg(reinterpret_cast<const unsigned short*>(cols.flag) + idx);
          cols.out_cat[p] = ct;
          cols.out_price[p] = pr;
          cols.out_supp[p] = sp;
          cols.out_flag[p] = fl;
        }
      }
    }
    __syncthreads();  // s_idx / s_row / s_w reused by the next tile
  }
}

// Pass 3 (C5): SUM(price) per category over the compacted selected rows --
// a coalesced read of the gathered category/price columns.  Warp-private
// fp64 shared bins; lanes of one category pre-sum with __match_any_sync +
// shuffles (shared fp64 atomics are CAS spin loops on sm_100a); one native
// global fp64 reduction per bin per CTA.
__global__ void __launch_bounds__(kThreads)
    k_category_sum(const int32_t* __restrict__ cat, const float* __restrict__ price,
                   const uint32_t* __restrict__ total, uint32_t n_categories,
                   double* __restrict__ sums) {
  extern __shared__ double s_bins[];  // [kWarps][n_categories] when small
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool smem = n_categories <= kSmemCategories;
  if (smem) {
    for (uint32_t i = threadIdx.x; i < kWarps * n_categories; i += kThreads) s_bins[i] = 0.0;
    __syncthreads();
  }
  constexpr int U = 8;  // rows per thread per iteration, loads issued first
  const uint64_t cnt = *total;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads * U;
  for (uint64_t j0 = (uint64_t)blockIdx.x * kThreads * U; j0 < cnt; j0 += stride) {  // uniform trips
    int32_t ct[U];
    float pr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t j = j0 + (uint64_t)u * kThreads + threadIdx.x;
      ct[u] = j < cnt ? __ldcs(cat + j) : -1;
      pr[u] = j < cnt ? __ldcs(price + j) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = (uint32_t)ct[u] < n_categories;
      const uint32_t peers = __match_any_sync(0xffffffffu, ok ? (uint32_t)ct[u] : 0xFFFFFFFFu);
      if (ok) {
        double grp = 0.0;
        for (uint32_t m = peers; m; m &= m - 1)
          grp += __shfl_sync(peers, (double)pr[u], __ffs(m) - 1);
        if (lane == __ffs(peers) - 1) {
          if (smem)
            s_bins[(size_t)w * n_categories + ct[u]] += grp;
          else
            atomicAdd(&sums[ct[u]], grp);
        }
      }
    }
  }
  if (smem) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n_categories; i += kThreads) {
      double v = 0.0;
      for (int ww = 0; ww < kWarps; ++ww) v += s_bins[(size_t)ww * n_categories + i];
      if (v != 0.0) atomicAdd(&sums[i], v);
    }
  }
}

// out bit r = pred(r) for r in [0, bits): one warp builds one u64 word from
// two ballots.  MODE 0: permute (pred = in bit offsets[r]-1); MODE 1: dim < thr.
template <int MODE>
__global__ void k_bitmap(const unsigned long long* __restrict__ in_words,
                         const uint32_t* __restrict__ offsets, const int32_t* __restrict__ dim,
                         int32_t thr, uint64_t bits, unsigned long long* __restrict__ out_words) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwords = (bits + 63) / 64;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t wd = warp; wd < nwords; wd += nwarps) {
    uint32_t half[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t r = wd * 64 + h * 32 + lane;
      bool b = false;
      if (r < bits) {
        if (MODE == 0) {
          const uint32_t i = offsets[r] - 1u;
          b = (in_words[i >> 6] >> (i & 63)) & 1ull;
        } else {
          b = dim[r] < thr;
        }
      }
      half[h] = __ballot_sync(0xffffffffu, b);
    }
    if (lane == 0) out_words[wd] = (unsigned long long)half[0] | ((unsigned long long)half[1] << 32);
  }
}

int select_impl(skx_ctx* ctx, bool fused, const uint32_t* fact, uint64_t n, const uint64_t* words,
                uint64_t bits, uint32_t base, uint32_t* out, Cols cols, uint64_t* count_dev,
                cudaStream_t s) {
  if (n > 0xFFFFFFFFull)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "select: fact row offsets exceed 32 bits");
  if (!count_dev) return set_error(ctx, SKX_INVALID_ARGUMENT, "select: null count pointer");
  ctx->last_domain = bits;
  cudaError_t e;
  if (fused && cols.sums && cols.n_categories) {
    e = cudaMemsetAsync(cols.sums, 0, (size_t)cols.n_categories * 8, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "select memset");
  }
  if (n == 0) {
    e = cudaMemsetAsync(count_dev, 0, 8, s);
    return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "select memset");
  }
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  // scratch: mask words [ntiles * 128] | tile counts | tile offsets | total
  uint32_t* sp = static_cast<uint32_t*>(scratch(ctx, 2, ntiles * (kTile / 32 + 2) * 4 + 256));
  if (!sp) return set_error(ctx, SKX_CUDA_ERROR, "select: out of device memory");
  uint32_t* mask = sp;
  uint32_t* counts = sp + ntiles * (kTile / 32);
  uint32_t* offs = counts + ntiles;
  uint32_t* total = offs + ntiles;
  const auto* wd = reinterpret_cast<const unsigned long long*>(words);
  // Optional bitmap prefix staged per CTA in shared memory.  Off: measured on
  // B200 at C5 (96 KB prefix, 2 CTAs/SM) 20.5 -> 38.2 ms -- the lost
  // occupancy and L1 capacity cost more than the on-chip probes save.
  const uint32_t sw = 0;
  const size_t smem1 = (size_t)sw * 8;
  cudaFuncSetAttribute(k_select_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  int per_sm1 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm1, k_select_count, kThreads, smem1);
  const unsigned grid1 = grid_for(ctx, ntiles, 1, per_sm1 < 1 ? 1 : per_sm1);
  k_select_count<<<grid1, kThreads, smem1, s>>>(fact, n, wd, bits, mask, counts, sw, ctx->err);
  ctx->launches++;
  int rc = launch_exclusive_scan_u32(ctx, counts, offs, ntiles, total, 3, s);
  if (rc) return rc;
  const size_t smem = (size_t)kTile * (4 + 2);
  int per_sm = 0;
  if (fused) {
    cudaFuncSetAttribute(k_select_write<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select_write<true>, kThreads, smem);
    const unsigned grid2 = grid_for(ctx, ntiles, 1, per_sm < 1 ? 1 : per_sm);
    k_select_write<true><<<grid2, kThreads, smem, s>>>(fact, n, mask, base, offs, total, out, cols,
                                                      reinterpret_cast<unsigned long long*>(count_dev));
    if (cols.n_categories) {
      const size_t bsmem =
          cols.n_categories <= kSmemCategories ? (size_t)kWarps * cols.n_categories * 8 : 0;
      cudaFuncSetAttribute(k_category_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
      int per_sm3 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3, k_category_sum, kThreads, bsmem);
      k_category_sum<<<(unsigned)ctx->num_sms * (per_sm3 < 1 ? 1 : per_sm3), kThreads, bsmem, s>>>(
          cols.out_cat, cols.out_price, total, cols.n_categories, cols.sums);
      ctx->launches++;
    }
  } else {
    cudaFuncSetAttribute(k_select_write<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select_write<false>, kThreads, smem);
    const unsigned grid2 = grid_for(ctx, ntiles, 1, per_sm < 1 ? 1 : per_sm);
    k_select_write<false><<<grid2, kThreads, smem, s>>>(fact, n, mask, base, offs, total, out, cols,
                                                       reinterpret_cast<unsigned long long*>(count_dev));
  }
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "select");
  return SKX_OK;
}

}  // namespace
}  // namespace skx

extern "C" {

int skx_select_offsets(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint64_t* words,
                       uint64_t bits, uint32_t base, uint32_t* out, uint64_t* count_dev,
                       void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::Cols cols{};
  return skx::select_impl(ctx, false, fact, n, words, bits, base, out, cols, count_dev,
                          skx::as_stream(stream));
}

int skx_select_gather_sum(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint64_t* words,
                          uint32_t d, const int32_t* cat, const float* price,
                          const uint64_t* supp, const uint16_t* flag, uint32_t base,
                          uint32_t n_categories, uint32_t* out_off, int32_t* out_cat,
                          float* out_price, uint64_t* out_supp, uint16_t* out_flag, double* sums,
                          uint64_t* count_dev, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (n && (!cat || !price || !supp || !flag || !out_cat || !out_price || !out_supp || !out_flag ||
            (n_categories && !sums)))
    return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "select_gather_sum: null column pointer");
  skx::Cols cols{cat, price, reinterpret_cast<const unsigned long long*>(supp), flag,
                 out_cat, out_price, reinterpret_cast<unsigned long long*>(out_supp), out_flag,
                 sums, n_categories};
  return skx::select_impl(ctx, true, fact, n, words, d, base, out_off, cols, count_dev,
                          skx::as_stream(stream));
}

int skx_permute_bitmap(skx_ctx* ctx, const uint64_t* words, uint64_t bits, const uint32_t* offsets,
                       uint32_t d, uint64_t* out_words, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (bits != d)
    return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "bitmap size does not match index cardinality");
  if (bits == 0) return SKX_OK;
  cudaStream_t s = skx::as_stream(stream);
  const uint64_t nwords = (bits + 63) / 64;
  skx::k_bitmap<0><<<skx::grid_for(ctx, nwords * 32, 256, 8), 256, 0, s>>>(
      reinterpret_cast<const unsigned long long*>(words), offsets, nullptr, 0, bits,
      reinterpret_cast<unsigned long long*>(out_words));
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "permute_bitmap");
  return SKX_OK;
}

int skx_build_bitmap_lt_i32(skx_ctx* ctx, const int32_t* dim, uint64_t d, int32_t threshold,
                            uint64_t* out_words, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  if (d == 0) return SKX_OK;
  cudaStream_t s = skx::as_stream(stream);
  const uint64_t nwords = (d + 63) / 64;
  skx::k_bitmap<1><<<skx::grid_for(ctx, nwords * 32, 256, 8), 256, 0, s>>>(
      nullptr, nullptr, dim, threshold, d, reinterpret_cast<unsigned long long*>(out_words));
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "build_bitmap");
  return SKX_OK;
}

}  // extern "C"

// select.cu -- Q2 selection (K8 in SURVEY.md §2.1): bitmap probe plus
// order-preserving compaction, optionally fused with the config-5 four-column
// gather and per-category fp64 SUM(price); plus the bitmap helpers.
//
// Reference: KernelTable::select_offsets (proj/src/kernels/scalar.cpp:31-42,
// avx2.cpp:59-98), select (operators.cpp:87-98), parallel_select
// (parallel.cpp:102-129: per-thread results concatenated in chunk order),
// permute_bitmap (operators.cpp:21-30), build_bitmap (operators.hpp:38-45).
//
// B200 design: single pass over the FK column
// with decoupled look-back.  A persistent grid takes 4096-row tiles from an
// atomic ticket (so every predecessor tile is already running), computes the
// tile's selected count with warp ballots, publishes its aggregate, looks
// back over predecessors' published prefixes (acquire/release at gpu scope)
// and writes the selected rows' offsets (and, fused, their gathered
// category/price/supplier/flag) at prefix + local rank -- ascending row
// order, exactly the reference's concatenation order.  Per-category sums
// live in shared memory (fp64) for the CTA's lifetime and are flushed once.
#include "scan.cuh"

namespace skx {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 rows
constexpr int kWarps = kThreads / 32;
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;
constexpr uint32_t kSmemCategories = 8192;

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

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

template <bool FUSED>
__global__ void __launch_bounds__(kThreads)
    k_select(const uint32_t* __restrict__ fact, uint64_t n, const unsigned long long* __restrict__ words,
             uint64_t bits, uint32_t base_off, uint32_t* __restrict__ out_off, Cols cols,
             unsigned long long* __restrict__ status, unsigned int* __restrict__ ticket,
             unsigned long long* __restrict__ count_dev, DevErr* err) {
  extern __shared__ double s_sums[];  // [n_categories] when FUSED and small
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_wtot[kWarps];
  __shared__ unsigned long long s_excl;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool smem_sums = FUSED && cols.n_categories <= kSmemCategories;
  if (smem_sums) {
    for (uint32_t i = threadIdx.x; i < cols.n_categories; i += kThreads) s_sums[i] = 0.0;
  }
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t pol = policy_evict_first();
  const uint32_t lt = lanemask_lt();
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint64_t row0 = tile * kTile + (uint64_t)w * (kItems * 32);
    uint32_t sel[kItems];
    uint32_t idxs[kItems];
    uint32_t wcount = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint64_t k = row0 + i * 32 + lane;
      bool s = false;
      uint32_t idx = 0;
      if (k < n) {
        const uint32_t id = ld_stream_u32(fact + k, pol);
        idx = id - 1u;
        if (idx < bits) {
          s = (__ldg(words + (idx >> 6)) >> (idx & 63)) & 1ull;
        } else {
          record_violation(err, k, id);
        }
      }
      idxs[i] = idx;
      sel[i] = __ballot_sync(0xffffffffu, s);
      wcount += __popc(sel[i]);
    }
    if (lane == 0) s_wtot[w] = wcount;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long agg = 0;
      for (int i = 0; i < kWarps; ++i) agg += s_wtot[i];
      unsigned long long excl = 0;
      if (tile == 0) {
        st_release(&status[0], kFlagInc | agg);
      } else {
        st_release(&status[tile], kFlagAgg | agg);
        int64_t j = (int64_t)tile - 1;
        for (;;) {
          const unsigned long long st = ld_acquire(&status[j]);
          const unsigned long long flag = st & ~kValMask;
          if (flag == 0) continue;  // predecessor still counting
          excl += st & kValMask;
          if (flag == kFlagInc) break;
          --j;
        }
        st_release(&status[tile], kFlagInc | (excl + agg));
      }
      if (tile == ntiles - 1) *count_dev = excl + agg;
      s_excl = excl;
    }
    __syncthreads();
    uint64_t pos = s_excl;
    for (int i = 0; i < w; ++i) pos += s_wtot[i];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      if ((sel[i] >> lane) & 1u) {
        const uint64_t p = pos + __popc(sel[i] & lt);
        const uint64_t k = row0 + i * 32 + lane;
        out_off[p] = base_off + (uint32_t)k;
        if (FUSED) {
          const uint32_t idx = idxs[i];
          const int32_t c = __ldg(cols.cat + idx);
          const float pr = __ldg(cols.price + idx);
          cols.out_cat[p] = c;
          cols.out_price[p] = pr;
          cols.out_supp[p] = __ldg(cols.supp + idx);
          cols.out_flag[p] = __ldg(reinterpret_cast<const unsigned short*>(cols.flag) + idx);
          if ((uint32_t)c < cols.n_categories) {
            if (smem_sums)
              atomicAdd(&s_sums[c], (double)pr);
            else
              atomicAdd(&cols.sums[c], (double)pr);
          }
        }
      }
      pos += __popc(sel[i]);
    }
  }
  if (smem_sums) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cols.n_categories; i += kThreads) {
      const double v = s_sums[i];
      if (v != 0.0) atomicAdd(&cols.sums[i], v);
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
  char* sp = static_cast<char*>(scratch(ctx, 2, ntiles * 8 + 256));
  if (!sp) return set_error(ctx, SKX_CUDA_ERROR, "select: out of device memory");
  unsigned int* ticket = reinterpret_cast<unsigned int*>(sp);
  unsigned long long* status = reinterpret_cast<unsigned long long*>(sp + 256);
  e = cudaMemsetAsync(sp, 0, ntiles * 8 + 256, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "select memset");
  const size_t smem =
      (fused && cols.n_categories <= kSmemCategories) ? (size_t)cols.n_categories * 8 : 0;
  // Persistent grid: all CTAs resident, so look-back always makes progress.
  int per_sm = 0;
  if (fused) {
    cudaFuncSetAttribute(k_select<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select<true>, kThreads, smem);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select<false>, kThreads, 0);
  }
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)ctx->num_sms * per_sm;
  if (grid > ntiles) grid = ntiles;
  if (fused)
    k_select<true><<<(unsigned)grid, kThreads, smem, s>>>(
        fact, n, reinterpret_cast<const unsigned long long*>(words), bits, base, out, cols, status,
        ticket, reinterpret_cast<unsigned long long*>(count_dev), ctx->err);
  else
    k_select<false><<<(unsigned)grid, kThreads, 0, s>>>(
        fact, n, reinterpret_cast<const unsigned long long*>(words), bits, base, out, cols, status,
        ticket, reinterpret_cast<unsigned long long*>(count_dev), ctx->err);
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

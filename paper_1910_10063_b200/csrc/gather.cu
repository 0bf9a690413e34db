// gather.cu -- Q1 FK-join gather out[k] = dim[fact[k]-1] (K4/K5/K6 in
// SURVEY.md §2.1), also used for recode_fact (ranks as the dimension) and
// permute_dimension (offsets as the fact column).
//
// Reference semantics: KernelTable::gather_u32 (proj/src/kernels/scalar.cpp:13-29,
// avx2.cpp:43-57) behind materialize (operators.cpp:60-66), which first runs
// find_domain_violation (operators.cpp:32-41).  Here the domain check is fused
// into the gather pass (first offending row recorded with atomicMin, reported
// at skx_sync), so the FK column is streamed once.
//
// B200 design:
//  * HBM roofline: algorithmic bytes per row = 4 (FK) + w (output).  The
//    dimension reads are data-dependent and are what the skew-aware index
//    turns into L2 hits: the reordered hot ids form a contiguous prefix.
//  * FK stream: 128-bit ld.global.nc.L1::no_allocate with an L2 evict_first
//    policy; output: 128-bit st.global with evict_first.  Dimension loads take
//    the read-only path with L2 evict_last so the hot prefix survives the
//    streams.
//  * Each thread keeps UNROLL x 4 independent dimension loads in flight;
//    persistent grid-stride loop, grid = 148 x resident blocks.
#include "skx_internal.cuh"

namespace skx {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;  // uint4 FK vectors per thread per iteration (16 rows)

template <typename V>
struct Pack4;  // 4 values of width V as 16B/8B stores

template <>
struct Pack4<uint32_t> {
  static __device__ __forceinline__ void store(uint32_t* out, const uint32_t (&v)[4], uint64_t pol) {
    st_stream_v4(out, make_uint4(v[0], v[1], v[2], v[3]), pol);
  }
};
template <>
struct Pack4<uint64_t> {
  static __device__ __forceinline__ void store(uint64_t* out, const uint64_t (&v)[4], uint64_t pol) {
    st_stream_v4(out, make_uint4((uint32_t)v[0], (uint32_t)(v[0] >> 32), (uint32_t)v[1],
                                 (uint32_t)(v[1] >> 32)),
                 pol);
    st_stream_v4(out + 2, make_uint4((uint32_t)v[2], (uint32_t)(v[2] >> 32), (uint32_t)v[3],
                                     (uint32_t)(v[3] >> 32)),
                 pol);
  }
};
template <>
struct Pack4<uint16_t> {
  static __device__ __forceinline__ void store(uint16_t* out, const uint16_t (&v)[4], uint64_t pol) {
    st_stream_v2(out, make_uint2((uint32_t)v[0] | ((uint32_t)v[1] << 16),
                                 (uint32_t)v[2] | ((uint32_t)v[3] << 16)),
                 pol);
  }
};

// Vector body: rows [head, head + 4*nvec) where fact + head is 16B aligned.
// OUT_VEC: out + head is aligned for Pack4 stores.
template <typename V, bool OUT_VEC, bool POL>
__global__ void __launch_bounds__(kThreads)
    k_gather_vec(const uint32_t* __restrict__ fact, uint64_t head, uint64_t nvec,
                 const V* __restrict__ dim, uint64_t dim_len, V* __restrict__ out, DevErr* err) {
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_d = policy_evict_last();
  const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
  V* o = out + head;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads * kUnroll;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads * kUnroll + threadIdx.x; base < nvec;
       base += stride) {
    uint4 f[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      f[u] = vi < nvec ? ld_stream_v4(fv + vi, pol_s) : make_uint4(1, 1, 1, 1);
    }
    V v[kUnroll][4];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t ids[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idx = ids[j] - 1u;
        if (idx < dim_len) {
          v[u][j] = ld_dim<V>(dim + idx, pol_d, POL);
        } else {
          v[u][j] = 0;
          const uint64_t vi = base + (uint64_t)u * kThreads;
          if (vi < nvec) record_violation(err, head + vi * 4 + j, ids[j]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      if (vi < nvec) {
        if (OUT_VEC) {
          Pack4<V>::store(o + vi * 4, v[u], pol_s);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) o[vi * 4 + j] = v[u][j];
        }
      }
    }
  }
}

// Scalar rows [b, e) -- the unaligned head and the ragged tail (< 4 rows each).
template <typename V>
__global__ void k_gather_scalar(const uint32_t* __restrict__ fact, uint64_t b, uint64_t e,
                                const V* __restrict__ dim, uint64_t dim_len, V* __restrict__ out,
                                DevErr* err) {
  const uint64_t k = b + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= e) return;
  const uint32_t id = fact[k];
  const uint32_t idx = id - 1u;
  if (idx < dim_len) {
    out[k] = dim[idx];
  } else {
    out[k] = 0;
    record_violation(err, k, id);
  }
}

template <typename V>
int gather_impl(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const V* dim, uint64_t dim_len,
                V* out, cudaStream_t s) {
  if (n == 0) return SKX_OK;
  ctx->last_domain = dim_len;
  const uintptr_t fa = reinterpret_cast<uintptr_t>(fact);
  if (fa % 4 != 0) return set_error(ctx, SKX_INVALID_ARGUMENT, "fact pointer not 4-byte aligned");
  uint64_t head = ((16 - fa % 16) % 16) / 4;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 4;
  const uint64_t tail_b = head + nvec * 4;
  if (head > 0) {
    k_gather_scalar<V><<<1, 32, 0, s>>>(fact, 0, head, dim, dim_len, out, ctx->err);
    ctx->launches++;
  }
  if (nvec > 0) {
    const uintptr_t oa = reinterpret_cast<uintptr_t>(out + head);
    const bool out_vec = (sizeof(V) == 2) ? (oa % 8 == 0) : (oa % 16 == 0);
    const unsigned grid = grid_for(ctx, nvec, kThreads * kUnroll, 8);
    const bool pol = ctx->gather_policy == 1;
    if (out_vec) {
      if (pol)
        k_gather_vec<V, true, true><<<grid, kThreads, 0, s>>>(fact, head, nvec, dim, dim_len, out, ctx->err);
      else
        k_gather_vec<V, true, false><<<grid, kThreads, 0, s>>>(fact, head, nvec, dim, dim_len, out, ctx->err);
    } else {
      if (pol)
        k_gather_vec<V, false, true><<<grid, kThreads, 0, s>>>(fact, head, nvec, dim, dim_len, out, ctx->err);
      else
        k_gather_vec<V, false, false><<<grid, kThreads, 0, s>>>(fact, head, nvec, dim, dim_len, out, ctx->err);
    }
    ctx->launches++;
  }
  if (tail_b < n) {
    k_gather_scalar<V><<<1, 32, 0, s>>>(fact, tail_b, n, dim, dim_len, out, ctx->err);
    ctx->launches++;
  }
  SKX_CHECK_LAUNCH(ctx, "gather");
  return SKX_OK;
}

}  // namespace

int launch_gather(skx_ctx* ctx, int width, const uint32_t* fact, uint64_t n, const void* dim,
                  uint64_t dim_len, void* out, cudaStream_t s) {
  if (n > (uint64_t(1) << 34))
    return set_error(ctx, SKX_INVALID_ARGUMENT, "gather: more than 2^34 rows per call");
  if (n > 0 && (fact == nullptr || out == nullptr || (dim == nullptr && dim_len > 0)))
    return set_error(ctx, SKX_INVALID_ARGUMENT, "gather: null pointer");
  switch (width) {
    case 2:
      return gather_impl<uint16_t>(ctx, fact, n, static_cast<const uint16_t*>(dim), dim_len,
                                   static_cast<uint16_t*>(out), s);
    case 4:
      return gather_impl<uint32_t>(ctx, fact, n, static_cast<const uint32_t*>(dim), dim_len,
                                   static_cast<uint32_t*>(out), s);
    case 8:
      return gather_impl<uint64_t>(ctx, fact, n, static_cast<const uint64_t*>(dim), dim_len,
                                   static_cast<uint64_t*>(out), s);
  }
  return set_error(ctx, SKX_INVALID_ARGUMENT, "gather: value width must be 2, 4 or 8");
}

}  // namespace skx

extern "C" {

int skx_gather_u16(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint16_t* dim,
                   uint64_t dim_len, uint16_t* out, void* stream) {
  return skx::launch_gather(ctx, 2, fact, n, dim, dim_len, out, skx::as_stream(stream));
}
int skx_gather_u32(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint32_t* dim,
                   uint64_t dim_len, uint32_t* out, void* stream) {
  return skx::launch_gather(ctx, 4, fact, n, dim, dim_len, out, skx::as_stream(stream));
}
int skx_gather_u64(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint64_t* dim,
                   uint64_t dim_len, uint64_t* out, void* stream) {
  return skx::launch_gather(ctx, 8, fact, n, dim, dim_len, out, skx::as_stream(stream));
}

int skx_recode_fact(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint32_t* ranks,
                    uint32_t d, uint32_t* out, void* stream) {
  // permindex.cpp:60-64: recode is materialize(fact, ranks).
  return skx::launch_gather(ctx, 4, fact, n, ranks, d, out, skx::as_stream(stream));
}

#define SKX_PERMUTE(W, T)                                                                  \
  int skx_permute_dimension_u##W(skx_ctx* ctx, const T* dim, uint64_t dim_len,             \
                                 const uint32_t* offsets, uint32_t d, T* out, void* stream) { \
    if (dim_len != d)                                                                      \
      return skx::set_error(ctx, SKX_INVALID_ARGUMENT,                                     \
                            "dimension length %llu does not match index cardinality %u",   \
                            (unsigned long long)dim_len, d);                               \
    return skx::launch_gather(ctx, W / 8, offsets, d, dim, dim_len, out,                    \
                              skx::as_stream(stream));                                     \
  }
SKX_PERMUTE(16, uint16_t)
SKX_PERMUTE(32, uint32_t)
SKX_PERMUTE(64, uint64_t)

}  // extern "C"

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
//    turns into on-chip hits: the reordered hot ids form a contiguous prefix.
//  * Default policy 129 (profiles/r1_experiments.md): FK stream as 128-bit
//    ld.global.cs, output as 128-bit st.global.cs, dimension loads on the
//    read-only path (ld.global.nc, L1-allocating) with an L2 evict_last hint.
//    The other policy bits are measured alternatives kept for tuning:
//  * Hot prefix (policy bit 2): the first `hot` dimension values are staged
//    in shared memory once per CTA (one 1024-thread CTA per SM) and served
//    from there -- slower in practice: the carve-out starves L1.
//  * L1 no-allocate / coherent / L2-only dimension loads, an L2 persisting
//    window, per-id tiered priorities, FK software prefetch: no gain on B200.
//  * Each thread keeps 32 independent dimension loads in flight (8 FK
//    vectors); persistent grid-stride loop, 2 CTAs/SM (8/SM for long columns).
#include "skx_internal.cuh"

namespace skx {
namespace {

constexpr int kThreads = 256;      // plain variant: several CTAs per SM
constexpr int kThreadsHot = 1024;  // hot-prefix variant: one CTA per SM owns the smem copy
constexpr int kUnroll = 8;         // uint4 FK vectors per thread per iteration (32 rows)
#ifndef SKX_GATHER_MINB
#define SKX_GATHER_MINB 2     // resident CTAs per SM the registers must allow
#endif
#ifndef SKX_GATHER_SMALL_CTAS
#define SKX_GATHER_SMALL_CTAS 2    // CTAs per SM for small columns
#endif

// Policy bits (skx_set_gather_policy).
constexpr int kPolHints = 1;   // evict_first streams, evict_last dimension
constexpr int kPolHot = 2;     // shared-memory hot prefix
constexpr int kPolWindow = 4;  // L2 persisting access-policy window over the dimension
constexpr int kPolNoL1 = 8;    // dimension loads bypass L1 allocation
constexpr int kPolPrefetch = 16;  // software-pipeline the FK stream one iteration ahead
constexpr int kPolTiered = 32;    // per-access cache class from the reordered id (see below)
constexpr int kPolBulkOut = 2048;  // output staged in shared memory, 8 KB cp.async.bulk stores
constexpr int kPolSt256 = 4096;    // 256-bit output stores (one per 4-row vector of int64)
constexpr int kBulkRing = 4;       // 8 KB staging buffers per CTA (kPolBulkOut)

// Cache tiers of a skew-reordered dimension (policy bit 32).  After the
// index, popularity decreases with the id, so the id alone says how hot an
// access is -- the GPU form of the paper's hot/cold threshold t
// (§4.2.1, operators.cpp:68-85):
//   idx <  hot: shared memory                          (policy bit 2)
//   idx <  t1 : L1 evict_last,  L2 evict_last          (per-SM hot tier)
//   idx <  t2 : L1 evict_first, L2 evict_last          (chip-wide warm tier)
//   otherwise : L1 evict_first, L2 evict_first         (cold: must not evict
//               the warmer tiers -- untiered, every cold miss displaces them)
struct GatherTiers {
  uint32_t hot;  // shared-memory tier (policy bit 2)
  uint64_t t1;
  uint64_t t2;
};

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

// Dimension load without L1 allocation (L2 evict_last).
template <typename V>
__device__ __forceinline__ V ld_dim_nol1(const V* p, uint64_t pol);
template <>
__device__ __forceinline__ uint32_t ld_dim_nol1<uint32_t>(const uint32_t* p, uint64_t pol) {
  return ld_stream_u32(p, pol);
}
template <>
__device__ __forceinline__ uint64_t ld_dim_nol1<uint64_t>(const uint64_t* p, uint64_t pol) {
  return ld_stream_u64(p, pol);
}
template <>
__device__ __forceinline__ uint16_t ld_dim_nol1<uint16_t>(const uint16_t* p, uint64_t pol) {
  unsigned short r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
               : "=h"(r)
               : "l"(p), "l"(pol));
  return r;
}

// Dimension load with an L1 eviction priority (allocating) and an L2 policy.
template <typename V, bool LAST>
__device__ __forceinline__ V ld_dim_l1p(const V* p, uint64_t pol) {
  if constexpr (sizeof(V) == 8) {
    uint64_t r;
    if (LAST)
      asm volatile("ld.global.nc.L1::evict_last.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
    else
      asm volatile("ld.global.nc.L1::evict_first.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
    return (V)r;
  } else if constexpr (sizeof(V) == 4) {
    uint32_t r;
    if (LAST)
      asm volatile("ld.global.nc.L1::evict_last.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    else
      asm volatile("ld.global.nc.L1::evict_first.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return (V)r;
  } else {
    unsigned short r;
    if (LAST)
      asm volatile("ld.global.nc.L1::evict_last.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
    else
      asm volatile("ld.global.nc.L1::evict_first.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
    return (V)r;
  }
}

// Vector body: rows [head, head + 4*nvec) where fact + head is 16B aligned.
// OUT_VEC: out + head is aligned for Pack4 stores.
template <typename V, bool OUT_VEC, int F>
__global__ void __launch_bounds__((F & kPolHot) ? kThreadsHot : kThreads, (F & kPolHot) ? 1 : SKX_GATHER_MINB)
    k_gather_vec(const uint32_t* __restrict__ fact, uint64_t head, uint64_t nvec,
                 const V* __restrict__ dim, uint64_t dim_len, V* __restrict__ out, DevErr* err,
                 GatherTiers tiers) {
  constexpr bool HOT = (F & kPolHot) != 0;
  constexpr bool HINTS = (F & kPolHints) != 0;
  constexpr bool NOL1 = (F & kPolNoL1) != 0;
  constexpr bool PREF = (F & kPolPrefetch) != 0;
  constexpr bool TIER = (F & kPolTiered) != 0;
  const uint32_t hot = tiers.hot;
  constexpr int NT = HOT ? kThreadsHot : kThreads;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* s_hot = reinterpret_cast<V*>(smem_raw);
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_d = policy_evict_last();
  if (HOT) {
    // 16-byte cooperative copy of dim[0, hot) (hot * sizeof(V) is a multiple of 16).
    const uint4* src = reinterpret_cast<const uint4*>(dim);
    uint4* dst = reinterpret_cast<uint4*>(s_hot);
    const uint32_t nv = (uint32_t)((uint64_t)hot * sizeof(V) / 16);
    for (uint32_t i = threadIdx.x; i < nv; i += NT) dst[i] = __ldg(src + i);
    __syncthreads();
  }
  const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
  V* o = out + head;
  constexpr bool BULK = (F & kPolBulkOut) != 0 && !HOT && OUT_VEC;  // bulk stores: 16 B aligned
  // kPolBulkOut: for each u the CTA's NT vectors are one contiguous run of
  // NT * 4 rows (8 KB of int64), staged in a ring of kBulkRing buffers and
  // written by one cp.async.bulk store with an L2 evict_first hint.
  V* s_ring = reinterpret_cast<V*>(smem_raw);
  uint32_t ring_n = 0;
  const uint64_t stride = (uint64_t)gridDim.x * NT * kUnroll;
  uint64_t base = (uint64_t)blockIdx.x * NT * kUnroll + threadIdx.x;
  uint4 f[kUnroll];
  uint64_t dbg = 0;
  if (PREF) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * NT;
      f[u] = vi < nvec ? ld_stream_v4(fv + vi, pol_s) : make_uint4(1, 1, 1, 1);
    }
  }
  // BULK: CTA-uniform trip count (the staging barriers)
  for (; (BULK ? base - threadIdx.x : base) < nvec; base += stride) {
    uint4 fn[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      // PREF: next iteration's FK vectors are in flight while this one's
      // dimension loads resolve.
      const uint64_t vi = PREF ? base + stride + (uint64_t)u * NT : base + (uint64_t)u * NT;
      if (F & 128)
        fn[u] = vi < nvec ? __ldcs(fv + vi) : make_uint4(1, 1, 1, 1);
      else
        fn[u] = vi < nvec ? ld_stream_v4(fv + vi, pol_s) : make_uint4(1, 1, 1, 1);
    }
    if (!PREF) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) f[u] = fn[u];
    }
    V v[kUnroll][4];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t ids[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idx = ids[j] - 1u;
        if (HOT && idx < hot) {
          v[u][j] = s_hot[idx];
        } else if (idx < dim_len) {
          if (TIER) {
            if (idx < tiers.t1)
              v[u][j] = ld_dim_l1p<V, true>(dim + idx, pol_d);
            else
              v[u][j] = ld_dim_l1p<V, false>(dim + idx, idx < tiers.t2 ? pol_d : pol_s);
          } else if (NOL1) {
            v[u][j] = ld_dim_nol1<V>(dim + idx, pol_d);
          } else {
            if constexpr ((F & 1024) != 0 && sizeof(V) == 8) {  // coherent, no L1 allocation
              uint64_t r;
              asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(r) : "l"(dim + idx));
              v[u][j] = (V)r;
            } else if constexpr ((F & 512) != 0 && sizeof(V) == 8) {  // .cg: cache in L2 only
              v[u][j] = (V)__ldcg(reinterpret_cast<const unsigned long long*>(dim + idx));
            } else if constexpr ((F & 256) != 0 && sizeof(V) == 8) {  // coherent (non-.nc) load path
              uint64_t r;
              asm volatile("ld.global.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(dim + idx), "l"(pol_d));
              v[u][j] = (V)r;
            } else {
              v[u][j] = ld_dim<V>(dim + idx, pol_d, HINTS);
            }
          }
        } else {
          v[u][j] = 0;
          const uint64_t vi = base + (uint64_t)u * NT;
          if (vi < nvec) record_violation(err, head + vi * 4 + j, ids[j]);
        }
      }
    }
    if constexpr (BULK) {
      const uint64_t cta0 = base - threadIdx.x;  // first vector of this CTA iteration
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t v0 = cta0 + (uint64_t)u * NT;  // CTA-uniform
        const uint64_t vi = v0 + threadIdx.x;
        if (v0 + NT <= nvec) {
          V* buf = s_ring + (size_t)(ring_n % kBulkRing) * NT * 4;
          if (threadIdx.x == 0)  // the buffer's previous store has finished reading it
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kBulkRing - 1) : "memory");
          __syncthreads();
#pragma unroll
          for (int j = 0; j < 4; ++j) buf[threadIdx.x * 4 + j] = v[u][j];
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncthreads();
          if (threadIdx.x == 0) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(buf);
            asm volatile(
                "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                ::"l"(o + v0 * 4), "r"(sa), "r"((uint32_t)(NT * 4 * sizeof(V))), "l"(pol_s)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          ++ring_n;
        } else if (vi < nvec) {
#pragma unroll
          for (int j = 0; j < 4; ++j) o[vi * 4 + j] = v[u][j];
        }
      }
    } else {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * NT;
      if (vi < nvec) {
        if ((F & kPolSt256) && sizeof(V) == 8 && OUT_VEC) {  // one 256-bit store per vector
          asm volatile("st.global.cs.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(o + vi * 4),
                       "l"((uint64_t)v[u][0]), "l"((uint64_t)v[u][1]), "l"((uint64_t)v[u][2]),
                       "l"((uint64_t)v[u][3])
                       : "memory");
        } else if (F & 64) {  // diagnostic: keep the loads, drop the output stream
          dbg ^= (uint64_t)v[u][0] ^ (uint64_t)v[u][1] ^ (uint64_t)v[u][2] ^ (uint64_t)v[u][3];
        } else if (OUT_VEC) {
          if (F & 128) {  // .cs (streaming) cache operator instead of an L2 policy
            if constexpr (sizeof(V) == 8) {
              __stcs(reinterpret_cast<ulonglong2*>(o + vi * 4), make_ulonglong2(v[u][0], v[u][1]));
              __stcs(reinterpret_cast<ulonglong2*>(o + vi * 4) + 1, make_ulonglong2(v[u][2], v[u][3]));
            } else {
              Pack4<V>::store(o + vi * 4, v[u], pol_s);
            }
          } else {
            Pack4<V>::store(o + vi * 4, v[u], pol_s);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) o[vi * 4 + j] = v[u][j];
        }
      }
    }
    }  // !BULK
    if (PREF) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) f[u] = fn[u];
    }
  }
  if ((F & 64) && dbg == 0x5eed5eed5eedull) o[threadIdx.x] = (V)dbg;
  if (BULK && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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

template <typename V, bool OUT_VEC, int F>
cudaError_t launch_vec(skx_ctx* ctx, const uint32_t* fact, uint64_t head, uint64_t nvec,
                       const V* dim, uint64_t dim_len, V* out, GatherTiers tiers, cudaStream_t s) {
  const uint32_t hot = tiers.hot;
  constexpr bool HOT = (F & kPolHot) != 0;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(HOT ? kThreadsHot : kThreads);
  cfg.gridDim = dim3(HOT ? grid_for(ctx, nvec, kThreadsHot * kUnroll, 1)
                         // small columns: exactly the 2 resident CTAs/SM (no tail wave);
                         // large ones: 8/SM so the scheduler balances SM speed differences
                         : grid_for(ctx, nvec, kThreads * kUnroll,
                                    nvec / (kThreads * kUnroll) < 16u * 2u * ctx->num_sms
                                        ? SKX_GATHER_SMALL_CTAS : 8));
  cfg.dynamicSmemBytes = HOT ? (size_t)hot * sizeof(V)
                             : ((F & kPolBulkOut) ? (size_t)kBulkRing * kThreads * 4 * sizeof(V) : 0);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  const uint64_t dim_bytes = dim_len * sizeof(V);
  if ((F & kPolWindow) && ctx->persist_max > 0 && dim_bytes > cfg.dynamicSmemBytes) {
    // Persist the bytes right after the shared-memory tier, as far as the
    // L2 set-aside allows (hitRatio 1: a window no larger than the set-aside).
    const uint64_t skip = cfg.dynamicSmemBytes & ~uint64_t(127);
    uint64_t win = dim_bytes - skip;
    const uint64_t cap = (uint64_t)((double)ctx->persist_max * ctx->tier_l2_frac);
    if (win > cap) win = cap;
    if (win > ctx->window_max) win = ctx->window_max;
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr =
        const_cast<char*>(reinterpret_cast<const char*>(dim) + skip);
    attr[0].val.accessPolicyWindow.num_bytes = (size_t)win;
    attr[0].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.numAttrs = 1;
  }
  if (HOT || (F & kPolBulkOut))
    cudaFuncSetAttribute(k_gather_vec<V, OUT_VEC, F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)cfg.dynamicSmemBytes);
  return cudaLaunchKernelEx(&cfg, k_gather_vec<V, OUT_VEC, F>, fact, head, nvec, dim, dim_len, out,
                            ctx->err, tiers);
}

template <typename V, bool OUT_VEC>
cudaError_t dispatch_vec(skx_ctx* ctx, int F, const uint32_t* fact, uint64_t head, uint64_t nvec,
                         const V* dim, uint64_t dim_len, V* out, GatherTiers t, cudaStream_t s) {
  // Bit 4 (window) is a launch attribute; instantiate the useful variants only.
  const bool win = (F & kPolWindow) != 0;
#define SKX_F(x)                                                                            \
  if ((F & ~kPolWindow) == (x))                                                             \
    return win ? launch_vec<V, OUT_VEC, (x) | kPolWindow>(ctx, fact, head, nvec, dim, dim_len, \
                                                          out, t, s)                        \
               : launch_vec<V, OUT_VEC, (x)>(ctx, fact, head, nvec, dim, dim_len, out, t, s);
  SKX_F(0) SKX_F(1) SKX_F(3) SKX_F(9) SKX_F(17) SKX_F(19)
  SKX_F(33) SKX_F(35) SKX_F(49) SKX_F(51) SKX_F(65) SKX_F(97) SKX_F(69) SKX_F(129) SKX_F(128)
  SKX_F(131) SKX_F(385) SKX_F(641) SKX_F(1153) SKX_F(2177) SKX_F(4225)
#undef SKX_F
  return cudaErrorInvalidValue;
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
    int F = ctx->gather_policy;
    // Shared-memory tier: as many leading dimension values as fit.
    uint32_t hot = 0;
    if ((F & kPolHot) && (reinterpret_cast<uintptr_t>(dim) % 16) == 0) {
      size_t budget = ctx->smem_optin > 4096 ? ctx->smem_optin - 4096 : 0;
      if (ctx->tier_smem_bytes && ctx->tier_smem_bytes < budget) budget = ctx->tier_smem_bytes;
      uint64_t h = budget / sizeof(V);
      if (h > dim_len) h = dim_len;
      h &= ~uint64_t(32 / sizeof(V) - 1);  // hot * sizeof(V) a multiple of 32
      if (h >= 1024) hot = (uint32_t)h;
    }
    if (!hot) F &= ~kPolHot;
    GatherTiers t{hot, 0, 0};
    if (F & kPolTiered) {
      // t1: what one SM's L1 can hold (minus the smem tier); t2: the share of
      // L2 the warm tier may occupy (the rest carries the streams).
      t.t1 = hot + (uint64_t)ctx->tier_l1_bytes / sizeof(V);
      t.t2 = (uint64_t)((double)ctx->l2_bytes * ctx->tier_l2_frac) / sizeof(V);
    }
    const cudaError_t e =
        out_vec ? dispatch_vec<V, true>(ctx, F, fact, head, nvec, dim, dim_len, out, t, s)
                : dispatch_vec<V, false>(ctx, F, fact, head, nvec, dim, dim_len, out, t, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gather launch");
    ctx->launches++;
  }
  if (tail_b < n) {
    k_gather_scalar<V><<<1, 32, 0, s>>>(fact, tail_b, n, dim, dim_len, out, ctx->err);
    ctx->launches++;
  }
  SKX_CHECK_LAUNCH(ctx, "gather");
  return SKX_OK;
}

// ---- threshold-split materialize -------------------------
// Reference: materialize_split (operators.cpp:68-85) with the table entry
// gather_split_pass1 (kernels.hpp:32-39, scalar.cpp:44-61, avx2.cpp:100-143):
// pass 1 gathers the rows whose id <= t (the hot prefix of a reordered
// dimension) and writes 0 for the others while appending (row, id) to a miss
// list; pass 2 patches the misses.  On the CPU this keeps the hot gather free
// of the cold rows' cache pollution.  On B200 pass 1 streams exactly like the
// one-pass gather; the miss list is compacted per warp (ballot + one atomic),
// so its order across warps is arbitrary -- pass 2's result does not depend on
// it (every miss writes its own row).  Pass 2 reads the list coalesced, the
// dimension at random and stores 8 bytes at random rows (a sector
// read-modify-write each): measured against the one-pass gather in
// profiles/r2_experiments.md.
template <typename V>
__global__ void __launch_bounds__(256)
    k_split_pass1(const uint32_t* __restrict__ fact, uint64_t n, const V* __restrict__ dim,
                  uint64_t dim_len, uint32_t t, V* __restrict__ out, uint2* __restrict__ miss,
                  unsigned long long* __restrict__ nmiss, DevErr* err) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol_d = policy_evict_last();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t n_round = (n + 31) / 32 * 32;  // warp-uniform trips (ballots)
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_round; k += stride) {
    const bool live = k < n;
    const uint32_t id = live ? __ldcs(fact + k) : 1u;
    const uint32_t idx = id - 1u;
    const bool in = idx < dim_len;
    if (live && !in) record_violation(err, k, id);
    const bool cold = live && in && id > t;
    V v = 0;
    if (live && in && !cold) v = ld_dim<V>(dim + idx, pol_d, true);
    if (live) __stcs(out + k, v);
    const uint32_t m = __ballot_sync(0xffffffffu, cold);
    if (m) {
      unsigned long long at = 0;
      const int first = __ffs(m) - 1;
      if (lane == first) at = atomicAdd(nmiss, (unsigned long long)__popc(m));
      at = __shfl_sync(0xffffffffu, at, first);
      if (cold) miss[at + __popc(m & lanemask_lt())] = make_uint2((uint32_t)k, id);
    }
  }
}

template <typename V>
__global__ void __launch_bounds__(256)
    k_split_pass2(const uint2* __restrict__ miss, const unsigned long long* __restrict__ nmiss,
                  const V* __restrict__ dim, V* __restrict__ out) {
  const uint64_t m = *nmiss;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint2 e = __ldcs(miss + i);
    out[e.x] = __ldg(dim + (e.y - 1u));
  }
}

template <typename V>
int gather_split_impl(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const V* dim,
                      uint64_t dim_len, uint32_t t, V* out, cudaStream_t s) {
  if (t == 0 || t > dim_len)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "split threshold must lie in 1..D");
  if (n > 0xFFFFFFFFull)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "gather_split: row positions exceed 32 bits");
  if (n == 0) return SKX_OK;
  ctx->last_domain = dim_len;
  char* sp = static_cast<char*>(scratch(ctx, 1, 256 + n * sizeof(uint2), s));
  if (!sp) return set_error(ctx, SKX_CUDA_ERROR, "gather_split: out of device memory");
  auto* nmiss = reinterpret_cast<unsigned long long*>(sp);
  auto* miss = reinterpret_cast<uint2*>(sp + 256);
  cudaError_t e = cudaMemsetAsync(nmiss, 0, 8, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gather_split memset");
  k_split_pass1<V><<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(fact, n, dim, dim_len, t, out, miss,
                                                            nmiss, ctx->err);
  k_split_pass2<V><<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(miss, nmiss, dim, out);
  ctx->launches += 2;
  SKX_CHECK_LAUNCH(ctx, "gather_split");
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

int skx_gather_split_u32(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint32_t* dim,
                         uint64_t dim_len, uint32_t threshold, uint32_t* out, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  return skx::gather_split_impl<uint32_t>(ctx, fact, n, dim, dim_len, threshold, out,
                                          skx::as_stream(stream));
}
int skx_gather_split_u64(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint64_t* dim,
                         uint64_t dim_len, uint32_t threshold, uint64_t* out, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  return skx::gather_split_impl<uint64_t>(ctx, fact, n, dim, dim_len, threshold, out,
                                          skx::as_stream(stream));
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

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

// Control word of the partitioned gather (below): the plan kernel's verdict and
// sample (copied to the host's plan cache), and the fill pass's work counter.
struct PgCtrl {
  uint32_t mode;          // plan: 1 = partition this column
  uint32_t items;         // fill work-item counter
  uint32_t sample_first;  // plan: sampled rows that were miss candidates (of 65536)
  uint32_t sample_asc;    // plan: ascending adjacent id pairs within the sampled vectors (of 49152)
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
  else  // no shared memory: ask for the whole unified array as L1 whatever ran before
    cudaFuncSetAttribute(k_gather_vec<V, OUT_VEC, F>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxL1);
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
                                                          out, t, s)                  \
               : launch_vec<V, OUT_VEC, (x)>(ctx, fact, head, nvec, dim, dim_len, out, t, s);
  SKX_F(0) SKX_F(1) SKX_F(3) SKX_F(9) SKX_F(17) SKX_F(19)
  SKX_F(33) SKX_F(35) SKX_F(49) SKX_F(51) SKX_F(65) SKX_F(97) SKX_F(69) SKX_F(129) SKX_F(128)
  SKX_F(131) SKX_F(385) SKX_F(641) SKX_F(1153) SKX_F(2177) SKX_F(4225)
#undef SKX_F
  return cudaErrorInvalidValue;
}

// ---- partitioned gather (policy bit kPolPart) --------------------------------
// Same result as the one-pass gather; what changes is how the cold rows meet
// the dimension.  A row whose id lies past the L2-resident prefix (idx >= t)
// costs the one-pass kernel a random HBM access, and random accesses complete
// at ~43 G/s whatever their size: at C2 s=1.0 the ~200 M cold
// rows are two thirds of the launch.  Here they are radix-partitioned by key
// range instead, so each partition's dimension slice is read while it sits in
// L2 -- the GPU form of a partitioned hash join.  Over 8192-row chunks:
//   plan : beside a column's first (one-pass) launch one CTA samples 64 K rows and
//          decides whether enough of them would miss L2 in the one-pass kernel
//          to pay for the extra passes (k_pg_plan below); the decision reaches
//          the host asynchronously and later launches over the column follow it;
//   part : FK through a double-buffered 1-D TMA ring in shared memory; the
//          chunk's cold keys go to its record segment grouped by partition
//          (keys[]), and every row gets a translated word tr[] = its id - 1
//          (hot), 2^31 | its record slot (cold) or ~0 (out of domain);
//   fill : partition by partition (work items handed out in order by one
//          counter, so all CTAs share one slice), vals[i] = dim[keys[i]];
//   emit : the one-pass gather's streaming loop over tr: hot rows read the
//          dimension, cold rows their chunk's vals.
// Slots inside a chunk: each thread owns fixed rows and ranks its cold rows
// per partition with shared atomics on a private column (one thread per
// address, so program order, and pipelined -- a read-modify-write would chain
// every row behind the previous one); an exclusive scan over (partition,
// thread) turns the counts into slots.
constexpr int kPolPart = 8192;
constexpr int kPolPartForce = 16384;  // with kPolPart: partition at once, no plan (tests, measurements)
constexpr int kPgT = 256;                         // threads per CTA (part)
constexpr int kPgU = 8;                           // FK vectors per thread per chunk
constexpr uint32_t kPgChunkVec = kPgT * kPgU;     // 2048 vectors = 8192 rows
constexpr uint32_t kPgChunkRows = kPgChunkVec * 4;
constexpr int kPgChunkShift = 13;
constexpr int kPgRows = 32;                       // count rows: partitions + 1 dummy
constexpr uint32_t kPgMaxParts = kPgRows - 1;
constexpr int kPgFillChunks = 64;                 // chunks per fill work item
constexpr uint32_t kPgCold = 0x80000000u;         // tr: cold row, low bits = record slot
#ifndef SKX_PG_HOT_MB
#define SKX_PG_HOT_MB 32                          // direct (L2-resident) dimension prefix
#endif
#ifndef SKX_PG_SLICE_MB
#define SKX_PG_SLICE_MB 32                        // dimension bytes per partition
#endif
#ifndef SKX_PG_FILL_CTAS
#define SKX_PG_FILL_CTAS 6                        // fill CTAs per SM (what its 40 registers allow)
#endif
#ifndef SKX_PG_EMIT_STAGED
#define SKX_PG_EMIT_STAGED 1                      // emit reads a chunk's records through shared memory
#endif
#ifndef SKX_PG_MIN_COLD_PERMILLE
#define SKX_PG_MIN_COLD_PERMILLE 300
#endif
// part: ring[2][2048] uint4 | cnt[32][256] | base[64] | bar[2]
constexpr int kPgRing = 2 * kPgChunkVec * 16;
constexpr int kPgCnt = kPgRows * kPgT * 4;
constexpr int kPgPartSmem = kPgRing + kPgCnt + 64 * 4 + 16;

struct PgPlan {
  uint32_t t;        // idx < t: direct gather
  uint32_t dl;       // dimension length (<= 2^32 - 1)
  uint32_t shift;    // partition of a cold idx: (idx - t) >> shift
  uint32_t nparts;   // <= kPgMaxParts
  uint32_t nchunks;
  uint32_t* keys;    // [nchunks * kPgChunkRows]: chunk c's records start at c * kPgChunkRows
  void* vals;        // same layout, of V
  uint32_t* tr;      // [nvec * 4] translated FK words
  uint16_t* ends;    // [nchunks][32] end of partition p's records within the chunk
  PgCtrl* ctrl;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ bool pg_cold(const PgPlan& pl, uint32_t idx) {
  return idx - pl.t < pl.dl - pl.t;  // t <= idx < dl
}

// plan: should this launch take the partitioned path?  It pays when many rows
// would miss L2 in the one-pass kernel AND the partitions see each dimension
// line several times.  A sample of kPlanRuns runs of 64 consecutive rows,
// spread evenly over the column, is hashed by 128-byte dimension line into a
// 2^20-bit shared-memory set: a sampled row counts as a miss candidate when
// its id lies past the L2-resident prefix (idx >= t) and it is the first of
// the sample on its line.  Hot ids of a skewed column repeat within the
// sample and rows that walk the dimension in order (permute_dimension over
// count ties) share lines within their run, so neither counts; uniform or
// weakly skewed ids do.  The path turns on when the candidates are at least
// SKX_PG_MIN_COLD_PERMILLE of the sample and the launch's estimated cold rows
// touch each cold dimension line >= kPlanMinTouch times (fewer: the fill pass
// would fetch as many HBM lines as the one-pass kernel misses), unless >= 80% of
// the adjacent id pairs inside the sampled vectors ascend (an in-order walk).
constexpr uint32_t kPlanRuns = 1024, kPlanRunVec = 16;
constexpr uint32_t kPlanRows = kPlanRuns * kPlanRunVec * 4;  // 65536 sampled rows
constexpr uint32_t kPlanBitsLog2 = 20;
constexpr int kPlanSmem = (1 << kPlanBitsLog2) / 8;          // 128 KB
constexpr uint32_t kPlanMinTouch = 4;

__global__ void __launch_bounds__(1024) k_pg_plan(const uint4* __restrict__ fv, uint64_t nvec,
                                                  PgPlan pl, uint32_t line_shift, uint32_t force) {
  extern __shared__ __align__(16) uint32_t plan_bits[];
  __shared__ uint32_t wsum[32], wasc[32];
  const uint32_t tid = threadIdx.x;
  constexpr int kB = 8;  // sampled vectors in flight per thread
  const uint64_t span = nvec - kPlanRunVec;  // nvec >= 2^20 (pgather_impl)
  uint4 q[kB];
#pragma unroll
  for (int k = 0; k < kB; ++k)
    q[k] = fv[(uint64_t)((tid >> 4) + 64 * k) * span / (kPlanRuns - 1) + (tid & 15)];
  for (uint32_t i = tid; i < (1u << kPlanBitsLog2) / 128; i += 1024)
    reinterpret_cast<uint4*>(plan_bits)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  uint32_t first = 0, asc = 0;
  for (int half = 0; half < 2; ++half) {
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const uint32_t ids[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
      asc += (ids[1] > ids[0]) + (ids[2] > ids[1]) + (ids[3] > ids[2]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idx = ids[j] - 1u;
        if (pg_cold(pl, idx)) {
          const uint32_t h = ((idx >> line_shift) * 0x9E3779B1u) >> (32 - kPlanBitsLog2);
          const uint32_t bit = 1u << (h & 31);
          first += (atomicOr(plan_bits + (h >> 5), bit) & bit) == 0;
        }
      }
    }
    if (half == 0) {
#pragma unroll
      for (int k = 0; k < kB; ++k)
        q[k] = fv[(uint64_t)((tid >> 4) + 64 * (k + kB)) * span / (kPlanRuns - 1) + (tid & 15)];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    first += __shfl_down_sync(0xffffffffu, first, o);
    asc += __shfl_down_sync(0xffffffffu, asc, o);
  }
  if ((tid & 31) == 0) {
    wsum[tid >> 5] = first;
    wasc[tid >> 5] = asc;
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t c = 0, a = 0;
    for (int w = 0; w < 32; ++w) {
      c += wsum[w];
      a += wasc[w];
    }
    const uint64_t cold_rows = nvec * 4 / kPlanRows * c;  // estimate for the whole column
    const uint64_t lines = ((uint64_t)(pl.dl - pl.t) >> line_shift) + 1;
    // A column that walks the dimension upwards (permute_dimension over runs of
    // equal counts: ids ascending within a run) fetches each line once, in
    // address order, in the one-pass kernel: not a case for partitioning.
    const bool in_order = (uint64_t)a * 10u >= (uint64_t)(kPlanRows / 4 * 3) * 8u;
    const bool on = (uint64_t)c * 1000u >= (uint64_t)kPlanRows * SKX_PG_MIN_COLD_PERMILLE &&
                    cold_rows >= lines * kPlanMinTouch && !in_order;
    pl.ctrl->mode = (on || force) ? 1u : 0u;
    pl.ctrl->items = 0;
    pl.ctrl->sample_first = c;
    pl.ctrl->sample_asc = a;
  }
}

// Before the three passes: reset the fill pass's work-item counter.
__global__ void k_pg_arm(PgCtrl* ctrl) {
  ctrl->mode = 1u;
  ctrl->items = 0;
}

__device__ __forceinline__ uint32_t pg_chunk_vecs(uint64_t nvec, uint32_t c) {
  const uint64_t left = nvec - (uint64_t)c * kPgChunkVec;
  return left < kPgChunkVec ? (uint32_t)left : kPgChunkVec;
}

// One 1-D TMA copy of chunk c's FK vectors into ring buffer b.
__device__ __forceinline__ void pg_issue(uint4* ring, uint64_t* bar, int b, const uint4* fv,
                                         uint64_t nvec, uint32_t c, uint64_t pol) {
  const uint32_t bytes = pg_chunk_vecs(nvec, c) * 16;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + b)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(ring + (size_t)b * kPgChunkVec)),
      "l"(fv + (uint64_t)c * kPgChunkVec), "r"(bytes), "r"(smem_u32(bar + b)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void pg_wait(uint64_t* bar, int b, uint32_t parity) {
  asm volatile(
      "{ .reg .pred p;\n\t"
      "PG_WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra PG_WAIT_%=; }" ::"r"(smem_u32(bar + b)),
      "r"(parity)
      : "memory");
}

// part: per chunk, the cold keys grouped by partition and the translated FK.
__global__ void __launch_bounds__(kPgT, 2)
    k_pg_part(const uint4* __restrict__ fv, uint64_t head, uint64_t nvec, PgPlan pl, DevErr* err) {
  extern __shared__ __align__(128) unsigned char pg_raw[];
  uint4* ring = reinterpret_cast<uint4*>(pg_raw);  // [2][kPgChunkVec]
  uint32_t* cnt = reinterpret_cast<uint32_t*>(pg_raw + kPgRing);
  uint32_t* base = cnt + kPgRows * kPgT;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 64);
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t* dummy = cnt + kPgMaxParts * kPgT + tid;  // sink of the other rows' updates
  const uint64_t pol = policy_evict_first();
  uint4* trv = reinterpret_cast<uint4*>(pl.tr);
  for (uint32_t i = tid; i < kPgRows * kPgT; i += kPgT) cnt[i] = 0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + 1)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t c = blockIdx.x;
  if (tid == 0 && c < pl.nchunks) pg_issue(ring, bar, 0, fv, nvec, c, pol);
  for (uint32_t k = 0; c < pl.nchunks; ++k, c += gridDim.x) {
    const int cur = k & 1;
    if (tid == 0 && c + gridDim.x < pl.nchunks) pg_issue(ring, bar, cur ^ 1, fv, nvec, c + gridDim.x, pol);
    pg_wait(bar, cur, (k >> 1) & 1);
    const uint32_t nv = pg_chunk_vecs(nvec, c);
    const uint64_t v0 = (uint64_t)c * kPgChunkVec;
    const uint4* fk = ring + (size_t)cur * kPgChunkVec;
    uint4 q[kPgU];
    uint32_t rk[kPgU];  // four 8-bit ranks per vector
#pragma unroll
    for (int u = 0; u < kPgU; ++u) {
      const uint32_t vi = tid + u * kPgT;
      q[u] = vi < nv ? fk[vi] : make_uint4(0, 0, 0, 0);
      const uint32_t ids[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
      rk[u] = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idx = ids[j] - 1u;
        uint32_t* a = pg_cold(pl, idx) ? cnt + ((idx - pl.t) >> pl.shift) * kPgT + tid : dummy;
        rk[u] |= (atomicAdd(a, 1u) & 0xffu) << (8 * j);  // the dummy's count is garbage
      }
      const uint32_t mx = max(max(ids[0] - 1u, ids[1] - 1u), max(ids[2] - 1u, ids[3] - 1u));
      if (vi < nv && mx >= pl.dl) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (ids[j] - 1u >= pl.dl) record_violation(err, head + (v0 + vi) * 4 + j, ids[j]);
      }
    }
    // counts -> slots: warp w scans rows w, w+8, ... over the 256 thread
    // columns; row bases are added once the row totals are known.
    __syncthreads();
    uint4 ex[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t r = w + 8 * i;
      uint32_t tot = 0;
      ex[i][0] = ex[i][1] = make_uint4(0, 0, 0, 0);
      if (r < pl.nparts) {
        const uint4* row = reinterpret_cast<const uint4*>(cnt + r * kPgT) + 2 * lane;
        const uint4 x0 = row[0], x1 = row[1];
        const uint32_t ls = x0.x + x0.y + x0.z + x0.w + x1.x + x1.y + x1.z + x1.w;
        uint32_t inc = ls;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        uint32_t x = inc - ls;
        ex[i][0].x = x; x += x0.x; ex[i][0].y = x; x += x0.y; ex[i][0].z = x; x += x0.z;
        ex[i][0].w = x; x += x0.w; ex[i][1].x = x; x += x1.x; ex[i][1].y = x; x += x1.y;
        ex[i][1].z = x; x += x1.z; ex[i][1].w = x;
        tot = __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) base[r] = tot;
    }
    __syncthreads();
    if (w == 0) {
      const uint32_t v = base[lane];
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      base[32 + lane] = inc - v;
      if (lane == 31) base[32] = inc;  // base[32] = total, base[33 + r] = start of row r + 1
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t r = w + 8 * i;
      if (r < pl.nparts) {
        const uint32_t b = r ? base[32 + r] : 0u;
        uint4* row = reinterpret_cast<uint4*>(cnt + r * kPgT) + 2 * lane;
        row[0] = make_uint4(ex[i][0].x + b, ex[i][0].y + b, ex[i][0].z + b, ex[i][0].w + b);
        row[1] = make_uint4(ex[i][1].x + b, ex[i][1].y + b, ex[i][1].z + b, ex[i][1].w + b);
      }
    }
    const uint32_t total = base[32];
    if (tid < 32) pl.ends[(size_t)c * 32 + tid] = (uint16_t)(tid + 1 < pl.nparts ? base[33 + tid] : total);
    __syncthreads();
    // keys in slot order over this chunk's ring buffer; tr in row order
    uint32_t* stage = reinterpret_cast<uint32_t*>(ring + (size_t)cur * kPgChunkVec);
#pragma unroll
    for (int u = 0; u < kPgU; ++u) {
      const uint32_t vi = tid + u * kPgT;
      const uint32_t ids[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idx = ids[j] - 1u;
        const bool cold = pg_cold(pl, idx);
        const uint32_t p = cold ? (idx - pl.t) >> pl.shift : kPgMaxParts;
        const uint32_t slot = cnt[p * kPgT + tid] + ((rk[u] >> (8 * j)) & 0xffu);
        *(cold ? stage + slot : dummy) = idx;
        o[j] = cold ? kPgCold | slot : (idx < pl.t ? idx : 0xffffffffu);
      }
      if (vi < nv) st_stream_v4(trv + v0 + vi, make_uint4(o[0], o[1], o[2], o[3]), pol);
    }
    __syncthreads();
    const uint64_t r0 = (uint64_t)c * kPgChunkRows;
    for (uint32_t i = tid; i < total; i += kPgT) pl.keys[r0 + i] = stage[i];
    for (uint32_t i = tid; i < pl.nparts * kPgT; i += kPgT) cnt[i] = 0;
    __syncthreads();  // ring buffer cur is refilled next iteration
  }
}

// fill: vals[i] = dim[keys[i]], partition-major: the work items (partition,
// 64 chunks) are handed out in order by one counter, so the CTAs stay within
// one or two partitions and each dimension slice is read while L2-resident.
template <typename V>
__global__ void __launch_bounds__(256)
    k_pg_fill(const V* __restrict__ dim, PgPlan pl) {
  __shared__ uint32_t sb[kPgFillChunks];  // first record of the chunk's run of partition p
  __shared__ uint32_t sn[kPgFillChunks];  // its length
  __shared__ uint32_t s_item;
  const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t nblk = (pl.nchunks + kPgFillChunks - 1) / kPgFillChunks;
  const uint32_t items = nblk * pl.nparts;
  V* vals = static_cast<V*>(pl.vals);
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_d = policy_evict_last();
  constexpr int kR = 4;  // runs a warp walks side by side (independent loads in flight per lane)
  static_assert(kPgFillChunks % (8 * kR) == 0, "8 warps x kR runs per pass");
  for (;;) {
    if (tid == 0) s_item = atomicAdd(&pl.ctrl->items, 1u);
    __syncthreads();
    const uint32_t it = s_item;
    if (it >= items) break;
    const uint32_t p = it / nblk, blk = it % nblk;
    if (tid < kPgFillChunks) {
      const uint32_t c = blk * kPgFillChunks + tid;
      uint32_t n = 0, b = 0;
      if (c < pl.nchunks) {
        const uint32_t st = p ? pl.ends[(size_t)c * 32 + p - 1] : 0u;
        n = pl.ends[(size_t)c * 32 + p] - st;
        b = c * kPgChunkRows + st;
      }
      sb[tid] = b;
      sn[tid] = n;
    }
    __syncthreads();
    // The runs of one partition in neighbouring chunks have similar lengths: a warp walks kR
    // of them in step, 32 records of each per iteration (coalesced key loads and record
    // stores, no search for a record's run).
#pragma unroll 1
    for (int j0 = w * kR; j0 < kPgFillChunks; j0 += 8 * kR) {
      uint32_t b[kR], n[kR], nmax = 0;
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        b[r] = sb[j0 + r];
        n[r] = sn[j0 + r];
        nmax = max(nmax, n[r]);
      }
      for (uint32_t i = lane; i - lane < nmax; i += 32) {
        uint32_t key[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r)
          if (i < n[r]) key[r] = ld_stream_u32(pl.keys + b[r] + i, pol_s);
        // the slice must outlive the record streams in L2: evict_last loads (L1-allocating:
        // the hot ids of a scattered skewed column repeat), streaming stores
        V v[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r)
          if (i < n[r]) v[r] = ld_dim<V>(dim + key[r], pol_d, true);
#pragma unroll
        for (int r = 0; r < kR; ++r)
          if (i < n[r]) __stcs(vals + b[r] + i, v[r]);
      }
    }
    __syncthreads();  // sb / sn / s_item are rewritten for the next item
  }
}

// emit: the one-pass gather's loop over the translated column.
template <typename V>
__global__ void __launch_bounds__(kThreads, SKX_GATHER_MINB)
    k_pg_emit(uint64_t nvec, const V* __restrict__ dim, V* __restrict__ o, PgPlan pl) {
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_d = policy_evict_last();
  const uint4* trv = reinterpret_cast<const uint4*>(pl.tr);
  const V* vals = static_cast<const V*>(pl.vals);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads * kUnroll;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads * kUnroll + threadIdx.x; base < nvec;
       base += stride) {
    uint4 f[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      f[u] = vi < nvec ? __ldcs(trv + vi) : make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    V v[kUnroll][4];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      const V* cv = vals + ((vi * 4) >> kPgChunkShift << kPgChunkShift);  // the chunk's records
      const uint32_t w[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t x = w[j];
        if (x < kPgCold)
          v[u][j] = ld_dim<V>(dim + x, pol_d, true);
        else if (x != 0xffffffffu)
          v[u][j] = ld_dim<V>(cv + (x & ~kPgCold), pol_s, true);
        else
          v[u][j] = 0;  // out of domain (recorded by part)
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      if (vi < nvec) {
        if constexpr (sizeof(V) == 8) {
          __stcs(reinterpret_cast<ulonglong2*>(o + vi * 4), make_ulonglong2(v[u][0], v[u][1]));
          __stcs(reinterpret_cast<ulonglong2*>(o + vi * 4) + 1, make_ulonglong2(v[u][2], v[u][3]));
        } else {
          Pack4<V>::store(o + vi * 4, v[u], pol_s);
        }
      }
    }
  }
}

// emit, records staged: the chunk's records come into shared memory with one 1-D TMA copy (each
// byte read once, however the CTA's lanes then address them), overlapped with the chunk's
// translated-column loads and hot dimension reads.  One CTA per chunk at a time.
template <typename V>
__global__ void __launch_bounds__(kThreads)
    k_pg_emit_s(uint64_t nvec, const V* __restrict__ dim, V* __restrict__ o, PgPlan pl) {
  static_assert(kThreads * kUnroll == (int)kPgChunkVec, "one emit iteration is one chunk");
  extern __shared__ __align__(128) unsigned char pg_raw[];
  V* rec = reinterpret_cast<V*>(pg_raw);                                   // [kPgChunkRows]
  uint64_t* bar = reinterpret_cast<uint64_t*>(pg_raw + kPgChunkRows * sizeof(V));
  const uint32_t tid = threadIdx.x;
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_d = policy_evict_last();
  const uint4* trv = reinterpret_cast<const uint4*>(pl.tr);
  const V* vals = static_cast<const V*>(pl.vals);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t k = 0;
  for (uint32_t c = blockIdx.x; c < pl.nchunks; c += gridDim.x, ++k) {
    if (tid == 0) {
      const uint32_t total = pl.ends[(size_t)c * 32 + pl.nparts - 1];
      uint32_t bytes = (uint32_t)((total * sizeof(V) + 15) & ~size_t(15));  // inside the chunk's region
      if (bytes == 0) bytes = 16;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                   "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
          "[%1], %2, [%3], %4;" ::"r"(smem_u32(rec)),
          "l"(vals + (uint64_t)c * kPgChunkRows), "r"(bytes), "r"(smem_u32(bar)), "l"(pol_s)
          : "memory");
    }
    const uint64_t base = (uint64_t)c * kPgChunkVec + tid;
    uint4 f[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      f[u] = vi < nvec ? __ldcs(trv + vi) : make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    V v[kUnroll][4];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t w[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) v[u][j] = w[j] < kPgCold ? ld_dim<V>(dim + w[j], pol_d, true) : (V)0;
    }
    pg_wait(bar, 0, k & 1);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t w[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (w[j] >= kPgCold && w[j] != 0xffffffffu) v[u][j] = rec[w[j] & ~kPgCold];
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      if (vi < nvec) {
        if constexpr (sizeof(V) == 8) {
          __stcs(reinterpret_cast<ulonglong2*>(o + vi * 4), make_ulonglong2(v[u][0], v[u][1]));
          __stcs(reinterpret_cast<ulonglong2*>(o + vi * 4) + 1, make_ulonglong2(v[u][2], v[u][3]));
        } else {
          Pack4<V>::store(o + vi * 4, v[u], pol_s);
        }
      }
    }
    __syncthreads();  // every lane has read its records before the next chunk's copy lands
  }
}

// ---- plan cache (skx_internal.cuh: PgCacheEntry) ------------------------------
// A launch never waits for its own plan: the first launch over a column runs
// the one-pass kernel and, beside it, the plan kernel, whose control word is
// copied back asynchronously; once the copy has landed, later launches over the
// same (fact, rows, dimension, length) take the planned path with no plan
// kernel and no scratch unless the plan says "partitioned".  Every
// kPgCacheUses launches the plan is refreshed in the background (the cached
// decision keeps serving until the new one lands).
static bool pg_same(const PgCacheEntry& e, const void* fact, uint64_t nvec, const void* dim,
                    uint64_t dim_len, int width) {
  return e.state != 0 && e.fact == fact && e.dim == dim && e.nvec == nvec &&
         e.dim_len == dim_len && e.width == width;
}

// The entry's copy has landed?  Then its decision becomes the served one.
static void pg_settle(skx_ctx* ctx, int i) {
  PgCacheEntry& e = ctx->pg_cache[i];
  if (!e.pending) return;
  const cudaError_t q = cudaEventQuery(e.ev);
  if (q == cudaErrorNotReady) return;
  e.pending = false;
  if (q != cudaSuccess) {
    cudaGetLastError();
    if (!e.known) e.state = 0;
    return;
  }
  e.known = true;
  e.mode = ctx->pg_host[i * 4];
  e.first = ctx->pg_host[i * 4 + 2];
  e.asc = ctx->pg_host[i * 4 + 3];
  e.uses = 0;
}

static bool pg_cache_init(skx_ctx* ctx) {
  if (ctx->pg_host && ctx->pg_dev) return true;
  if (!ctx->pg_host && cudaHostAlloc(reinterpret_cast<void**>(&ctx->pg_host), kPgCacheSlots * 16,
                                     cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    ctx->pg_host = nullptr;
    return false;
  }
  if (!ctx->pg_dev && cudaMalloc(reinterpret_cast<void**>(&ctx->pg_dev), kPgCacheSlots * 16) !=
                          cudaSuccess) {
    cudaGetLastError();
    ctx->pg_dev = nullptr;
    return false;
  }
  return true;
}

// Launches the plan kernel for entry i and the copy of its control word.
template <typename V>
static void pg_plan_launch(skx_ctx* ctx, int i, const uint4* fv, uint64_t nvec, const PgPlan& base,
                           cudaStream_t s) {
  PgCacheEntry& e = ctx->pg_cache[i];
  if (!e.ev && cudaEventCreateWithFlags(&e.ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    e.ev = nullptr;
    if (!e.known) e.state = 0;
    return;
  }
  PgPlan pl = base;
  pl.ctrl = reinterpret_cast<PgCtrl*>(ctx->pg_dev + i * 4);
  uint32_t line_shift = 0;
  while ((sizeof(V) << line_shift) < 128) ++line_shift;
  static_assert(sizeof(PgCtrl) == 16, "PgCtrl is the 4-word record of the plan cache");
  k_pg_plan<<<1, 1024, kPlanSmem, s>>>(fv, nvec, pl, line_shift, 0u);
  ctx->launches++;
  if (cudaMemcpyAsync(ctx->pg_host + i * 4, pl.ctrl, 16, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaEventRecord(e.ev, s) != cudaSuccess) {
    cudaGetLastError();
    if (!e.known) e.state = 0;
    return;
  }
  e.pending = true;
}

// Returns 1 when the one-pass kernel must do this launch, 2 when the
// partitioned kernels did it, else an error status.
template <typename V>
int pgather_impl(skx_ctx* ctx, const uint32_t* fact, uint64_t head, uint64_t nvec, const V* dim,
                 uint64_t dim_len, V* out, cudaStream_t s) {
  if constexpr (sizeof(V) < 4) {
    return 1;
  } else {
    const uint64_t t = ((uint64_t)SKX_PG_HOT_MB << 20) / sizeof(V);
    if (dim_len <= 2 * t || dim_len > 0xFFFFFFFFull || nvec < (1u << 20)) return 1;
    const uint64_t nchunks = (nvec + kPgChunkVec - 1) / kPgChunkVec;
    if (nchunks * kPgChunkRows > 0xFFFFFFFFull) return 1;  // 32-bit record positions
    if (reinterpret_cast<uintptr_t>(out + head) % 16 != 0) return 1;
    const bool force = (ctx->gather_policy & kPolPartForce) != 0;
    uint32_t shift = 0;
    while (((uint64_t)1 << shift) < ((uint64_t)SKX_PG_SLICE_MB << 20) / sizeof(V)) ++shift;
    while (((dim_len - t + ((uint64_t)1 << shift) - 1) >> shift) > kPgMaxParts) ++shift;
    PgPlan pl{};
    pl.t = (uint32_t)t;
    pl.dl = (uint32_t)dim_len;
    pl.shift = shift;
    pl.nparts = (uint32_t)((dim_len - t + ((uint64_t)1 << shift) - 1) >> shift);
    pl.nchunks = (uint32_t)nchunks;
    const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
    if (!ctx->pg_attr_set) {  // per device, so per context
      cudaFuncSetAttribute(k_pg_part, cudaFuncAttributeMaxDynamicSharedMemorySize, kPgPartSmem);
      cudaFuncSetAttribute(k_pg_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlanSmem);
      ctx->pg_attr_set = true;
    }
    bool on = force;
    if (!force) {
      // The cache queries events and enqueues a copy: neither belongs in a captured graph.
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return 1;
      }
      if (!pg_cache_init(ctx)) return 1;
      int slot = -1;
      for (int i = 0; i < kPgCacheSlots && slot < 0; ++i)
        if (pg_same(ctx->pg_cache[i], fv, nvec, dim, dim_len, (int)sizeof(V))) slot = i;
      if (slot < 0) {  // a new column: take a slot whose copy is not in flight, plan, run one pass
        for (int k = 0; k < kPgCacheSlots && slot < 0; ++k) {
          const int i = (ctx->pg_next + k) % kPgCacheSlots;
          pg_settle(ctx, i);
          if (!ctx->pg_cache[i].pending) slot = i;
        }
        ctx->last_pg_slot = -1;
        if (slot < 0) return 1;
        ctx->pg_next = (slot + 1) % kPgCacheSlots;
        PgCacheEntry& e = ctx->pg_cache[slot];
        const cudaEvent_t ev = e.ev;
        e = PgCacheEntry{};
        e.ev = ev;
        e.fact = fv;
        e.dim = dim;
        e.nvec = nvec;
        e.dim_len = dim_len;
        e.width = (int)sizeof(V);
        e.state = 1;
        pg_plan_launch<V>(ctx, slot, fv, nvec, pl, s);
        ctx->last_pg_slot = slot;
        ctx->last_pg_path = 0;
        return 1;
      }
      PgCacheEntry& e = ctx->pg_cache[slot];
      pg_settle(ctx, slot);
      ctx->last_pg_slot = slot;
      ctx->last_pg_path = 0;
      if (e.state == 0 || !e.known) return 1;  // its first plan is still on its way
      if (!e.pending && ++e.uses > kPgCacheUses) {  // the column may have been rewritten
        e.uses = 0;
        pg_plan_launch<V>(ctx, slot, fv, nvec, pl, s);
      }
      on = e.mode != 0;
      if (!on) return 1;
    }
    const uint64_t recs = nchunks * kPgChunkRows;
    auto up = [](uint64_t b) { return (size_t)((b + 255) & ~uint64_t(255)); };
    const size_t ends_b = up(nchunks * 32 * 2), keys_b = up(recs * 4), tr_b = up(nvec * 16);
    char* sp = static_cast<char*>(
        scratch(ctx, 1, 256 + ends_b + keys_b + tr_b + recs * sizeof(V), s));
    if (!sp) {  // the path is an optimisation: without room for its records the one-pass kernel runs
      cudaGetLastError();
      return 1;
    }
    pl.ctrl = reinterpret_cast<PgCtrl*>(sp);
    pl.ends = reinterpret_cast<uint16_t*>(sp + 256);
    pl.keys = reinterpret_cast<uint32_t*>(sp + 256 + ends_b);
    pl.tr = reinterpret_cast<uint32_t*>(sp + 256 + ends_b + keys_b);
    pl.vals = sp + 256 + ends_b + keys_b + tr_b;
    k_pg_arm<<<1, 1, 0, s>>>(pl.ctrl);
    k_pg_part<<<grid_for(ctx, nchunks, 1, 2), kPgT, kPgPartSmem, s>>>(fv, head, nvec, pl, ctx->err);
    k_pg_fill<V><<<grid_for(ctx, (uint64_t)pl.nparts * nchunks, kPgFillChunks, SKX_PG_FILL_CTAS), 256, 0, s>>>(
        dim, pl);
#if SKX_PG_EMIT_STAGED
    constexpr int kEmitSmem = (int)(kPgChunkRows * sizeof(V)) + 16;
    cudaFuncSetAttribute(k_pg_emit_s<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, kEmitSmem);
    k_pg_emit_s<V><<<grid_for(ctx, nchunks, 1, 8), kThreads, kEmitSmem, s>>>(nvec, dim, out + head, pl);
#else
    k_pg_emit<V><<<grid_for(ctx, nvec, kThreads * kUnroll, 8), kThreads, 0, s>>>(nvec, dim,
                                                                                out + head, pl);
#endif
    ctx->launches += 4;
    ctx->last_pg_path = 1;
    if (force) ctx->last_pg_slot = -1;
    return 2;
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
    int F = ctx->gather_policy;
    int pg = 1;
    ctx->last_pg_slot = -1;
    ctx->last_pg_path = 0;
    if (F & kPolPart) {
      pg = pgather_impl<V>(ctx, fact, head, nvec, dim, dim_len, out, s);
      if (pg != 1 && pg != 2) return pg;
    }
    F &= ~(kPolPart | kPolPartForce);
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
    if (pg != 2) {  // 2: a cached plan sent the whole launch down the partitioned path
      const cudaError_t e =
          out_vec ? dispatch_vec<V, true>(ctx, F, fact, head, nvec, dim, dim_len, out, t, s)
                  : dispatch_vec<V, false>(ctx, F, fact, head, nvec, dim, dim_len, out, t, s);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "gather launch");
      ctx->launches++;
    }
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

int skx_gather_last_plan(skx_ctx* ctx, uint32_t* info, void* stream) {
  if (!ctx || !info) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  info[0] = ctx->last_pg_path;
  info[1] = info[2] = 0;
  info[3] = ctx->last_pg_path;  // a forced launch has no plan: it took the path it was told to
  const int i = ctx->last_pg_slot;
  if (i < 0) return SKX_OK;
  const cudaError_t e = cudaStreamSynchronize(skx::as_stream(stream));
  if (e != cudaSuccess) return skx::cuda_fail(ctx, e, "gather_last_plan");
  skx::PgCacheEntry& pe = ctx->pg_cache[i];
  if (pe.pending && pe.ev) cudaEventSynchronize(pe.ev);
  skx::pg_settle(ctx, i);
  info[1] = pe.first;
  info[2] = pe.asc;
  info[3] = pe.known ? pe.mode : 0;
  return SKX_OK;
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

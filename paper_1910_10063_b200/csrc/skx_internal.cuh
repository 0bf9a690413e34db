// skx_internal.cuh -- shared device helpers and the context object behind
// include/skx.h.  sm_100a only (built with -gencode arch=compute_100a,code=sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstring>

#include "skx.h"

namespace skx {

// ---------------------------------------------------------------------------
// Device error block.  Domain violations are recorded as
//   viol[k >> 32] = min over violating rows of ((k & 0xffffffff) << 32 | value)
// so the FIRST offending row (and its value) survives an unordered parallel
// scan: the reference reports exactly that row (operators.cpp:32-41).
// ---------------------------------------------------------------------------
constexpr int kViolSlots = 4;  // rows up to 2^34 per operator
struct DevErr {
  unsigned long long viol[kViolSlots];
  unsigned int invalid;  // build_index: counts do not sum to total
  unsigned int pad;
  unsigned long long sum;  // scratch: Σ counts for the build_index check
};

__device__ __forceinline__ void record_violation(DevErr* err, uint64_t k, uint32_t value) {
  const unsigned long long rec = ((k & 0xffffffffull) << 32) | value;
  atomicMin(&err->viol[(k >> 32) & (kViolSlots - 1)], rec);
}

// ---------------------------------------------------------------------------
// Cache-policy loads/stores (PTX ISA: createpolicy, ld/st .L2::cache_hint).
// Streams (FK columns, outputs) are evict_first so the reused dimension
// prefix -- which the skew-aware index makes contiguous -- stays L2 resident.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint4 ld_stream_v4(const void* ptr, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr), "l"(pol));
  return r;
}
// Streaming loads with the .cs cache operator (evict-first in L1 and L2).
__device__ __forceinline__ uint4 ld_cs_v4(const void* ptr) {
  uint4 r;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const void* ptr, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(r)
               : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t ld_stream_u64(const void* ptr, uint64_t pol) {
  uint64_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;"
               : "=l"(r)
               : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_stream_v4(void* ptr, uint4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
               :
               : "l"(ptr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_stream_v2(void* ptr, uint2 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.u32 [%0], {%1,%2}, %3;"
               :
               : "l"(ptr), "r"(v.x), "r"(v.y), "l"(pol)
               : "memory");
}

// Dimension (random) loads: read-only path, optionally evict_last in L2.
template <typename V>
__device__ __forceinline__ V ld_dim(const V* p, uint64_t pol, bool use_pol);

template <>
__device__ __forceinline__ uint32_t ld_dim<uint32_t>(const uint32_t* p, uint64_t pol, bool use_pol) {
  uint32_t r;
  if (use_pol)
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  else
    r = __ldg(p);
  return r;
}
template <>
__device__ __forceinline__ uint64_t ld_dim<uint64_t>(const uint64_t* p, uint64_t pol, bool use_pol) {
  uint64_t r;
  if (use_pol)
    asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
  else
    r = __ldg(reinterpret_cast<const unsigned long long*>(p));
  return r;
}
template <>
__device__ __forceinline__ uint16_t ld_dim<uint16_t>(const uint16_t* p, uint64_t pol, bool use_pol) {
  unsigned short r;
  if (use_pol)
    asm volatile("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
  else
    r = __ldg(reinterpret_cast<const unsigned short*>(p));
  return r;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------
// Host-side context.
// ---------------------------------------------------------------------------
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
};
// Scratch arenas are kept per stream: an operator only ever touches the set of
// the stream it is enqueued on, and a set grows with stream-ordered
// cudaFreeAsync / cudaMallocAsync on that stream -- no device-wide
// synchronisation, and two host streams of one context never share scratch.
constexpr int kScratchSlots = 4;
constexpr int kScratchSets = 6;
struct ScratchSet {
  bool used = false;
  cudaStream_t stream = nullptr;
  Scratch slot[kScratchSlots];
  // the last fused selection on this stream (skx_select_sum_partials)
  void* sel_acc = nullptr;
  void* sel_ctl = nullptr;
  uint32_t sel_ncat = 0;
};

// Plan cache of the partitioned gather (gather.cu): the device-side plan of a
// (fact column, dimension) pair is copied back asynchronously, and once it has
// arrived launches over the same pair follow it -- a stale entry can only cost
// time, never change a result (both paths compute the same bytes); plans are
// refreshed every kPgCacheUses launches (a buffer reused for another column is
// re-planned soon) and skx_set_gather_policy drops them all.
constexpr int kPgCacheSlots = 8;
constexpr uint32_t kPgCacheUses = 16;
struct PgCacheEntry {
  const void* fact = nullptr;
  const void* dim = nullptr;
  uint64_t nvec = 0, dim_len = 0;
  int width = 0;
  int state = 0;         // 0 empty, 1 in use
  bool known = false;    // mode / first / asc hold a landed plan
  bool pending = false;  // a plan's copy is in flight (event ev)
  uint32_t mode = 0, first = 0, asc = 0;
  uint32_t uses = 0;
  cudaEvent_t ev = nullptr;
};

}  // namespace skx

struct skx_ctx {
  int device = 0;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  size_t l2_bytes = 0;
  skx::DevErr* err = nullptr;       // device
  skx::DevErr* err_host = nullptr;  // pinned mirror
  uint64_t last_domain = 0;
  bool pg_attr_set = false;            // shared-memory opt-in of the k_pg_* kernels done
  skx::PgCacheEntry pg_cache[skx::kPgCacheSlots];
  uint32_t* pg_host = nullptr;         // pinned: 4 words (PgCtrl) per cache slot
  uint32_t* pg_dev = nullptr;          // device: the plan kernels' control words, same layout
  int pg_next = 0;                     // next slot to evict
  int last_pg_slot = -1;               // cache slot of the last gather launch (-1: none)
  uint32_t last_pg_path = 0;           // 1: the last gather launch ran the partitioned kernels
  int gather_policy = 129 | 8192;  // L2 hints + .cs streams + partitioned cold rows
  size_t persist_max = 0;  // cudaDevAttrMaxPersistingL2CacheSize (0: no windows)
  size_t window_max = 0;   // cudaDevAttrMaxAccessPolicyWindowSize
  bool setaside_on = false;  // cudaLimitPersistingL2CacheSize currently reserved
  size_t tier_smem_bytes = 0;         // gather shared-memory tier cap (0: all opt-in smem)
  size_t tier_l1_bytes = 160 * 1024;  // gather tier t1 (bytes of the dimension prefix)
  double tier_l2_frac = 0.6;          // gather tier t2 (share of L2)
  int hist_mode = 0;  // histogram cold keys: 0 packed 16-bit + check, 1 staged buckets, 2 direct
  int agg_mode = 0;  // group-by cold tail: 0 packed + exact fallback, 1 staged, 2 direct pairs
  std::atomic<uint64_t> launches{0};
  skx_error_info last{};
  // scratch arenas (grow-only, stream-ordered), one set per stream
  skx::ScratchSet sets[skx::kScratchSets];
  // host-buffer pipeline buffers (grown on hstream[0] by the _host entries)
  skx::Scratch hb[6];
  cudaStream_t hstream[2] = {nullptr, nullptr};
  cudaEvent_t hevent[4] = {};
};

namespace skx {

int set_error(skx_ctx* ctx, int status, const char* fmt, ...);
int cuda_fail(skx_ctx* ctx, cudaError_t e, const char* where);
// Ensures scratch arena `slot` of stream s's set holds >= bytes (growing it in
// stream order on s); returns the device pointer, or null when out of memory.
void* scratch(skx_ctx* ctx, int slot, size_t bytes, cudaStream_t s);
void* host_scratch_dev(skx_ctx* ctx, int slot, size_t bytes, cudaStream_t s);
// The scratch set of stream s (created on first use).
ScratchSet* scratch_set(skx_ctx* ctx, cudaStream_t s);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Makes the context's device current for the calling thread (an entry point
// may be called from a thread whose current device is another one, e.g. the
// C++ drop-in's multi-device overloads).
inline void bind(const skx_ctx* c) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != c->device) cudaSetDevice(c->device);
}

#define SKX_CHECK_LAUNCH(ctx, where)                              \
  do {                                                            \
    cudaError_t e_ = cudaGetLastError();                          \
    if (e_ != cudaSuccess) return ::skx::cuda_fail(ctx, e_, where); \
  } while (0)

// Grid for a persistent grid-stride kernel.
inline unsigned grid_for(const skx_ctx* ctx, uint64_t work_items, unsigned per_block,
                         unsigned blocks_per_sm) {
  const uint64_t need = (work_items + per_block - 1) / per_block;
  const uint64_t cap = static_cast<uint64_t>(ctx->num_sms) * blocks_per_sm;
  uint64_t g = need < cap ? need : cap;
  return static_cast<unsigned>(g == 0 ? 1 : g);
}

// Internal launchers shared between translation units.
// fresh: the caller zeroed `counts` (enables the packed 16-bit cold path).
int launch_histogram(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d, void* counts,
                     int counter_bytes, bool fresh, cudaStream_t s);
int launch_gather(skx_ctx* ctx, int width, const uint32_t* fact, uint64_t n, const void* dim,
                  uint64_t dim_len, void* out, cudaStream_t s);
int launch_build_index(skx_ctx* ctx, const void* counts, int counter_bytes, uint32_t d,
                       uint64_t total, uint32_t* offsets, uint32_t* ranks, cudaStream_t s);
int launch_aggregate(skx_ctx* ctx, const uint32_t* fact, const void* measure, int mw, uint64_t n,
                     uint32_t d, uint32_t hot, uint64_t* counts, uint64_t* sums, cudaStream_t s);
// Exclusive scan of u32 in[0..m) -> out (may alias); total written to *total_dev if non-null.
int launch_exclusive_scan_u32(skx_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t m,
                              uint32_t* total_dev, int scratch_slot, cudaStream_t s);

}  // namespace skx

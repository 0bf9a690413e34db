// aggregate.cu -- Q3 group-by COUNT / SUM(measure) per key (K7 in SURVEY.md
// §2.1) and Q3a heavy-hitter counting.
//
// Reference: aggregate_count / aggregate_sum (proj/src/operators.cpp:100-118),
// the hybrid strategy of parallel_aggregate (proj/src/parallel.cpp:178-207:
// private per-thread bins for ids <= h, shared relaxed atomics for the tail,
// serial fold), the lane-copy variant (operators.cpp:120-165) and
// heavy_hitter_count (operators.cpp:184-203).
//
// B200 design.  On a recoded (skew-reordered)
// FK column the hot keys are the ids 1..H, so each CTA (one per SM) holds
// private shared-memory bins for them -- the GPU form of the hybrid plan's
// private hot region.  Bins use 32-bit shared atomics only: sm_100a has no
// native 64-bit shared add (it compiles to a compare-and-swap spin loop that
// serialises on the hottest keys), while 32-bit adds are native and merge
// same-address lanes.  A bin is {u32 count, u32 sum lo}; the rare bits above
// 32 go straight to the key's global sum.  In the packed mode only the 1024
// hottest keys get such bins; the rest of the shared memory holds 4-byte warm
// bins (count << 22 | sum, carries and wraps corrected from the returned word),
// twice the keys per byte.
//
// Tail keys (id > H), default "packed" mode: ONE fire-and-forget 64-bit
// reduction of (1 << 40 | m) per cold row into an 8 B/key accumulator, so a
// key's count lands in bits 40..63 and its sum in bits 0..39.  That halves
// both the reductions and the accumulator footprint of the {count, sum} pair
// layout (tools/probe/agg_probe.cu: 9.6 -> 5.9 ms at C3).  Exactness is
// proved on the device, not assumed: every CTA also counts its packed rows
// and their measure sum exactly; the decode pass sums the decoded fields and
// both totals must match.  The argument, for a key with true count C and sum
// S whose word is W = (C << 40) + S mod 2^64: the decoded sum is S mod 2^40
// <= S, with equality iff S < 2^40; the totals cannot wrap (rows with
// m >= 2^16 are not packed and flag the launch, so the exact sum stays below
// 2^50), hence equal sum totals prove S < 2^40 for EVERY key.  Only then is
// there no carry from the sum field into the count field, so the decoded
// count is C mod 2^24 <= C, with equality iff C < 2^24, and equal count
// totals prove every count exact.  (Without the sum check a carry could make
// a decoded count LARGER than C; the count check alone would not be sound.)  On any flag or
// mismatch three gated kernels, already queued behind the decode, redo the
// whole call with two exact reductions per cold row on an interleaved
// {count, sum} pair (mode 2); otherwise they exit at once.  No host sync.
// For domains above 2^22 the rarest keys (ids >= 2^18 per 2^30 rows) use
// 4-byte words (count << 21 | sum) under the same check, so the accumulator
// set fits the ~64 MB the L2 offers random accesses.  COUNT-only calls count
// into exact u32 counters (below 2^32 rows) widened at the end.
#include "skx_internal.cuh"

#ifndef SKX_AGG_RED_HINT
#define SKX_AGG_RED_HINT 1  // packed tail: evict_last reductions (C3 3.86 -> 3.78 ms)
#endif

namespace skx {
namespace {

constexpr int kThreads = 1024;
constexpr int kMaxBuckets = 64;
#ifndef SKX_AGG_UNROLL
#define SKX_AGG_UNROLL 1
#endif
constexpr int kAggUnroll = SKX_AGG_UNROLL;

template <int MW>
__device__ __forceinline__ void load_measure4(const void* measure, uint64_t row, bool vec,
                                              uint64_t pol, unsigned long long (&m)[4]) {
  if (MW == 8) {
    const unsigned long long* p = static_cast<const unsigned long long*>(measure) + row;
    if (vec) {
      const uint4 a = ld_cs_v4(p), b = ld_cs_v4(p + 2);
      m[0] = a.x | ((unsigned long long)a.y << 32);
      m[1] = a.z | ((unsigned long long)a.w << 32);
      m[2] = b.x | ((unsigned long long)b.y << 32);
      m[3] = b.z | ((unsigned long long)b.w << 32);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) m[j] = ld_stream_u64(p + j, pol);
    }
  } else if (MW == 4) {
    const uint32_t* p = static_cast<const uint32_t*>(measure) + row;
    if (vec) {
      const uint4 a = ld_cs_v4(p);
      m[0] = a.x, m[1] = a.y, m[2] = a.z, m[3] = a.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) m[j] = ld_stream_u32(p + j, pol);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = 0;
  }
}

template <int MW>
__device__ __forceinline__ unsigned long long load_measure1(const void* measure, uint64_t row) {
  if (MW == 8) return static_cast<const unsigned long long*>(measure)[row];
  if (MW == 4) return static_cast<const uint32_t*>(measure)[row];
  return 0;
}

struct HotBins {
  uint32_t* cnt;
  uint32_t* lo;
  uint32_t* hi;
  uint32_t* warm;  // packed mode: 4-byte warm bins for ids [hot8, hot)
  uint32_t hot8;   // packed mode: ids below get the 8-byte {count, sum lo} bins
};

// Packed mode: past the hottest kHot8 keys, a shared bin is ONE 32-bit word
// (count << 22 | sum), twice the keys per byte of shared memory, so fewer rows
// reach the global tail.  The add returns the old word: a sum field that
// carried into the count field, or a count field that wrapped out of the
// word, is corrected in the key's global pair right away -- exact for any
// input; at C3 a warm key sees a few hundred rows per CTA, so corrections
// are rare.
#ifndef SKX_AGG_WARM
#define SKX_AGG_WARM 1
#endif
#ifndef SKX_AGG_HOT8
#define SKX_AGG_HOT8 1024
#endif
constexpr uint32_t kHot8 = SKX_AGG_HOT8;
constexpr int kWarmSumBits = 22;
constexpr uint32_t kWarmMask = (1u << kWarmSumBits) - 1u;

__device__ __forceinline__ void warm_add(const HotBins& b, uint32_t idx, unsigned long long m,
                                         unsigned long long* gpairs) {
  if (m > kWarmMask) {  // wide measure: straight to the exact global pair
    atomicAdd(&gpairs[2 * (uint64_t)idx], 1ull);
    atomicAdd(&gpairs[2 * (uint64_t)idx + 1], m);
    return;
  }
  const uint32_t inc = (1u << kWarmSumBits) | (uint32_t)m;
  const uint32_t old = atomicAdd(&b.warm[idx - b.hot8], inc);
  const uint32_t carry = ((old & kWarmMask) + (uint32_t)m) >> kWarmSumBits;  // sum -> count field
  const bool wrap = (uint32_t)(old + inc) < old;                               // count field -> out
  if (carry | (uint32_t)wrap) {
    const long long dc = (wrap ? (1ll << (32 - kWarmSumBits)) : 0ll) - (long long)carry;
    if (dc) atomicAdd(&gpairs[2 * (uint64_t)idx], (unsigned long long)dc);
    if (carry) atomicAdd(&gpairs[2 * (uint64_t)idx + 1], 1ull << kWarmSumBits);
  }
}

// Device-side exactness check of the packed tail (see the header).
struct AggCheck {
  unsigned long long tail_rows;  // rows reduced into acc (exact)
  unsigned long long tail_sum;   // their measure sum (exact, < 2^50)
  unsigned long long dec_rows;   // sum of decoded counts
  unsigned long long dec_sum;    // sum of decoded sums
  unsigned int big;              // a cold row had m >= 2^16 (not packed)
  unsigned int pad[7];
};
constexpr unsigned long long kPackOne = 1ull << 40;
constexpr unsigned long long kPackMax = 1ull << 16;  // packed measures are < 2^16
constexpr unsigned long long kPackMask = kPackOne - 1;
// Far tail (ids >= Tail::far, the rarest keys): 4-byte packed accumulators,
// count in bits 21..31, sum in bits 0..20 -- half the footprint again, so the
// accumulators of a 2^24-key domain fit the half of L2 the streams leave
// (C3 s=1.0 5.85 -> 3.8 ms).  The same exact-totals check covers them; the
// boundary (2^18 for 2^30 rows, scaled with the row count) keeps a Zipf key's
// expected count there in the low hundreds for s in [0.5, 1.5].
constexpr int kFarSumBits = 21;
constexpr unsigned int kFarOne = 1u << kFarSumBits;
constexpr unsigned int kFarMask = kFarOne - 1u;
#ifndef SKX_AGG_FAR
#define SKX_AGG_FAR 1
#endif

__device__ __forceinline__ bool agg_ok(const AggCheck* c) {
  return c->big == 0 && c->dec_rows == c->tail_rows && c->dec_sum == c->tail_sum;
}

// Global accumulators: MW ? interleaved {count, sum} pairs[limit][2] (packed
// mode: the hot keys' pairs only) : the caller's counts[limit] (one RED per
// tail row).
struct Tail {
  unsigned long long* pairs;
  unsigned long long* acc;  // packed mode: [far] (count << 40 | sum) for ids < far
  AggCheck* chk;            // packed mode
  unsigned int* acc32;      // packed mode: [d - far] (count << 21 | sum) for ids >= far
  uint32_t far;             // packed mode: first id of the far tail (d = none)
  unsigned int* cnt32;      // COUNT only, < 2^32 rows: u32 counts (half the footprint)
  // Staged tail (STG): rows of cold keys are appended per key-range bucket
  // and folded by k_agg_fold while the bucket's pairs are L2-resident.
  unsigned long long* cursors;  // [nb]
  uint32_t* keys;               // [nb][cap]
  unsigned long long* ms;       // [nb][cap]
  uint64_t cap;
  uint32_t nb;
  uint32_t wshift;              // bucket = (idx - hot) >> wshift
  unsigned long long pol_acc;   // packed mode: L2 policy of the reductions (set on the device)
};

#ifndef SKX_AGG_BIN_BYTES
#define SKX_AGG_BIN_BYTES 8
#endif
constexpr int kBinBytes = SKX_AGG_BIN_BYTES;  // 8: {count, sum lo}; 12: + sum hi

// Hot row: 32-bit shared count and sum-lo adds; the bits above 32 (the
// measure's high word plus the lo word's carry, decided from the returned
// old value) go straight to the key's global sum when they occur (8-byte
// bins) or to a third shared word (12-byte bins).
__device__ __forceinline__ void hot_add(const HotBins& b, uint32_t idx, unsigned long long m,
                                        bool with_sum, unsigned long long* gpairs) {
  atomicAdd(&b.cnt[idx], 1u);
  if (with_sum) {
    const uint32_t ml = (uint32_t)m;
    const uint32_t old = atomicAdd(&b.lo[idx], ml);
    const uint32_t hi_add = (uint32_t)(m >> 32) + ((uint32_t)(old + ml) < old ? 1u : 0u);
    if (hi_add) {
      if (kBinBytes == 8)
        atomicAdd(&gpairs[2 * (uint64_t)idx + 1], (unsigned long long)hi_add << 32);
      else
        atomicAdd(&b.hi[idx], hi_add);
    }
  }
}

__device__ __forceinline__ void tail_add(const Tail& t, uint32_t idx, unsigned long long m) {
  atomicAdd(&t.pairs[2 * (uint64_t)idx], 1ull);
  atomicAdd(&t.pairs[2 * (uint64_t)idx + 1], m);
}

// Per-thread exact totals of the packed rows.
struct PackTally {
  uint32_t rows = 0;
  unsigned long long sum = 0;
  bool big = false;
};

// One row: idx = id - 1 already domain-checked (idx < d).
template <int MW, bool PACK>
__device__ __forceinline__ void agg_row(uint32_t idx, unsigned long long m, uint32_t hot,
                                        uint32_t limit, const HotBins& b, const Tail& t,
                                        PackTally& pt) {
  if (idx < hot) {
    if (PACK && MW && SKX_AGG_WARM && idx >= b.hot8)
      warm_add(b, idx, m, t.pairs);
    else
      hot_add(b, idx, m, MW != 0, t.pairs);
  } else if (idx < limit) {
    if (!MW) {
      if (t.cnt32)
        atomicAdd(&t.cnt32[idx], 1u);
      else
        atomicAdd(&t.pairs[idx], 1ull);
    } else if (PACK) {
      if (m < kPackMax) {
#if SKX_AGG_RED_HINT
        // the accumulators before the streams in L2 (evict_last reductions)
        if (idx < t.far)
          asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(t.acc + idx),
                       "l"(kPackOne | m), "l"(t.pol_acc) : "memory");
        else
          asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(
                           t.acc32 + (idx - t.far)),
                       "r"(kFarOne | (unsigned int)m), "l"(t.pol_acc) : "memory");
#else
        if (idx < t.far)
          atomicAdd(&t.acc[idx], kPackOne | m);
        else
          atomicAdd(&t.acc32[idx - t.far], kFarOne | (unsigned int)m);
#endif
        ++pt.rows;
        pt.sum += m;
      } else {
        pt.big = true;
      }
    } else {
      tail_add(t, idx, m);
    }
  }
}

template <int MW, bool PACK>
__global__ void __launch_bounds__(kThreads, 1)
    k_aggregate(const uint32_t* __restrict__ fact, const void* __restrict__ measure, uint64_t head,
                uint64_t nvec, uint64_t n, uint32_t d, uint32_t limit, uint32_t hot, bool mvec,
                Tail t, DevErr* err, const AggCheck* gate) {
  // Exact fallback of the packed mode: nothing to do when the check passed.
  if (gate && agg_ok(gate)) return;
#if SKX_AGG_RED_HINT
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(t.pol_acc));
#endif
  extern __shared__ uint32_t smem_agg[];
  PackTally pt;
  // bins: cnt [hot8] | lo [hot8] (| hi [hot8]) | warm [hot - hot8] (packed mode)
  const uint32_t hot8 = PACK && MW && SKX_AGG_WARM && kBinBytes == 8 ? min(hot, kHot8) : hot;
  HotBins b{smem_agg, smem_agg + hot8, smem_agg + 2 * (size_t)hot8,
            smem_agg + (MW ? 2 * (size_t)hot8 : (size_t)hot8), hot8};
  for (uint32_t i = threadIdx.x; i < hot8; i += kThreads) {
    b.cnt[i] = 0u;
    if (MW) {
      b.lo[i] = 0u;
      if (kBinBytes == 12) b.hi[i] = 0u;
    }
  }
  for (uint32_t i = hot8 + threadIdx.x; i < hot; i += kThreads) b.warm[i - hot8] = 0u;
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
  constexpr int U = MW ? kAggUnroll : 2 * kAggUnroll;
  // U vectors of 4 rows per thread per iteration (COUNT-only: twice as many,
  // it streams 4 B/row): all loads first
  // (more bytes in flight per SM), then the updates.
  const uint64_t stride = (uint64_t)gridDim.x * kThreads * U;
#ifndef SKX_AGG_PIPE
#define SKX_AGG_PIPE 1
#endif
  // Block-uniform trip count: the warp collectives below need every lane.
  // The next iteration's FK and measure vectors are loaded before this one's
  // updates (software pipelining), so the streams stay in flight while the
  // shared-memory and global reductions issue.
  uint4 f[U];
  unsigned long long m[U][4];
  const uint64_t vstart = (uint64_t)blockIdx.x * kThreads * U;
  auto load = [&](uint64_t vb0, uint4 (&ff)[U], unsigned long long (&mm)[U][4]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = vb0 + threadIdx.x + (uint64_t)u * kThreads;
      if (vi < nvec) {
        ff[u] = ld_cs_v4(fv + vi);
        load_measure4<MW>(measure, head + vi * 4, mvec, pol, mm[u]);
      }
    }
  };
  if (SKX_AGG_PIPE && vstart < nvec) load(vstart, f, m);
  for (uint64_t vb0 = vstart; vb0 < nvec; vb0 += stride) {
    const uint64_t vb = vb0 + threadIdx.x;
    uint4 nf[U];
    unsigned long long nm[U][4];
    if (SKX_AGG_PIPE) {
      if (vb0 + stride < nvec) load(vb0 + stride, nf, nm);
    } else {
      load(vb0, f, m);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t vi = vb + (uint64_t)u * kThreads;
      const bool live = vi < nvec;  // warp-collective below: no early exit
      const uint32_t ids[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idx = ids[j] - 1u;
        const bool ok = live && idx < d;
        if (live && !ok) record_violation(err, head + vi * 4 + j, ids[j]);
        // (Warp pre-aggregation of equal hot keys with __match_any_sync +
        // __reduce_add_sync was measured 3.4x slower at Zipf 1.5: the
        // hardware already merges same-address 32-bit shared adds.)
        if (ok) agg_row<MW, PACK>(idx, m[u][j], hot, limit, b, t, pt);
      }
    }
    if (SKX_AGG_PIPE) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        f[u] = nf[u];
#pragma unroll
        for (int j = 0; j < 4; ++j) m[u][j] = nm[u][j];
      }
    }
  }
  if (blockIdx.x == 0) {
    const uint64_t tail_b = head + nvec * 4;
    const uint64_t extra = head + (n - tail_b);
    for (uint64_t k0 = threadIdx.x; k0 < extra; k0 += kThreads) {
      const uint64_t k = k0 < head ? k0 : tail_b + (k0 - head);
      const uint32_t id = fact[k];
      const uint32_t idx = id - 1u;
      if (idx < d)
        agg_row<MW, PACK>(idx, load_measure1<MW>(measure, k), hot, limit, b, t, pt);
      else
        record_violation(err, k, id);
    }
  }
  if (PACK) {
    unsigned long long r = pt.rows, sm = pt.sum;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r += __shfl_down_sync(0xffffffffu, r, o);
      sm += __shfl_down_sync(0xffffffffu, sm, o);
    }
    const bool big = __any_sync(0xffffffffu, pt.big);
    if ((threadIdx.x & 31) == 0) {
      if (r) atomicAdd(&t.chk->tail_rows, r);
      if (sm) atomicAdd(&t.chk->tail_sum, sm);
      if (big) atomicOr(&t.chk->big, 1u);
    }
  }
  __syncthreads();
  // Fold the CTA's private bins into the result (the reference's serial fold
  // of parallel.cpp:199-204, here one 64-bit atomic per live bin).
  for (uint32_t i = threadIdx.x; i < hot8; i += kThreads) {
    const unsigned long long c = b.cnt[i];
    if (c) {
      if (MW) {
        atomicAdd(&t.pairs[2 * (uint64_t)i], c);
        atomicAdd(&t.pairs[2 * (uint64_t)i + 1],
                  ((unsigned long long)(kBinBytes == 12 ? b.hi[i] : 0u) << 32) | b.lo[i]);
      } else {
        if (t.cnt32)
          atomicAdd(&t.cnt32[i], (unsigned int)c);
        else
          atomicAdd(&t.pairs[i], c);
      }
    }
  }
  for (uint32_t i = hot8 + threadIdx.x; i < hot; i += kThreads) {  // packed warm bins
    const uint32_t w = b.warm[i - hot8];
    if (w) {
      atomicAdd(&t.pairs[2 * (uint64_t)i], (unsigned long long)(w >> kWarmSumBits));
      atomicAdd(&t.pairs[2 * (uint64_t)i + 1], (unsigned long long)(w & kWarmMask));
    }
  }
}

// Staged variant (MW != 0, tail pairs >> L2): block-synchronous rounds of
// kThreads x 4 rows.  Hot rows go to the shared bins; cold rows claim a slot
// in their key-range bucket with a shared atomic, one thread per bucket
// reserves the round's slots with ONE global atomic, and the rows are written
// to the bucket buffers.  k_agg_fold later applies them bucket by bucket.
template <int MW>
__global__ void __launch_bounds__(kThreads, 1)
    k_aggregate_staged(const uint32_t* __restrict__ fact, const void* __restrict__ measure,
                       uint64_t head, uint64_t nvec, uint64_t n, uint32_t d, uint32_t hot, bool mvec,
                       Tail t, DevErr* err) {
  extern __shared__ uint32_t smem_agg[];
  HotBins b{smem_agg, smem_agg + hot, smem_agg + 2 * (size_t)hot, nullptr, hot};
  __shared__ unsigned int s_cnt[kMaxBuckets];
  __shared__ unsigned long long s_base[kMaxBuckets];
  for (uint32_t i = threadIdx.x; i < hot; i += kThreads) {
    b.cnt[i] = 0u;
    b.lo[i] = 0u;
    if (kBinBytes == 12) b.hi[i] = 0u;
  }
  const uint64_t pol = policy_evict_first();
  const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t nvec_round = (nvec + kThreads - 1) / kThreads * kThreads;
  for (uint64_t base = (uint64_t)blockIdx.x * kThreads; base < nvec_round; base += stride) {
    if (threadIdx.x < t.nb) s_cnt[threadIdx.x] = 0u;
    __syncthreads();
    const uint64_t vi = base + threadIdx.x;
    const bool live = vi < nvec;
    uint4 f = make_uint4(0, 0, 0, 0);
    unsigned long long m[4] = {0, 0, 0, 0};
    if (live) {
      f = ld_stream_v4(fv + vi, pol);
      load_measure4<MW>(measure, head + vi * 4, mvec, pol, m);
    }
    const uint32_t ids[4] = {f.x, f.y, f.z, f.w};
    uint32_t slot[4], bk[4];
    bool staged[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      staged[j] = false;
      if (!live) continue;
      const uint32_t idx = ids[j] - 1u;
      if (idx >= d) {
        record_violation(err, head + vi * 4 + j, ids[j]);
      } else if (idx < hot) {
        hot_add(b, idx, m[j], true, t.pairs);
      } else {
        bk[j] = (idx - hot) >> t.wshift;
        slot[j] = atomicAdd(&s_cnt[bk[j]], 1u);
        staged[j] = true;
      }
    }
    __syncthreads();
    if (threadIdx.x < t.nb && s_cnt[threadIdx.x])
      s_base[threadIdx.x] = atomicAdd(&t.cursors[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!staged[j]) continue;
      const uint32_t idx = ids[j] - 1u;
      const unsigned long long pos = s_base[bk[j]] + slot[j];
      if (pos < t.cap) {
        const uint64_t at = (uint64_t)bk[j] * t.cap + pos;
        t.keys[at] = idx;
        t.ms[at] = m[j];
      } else {
        tail_add(t, idx, m[j]);  // bucket full: direct update
      }
    }
  }
  if (blockIdx.x == 0) {
    const uint64_t tail_b = head + nvec * 4;
    const uint64_t extra = head + (n - tail_b);
    for (uint64_t k0 = threadIdx.x; k0 < extra; k0 += kThreads) {
      const uint64_t k = k0 < head ? k0 : tail_b + (k0 - head);
      const uint32_t id = fact[k];
      const uint32_t idx = id - 1u;
      PackTally unused;
      if (idx < d)
        agg_row<MW, false>(idx, load_measure1<MW>(measure, k), hot, d, b, t, unused);
      else
        record_violation(err, k, id);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < hot; i += kThreads) {
    const unsigned long long c = b.cnt[i];
    if (c) {
      atomicAdd(&t.pairs[2 * (uint64_t)i], c);
      atomicAdd(&t.pairs[2 * (uint64_t)i + 1],
                ((unsigned long long)(kBinBytes == 12 ? b.hi[i] : 0u) << 32) | b.lo[i]);
    }
  }
}

// Apply the staged cold rows bucket by bucket: all CTAs sweep bucket b
// together, so the 16 B/key pairs they update (one bucket's key range) stay
// L2-resident instead of read-modify-writing HBM lines.
__global__ void __launch_bounds__(512)
    k_agg_fold(Tail t) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint32_t bk = 0; bk < t.nb; ++bk) {
    const uint64_t m = t.cursors[bk] < t.cap ? t.cursors[bk] : t.cap;
    const uint32_t* keys = t.keys + (uint64_t)bk * t.cap;
    const unsigned long long* ms = t.ms + (uint64_t)bk * t.cap;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
      const uint32_t idx = __ldcs(keys + i);
      const unsigned long long v = __ldcs(ms + i);
      atomicAdd(&t.pairs[2 * (uint64_t)idx], 1ull);
      atomicAdd(&t.pairs[2 * (uint64_t)idx + 1], v);
    }
  }
}

__global__ void k_deinterleave(const unsigned long long* __restrict__ pairs, uint32_t d,
                               unsigned long long* __restrict__ counts,
                               unsigned long long* __restrict__ sums, const AggCheck* gate) {
  if (gate && agg_ok(gate)) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += stride) {
    const ulonglong2 p = reinterpret_cast<const ulonglong2*>(pairs)[i];
    if (counts) counts[i] = p.x;
    if (sums) sums[i] = p.y;
  }
}

// Packed mode: counts/sums from the hot pairs (ids < hot) and the packed
// accumulators (ids >= hot), plus the decoded totals for the exactness check.
__global__ void __launch_bounds__(256)
    k_agg_decode(const unsigned long long* __restrict__ hotpairs,
                 const unsigned long long* __restrict__ acc,
                 const unsigned int* __restrict__ acc32, uint32_t far, uint32_t hot, uint32_t d,
                 unsigned long long* __restrict__ counts, unsigned long long* __restrict__ sums,
                 AggCheck* chk) {
  unsigned long long lr = 0, ls = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += stride) {
    unsigned long long c, sm;
    if (i < hot) {
      const ulonglong2 p = reinterpret_cast<const ulonglong2*>(hotpairs)[i];
      c = p.x;
      sm = p.y;
    } else if (i < far) {
      const unsigned long long x = __ldcs(acc + i);
      c = x >> 40;
      sm = x & kPackMask;
      lr += c;
      ls += sm;
    } else {
      const unsigned int x = __ldcs(acc32 + (i - far));
      c = x >> kFarSumBits;
      sm = x & kFarMask;
      lr += c;
      ls += sm;
    }
    if (counts) __stcs(counts + i, c);
    if (sums) __stcs(sums + i, sm);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lr += __shfl_down_sync(0xffffffffu, lr, o);
    ls += __shfl_down_sync(0xffffffffu, ls, o);
  }
  // one pair of same-address atomics per CTA, not per warp (they serialise)
  __shared__ unsigned long long s_r[8], s_s[8];
  if ((threadIdx.x & 31) == 0) s_r[threadIdx.x >> 5] = lr, s_s[threadIdx.x >> 5] = ls;
  __syncthreads();
  if (threadIdx.x == 0) {
    lr = ls = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) lr += s_r[w], ls += s_s[w];
    if (lr) atomicAdd(&chk->dec_rows, lr);
    if (ls) atomicAdd(&chk->dec_sum, ls);
  }
}

// Exact fallback, step 1: clear the pair accumulators unless the check passed.
__global__ void __launch_bounds__(256)
    k_agg_zero_if_failed(ulonglong2* __restrict__ pairs, uint64_t n2, const AggCheck* gate) {
  if (agg_ok(gate)) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride)
    pairs[i] = make_ulonglong2(0ull, 0ull);
}

__global__ void __launch_bounds__(256)
    k_widen_u32(const unsigned int* __restrict__ c32, uint32_t d,
                unsigned long long* __restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += stride)
    __stcs(counts + i, (unsigned long long)__ldcs(c32 + i));
}

// Keys with private shared-memory bins.  Packed mode (pack, MW != 0): kHot8
// 8-byte bins, then 4-byte warm bins for the rest of the budget.
uint32_t hot_keys(const skx_ctx* ctx, int mw, uint32_t hot_req, uint32_t limit, bool pack = false) {
  const size_t budget = ctx->smem_optin > 2048 ? ctx->smem_optin - 2048 : 0;
  uint32_t hot;
  if (pack && mw && SKX_AGG_WARM && kBinBytes == 8 && budget >= (size_t)kHot8 * 8 + 4)
    hot = kHot8 + (uint32_t)((budget - (size_t)kHot8 * 8) / 4);
  else
    hot = (uint32_t)(budget / (mw ? kBinBytes : 4));
  if (hot_req && hot_req < hot) hot = hot_req;
  if (hot > limit) hot = limit;
  return hot;
}

size_t hot_smem(int mw, bool pack, uint32_t hot) {
  if (pack && mw && SKX_AGG_WARM && kBinBytes == 8) {
    const uint32_t h8 = hot < kHot8 ? hot : kHot8;
    return (size_t)h8 * 8 + (size_t)(hot - h8) * 4;
  }
  return (size_t)hot * (mw ? kBinBytes : 4);
}

template <int MW, bool PACK>
int aggregate_impl(skx_ctx* ctx, const uint32_t* fact, const void* measure, uint64_t n, uint32_t d,
                   uint32_t limit, uint32_t hot_req, Tail t, cudaStream_t s,
                   const AggCheck* gate = nullptr) {
  const uintptr_t fa = reinterpret_cast<uintptr_t>(fact);
  if (fa % 4 != 0) return set_error(ctx, SKX_INVALID_ARGUMENT, "fact pointer not 4-byte aligned");
  uint64_t head = ((16 - fa % 16) % 16) / 4;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 4;
  bool mvec = true;
  if (MW) mvec = (reinterpret_cast<uintptr_t>(static_cast<const char*>(measure) + head * MW) % 16) == 0;
  const unsigned grid = grid_for(ctx, nvec ? nvec : 1, kThreads, 1);
  // Per-CTA counts must fit the u32 bins.
  if (n / grid + 4 * (uint64_t)kThreads >= (uint64_t(1) << 32))
    return set_error(ctx, SKX_INVALID_ARGUMENT, "aggregate: too many rows per call");
  const uint32_t hot = hot_keys(ctx, MW, hot_req, limit, PACK);
  const size_t smem = hot_smem(MW, PACK, hot);
  // Stage the cold tail when its pairs overflow half of L2 (MW != 0 only).
  const uint64_t tail_keys = limit > hot ? limit - hot : 0;
  if (MW && !PACK && !gate && limit == d && ctx->agg_mode == 1 &&
      tail_keys * 16 > ctx->l2_bytes / 2 && n >= (uint64_t(1) << 20)) {
    uint32_t wshift = 20;  // 1M keys x 16 B = 16 MiB of pairs per bucket
    while (((tail_keys + (uint64_t(1) << wshift) - 1) >> wshift) > (uint64_t)kMaxBuckets) ++wshift;
    t.nb = (uint32_t)((tail_keys + (uint64_t(1) << wshift) - 1) >> wshift);
    t.wshift = wshift;
    t.cap = n / (2 * (uint64_t)t.nb) + 4096;
    const uint64_t kb = ((uint64_t)t.nb * t.cap * 4 + 255) & ~uint64_t(255);
    char* sp = static_cast<char*>(scratch(ctx, 0, 256 + kb + (uint64_t)t.nb * t.cap * 8, s));
    if (!sp) return set_error(ctx, SKX_CUDA_ERROR, "aggregate: out of device memory for staging");
    t.cursors = reinterpret_cast<unsigned long long*>(sp);
    t.keys = reinterpret_cast<uint32_t*>(sp + 256);
    t.ms = reinterpret_cast<unsigned long long*>(sp + 256 + kb);
    cudaError_t e = cudaMemsetAsync(t.cursors, 0, 256, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "aggregate memset");
    cudaFuncSetAttribute(k_aggregate_staged<MW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_aggregate_staged<MW><<<grid, kThreads, smem, s>>>(fact, measure, head, nvec, n, d, hot, mvec,
                                                        t, ctx->err);
    k_agg_fold<<<grid_for(ctx, n, 512, 4), 512, 0, s>>>(t);
    ctx->launches += 2;
  } else {
    cudaFuncSetAttribute(k_aggregate<MW, PACK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k_aggregate<MW, PACK><<<grid, kThreads, smem, s>>>(fact, measure, head, nvec, n, d, limit, hot,
                                                       mvec, t, ctx->err, gate);
    ctx->launches++;
  }
  SKX_CHECK_LAUNCH(ctx, "aggregate");
  return SKX_OK;
}

}  // namespace

int launch_aggregate(skx_ctx* ctx, const uint32_t* fact, const void* measure, int mw, uint64_t n,
                     uint32_t d, uint32_t hot_req, uint64_t* counts, uint64_t* sums,
                     cudaStream_t s) {
  if (mw != 0 && mw != 4 && mw != 8)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "aggregate: measure width must be 0, 4 or 8");
  if (mw && !measure && n) return set_error(ctx, SKX_INVALID_ARGUMENT, "aggregate: null measure");
  if (n > (uint64_t(1) << 34))
    return set_error(ctx, SKX_INVALID_ARGUMENT, "aggregate: more than 2^34 rows per call");
  ctx->last_domain = d;
  if (mw == 0 || !sums) {
    // COUNT only: accumulate straight into the caller's counts.
    if (!counts) return SKX_OK;
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)d * 8, s);
    if (sums && e == cudaSuccess) e = cudaMemsetAsync(sums, 0, (size_t)d * 8, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "aggregate memset");
    if (n == 0) return SKX_OK;
    if (n < 0xFFFFFFFFull && d >= (1u << 20)) {
      // u32 counts are exact below 2^32 rows and halve the tail's footprint
      unsigned int* c32 = static_cast<unsigned int*>(scratch(ctx, 1, (size_t)d * 4, s));
      if (!c32) return set_error(ctx, SKX_CUDA_ERROR, "aggregate: out of device memory");
      e = cudaMemsetAsync(c32, 0, (size_t)d * 4, s);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "aggregate memset");
      Tail t{nullptr, nullptr, nullptr, nullptr, 0, c32, nullptr, nullptr, nullptr, 0, 0, 0};
      const int rc = aggregate_impl<0, false>(ctx, fact, nullptr, n, d, d, hot_req, t, s);
      if (rc) return rc;
      k_widen_u32<<<grid_for(ctx, d, 256, 8), 256, 0, s>>>(c32, d,
                                                          reinterpret_cast<unsigned long long*>(counts));
      ctx->launches++;
      SKX_CHECK_LAUNCH(ctx, "aggregate widen");
      return SKX_OK;
    }
    Tail t{reinterpret_cast<unsigned long long*>(counts), nullptr, nullptr, nullptr, 0, nullptr,
           nullptr, nullptr, nullptr, 0, 0, 0};
    return aggregate_impl<0, false>(ctx, fact, nullptr, n, d, d, hot_req, t, s);
  }
  const bool pack = ctx->agg_mode == 0 && n > 0;
  const uint32_t hot = hot_keys(ctx, mw, hot_req, d, pack);
  // Far tail for domains whose 8-byte accumulators would not fit half of L2.
  uint32_t far = d;
#ifndef SKX_AGG_FAR_BITS
#define SKX_AGG_FAR_BITS 18
#endif
  if (SKX_AGG_FAR && d > (1u << 22)) {
    uint64_t first = uint64_t(1) << SKX_AGG_FAR_BITS;  // for <= 2^30 rows
    for (uint64_t r = uint64_t(1) << 30; r < n && first < (uint64_t(1) << 22); r <<= 1) first <<= 1;
    far = hot > first ? hot : (uint32_t)first;
  }
  // Slot-1 layout: [AggCheck 256 B][hot pairs hot x 16 B][acc far x 8 B]
  //                [acc32 (d - far) x 4 B][pairs d x 16 B]
  auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t chk_b = 256, hp_b = up((size_t)hot * 16), acc_b = up((size_t)far * 8);
  const size_t acc32_b = up((size_t)(d - far) * 4);
  const size_t pairs_off = pack ? chk_b + hp_b + acc_b + acc32_b : 0;
  char* base = static_cast<char*>(scratch(ctx, 1, pairs_off + (size_t)d * 16 + 16, s));
  if (!base) return set_error(ctx, SKX_CUDA_ERROR, "aggregate: out of device memory");
  unsigned long long* pairs = reinterpret_cast<unsigned long long*>(base + pairs_off);
  unsigned long long* counts64 = reinterpret_cast<unsigned long long*>(counts);
  unsigned long long* sums64 = reinterpret_cast<unsigned long long*>(sums);
  if (pack) {
    AggCheck* chk = reinterpret_cast<AggCheck*>(base);
    unsigned long long* hotpairs = reinterpret_cast<unsigned long long*>(base + chk_b);
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(base + chk_b + hp_b);
    unsigned int* acc32 = reinterpret_cast<unsigned int*>(base + chk_b + hp_b + acc_b);
    cudaError_t e = cudaMemsetAsync(base, 0, pairs_off, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "aggregate memset");
    Tail tp{hotpairs, acc, chk, acc32, far, nullptr, nullptr, nullptr, nullptr, 0, 0, 0};
    int rc = mw == 8 ? aggregate_impl<8, true>(ctx, fact, measure, n, d, d, hot_req, tp, s)
                     : aggregate_impl<4, true>(ctx, fact, measure, n, d, d, hot_req, tp, s);
    if (rc) return rc;
    k_agg_decode<<<grid_for(ctx, d, 256, 8), 256, 0, s>>>(hotpairs, acc, acc32, far, hot, d,
                                                         counts64, sums64, chk);
    // Exact fallback, queued now and skipped on the device when the check passed.
    k_agg_zero_if_failed<<<grid_for(ctx, d, 256, 8), 256, 0, s>>>(
        reinterpret_cast<ulonglong2*>(pairs), d, chk);
    ctx->launches += 2;
    Tail t{pairs, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr, 0, 0, 0};
    rc = mw == 8 ? aggregate_impl<8, false>(ctx, fact, measure, n, d, d, hot_req, t, s, chk)
                 : aggregate_impl<4, false>(ctx, fact, measure, n, d, d, hot_req, t, s, chk);
    if (rc) return rc;
    k_deinterleave<<<grid_for(ctx, d, 256, 8), 256, 0, s>>>(pairs, d, counts64, sums64, chk);
    ctx->launches++;
    SKX_CHECK_LAUNCH(ctx, "aggregate decode");
    return SKX_OK;
  }
  cudaError_t e = cudaMemsetAsync(pairs, 0, (size_t)d * 16, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "aggregate memset");
  Tail t{pairs, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr, 0, 0, 0};
  int rc = SKX_OK;
  if (n > 0) {
    rc = mw == 8 ? aggregate_impl<8, false>(ctx, fact, measure, n, d, d, hot_req, t, s)
                 : aggregate_impl<4, false>(ctx, fact, measure, n, d, d, hot_req, t, s);
    if (rc) return rc;
  }
  if (d > 0) {
    k_deinterleave<<<grid_for(ctx, d, 256, 8), 256, 0, s>>>(pairs, d, counts64, sums64, nullptr);
    ctx->launches++;
  }
  SKX_CHECK_LAUNCH(ctx, "aggregate deinterleave");
  return SKX_OK;
}

}  // namespace skx

extern "C" {

int skx_aggregate(skx_ctx* ctx, const uint32_t* fact, const void* measure, int measure_width,
                  uint64_t n, uint32_t d, uint32_t hot_threshold, uint64_t* counts, uint64_t* sums,
                  void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  return skx::launch_aggregate(ctx, fact, measure, measure_width, n, d, hot_threshold, counts,
                               sums, skx::as_stream(stream));
}

int skx_heavy_hitter_count(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d, uint32_t k,
                           uint64_t* counts, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  if (k == 0) return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "heavy_hitter_count: k must be at least 1");
  cudaStream_t s = skx::as_stream(stream);
  const uint32_t cutoff = k < d ? k : d;
  ctx->last_domain = d;
  if (cutoff > 0) {
    cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)cutoff * 8, s);
    if (e != cudaSuccess) return skx::cuda_fail(ctx, e, "heavy_hitter memset");
  }
  if (n == 0) return SKX_OK;
  skx::Tail t{reinterpret_cast<unsigned long long*>(counts), nullptr, nullptr, nullptr, 0,
              nullptr, nullptr, nullptr, nullptr, 0, 0, 0};
  return skx::aggregate_impl<0, false>(ctx, fact, nullptr, n, d, cutoff, cutoff, t, s);
}

}  // extern "C"

// histogram.cu -- frequency histogram counts[id-1] += 1 (K1 in SURVEY.md §2.1).
//
// Reference: count_frequencies (proj/src/permindex.cpp:18-30): a single-thread
// scattered increment that throws DomainViolation at the first bad row.
//
// B200 design.  Before the reorder the hot
// keys are scattered ids (a Zipf(1.25) key alone is ~22% of all rows), so:
//  1. every lane adds 1 to a per-CTA shared-memory table (key -> count)
//     that captures the keys the CTA sees first -- for skewed data the hot
//     ones -- claiming slots with CAS.  Each key has two candidate slots,
//     read together (no probe loop for the warp to diverge on); same-key
//     lanes of a warp are merged by the shared-memory atomic unit itself (a
//     __match_any_sync pre-aggregation was measured 2.4x slower at C4);
//  2. a key with neither slot is cold: a global red.add into the counters
//     (direct, default), or into packed 16-bit halves for counter arrays
//     beyond 3x L2 (that mode keeps linear probing, see SKX_HIST_2CHOICE);
//  3. opt-in (skx_set_histogram_mode(1)): for large domains the CTA collects
//     the cold (key, count) pairs of each 4096-row tile in shared memory,
//     partitions them by key range (64 ranges) and appends each range's run
//     to that range's global bucket with one cursor atomic; a second kernel
//     applies each bucket while its counter slice is L2-resident -- so no
//     cold update read-modify-writes an HBM line (on B200 every L2 miss
//     moves a 128-byte line, profiles/r1_experiments.md §7);
//  4. each CTA flushes its table once.
// The FK column is streamed once with 128-bit evict_first loads; the domain
// check is fused (first bad row via atomicMin, reported at skx_sync).
#include "skx_internal.cuh"

namespace skx {
namespace {

#ifndef SKX_HIST_THREADS
#define SKX_HIST_THREADS 512
#endif
#ifndef SKX_HIST_TBITS
#define SKX_HIST_TBITS 13
#endif
#ifndef SKX_HIST_PASS_BYTES
// C16 key-range pass size: packed cold counters per pass (the reductions'
// L2-resident working set).  C2 index (D=2^27, 256 MB of packed counters):
// 1 pass 15.2 ms, 2 passes (128 MB) 11.3, 3 (~85 MB) 10.8, 4 13.9, 8 24.8.
#define SKX_HIST_PASS_BYTES (96ull << 20)
#endif
#ifndef SKX_HIST_SAMPLED
#define SKX_HIST_SAMPLED 1  // direct counters: sampled read-only hot set (k_histogram_seeded)
#endif
#ifndef SKX_HIST_TOPREG
#define SKX_HIST_TOPREG 1  // sampled path: the hottest key counts in a register
#endif
#ifndef SKX_HIST_RED_HINT
#define SKX_HIST_RED_HINT 1  // global counter reductions with an evict_last L2 policy (C4 histogram -4%)
#endif
#ifndef SKX_HIST_CTAS
#define SKX_HIST_CTAS 3
#endif
constexpr int kThreads = SKX_HIST_THREADS;
constexpr int kTableBits = SKX_HIST_TBITS;  // default 8192 slots x 8 B = 64 KB per CTA
constexpr int kTable = 1 << kTableBits;
// Two-choice table (default): each key has two candidate slots, read at once,
// no probe loop -- the warp no longer pays a divergent probe sequence for its
// cold lanes (C4 histogram 2.52 -> 2.15 ms; 16K slots at 1 CTA/SM 2.44,
// 4K slots at 6 CTAs/SM 3.36).  The packed 16-bit cold counters keep the
// linear probes: with two choices their halves wrap and the exact recount
// runs (C2 index 15.3 -> 33 ms).
#ifndef SKX_HIST_2CHOICE_C16
#define SKX_HIST_2CHOICE_C16 0
#endif
#ifndef SKX_HIST_2CHOICE
#define SKX_HIST_2CHOICE 1
#endif
#ifndef SKX_HIST_PROBES
#define SKX_HIST_PROBES 3
#endif
// Slots tried before a key counts as cold.  Every probe is paid by the whole
// warp whenever one lane is cold (divergence), so fewer is faster (C4
// histogram: 4 probes 2.90 ms, 3 2.51, 2 2.59, 1 3.53) -- but the packed
// 16-bit cold counters (C16) need hot keys to stay in the table: with 3
// probes displaced hot keys wrap their halves and the exact fallback recount
// runs (C2 index 15.3 -> 33 ms), so C16 keeps 4.
constexpr int kProbe = SKX_HIST_PROBES;
constexpr int kProbeC16 = 4;
constexpr int kUnroll = 2;        // uint4 per thread per iteration
constexpr int kTileRows = kThreads * kUnroll * 4;  // rows per CTA iteration
constexpr int kNB = 64;           // key-range buckets (staged cold path)
constexpr int kLocalBits = 26;    // entry = (count << 26) | (idx - bucket base)

__device__ __forceinline__ uint32_t slot_hash(uint32_t id) {
  return (id * 0x9E3779B1u) >> (32 - kTableBits);
}
__device__ __forceinline__ uint32_t slot_hash2(uint32_t id) {
  return (id * 0x85EBCA77u + 0x6A09E667u) >> (32 - kTableBits);
}

template <typename CT>
__device__ __forceinline__ void global_add(CT* counts, uint32_t idx, uint32_t c);
template <>
__device__ __forceinline__ void global_add<uint32_t>(uint32_t* counts, uint32_t idx, uint32_t c) {
#if SKX_HIST_RED_HINT
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(counts + idx),
               "r"(c), "l"(pol) : "memory");
#else
  atomicAdd(counts + idx, c);
#endif
}
template <>
__device__ __forceinline__ void global_add<unsigned long long>(unsigned long long* counts,
                                                               uint32_t idx, uint32_t c) {
#if SKX_HIST_RED_HINT
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(counts + idx),
               "l"((unsigned long long)c), "l"(pol) : "memory");
#else
  atomicAdd(counts + idx, (unsigned long long)c);
#endif
}

struct Buckets {
  unsigned int* cursors;  // [kNB]
  uint32_t* buf;          // [kNB][cap]: (count << 26) | (idx - (b << shift))
  uint64_t cap;
  uint32_t shift;         // bucket = idx >> shift
};

// Packed 16-bit cold counters (C16): two keys per 32-bit word, half the
// footprint of u32 counters so more of the cold keys' lines stay in L2.  A
// wrap of a half is caught on the device: the merged halves fall short of the
// exact number of cold rows (each half <= its true count, equality iff it
// did not wrap); gated kernels then redo the call with direct counters.
struct HistCheck {
  unsigned long long cold_rows;  // rows counted into the 16-bit halves (exact)
  unsigned long long merged;     // sum of the merged halves
};

__device__ __forceinline__ bool hist_ok(const HistCheck* c) { return c->cold_rows == c->merged; }

// Shared-memory state of the bucketed (BK) path: the tile's cold pairs and
// its per-range counts / global bases.
struct TileCold {
  unsigned long long* pairs;  // [kTileRows]: (count << 32) | idx
  unsigned int* n;            // number of pairs
  unsigned int* cnt;          // [kNB]
  unsigned int* base;         // [kNB]
};

// Warp-collective: every lane calls it (invalid lanes with valid = false).
template <typename CT, bool BK, bool C16>
__device__ __forceinline__ void count_one(uint32_t id, bool valid, uint32_t* keys, uint32_t* cnts,
                                          CT* counts, const TileCold& tc, unsigned int* c16,
                                          unsigned long long& cold_rows) {
  const uint32_t key = valid ? id : 0u;
  // Every lane updates on its own: same-address 32-bit shared adds from one
  // warp merge in hardware, so warp pre-aggregation with __match_any_sync
  // only adds latency (C4 histogram 6.86 -> 2.88 ms without it).
  const bool leader = key != 0u;
  const uint32_t c = 1u;
  bool cold = false;
#if SKX_HIST_2CHOICE
  if (leader && (!C16 || SKX_HIST_2CHOICE_C16)) {
    // Two-choice table: both candidate slots read at once, no probe loop.
    // A key may end up in both slots after a race; every row still adds to
    // exactly one slot or counter, and the flush adds every slot.
    const uint32_t h1 = slot_hash(key), h2 = slot_hash2(key);
    const uint32_t k1 = keys[h1], k2 = keys[h2];
    int slot = k1 == key ? (int)h1 : (k2 == key ? (int)h2 : -1);
    if (slot < 0 && k1 == 0u) {
      const uint32_t o = atomicCAS(&keys[h1], 0u, key);
      if (o == 0u || o == key) slot = (int)h1;
    }
    if (slot < 0 && k2 == 0u) {
      const uint32_t o = atomicCAS(&keys[h2], 0u, key);
      if (o == 0u || o == key) slot = (int)h2;
    }
    if (slot >= 0) {
      atomicAdd(&cnts[slot], c);
    } else if (!BK) {
      if (C16) {
        const uint32_t idx = key - 1u;
        atomicAdd(&c16[idx >> 1], 1u << ((idx & 1u) * 16));
        ++cold_rows;
      } else {
        global_add<CT>(counts, key - 1, c);
      }
    }
    cold = slot < 0;
  } else
#endif
  if (leader) {
    uint32_t h = slot_hash(key);
    cold = true;
#pragma unroll
    for (int p = 0; p < (C16 ? kProbeC16 : kProbe); ++p) {
      uint32_t k = keys[h];
      if (k == 0u) {
        k = atomicCAS(&keys[h], 0u, key);
        if (k == 0u) k = key;
      }
      if (k == key) {
        atomicAdd(&cnts[h], c);
        cold = false;
        break;
      }
      h = (h + 1) & (kTable - 1);
    }
    if (cold && !BK) {
      if (C16) {
        const uint32_t idx = key - 1u;
        atomicAdd(&c16[idx >> 1], 1u << ((idx & 1u) * 16));
        ++cold_rows;
      } else {
        global_add<CT>(counts, key - 1, c);
      }
    }
  }
  if (BK) {  // warp-aggregated append to the tile's cold list
    const uint32_t m = __ballot_sync(0xffffffffu, cold);
    if (m) {
      const int lane = threadIdx.x & 31;
      const int first = __ffs(m) - 1;
      unsigned int at = 0;
      if (lane == first) at = atomicAdd(tc.n, (unsigned int)__popc(m));
      at = __shfl_sync(0xffffffffu, at, first);
      if (cold)
        tc.pairs[at + __popc(m & lanemask_lt())] = ((unsigned long long)c << 32) | (key - 1u);
    }
  }
}

// BK: partition the tile's cold pairs by key range and append each range's
// run to its global bucket (one cursor atomic per range per tile).  Called
// by the whole CTA between barriers.
template <typename CT>
__device__ __forceinline__ void flush_tile(const TileCold& tc, const Buckets& bk, CT* counts) {
  __syncthreads();
  const unsigned int m = *tc.n;
  for (unsigned int i = threadIdx.x; i < m; i += kThreads)
    atomicAdd(&tc.cnt[(uint32_t)tc.pairs[i] >> bk.shift], 1u);
  __syncthreads();
  if (threadIdx.x < kNB) {
    const unsigned int c = tc.cnt[threadIdx.x];
    tc.base[threadIdx.x] = c ? atomicAdd(&bk.cursors[threadIdx.x], c) : 0u;
    tc.cnt[threadIdx.x] = 0u;
  }
  __syncthreads();
  for (unsigned int i = threadIdx.x; i < m; i += kThreads) {
    const unsigned long long p = tc.pairs[i];
    const uint32_t idx = (uint32_t)p, c = (uint32_t)(p >> 32);
    const uint32_t b = idx >> bk.shift;
    const uint64_t pos = (uint64_t)tc.base[b] + atomicAdd(&tc.cnt[b], 1u);
    if (pos < bk.cap)
      bk.buf[(uint64_t)b * bk.cap + pos] = (c << kLocalBits) | (idx - (b << bk.shift));
    else
      global_add<CT>(counts, idx, c);  // bucket full: direct reduction
  }
  __syncthreads();
  if (threadIdx.x < kNB) tc.cnt[threadIdx.x] = 0u;
  if (threadIdx.x == 0) *tc.n = 0u;
  __syncthreads();  // resets visible before the next tile's appends
}

template <typename CT, bool BK, bool C16>
__global__ void __launch_bounds__(kThreads)
    k_histogram(const uint32_t* __restrict__ fact, uint64_t head, uint64_t nvec, uint64_t n,
                uint32_t d, CT* __restrict__ counts, Buckets bk, DevErr* err,
                unsigned int* __restrict__ c16, HistCheck* chk, const HistCheck* gate,
                uint32_t lo = 0u, uint32_t span = 0xFFFFFFFFu) {
  // Key-range pass (C16 at very large domains): only ids with id - 1 in
  // [lo, lo + span) are counted; violations are reported by the pass with err.
  if (gate && hist_ok(gate)) return;  // C16 fallback: nothing to redo
  unsigned long long cold_rows = 0;
  extern __shared__ __align__(16) uint32_t smem_tab[];
  uint32_t* keys = smem_tab;
  uint32_t* cnts = smem_tab + kTable;
  // BK: [pairs kTileRows x u64][n][cnt kNB][base kNB] after the table
  TileCold tc{reinterpret_cast<unsigned long long*>(smem_tab + 2 * kTable),
              smem_tab + 2 * kTable + 2 * kTileRows, smem_tab + 2 * kTable + 2 * kTileRows + 1,
              smem_tab + 2 * kTable + 2 * kTileRows + 1 + kNB};
  for (int i = threadIdx.x; i < kTable; i += kThreads) {
    keys[i] = 0u;
    cnts[i] = 0u;
  }
  if (BK && threadIdx.x <= kNB) tc.n[threadIdx.x] = 0u;  // n and cnt[]
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
  const uint64_t per_iter = (uint64_t)kThreads * kUnroll;
  const uint64_t stride = (uint64_t)gridDim.x * per_iter;
  // Vector body; every lane of a warp runs the same trip count (warp collectives).
  const uint64_t nvec_round = (nvec + per_iter - 1) / per_iter * per_iter;
  for (uint64_t base = (uint64_t)blockIdx.x * per_iter + threadIdx.x; base < nvec_round;
       base += stride) {
    uint4 f[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      f[u] = vi < nvec ? ld_stream_v4(fv + vi, pol) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      const bool live = vi < nvec;
      const uint32_t ids[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool ok = (ids[j] - 1u) < d;
        if (live && !ok && (!C16 || err)) record_violation(err, head + vi * 4 + j, ids[j]);
        const bool inr = !C16 || (ids[j] - 1u - lo) < span;  // passes: C16 only
        count_one<CT, BK, C16>(ids[j], live && ok && inr, keys, cnts, counts, tc, c16, cold_rows);
      }
    }
    if (BK) flush_tile<CT>(tc, bk, counts);
  }
  // Scalar head [0, head) and tail [head + 4*nvec, n): block 0, warp-uniform trips.
  if (blockIdx.x == 0) {
    const uint64_t tail_b = head + nvec * 4;
    const uint64_t extra = head + (n - tail_b);  // < 8 rows
    for (uint64_t t0 = 0; t0 < extra; t0 += kThreads) {
      const uint64_t t = t0 + threadIdx.x;
      uint64_t k = 0;
      const bool live = t < extra;
      if (live) k = t < head ? t : tail_b + (t - head);
      const uint32_t id = live ? fact[k] : 0u;
      const bool ok = (id - 1u) < d;
      if (live && !ok && (!C16 || err)) record_violation(err, k, id);
      const bool inr = !C16 || (id - 1u - lo) < span;
      count_one<CT, BK, C16>(id, live && ok && inr, keys, cnts, counts, tc, c16, cold_rows);
    }
  }
  if (BK) flush_tile<CT>(tc, bk, counts);  // block-uniform: also blocks != 0
  if (C16) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cold_rows += __shfl_down_sync(0xffffffffu, cold_rows, o);
    if ((threadIdx.x & 31) == 0 && cold_rows) atomicAdd(&chk->cold_rows, cold_rows);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kTable; i += kThreads) {
    const uint32_t k = keys[i];
    if (k != 0u && cnts[i] != 0u) global_add<CT>(counts, k - 1, cnts[i]);
  }
}

// ---- sampled hot set (direct counters) -------------------------------------
// The dynamic table above keeps the first keys a CTA sees: under Zipf(1.25)
// many are one-off tail keys, so ~21% of C4's rows still reached global
// reductions (ncu: 231 M RED sectors per 2^30 rows) although the 8192 most
// frequent keys carry ~92% of the rows.  Instead, a strided sample of the
// column is counted first (k_hist_sample, an L2-resident open-addressing
// table), the keys hit at least twice become the hot set (k_hist_pick), and
// every CTA loads that set into a read-only two-choice table: no slot claims
// in the main loop, and the cold reductions fall to the true tail.
constexpr int kSampleBits = 21;                     // 2M (key, hits) slots = 16 MB
constexpr uint32_t kHotCap = (kTable * 3) / 4;      // hot keys per table (load 0.75)
constexpr int kBands = 8;                           // sample-hit bands, hottest first
__constant__ uint32_t c_band_lo[kBands] = {4096, 512, 64, 16, 8, 4, 3, 2};
constexpr int kSampleSlots = 4096;                  // per-CTA pre-aggregation (32 KB)

__device__ __forceinline__ void sample_add(uint2* tab, uint32_t key, uint32_t c) {
  constexpr uint32_t mask = (1u << kSampleBits) - 1u;
  uint32_t h = (key * 0x9E3779B1u) >> (32 - kSampleBits);
  for (int p = 0; p < 64; ++p, h = (h + 1) & mask) {
    uint32_t k = tab[h].x;
    if (k == 0u) {
      k = atomicCAS(&tab[h].x, 0u, key);
      if (k == 0u) k = key;
    }
    if (k == key) {
      atomicAdd(&tab[h].y, c);
      return;
    }
  }
}

// Each CTA counts its share of the strided sample in shared memory first (a
// Zipf top key alone is ~22% of the samples: one global atomic per CTA
// instead of ~230K on one address), then merges its entries.
__global__ void __launch_bounds__(512)
    k_hist_sample(const uint32_t* __restrict__ fact, uint64_t step, uint32_t nsamp, uint32_t d,
                  uint2* __restrict__ tab) {
  __shared__ uint32_t s_key[kSampleSlots], s_cnt[kSampleSlots];
  for (int i = threadIdx.x; i < kSampleSlots; i += blockDim.x) s_key[i] = 0u, s_cnt[i] = 0u;
  __syncthreads();
  const uint32_t per = (nsamp + gridDim.x - 1) / gridDim.x;
  const uint32_t b = blockIdx.x * per, e = min(nsamp, b + per);
  for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    const uint32_t key = __ldg(fact + (uint64_t)i * step);
    if (key - 1u >= d) continue;  // violations are reported by the counting pass
    uint32_t h = (key * 0x9E3779B1u) >> (32 - 12);
    bool done = false;
    for (int p = 0; p < 8 && !done; ++p, h = (h + 1) & (kSampleSlots - 1)) {
      uint32_t k = s_key[h];
      if (k == 0u) {
        k = atomicCAS(&s_key[h], 0u, key);
        if (k == 0u) k = key;
      }
      if (k == key) {
        atomicAdd(&s_cnt[h], 1u);
        done = true;
      }
    }
    if (!done) sample_add(tab, key, 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSampleSlots; i += blockDim.x)
    if (s_cnt[i]) sample_add(tab, s_key[i], s_cnt[i]);
}

// One pass over the sample table: keys hit >= 2 times go to the list of their
// hit band (warp-aggregated cursor atomics); the seeded kernel takes bands in
// order, so a full hot set never drops a key hotter than one it holds.
__global__ void __launch_bounds__(256)
    k_hist_pick(const uint2* __restrict__ tab, uint32_t* __restrict__ band_keys,
                unsigned int* __restrict__ band_n) {
  const int lane = threadIdx.x & 31;
  const uint32_t total = 1u << kSampleBits;  // a multiple of 32: warp-uniform trips
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint2 e = tab[i];
#if SKX_HIST_TOPREG
    if (e.y >= c_band_lo[0])  // the most-sampled key, (hits << 32 | key) in band_n[8..9]
      atomicMax(reinterpret_cast<unsigned long long*>(band_n + kBands),
                ((unsigned long long)e.y << 32) | e.x);
#endif
    int band = kBands;
    if (e.x != 0u)
#pragma unroll
      for (int q = kBands - 1; q >= 0; --q)
        if (e.y >= c_band_lo[q]) band = q;
#pragma unroll
    for (int q = 0; q < kBands; ++q) {
      const uint32_t m = __ballot_sync(0xffffffffu, band == q);
      if (!m) continue;
      unsigned int at = 0;
      const int first = __ffs(m) - 1;
      if (lane == first) at = atomicAdd(&band_n[q], (unsigned int)__popc(m));
      at = __shfl_sync(0xffffffffu, at, first);
      if (band == q) {
        const unsigned int pos = at + __popc(m & lanemask_lt());
        if (pos < kHotCap) band_keys[q * kHotCap + pos] = e.x;
      }
    }
  }
}

template <typename CT>
__global__ void __launch_bounds__(kThreads)
    k_histogram_seeded(const uint32_t* __restrict__ fact, uint64_t head, uint64_t nvec, uint64_t n,
                       uint32_t d, CT* __restrict__ counts, DevErr* err,
                       const uint32_t* __restrict__ band_keys, const unsigned int* band_n) {
  extern __shared__ __align__(16) uint32_t smem_tab[];
  uint32_t* keys = smem_tab;
  uint32_t* cnts = smem_tab + kTable;
  __shared__ uint32_t s_bstart[kBands + 1];
  for (int i = threadIdx.x; i < kTable; i += kThreads) {
    keys[i] = 0u;
    cnts[i] = 0u;
  }
  if (threadIdx.x == 0) {  // bands concatenated hottest first, capped at kHotCap keys
    uint32_t acc = 0;
    for (int q = 0; q < kBands; ++q) {
      s_bstart[q] = acc;
      acc = min(kHotCap, acc + min(band_n[q], kHotCap));
    }
    s_bstart[kBands] = acc;
  }
  __syncthreads();
  const uint32_t nh = s_bstart[kBands];
#if SKX_HIST_TOPREG
  // the hottest key (~22% of C4's rows) counts in a register, not a shared slot
  const uint32_t top = (uint32_t)*reinterpret_cast<const unsigned long long*>(band_n + kBands);
  uint32_t topc = 0;
#endif
  for (uint32_t i = threadIdx.x; i < nh; i += kThreads) {  // fill once; read-only afterwards
    int q = 0;
    while (i >= s_bstart[q + 1]) ++q;
    const uint32_t key = __ldg(band_keys + q * kHotCap + (i - s_bstart[q]));
    if (atomicCAS(&keys[slot_hash(key)], 0u, key) != 0u) atomicCAS(&keys[slot_hash2(key)], 0u, key);
  }
  __syncthreads();
  auto count = [&](uint32_t key) {  // key already domain-checked
#if SKX_HIST_TOPREG
    if (key == top) {
      ++topc;
      return;
    }
#endif
    const uint32_t h1 = slot_hash(key), h2 = slot_hash2(key);
    const uint32_t k1 = keys[h1], k2 = keys[h2];
    if (k1 == key)
      atomicAdd(&cnts[h1], 1u);
    else if (k2 == key)
      atomicAdd(&cnts[h2], 1u);
    else
      global_add<CT>(counts, key - 1u, 1u);
  };
  const uint64_t pol = policy_evict_first();
  const uint4* fv = reinterpret_cast<const uint4*>(fact + head);
  const uint64_t per_iter = (uint64_t)kThreads * kUnroll;
  const uint64_t stride = (uint64_t)gridDim.x * per_iter;
  for (uint64_t base = (uint64_t)blockIdx.x * per_iter + threadIdx.x; base < nvec; base += stride) {
    uint4 f[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      f[u] = vi < nvec ? ld_stream_v4(fv + vi, pol) : make_uint4(1, 1, 1, 1);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t vi = base + (uint64_t)u * kThreads;
      const uint32_t ids[4] = {f[u].x, f[u].y, f[u].z, f[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if ((ids[j] - 1u) < d) {
          if (vi < nvec) count(ids[j]);
        } else if (vi < nvec) {
          record_violation(err, head + vi * 4 + j, ids[j]);
        }
      }
    }
  }
  if (blockIdx.x == 0) {  // scalar head [0, head) and tail [head + 4*nvec, n)
    const uint64_t tail_b = head + nvec * 4;
    const uint64_t extra = head + (n - tail_b);
    for (uint64_t t = threadIdx.x; t < extra; t += kThreads) {
      const uint64_t k = t < head ? t : tail_b + (t - head);
      const uint32_t id = fact[k];
      if ((id - 1u) < d)
        count(id);
      else
        record_violation(err, k, id);
    }
  }
#if SKX_HIST_TOPREG
  for (int o = 16; o > 0; o >>= 1) topc += __shfl_down_sync(0xffffffffu, topc, o);
  if ((threadIdx.x & 31) == 0 && topc) global_add<CT>(counts, top - 1u, topc);
#endif
  __syncthreads();
  for (int i = threadIdx.x; i < kTable; i += kThreads) {
    const uint32_t k = keys[i];
    if (k != 0u && cnts[i] != 0u) global_add<CT>(counts, k - 1, cnts[i]);
  }
}

// Second kernel: apply the buckets in key-range order; all CTAs sweep bucket
// b together, so its counter slice (2^shift counters) stays L2-resident and
// the reductions never read-modify-write HBM lines.
template <typename CT>
__global__ void __launch_bounds__(256)
    k_hist_fold(Buckets bk, CT* __restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint32_t b = 0; b < kNB; ++b) {
    const uint64_t m = bk.cursors[b] < bk.cap ? bk.cursors[b] : bk.cap;
    const uint32_t* src = bk.buf + (uint64_t)b * bk.cap;
    const uint32_t g0 = b << bk.shift;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
      const uint32_t v = __ldcs(src + i);
      global_add<CT>(counts, g0 + (v & ((1u << kLocalBits) - 1u)), v >> kLocalBits);
    }
  }
}

// C16: counts[i] += half i of the packed words; sums the halves for the check.
// Four counters per thread (two packed words), read and written whole: a
// store only where a half is non-zero leaves partial sectors that HBM must
// read back (0.49 ms at the C2 index before).
template <typename CT>
__device__ __forceinline__ void add4(CT* c, uint32_t a, uint32_t b, uint32_t e, uint32_t f);
template <>
__device__ __forceinline__ void add4<uint32_t>(uint32_t* c, uint32_t a, uint32_t b, uint32_t e,
                                               uint32_t f) {
  uint4 v = *reinterpret_cast<uint4*>(c);
  v.x += a, v.y += b, v.z += e, v.w += f;
  *reinterpret_cast<uint4*>(c) = v;
}
template <>
__device__ __forceinline__ void add4<unsigned long long>(unsigned long long* c, uint32_t a,
                                                         uint32_t b, uint32_t e, uint32_t f) {
  ulonglong2 v0 = reinterpret_cast<ulonglong2*>(c)[0], v1 = reinterpret_cast<ulonglong2*>(c)[1];
  v0.x += a, v0.y += b, v1.x += e, v1.y += f;
  reinterpret_cast<ulonglong2*>(c)[0] = v0;
  reinterpret_cast<ulonglong2*>(c)[1] = v1;
}

template <typename CT>
__global__ void __launch_bounds__(256)
    k_hist_merge16(const unsigned int* __restrict__ c16, uint32_t d, CT* __restrict__ counts,
                   HistCheck* chk) {
  unsigned long long tot = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(counts) % (4 * sizeof(CT))) == 0;
  const uint64_t nq = vec ? d / 4 : 0;  // whole groups of four counters
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const uint2 x = __ldcs(reinterpret_cast<const uint2*>(c16) + q);
    add4<CT>(counts + 4 * q, x.x & 0xFFFFu, x.x >> 16, x.y & 0xFFFFu, x.y >> 16);
    tot += (x.x & 0xFFFFu) + (x.x >> 16) + (x.y & 0xFFFFu) + (x.y >> 16);
  }
  for (uint64_t i = 4 * nq + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += stride) {
    const uint32_t h = (c16[i >> 1] >> ((i & 1u) * 16)) & 0xFFFFu;  // ragged tail / unaligned
    if (h) counts[i] += (CT)h;
    tot += h;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_down_sync(0xffffffffu, tot, o);
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(&chk->merged, tot);
}

template <typename CT>
__global__ void __launch_bounds__(256)
    k_hist_zero_if_failed(CT* __restrict__ counts, uint32_t d, const HistCheck* gate) {
  if (hist_ok(gate)) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += stride)
    counts[i] = 0;
}

template <typename CT>
int histogram_impl(skx_ctx* ctx, const uint32_t* fact, uint64_t head, uint64_t nvec, uint64_t n,
                   uint32_t d, CT* counts, bool fresh, cudaStream_t s) {
  const unsigned grid = grid_for(ctx, nvec ? nvec : 1, kThreads * kUnroll, SKX_HIST_CTAS);
  const size_t smem = size_t(2) * kTable * sizeof(uint32_t);
  // Stage the cold updates by key range when the counters overflow half of L2
  // -- opt-in (skx_set_histogram_mode(1)): the staging removes the HBM
  // read-modify-writes (C2 index: 40 -> 7 GB of DRAM traffic in the counting
  // kernel) but its per-tile partition work makes the kernel instruction-bound
  // and the L2-resident fold is reduction-rate bound, so the sum is slower
  // than direct reductions as measured (C4 6.86 -> 10.0 ms, C2 index
  // 17.6 -> 20.9 ms; profiles/r1_experiments.md).
  const bool bucketed = ctx->hist_mode == 1 && (uint64_t)d * sizeof(CT) > ctx->l2_bytes / 2 &&
                        n >= (uint64_t(1) << 20);
  Buckets bk{nullptr, nullptr, 0, 0};
  if (bucketed) {
    uint32_t shift = 0;
    while (((uint64_t)d + (uint64_t(1) << shift) - 1) >> shift > (uint64_t)kNB) ++shift;
    bk.shift = shift;
    // the fair share of all rows (overflow -> direct reductions); a multiple
    // of 4 so full 8-entry flushes can use 16-byte stores
    bk.cap = (n / kNB + 65536 + 3) & ~uint64_t(3);
    if (bk.cap > 0xFFFFFFFCull) bk.cap = 0xFFFFFFFCull;
    char* sp = static_cast<char*>(scratch(ctx, 0, (uint64_t)kNB * bk.cap * 4 + 512, s));
    if (!sp) return set_error(ctx, SKX_CUDA_ERROR, "histogram: out of device memory for buckets");
    bk.cursors = reinterpret_cast<unsigned int*>(sp);
    bk.buf = reinterpret_cast<uint32_t*>(sp + 512);
    cudaError_t e = cudaMemsetAsync(bk.cursors, 0, kNB * 4, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "histogram memset");
    const size_t bsmem = smem + (size_t)kTileRows * 8 + (1 + 2 * kNB) * 4;
    cudaFuncSetAttribute(k_histogram<CT, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)bsmem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_histogram<CT, true, false>, kThreads,
                                                  bsmem);
    const unsigned bgrid = grid_for(ctx, nvec ? nvec : 1, kThreads * kUnroll, per_sm < 1 ? 1 : per_sm);
    k_histogram<CT, true, false><<<bgrid, kThreads, bsmem, s>>>(fact, head, nvec, n, d, counts, bk,
                                                                ctx->err, nullptr, nullptr,
                                                                nullptr);
    k_hist_fold<CT><<<grid_for(ctx, n, 256, 8), 256, 0, s>>>(bk, counts);
    ctx->launches += 2;
  } else if (fresh && ctx->hist_mode == 0 && (uint64_t)d * sizeof(CT) > 3 * ctx->l2_bytes &&
             n >= (uint64_t(1) << 20)) {
    // C16 cold counters, for counter arrays beyond 3x L2 (C2 index, 512 MiB of
    // u32: 17.5 -> 14.6 ms; at 256 MiB the extra merge pass costs more than it
    // saves: C4 2.89 -> 3.38 ms).  counts were zeroed by the caller, so the
    // gated fallback may zero them again and recount directly.
    const size_t w16 = (((size_t)d + 1) / 2) * 4;
    char* sp = static_cast<char*>(scratch(ctx, 0, 256 + w16, s));
    if (!sp) return set_error(ctx, SKX_CUDA_ERROR, "histogram: out of device memory");
    HistCheck* chk = reinterpret_cast<HistCheck*>(sp);
    unsigned int* c16 = reinterpret_cast<unsigned int*>(sp + 256);
    cudaError_t e = cudaMemsetAsync(sp, 0, 256 + w16, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "histogram memset");
    cudaFuncSetAttribute(k_histogram<CT, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    // Key-range passes: each pass counts the ids of one slice of the domain,
    // so its packed cold counters (SKX_HIST_PASS_BYTES) stay L2-resident for
    // the reductions and the CTA tables hold only that slice's keys; the FK
    // column is re-streamed per pass.
    const uint64_t pass_keys = std::max<uint64_t>(uint64_t(SKX_HIST_PASS_BYTES) / 2, 1);
    const uint32_t passes = (uint32_t)(((uint64_t)d + pass_keys - 1) / pass_keys);
    const uint32_t span = (uint32_t)(((uint64_t)d + passes - 1) / passes);
    for (uint32_t p = 0; p < passes; ++p) {
      k_histogram<CT, false, true><<<grid, kThreads, smem, s>>>(
          fact, head, nvec, n, d, counts, bk, p == 0 ? ctx->err : nullptr, c16, chk, nullptr,
          p * span, span);
      ctx->launches++;
    }
    k_hist_merge16<CT><<<grid_for(ctx, (d + 1) / 2, 256, 8), 256, 0, s>>>(c16, d, counts, chk);
    k_hist_zero_if_failed<CT><<<grid_for(ctx, d, 256, 8), 256, 0, s>>>(counts, d, chk);
    cudaFuncSetAttribute(k_histogram<CT, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k_histogram<CT, false, false><<<grid, kThreads, smem, s>>>(fact, head, nvec, n, d, counts, bk,
                                                               ctx->err, nullptr, nullptr, chk);
    ctx->launches += 3;
  } else if (SKX_HIST_SAMPLED && n >= (uint64_t(1) << 22) && d > (uint32_t)kTable) {
    // sampled hot set: ~2^20 rows (strided over the whole column) counted
    // into an L2-resident table, banded by hits (>= 2) hottest first
    const uint32_t nsamp = (uint32_t)std::min<uint64_t>(n / 16, uint64_t(1) << 20);
    const uint64_t step = n / nsamp;
    const size_t tab_b = (size_t(1) << kSampleBits) * 8;
    const size_t band_b = (size_t)kBands * kHotCap * 4;
    char* sp = static_cast<char*>(scratch(ctx, 0, tab_b + 256 + band_b, s));
    if (!sp) return set_error(ctx, SKX_CUDA_ERROR, "histogram: out of device memory");
    uint2* tab = reinterpret_cast<uint2*>(sp);
    unsigned int* band_n = reinterpret_cast<unsigned int*>(sp + tab_b);
    uint32_t* band_keys = reinterpret_cast<uint32_t*>(sp + tab_b + 256);
    cudaError_t e = cudaMemsetAsync(sp, 0, tab_b + 256, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "histogram memset");
    k_hist_sample<<<ctx->num_sms, 512, 0, s>>>(fact, step, nsamp, d, tab);
    k_hist_pick<<<grid_for(ctx, size_t(1) << kSampleBits, 256, 8), 256, 0, s>>>(tab, band_keys,
                                                                                band_n);
    cudaFuncSetAttribute(k_histogram_seeded<CT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k_histogram_seeded<CT><<<grid, kThreads, smem, s>>>(fact, head, nvec, n, d, counts, ctx->err,
                                                        band_keys, band_n);
    ctx->launches += 3;
  } else {
    cudaFuncSetAttribute(k_histogram<CT, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    k_histogram<CT, false, false><<<grid, kThreads, smem, s>>>(fact, head, nvec, n, d, counts, bk,
                                                               ctx->err, nullptr, nullptr,
                                                               nullptr);
    ctx->launches++;
  }
  SKX_CHECK_LAUNCH(ctx, "histogram");
  return SKX_OK;
}

}  // namespace

int launch_histogram(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d, void* counts,
                     int counter_bytes, bool fresh, cudaStream_t s) {
  if (n == 0) return SKX_OK;
  if (n > (uint64_t(1) << 34))
    return set_error(ctx, SKX_INVALID_ARGUMENT, "histogram: more than 2^34 rows per call");
  if (counter_bytes == 4 && n > 0xFFFFFFFFull)
    return set_error(ctx, SKX_INVALID_ARGUMENT, "histogram_u32: more than 2^32-1 rows");
  const uintptr_t fa = reinterpret_cast<uintptr_t>(fact);
  if (fa % 4 != 0) return set_error(ctx, SKX_INVALID_ARGUMENT, "fact pointer not 4-byte aligned");
  uint64_t head = ((16 - fa % 16) % 16) / 4;
  if (head > n) head = n;
  const uint64_t nvec = (n - head) / 4;
  ctx->last_domain = d;
  if (counter_bytes == 4)
    return histogram_impl<uint32_t>(ctx, fact, head, nvec, n, d, static_cast<uint32_t*>(counts),
                                    fresh, s);
  return histogram_impl<unsigned long long>(ctx, fact, head, nvec, n, d,
                                            static_cast<unsigned long long*>(counts), fresh, s);
}

}  // namespace skx

extern "C" {

int skx_count_frequencies(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d,
                          uint64_t* counts, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  cudaStream_t s = skx::as_stream(stream);
  if (d > 0) {
    cudaError_t e = cudaMemsetAsync(counts, 0, uint64_t(d) * 8, s);
    if (e != cudaSuccess) return skx::cuda_fail(ctx, e, "count_frequencies memset");
  }
  return skx::launch_histogram(ctx, fact, n, d, counts, 8, true, s);
}

int skx_histogram_u32(skx_ctx* ctx, const uint32_t* fact, uint64_t n, uint32_t d,
                      uint32_t* counts, int accumulate, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  cudaStream_t s = skx::as_stream(stream);
  if (!accumulate && d > 0) {
    cudaError_t e = cudaMemsetAsync(counts, 0, uint64_t(d) * 4, s);
    if (e != cudaSuccess) return skx::cuda_fail(ctx, e, "histogram memset");
  }
  return skx::launch_histogram(ctx, fact, n, d, counts, 4, !accumulate, s);
}

}  // extern "C"

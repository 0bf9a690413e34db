// select.cu -- Q2 selection (K8 in SURVEY.md §2.1): bitmap probe plus
// order-preserving compaction, optionally fused with the config-5 four-column
// gather and per-category SUM(price); plus the bitmap helpers.
//
// Reference: KernelTable::select_offsets (proj/src/kernels/scalar.cpp:31-42,
// avx2.cpp:59-98), select (operators.cpp:87-98), parallel_select
// (parallel.cpp:102-129: per-thread results concatenated in chunk order),
// permute_bitmap (operators.cpp:21-30), build_bitmap (operators.hpp:38-45).
//
// B200 design: two passes with a device scan
// between them, no inter-CTA ordering inside a kernel.  Pass 1 streams the
// FK column once (one 256-bit load of 8 consecutive rows per lane; the bitmap
// prefix that holds the hot ids of a reordered column sits in shared memory);
// each warp owns a contiguous run of 256-row slices and appends their
// selected rows -- (dimension index, row), in row order (one warp scan of the
// lanes' popcounts per slice) -- densely to its own region, then writes the
// region's count.  The scan turns the region counts into output offsets.
// Pass 2 streams the regions: entry e of a region goes to its offset + e --
// ascending row order, exactly the reference's chunk-ordered concatenation --
// with 4 entries per lane loaded before their records and stores, so the FK
// column is read once.  A region whose selected rows overflow its capacity
// (a quarter of its rows: dense selections) is re-derived in pass 2 from the
// FK column and the bitmap.  (Single-pass decoupled look-back forms were
// measured slower on B200: profiles/r1_experiments.md,
// profiles/r2_experiments.md §11.)
//
// The C5 variant first interleaves the four dimension columns into 32-byte
// records (one 256-bit load and one sector per selected row instead of four
// separate lines -- an L2 miss costs a whole 128-byte line on B200) and sums
// price per category inside pass 2 in exact 96-bit fixed point: per-CTA
// shared bins updated with native 32-bit atomics (carries via the returned
// old value), folded once per CTA, converted to fp64 at the end.  The scale
// 2^S comes from the selected keys' price exponent range (|price * 2^S| < 2^62);
// non-finite prices, an exponent span above 2^30 or more than 4096
// categories switch, on the device, to an fp64 pass over the compacted
// columns (warp-private fp64 bins, __match_any_sync pre-sums).
#include "scan.cuh"

namespace skx {
namespace {

constexpr int kThreads = 256;                  // pass 2 / fallback sum CTAs
constexpr int kWarps = kThreads / 32;
constexpr int kWarpRows = 256;                 // rows per warp slice
constexpr int kItems = kWarpRows / 128;        // 4 items of 128 rows (4 per lane)
constexpr uint32_t kCap = 64;                  // compacted entries kept per slice
#ifndef SKX_SEL_P2_MINB
#define SKX_SEL_P2_MINB 2   // pass 2 CTAs per SM the registers must allow
#endif
#ifndef SKX_SEL_P1_PREF
#define SKX_SEL_P1_PREF 0   // pass 1: next slice's FKs in flight while probing
#endif
#ifndef SKX_SEL_OUT_CS
#define SKX_SEL_OUT_CS 1    // pass 2 output columns as streaming stores
#endif
#ifndef SKX_SEL_PER
#define SKX_SEL_PER 8
#endif
constexpr int kParts = 8;                      // pass 2: work items per pass-1 region
constexpr int kPer = SKX_SEL_PER;              // pass 2: entries per lane in flight
constexpr int kThreads1 = 1024;                // pass 1 CTA (shares one bitmap prefix)
constexpr uint32_t kSmemCategories = 2048;     // fp64 fallback: 8 warps x 2048 x 8 B
constexpr uint32_t kFixedCategories = 4096;    // fixed point: 3 x 4096 x 4 B per CTA
constexpr int kRangeLimit = 30;                // max exponent span for fixed point
#ifndef SKX_SEL_SMEM_KB
#define SKX_SEL_SMEM_KB 160
#endif

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
  const uint4* rec;          // [selected keys][2]: {cat, price, supp lo, supp hi}, {flag, 0, 0, 0}
  const uint2* dir;          // rank directory of the bitmap: key -> dense record index
  struct SumCtl* ctl;
  unsigned int* acc96;       // [n_categories][4]: lo, mid, hi, pad
  unsigned long long cap;    // output rows the caller's buffers hold
};

// Price exponent range for the fixed-point sums (frexp exponent + 1024).
struct SumCtl {
  unsigned int emax_b;    // max over finite nonzero |price|; 0 = none
  unsigned int emin_neg;  // max of 2048 - e_b (i.e. 2048 - min e_b); 0 = none
  unsigned int nonfinite;
  unsigned int pad;
};

__device__ __forceinline__ bool fixed_ok(const SumCtl* c, uint32_t ncat, int& S) {
  S = 0;
  if (c->nonfinite || ncat == 0 || ncat > kFixedCategories) return false;
  if (c->emax_b == 0) return true;  // every price is zero
  const int emax = (int)c->emax_b - 1024;
  const int emin = (int)(2048u - c->emin_neg) - 1024;
  if (emax - emin > kRangeLimit) return false;
  S = 62 - emax;  // |price| < 2^emax  =>  |price * 2^S| < 2^62
  return true;
}

// Rank directory of the selection bitmap: dir[w] = {word w, selected bits
// before word w}, so the dense record index of a selected key i -- its
// position among the selected keys -- is dir[i/32].y + popc(dir[i/32].x below
// bit i%32).
__device__ __forceinline__ uint32_t compact_index(uint2 pr, uint32_t idx) {
  return pr.y + __popc(pr.x & ((1u << (idx & 31)) - 1u));
}

__global__ void k_word_popc(const uint32_t* __restrict__ w, uint64_t nw, uint32_t* __restrict__ pc) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw;
       i += (uint64_t)gridDim.x * blockDim.x)
    pc[i] = __popc(__ldg(w + i));
}
__global__ void k_dir_fill(const uint32_t* __restrict__ w, const uint32_t* __restrict__ pre,
                           uint64_t nw, uint2* __restrict__ dir) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw;
       i += (uint64_t)gridDim.x * blockDim.x)
    dir[i] = make_uint2(__ldg(w + i), __ldg(pre + i));
}

__device__ __forceinline__ void price_exponent(float p, unsigned int& emax, unsigned int& eneg,
                                               unsigned int& nf) {
  if (!isfinite(p)) {
    nf = 1;
  } else if (p != 0.f) {
    int e;
    frexpf(p, &e);
    const unsigned int eb = (unsigned int)(e + 1024);
    emax = max(emax, eb);
    eneg = max(eneg, 2048u - eb);
  }
}

// C5 prologue: interleave the four dimension columns into 32-byte records for
// the SELECTED keys only, dense in key (= rank) order -- record c belongs to
// the c-th selected key, so the hot selected keys' records share lines -- and
// record the selected prices' exponent range.  Four keys per thread: the
// columns stream in with vector loads (every sector is touched anyway at ~10%
// selectivity) and only the records are scattered.
__global__ void __launch_bounds__(256)
    k_pack_records(const int32_t* __restrict__ cat, const float* __restrict__ price,
                   const unsigned long long* __restrict__ supp, const uint16_t* __restrict__ flag,
                   const uint2* __restrict__ dir, uint32_t d, bool vec, uint4* __restrict__ rec,
                   SumCtl* ctl) {
  unsigned int emax = 0, eneg = 0, nf = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t nq = d / 4;  // full quads
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
    const uint64_t i0 = q * 4;
    const uint2 pr = __ldg(dir + (i0 >> 5));
    const uint32_t bits4 = (pr.x >> (i0 & 31)) & 0xfu;
    if (!bits4) continue;
    int32_t cs[4];
    float ps[4];
    unsigned long long ss[4];
    uint32_t fs[4];
    if (vec) {  // 16-byte aligned columns (8-byte aligned flags)
      const int4 c4 = __ldcs(reinterpret_cast<const int4*>(cat) + q);
      const float4 p4 = __ldcs(reinterpret_cast<const float4*>(price) + q);
      const ulonglong2 sa = __ldcs(reinterpret_cast<const ulonglong2*>(supp) + 2 * q);
      const ulonglong2 sb = __ldcs(reinterpret_cast<const ulonglong2*>(supp) + 2 * q + 1);
      const uint2 f4 = __ldcs(reinterpret_cast<const uint2*>(flag) + q);
      cs[0] = c4.x, cs[1] = c4.y, cs[2] = c4.z, cs[3] = c4.w;
      ps[0] = p4.x, ps[1] = p4.y, ps[2] = p4.z, ps[3] = p4.w;
      ss[0] = sa.x, ss[1] = sa.y, ss[2] = sb.x, ss[3] = sb.y;
      fs[0] = f4.x & 0xffffu, fs[1] = f4.x >> 16, fs[2] = f4.y & 0xffffu, fs[3] = f4.y >> 16;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        cs[j] = cat[i0 + j], ps[j] = price[i0 + j], ss[j] = supp[i0 + j], fs[j] = flag[i0 + j];
      }
    }
    uint32_t c = compact_index(pr, (uint32_t)i0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!((bits4 >> j) & 1u)) continue;
      rec[2 * (uint64_t)c] = make_uint4((uint32_t)cs[j], __float_as_uint(ps[j]), (uint32_t)ss[j],
                                        (uint32_t)(ss[j] >> 32));
      rec[2 * (uint64_t)c + 1] = make_uint4(fs[j], 0u, 0u, 0u);
      price_exponent(ps[j], emax, eneg, nf);
      ++c;
    }
  }
  // the last d % 4 keys, one per thread of the first CTA
  if (blockIdx.x == 0 && threadIdx.x < d % 4) {
    const uint64_t i = nq * 4 + threadIdx.x;
    const uint2 pr = __ldg(dir + (i >> 5));
    if ((pr.x >> (i & 31)) & 1u) {
      const uint64_t c = compact_index(pr, (uint32_t)i);
      const float p = price[i];
      const unsigned long long sp = supp[i];
      rec[2 * c] = make_uint4((uint32_t)cat[i], __float_as_uint(p), (uint32_t)sp,
                              (uint32_t)(sp >> 32));
      rec[2 * c + 1] = make_uint4((uint32_t)flag[i], 0u, 0u, 0u);
      price_exponent(p, emax, eneg, nf);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    eneg = max(eneg, __shfl_xor_sync(0xffffffffu, eneg, o));
    nf |= __shfl_xor_sync(0xffffffffu, nf, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (emax) atomicMax(&ctl->emax_b, emax);
    if (eneg) atomicMax(&ctl->emin_neg, eneg);
    if (nf) atomicOr(&ctl->nonfinite, 1u);
  }
}

// 96-bit two's-complement add of v into {lo, mid, hi}[c] (shared or global):
// the carry out of each word is decided from the value the atomic returned.
__device__ __forceinline__ void add96(unsigned int* lo, unsigned int* mid, unsigned int* hi,
                                      long long v) {
  const unsigned int vl = (unsigned int)v;
  const unsigned int old = atomicAdd(lo, vl);
  const long long up = (v >> 32) + ((unsigned int)(old + vl) < old ? 1 : 0);
  if (up) {
    const unsigned int um = (unsigned int)up, uh = (unsigned int)((unsigned long long)up >> 32);
    const unsigned int old2 = atomicAdd(mid, um);
    const unsigned int h = uh + ((unsigned int)(old2 + um) < old2 ? 1u : 0u);
    if (h) atomicAdd(hi, h);
  }
}

// Probe helpers.  ids are u32: idx = id - 1 < bits32 <=> in domain (id 0
// wraps to 2^32 - 1).  One predicated shared or global load per probe.
__device__ __forceinline__ uint32_t probe_word(uint32_t wi, uint32_t sw, uint32_t s_base,
                                               const uint32_t* words32) {
  uint32_t wv;
  asm volatile(
      "{\n.reg .pred ps;\nsetp.lt.u32 ps, %1, %2;\n"
      "@ps ld.shared.u32 %0, [%3];\n@!ps ld.global.nc.u32 %0, [%4];\n}"
      : "=r"(wv)
      : "r"(wi), "r"(sw), "r"(s_base + 4 * wi), "l"(words32 + wi));
  return wv;
}

// Load the 16 FKs of lane `lane` in slice row0 (rows 128i + 4*lane + j):
// 128-bit loads when the slice is full and the column 16-byte aligned.
template <bool VEC>
__device__ __forceinline__ void load_slice(const uint32_t* __restrict__ fact, uint64_t n,
                                           uint64_t row0, bool full, int lane,
                                           uint32_t (&fk)[kItems][4]) {
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t r = row0 + (uint64_t)i * 128 + 4 * lane;
    if (VEC && full) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(fact + r));
      fk[i][0] = v.x, fk[i][1] = v.y, fk[i][2] = v.z, fk[i][3] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) fk[i][j] = r + j < n ? __ldcs(fact + r + j) : 1u;
    }
  }
}

// Selection bits of one slice: sel[i] bit j = row 128i + 4*lane + j selected.
// Records the first out-of-domain row of the slice (when err != nullptr).
template <bool FULL>
__device__ __forceinline__ void probe_slice(const uint32_t (&fk)[kItems][4], uint64_t row0,
                                            uint64_t n, uint32_t bits32, uint32_t sw,
                                            uint32_t s_base, const uint32_t* words32, int lane,
                                            DevErr* err, uint32_t (&sel)[kItems]) {
  bool anybad = false;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    sel[i] = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t idx = fk[i][j] - 1u;
      const bool live = FULL || row0 + (uint64_t)i * 128 + 4 * lane + j < n;
      const bool ok = live && idx < bits32;
      const uint32_t wv = probe_word(ok ? idx >> 5 : 0u, sw, s_base, words32);
      sel[i] |= (ok ? (wv >> (idx & 31)) & 1u : 0u) << j;
      anybad |= live && !ok;
    }
  }
  if (err != nullptr && __any_sync(0xffffffffu, anybad)) {
#pragma unroll
    for (int i = 0; i < kItems; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t k = row0 + (uint64_t)i * 128 + 4 * lane + j;
        if ((FULL || k < n) && fk[i][j] - 1u >= bits32) record_violation(err, k, fk[i][j]);
      }
  }
}

// Compact one 128-row item: rows before this lane's j-th row are the
// selected rows of lanes < lane (any j) and this lane's rows j' < j.
__device__ __forceinline__ uint32_t item_base(const uint32_t (&b)[4], uint32_t lt) {
  return __popc(b[0] & lt) + __popc(b[1] & lt) + __popc(b[2] & lt) + __popc(b[3] & lt);
}
__device__ __forceinline__ uint32_t item_count(const uint32_t (&b)[4]) {
  return __popc(b[0]) + __popc(b[1]) + __popc(b[2]) + __popc(b[3]);
}

// 8 consecutive FKs of one lane (16-byte aligned): one 256-bit load when
// 32-byte aligned, else two 128-bit loads.
__device__ __forceinline__ void load_rows8(const uint32_t* p, bool v8, uint32_t (&fk)[8]) {
  if (v8) {
    asm volatile("ld.global.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(fk[0]), "=r"(fk[1]), "=r"(fk[2]), "=r"(fk[3]), "=r"(fk[4]), "=r"(fk[5]),
                   "=r"(fk[6]), "=r"(fk[7])
                 : "l"(p));
  } else {
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(p));
    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(p) + 1);
    fk[0] = a.x, fk[1] = a.y, fk[2] = a.z, fk[3] = a.w;
    fk[4] = b.x, fk[5] = b.y, fk[6] = b.z, fk[7] = b.w;
  }
}

// Pass 1, any slice (unaligned column, empty domain): per-item ballots.
// Appends the slice's selected rows at region[wpos..] (while they fit the
// region's capacity) and returns the slice's count (warp-uniform).
template <bool VEC>
__device__ __forceinline__ uint32_t count_slice_generic(const uint32_t* __restrict__ fact,
                                                        uint64_t n, uint64_t sl,
                                                        const uint32_t* __restrict__ words32,
                                                        uint32_t bits32, uint32_t sw,
                                                        uint32_t s_base, uint2* __restrict__ region,
                                                        uint64_t wpos, uint64_t capw, DevErr* err) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const uint64_t row0 = sl * kWarpRows;
  const bool full = row0 + kWarpRows <= n;  // warp-uniform
  uint32_t fk[kItems][4];
  load_slice<VEC>(fact, n, row0, full, lane, fk);
  uint32_t sel[kItems];
  if (full)
    probe_slice<true>(fk, row0, n, bits32, sw, s_base, words32, lane, err, sel);
  else
    probe_slice<false>(fk, row0, n, bits32, sw, s_base, words32, lane, err, sel);
  const uint32_t row_l = (uint32_t)row0 + 4u * lane;  // n < 2^32
  uint32_t run = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    uint32_t b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = __ballot_sync(0xffffffffu, (sel[i] >> j) & 1u);
    if (sel[i]) {
      uint64_t pos = wpos + run + item_base(b, lt);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if ((sel[i] >> j) & 1u) {
          if (pos < capw) region[pos] = make_uint2(fk[i][j] - 1u, row_l + i * 128 + j);
          ++pos;
        }
      }
    }
    run += item_count(b);
  }
  return run;
}

// Pass 1: probe every row once.  Global warp g owns the contiguous slices
// [g * spw, (g + 1) * spw) and appends their selected rows -- (dimension
// index, row), in row order -- densely to its region entries[g * spw * kCap ..]
// (capacity spw * kCap, a quarter of its rows), then writes its count.  Row
// order across regions is warp order, so an exclusive scan of the counts
// gives every region's output offset, and pass 2 streams each region.
template <bool VEC, bool FAST>
__global__ void __launch_bounds__(kThreads1, 1)
    k_select_count(const uint32_t* __restrict__ fact, uint64_t n,
                   const uint32_t* __restrict__ words32, uint64_t bits,
                   uint2* __restrict__ entries, uint32_t* __restrict__ warp_counts, uint64_t spw,
                   uint32_t sw, DevErr* err) {
  extern __shared__ __align__(16) uint32_t s_words[];  // bitmap prefix [sw]
  const int lane = threadIdx.x & 31;
  const uint64_t nslices = (n + kWarpRows - 1) / kWarpRows;
  const uint32_t bits32 = bits < 0xFFFFFFFFull ? (uint32_t)bits : 0xFFFFFFFFu;
  const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(s_words);
  for (uint32_t i = threadIdx.x; i < sw; i += kThreads1) s_words[i] = __ldg(words32 + i);
  __syncthreads();
  const uint32_t maxw = bits32 ? (bits32 - 1u) >> 5 : 0u;
  const bool v8 = (reinterpret_cast<uintptr_t>(fact) & 31u) == 0;
  const uint64_t gw = (uint64_t)blockIdx.x * (kThreads1 / 32) + (threadIdx.x >> 5);
  const uint64_t s_begin = gw * spw < nslices ? gw * spw : nslices;
  const uint64_t s_end = s_begin + spw < nslices ? s_begin + spw : nslices;
  uint2* region = entries + gw * spw * kCap;
  const uint64_t capw = spw * kCap;
  uint64_t wpos = 0;  // warp-uniform: selected rows of the slices done so far
  if constexpr (!FAST) {
    for (uint64_t sl = s_begin; sl < s_end; ++sl)
      wpos += count_slice_generic<VEC>(fact, n, sl, words32, bits32, sw, s_base, region, wpos,
                                       capw, err);
    if (lane == 0) warp_counts[gw] = (uint32_t)wpos;  // < 2^32: n < 2^32
    return;
  }
  // Fast path: lane l owns the 8 consecutive rows row0 + 8l + j, so the
  // slice's row order is (lane, j) and one warp scan of the per-lane counts
  // places every selected row -- ~half the instructions of the per-item
  // ballots of the generic path (pass 1 is issue-bound).  Out-of-domain ids
  // read a clamped word; their rows are reported (the call fails), so their
  // selection bit does not matter.  The next slice's FKs are loaded before
  // this one is probed (SKX_SEL_P1_PREF).
  auto load8 = [&](uint64_t sl, uint32_t (&fk)[8]) -> uint32_t {  // returns the live-row mask
    const uint64_t row0 = sl * kWarpRows;
    if (sl >= nslices) {
#pragma unroll
      for (int j = 0; j < 8; ++j) fk[j] = 1u;
      return 0u;
    }
    if (row0 + kWarpRows <= n) {
      load_rows8(fact + row0 + 8 * lane, v8, fk);
      return 0xffu;
    }
    uint32_t live = 0u;  // the column's last slice
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t r = row0 + 8 * lane + j;
      fk[j] = r < n ? __ldcs(fact + r) : 1u;
      live |= (r < n ? 1u : 0u) << j;
    }
    return live;
  };
  uint32_t fk[8];
  uint32_t live = s_begin < s_end ? load8(s_begin, fk) : 0u;
  for (uint64_t sl = s_begin; sl < s_end; ++sl) {
    const uint64_t row0 = sl * kWarpRows;
#if SKX_SEL_P1_PREF
    uint32_t fkn[8];
    const uint32_t liven = load8(sl + 1 < s_end ? sl + 1 : nslices, fkn);
#endif
    uint32_t sel = 0;
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t idx = fk[j] - 1u;
      bad |= idx >= bits32;  // padding rows read id 1
      const uint32_t wv = probe_word(min(idx >> 5, maxw), sw, s_base, words32);
      sel |= ((wv >> (idx & 31)) & 1u) << j;
    }
    sel &= live;
    if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (((live >> j) & 1u) && fk[j] - 1u >= bits32)
          record_violation(err, row0 + 8 * lane + j, fk[j]);
    }
    const uint32_t c = __popc(sel);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t row_l = (uint32_t)row0 + 8u * lane;  // n < 2^32
    if (sel) {
      uint64_t pos = wpos + incl - c;
      uint2* o = region + pos;
      if (wpos + incl <= capw) {  // all of this lane's rows fit: predicated stores only
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if ((sel >> j) & 1u) *o++ = make_uint2(fk[j] - 1u, row_l + j);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if ((sel >> j) & 1u) {
            if (pos < capw) *o = make_uint2(fk[j] - 1u, row_l + j);
            ++o, ++pos;
          }
      }
    }
    wpos += __shfl_sync(0xffffffffu, incl, 31);
#if SKX_SEL_P1_PREF
#pragma unroll
    for (int j = 0; j < 8; ++j) fk[j] = fkn[j];
    live = liven;
#else
    live = load8(sl + 1 < s_end ? sl + 1 : nslices, fk);
#endif
  }
  if (lane == 0) warp_counts[gw] = (uint32_t)wpos;  // < 2^32: n < 2^32
}

struct Rec8 {
  uint32_t a0, a1, a2, a3, b0;
};

__device__ __forceinline__ Rec8 load_rec(const uint4* rec, uint32_t idx) {
  Rec8 r;
  uint32_t pad[3];  // record bytes 20..31 (unused)
  asm("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r.a0), "=r"(r.a1), "=r"(r.a2), "=r"(r.a3), "=r"(r.b0), "=r"(pad[0]), "=r"(pad[1]),
        "=r"(pad[2])
      : "l"(rec + 2 * (uint64_t)idx));
  (void)pad;
  return r;
}

// One selected row: offset, and (FUSED) the four output columns and the
// fixed-point category sum from its record.
template <bool FUSED>
__device__ __forceinline__ void emit_row(uint64_t p, uint32_t row, const Rec8& r,
                                         uint32_t base_off, uint32_t* __restrict__ out_off,
                                         const Cols& cols, bool fixed, int S, unsigned int* s_acc) {
  const bool fits = p < cols.cap;  // rows past the caller's capacity are counted, not written
#if SKX_SEL_OUT_CS
  // output columns: streaming (.cs) stores, so they do not displace the records in L2
  if (fits) __stcs(out_off + p, base_off + row);
#else
  if (fits) out_off[p] = base_off + row;
#endif
  if (FUSED) {
    const int32_t ct = (int32_t)r.a0;
    const float pr = __uint_as_float(r.a1);
    if (fits) {
#if SKX_SEL_OUT_CS
      __stcs(cols.out_cat + p, ct);
      __stcs(cols.out_price + p, pr);
      __stcs(cols.out_supp + p, (unsigned long long)r.a2 | ((unsigned long long)r.a3 << 32));
      __stcs(reinterpret_cast<unsigned short*>(cols.out_flag) + p, (unsigned short)r.b0);
#else
      cols.out_cat[p] = ct;
      cols.out_price[p] = pr;
      cols.out_supp[p] = (unsigned long long)r.a2 | ((unsigned long long)r.a3 << 32);
      cols.out_flag[p] = (uint16_t)r.b0;
#endif
    }
    const uint32_t ncat = cols.n_categories;
    if (fixed && (uint32_t)ct < ncat) {
      const long long v = __double2ll_rn(ldexp((double)pr, S));
      add96(&s_acc[ct], &s_acc[ncat + ct], &s_acc[2 * ncat + ct], v);
    }
  }
}

// Pass 2: streams the regions of pass 1 (each split into kParts work items for
// balance): a region's entries are the selected rows of a contiguous run of
// slices, already dense and in row order, so entry e goes to region_off + e.  kPer entries per lane are loaded
// (coalesced) before their records (C5) and before any store, so each warp
// keeps 32 x kPer independent record loads in flight.  A region whose rows
// overflowed its capacity (dense selections) is re-derived from the FK column
// and the bitmap, slice by slice.
template <bool FUSED, bool VEC>
__global__ void __launch_bounds__(kThreads, SKX_SEL_P2_MINB)
    k_select_emit(const uint32_t* __restrict__ fact, uint64_t n,
                  const uint32_t* __restrict__ words32, uint64_t bits,
                  const uint2* __restrict__ entries, const uint32_t* __restrict__ warp_counts,
                  const uint32_t* __restrict__ warp_off, uint64_t nregions, uint64_t spw,
                  uint32_t base_off, const uint32_t* __restrict__ total,
                  uint32_t* __restrict__ out_off, Cols cols,
                  unsigned long long* __restrict__ count_dev) {
  extern __shared__ __align__(16) unsigned int s_acc[];  // [3][ncat] (fixed-point sums)
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count_dev = *total;
  const uint32_t ncat = cols.n_categories;
  int S = 0;
#ifdef SKX_SEL_DIAG_NOSUM
  const bool fixed = false;  // diagnostic build: no category sums
#else
  const bool fixed = FUSED && cols.sums && fixed_ok(cols.ctl, ncat, S);
#endif
  if (fixed) {
    for (uint32_t i = threadIdx.x; i < 3 * ncat; i += kThreads) s_acc[i] = 0u;
    __syncthreads();
  }
  const uint64_t nslices = (n + kWarpRows - 1) / kWarpRows;
  const uint32_t bits32 = bits < 0xFFFFFFFFull ? (uint32_t)bits : 0xFFFFFFFFu;
  const uint32_t lt = lanemask_lt();
  const uint64_t capw = spw * kCap;
  const uint64_t warps = (uint64_t)gridDim.x * kWarps;
  // work item = (region, part): a region's entries split into kParts even runs
  const uint64_t items = nregions * kParts;
  for (uint64_t it = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); it < items; it += warps) {
    const uint64_t r = it / kParts;
    const uint32_t part = (uint32_t)(it % kParts);
    const uint32_t cnt = __ldg(warp_counts + r);
    const uint64_t ob = __ldg(warp_off + r);
    if (cnt <= capw) {
      const uint2* src = entries + r * capw;
      const uint32_t e_end = (uint32_t)((uint64_t)cnt * (part + 1) / kParts);
      for (uint32_t j0 = (uint32_t)((uint64_t)cnt * part / kParts); j0 < e_end; j0 += 32 * kPer) {
        uint2 e[kPer];
        Rec8 rc[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const uint32_t f = j0 + u * 32 + lane;
          e[u] = f < e_end ? __ldcs(src + f) : make_uint2(0u, 0u);
        }
        if (FUSED) {  // key -> dense record index (the directory is L2-resident) -> record
          uint2 pr[kPer];
#pragma unroll
          for (int u = 0; u < kPer; ++u)
            pr[u] = j0 + u * 32 + lane < e_end ? __ldg(cols.dir + (e[u].x >> 5)) : make_uint2(0u, 0u);
#pragma unroll
          for (int u = 0; u < kPer; ++u) {
            rc[u] = Rec8{};
            if (j0 + u * 32 + lane < e_end) rc[u] = load_rec(cols.rec, compact_index(pr[u], e[u].x));
          }
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const uint32_t f = j0 + u * 32 + lane;
          if (f < e_end)
            emit_row<FUSED>(ob + f, e[u].y, rc[u], base_off, out_off, cols, fixed, S, s_acc);
        }
      }
      continue;
    }
    if (part != 0) continue;  // an overflowed region is re-derived by its first item
    // overflowed region: every slice re-derived (domain already checked in pass 1)
    const uint64_t s_begin = r * spw < nslices ? r * spw : nslices;
    const uint64_t s_end = s_begin + spw < nslices ? s_begin + spw : nslices;
    uint64_t run = 0;
    for (uint64_t sl = s_begin; sl < s_end; ++sl) {
      const uint64_t row0 = sl * kWarpRows;
      const bool full = row0 + kWarpRows <= n;
      uint32_t fk[kItems][4];
      load_slice<VEC>(fact, n, row0, full, lane, fk);
      uint32_t sel[kItems];
      if (full)
        probe_slice<true>(fk, row0, n, bits32, 0u, 0u, words32, lane, nullptr, sel);
      else
        probe_slice<false>(fk, row0, n, bits32, 0u, 0u, words32, lane, nullptr, sel);
      const uint32_t row_l = (uint32_t)row0 + 4u * lane;
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        uint32_t b[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = __ballot_sync(0xffffffffu, (sel[i] >> j) & 1u);
        uint64_t pos = run + item_base(b, lt);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if ((sel[i] >> j) & 1u) {
            Rec8 rr{};
            if (FUSED) {
              const uint32_t idx = fk[i][j] - 1u;
              rr = load_rec(cols.rec, compact_index(__ldg(cols.dir + (idx >> 5)), idx));
            }
            emit_row<FUSED>(ob + pos, row_l + i * 128 + j, rr, base_off, out_off, cols, fixed, S,
                            s_acc);
            ++pos;
          }
        }
        run += item_count(b);
      }
    }
  }
  if (fixed) {
    __syncthreads();
    for (uint32_t c2 = threadIdx.x; c2 < ncat; c2 += kThreads) {
      const unsigned int L = s_acc[c2], M = s_acc[ncat + c2], H = s_acc[2 * ncat + c2];
      if ((L | M | H) == 0u) continue;
      unsigned int* g = cols.acc96 + 4 * (uint64_t)c2;
      const unsigned int old = atomicAdd(&g[0], L);
      const unsigned int c1 = (unsigned int)(old + L) < old ? 1u : 0u;
      const unsigned int m2 = M + c1;
      unsigned int h = H + (m2 < M ? 1u : 0u);
      const unsigned int old2 = atomicAdd(&g[1], m2);
      h += (unsigned int)(old2 + m2) < old2 ? 1u : 0u;
      if (h) atomicAdd(&g[2], h);
    }
  }
}

// C5 epilogue (fixed point): 96-bit sums -> fp64.  No-op on the fp64 path.
__global__ void k_sum_finalize(const unsigned int* __restrict__ acc96, const SumCtl* ctl,
                               uint32_t ncat, double* __restrict__ sums) {
  int S = 0;
  if (!fixed_ok(ctl, ncat, S)) return;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncat; c += gridDim.x * blockDim.x) {
    const unsigned int* g = acc96 + 4 * (uint64_t)c;
    const long long hi64 = (long long)(((unsigned long long)g[2] << 32) | g[1]);  // bits 32..95
    sums[c] = ldexp(ldexp((double)hi64, 32) + (double)g[0], -S);
  }
}

// Cross-GPU combine of the fixed-point sums (skx_select_sum_partials): the
// three 32-bit limbs of each category's 96-bit sum, widened to int64 (low and
// middle unsigned, high signed) so an element-wise integer SUM over ranks is
// exact; out[0] = 1 when this rank summed in fixed point, out[1] = its scale.
__global__ void k_sum_partials(const unsigned int* __restrict__ acc96, const SumCtl* ctl,
                               uint32_t ncat, long long* __restrict__ out) {
  int S = 0;
  const bool fx = ctl != nullptr && fixed_ok(ctl, ncat, S);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) {
    out[0] = fx ? 1 : 0;
    out[1] = fx ? S : 0;
  }
  for (uint32_t c = t; c < ncat; c += gridDim.x * blockDim.x) {
    const unsigned int* g = acc96 + 4 * (uint64_t)c;
    out[2 + 3 * (uint64_t)c] = fx ? (long long)g[0] : 0;
    out[3 + 3 * (uint64_t)c] = fx ? (long long)g[1] : 0;
    out[4 + 3 * (uint64_t)c] = fx ? (long long)(int)g[2] : 0;
  }
}

// After the SUM over `nranks` partials: when every rank summed in fixed point
// with one scale S, sums[c] = (lo + mid 2^32 + hi 2^64) 2^-S, carried exactly
// in 128 bits and rounded once per part; else the fp64 sums stay as they are.
__global__ void k_sums_from_partials(const long long* __restrict__ p, uint32_t ncat,
                                     uint32_t nranks, double* __restrict__ sums) {
  if (p[0] != (long long)nranks || p[1] % (long long)nranks != 0) return;
  const int S = (int)(p[1] / (long long)nranks);
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncat; c += gridDim.x * blockDim.x) {
    const __int128 v = (__int128)p[2 + 3 * (uint64_t)c] + ((__int128)p[3 + 3 * (uint64_t)c] << 32) +
                       ((__int128)p[4 + 3 * (uint64_t)c] << 64);
    const double top = (double)(long long)(v >> 64);
    const double mid = (double)(unsigned long long)((unsigned long long)(v >> 32) & 0xffffffffull);
    const double low = (double)(unsigned long long)((unsigned long long)v & 0xffffffffull);
    sums[c] = ldexp(ldexp(top, 64) + (ldexp(mid, 32) + low), -S);
  }
}

// Pass 3 (C5): SUM(price) per category over the compacted selected rows --
// a coalesced read of the gathered category/price columns.  Warp-private
// fp64 shared bins; lanes of one category pre-sum with __match_any_sync +
// shuffles (shared fp64 atomics are CAS spin loops on sm_100a); one native
// global fp64 reduction per bin per CTA.
__global__ void __launch_bounds__(kThreads)
    k_category_sum(const int32_t* __restrict__ cat, const float* __restrict__ price,
                   const uint32_t* __restrict__ total, uint64_t cap, uint32_t n_categories,
                   double* __restrict__ sums, const SumCtl* ctl) {
  int S_unused = 0;
  if (fixed_ok(ctl, n_categories, S_unused)) return;  // summed in pass 2
  extern __shared__ double s_bins[];  // [kWarps][n_categories] when small
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool smem = n_categories <= kSmemCategories;
  if (smem) {
    for (uint32_t i = threadIdx.x; i < kWarps * n_categories; i += kThreads) s_bins[i] = 0.0;
    __syncthreads();
  }
  constexpr int U = 8;  // rows per thread per iteration, loads issued first
  const uint64_t cnt = *total < cap ? *total : cap;
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
  const bool sums_on = fused && cols.sums && cols.n_categories;
  if (sums_on) {
    e = cudaMemsetAsync(cols.sums, 0, (size_t)cols.n_categories * 8, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "select memset");
  }
  if (n == 0 && !fused) {
    e = cudaMemsetAsync(count_dev, 0, 8, s);
    return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "select memset");
  }
  const uint64_t nslices = (n + kWarpRows - 1) / kWarpRows;
  // pass 1 grid: one CTA per SM (they share nothing but the bitmap prefix);
  // global warp g owns the slices [g * spw, (g + 1) * spw)
  const uint64_t cta1 = (nslices + kThreads1 / 32 - 1) / (kThreads1 / 32);
  const unsigned grid1 = (unsigned)(cta1 < (uint64_t)ctx->num_sms ? cta1 : ctx->num_sms);
  const uint64_t nregions = (uint64_t)grid1 * (kThreads1 / 32);
  const uint64_t spw = (nslices + nregions - 1) / nregions;
  // scratch: entries [nregions][spw * kCap] | region counts | region offsets | total |
  //          (fused) SumCtl 256 B | acc96 [ncat][4] | records [d][32 B]
  const uint64_t ent_b = nregions * spw * kCap * 8;
  const uint64_t base_b = (ent_b + nregions * 8 + 256 + 255) & ~uint64_t(255);
  const uint64_t acc_b = fused ? (((uint64_t)cols.n_categories * 16 + 255) & ~uint64_t(255)) : 0;
  const uint64_t rec_b = fused ? bits * 32 : 0;
  const uint64_t nw32 = (bits + 31) / 32;
  const uint64_t dir_b = fused ? ((nw32 * 8 + 255) & ~uint64_t(255)) : 0;
  const uint64_t pc_b = fused ? ((nw32 * 4 + 255) & ~uint64_t(255)) : 0;
  // (fused) ... | rank directory [nw32] | word popcounts [nw32]
  char* raw = static_cast<char*>(
      scratch(ctx, 2, base_b + (fused ? 256 : 0) + acc_b + rec_b + dir_b + pc_b, s));
  if (!raw) return set_error(ctx, SKX_CUDA_ERROR, "select: out of device memory");
  uint2* entries = reinterpret_cast<uint2*>(raw);
  uint32_t* counts = reinterpret_cast<uint32_t*>(raw + ent_b);
  uint32_t* offs = counts + nregions;
  uint32_t* total = offs + nregions;
  if (fused) {
    cols.ctl = reinterpret_cast<SumCtl*>(raw + base_b);
    cols.acc96 = reinterpret_cast<unsigned int*>(raw + base_b + 256);
    cols.rec = reinterpret_cast<const uint4*>(raw + base_b + 256 + acc_b);
    cols.dir = reinterpret_cast<const uint2*>(raw + base_b + 256 + acc_b + rec_b);
    ScratchSet* ss = scratch_set(ctx, s);
    ss->sel_acc = cols.acc96;
    ss->sel_ctl = cols.ctl;
    ss->sel_ncat = cols.n_categories;
    e = cudaMemsetAsync(raw + base_b, 0, 256 + acc_b, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "select memset");
    if (bits) {
      // rank directory: per 32-bit word, the selected bits before it
      uint32_t* pc = reinterpret_cast<uint32_t*>(raw + base_b + 256 + acc_b + rec_b + dir_b);
      const auto* w32 = reinterpret_cast<const uint32_t*>(words);
      k_word_popc<<<grid_for(ctx, nw32, 256, 8), 256, 0, s>>>(w32, nw32, pc);
      ctx->launches++;
      int rc = launch_exclusive_scan_u32(ctx, pc, pc, nw32, nullptr, 3, s);
      if (rc) return rc;
      k_dir_fill<<<grid_for(ctx, nw32, 256, 8), 256, 0, s>>>(w32, pc, nw32,
                                                             const_cast<uint2*>(cols.dir));
      const bool cvec = ((reinterpret_cast<uintptr_t>(cols.cat) | reinterpret_cast<uintptr_t>(cols.price) |
                          reinterpret_cast<uintptr_t>(cols.supp)) % 16 == 0) &&
                        reinterpret_cast<uintptr_t>(cols.flag) % 8 == 0;
      k_pack_records<<<grid_for(ctx, (bits + 3) / 4, 256, 8), 256, 0, s>>>(
          cols.cat, cols.price, cols.supp, cols.flag, cols.dir, (uint32_t)bits, cvec,
          const_cast<uint4*>(cols.rec), cols.ctl);
      ctx->launches += 2;
    }
    if (n == 0) {  // no rows: zero sums and count; the scale is still recorded for combining
      e = cudaMemsetAsync(count_dev, 0, 8, s);
      return e == cudaSuccess ? SKX_OK : cuda_fail(ctx, e, "select memset");
    }
  }
  const bool vec = reinterpret_cast<uintptr_t>(fact) % 16 == 0;
  const auto* w32 = reinterpret_cast<const uint32_t*>(words);
  // Pass 1 with the bitmap prefix staged per CTA in shared memory.
  size_t sbytes = (size_t)SKX_SEL_SMEM_KB * 1024;
  if (sbytes > ctx->smem_optin - 1024) sbytes = ctx->smem_optin - 1024;
  const uint32_t sw = (uint32_t)(nw32 < sbytes / 4 ? nw32 : sbytes / 4);
  const size_t smem1 = (size_t)sw * 4;
  auto k1 = vec ? (bits ? k_select_count<true, true> : k_select_count<true, false>)
                : k_select_count<false, false>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  k1<<<grid1, kThreads1, smem1, s>>>(fact, n, w32, bits, entries, counts, spw, sw, ctx->err);
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "select pass 1");
  int rc = launch_exclusive_scan_u32(ctx, counts, offs, nregions, total, 3, s);
  if (rc) return rc;
  const size_t smem = sums_on && cols.n_categories <= kFixedCategories
                          ? (size_t)cols.n_categories * 12 : 0;
  auto k2 = fused ? (vec ? k_select_emit<true, true> : k_select_emit<true, false>)
                  : (vec ? k_select_emit<false, true> : k_select_emit<false, false>);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2, kThreads, smem);
  const unsigned grid2 = grid_for(ctx, (nregions + kWarps - 1) / kWarps, 1, per_sm < 1 ? 1 : per_sm);
  k2<<<grid2, kThreads, smem, s>>>(fact, n, w32, bits, entries, counts, offs, nregions, spw, base,
                                   total, out, cols,
                                   reinterpret_cast<unsigned long long*>(count_dev));
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "select pass 2");
  if (sums_on) {
    k_sum_finalize<<<(cols.n_categories + 255) / 256, 256, 0, s>>>(cols.acc96, cols.ctl,
                                                                   cols.n_categories, cols.sums);
    // fp64 fallback over the compacted columns; exits at once on the fixed path.
    const size_t bsmem =
        cols.n_categories <= kSmemCategories ? (size_t)kWarps * cols.n_categories * 8 : 0;
    cudaFuncSetAttribute(k_category_sum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
    int per_sm3 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3, k_category_sum, kThreads, bsmem);
    k_category_sum<<<(unsigned)ctx->num_sms * (per_sm3 < 1 ? 1 : per_sm3), kThreads, bsmem, s>>>(
        cols.out_cat, cols.out_price, total, cols.cap, cols.n_categories, cols.sums, cols.ctl);
    ctx->launches += 2;
  }
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
  skx::bind(ctx);
  skx::Cols cols{};
  cols.cap = n;  // KernelTable::select_offsets contract: out holds n entries
  return skx::select_impl(ctx, false, fact, n, words, bits, base, out, cols, count_dev,
                          skx::as_stream(stream));
}

int skx_select_gather_sum(skx_ctx* ctx, const uint32_t* fact, uint64_t n, const uint64_t* words,
                          uint32_t d, const int32_t* cat, const float* price,
                          const uint64_t* supp, const uint16_t* flag, uint32_t base,
                          uint32_t n_categories, uint64_t capacity, uint32_t* out_off,
                          int32_t* out_cat, float* out_price, uint64_t* out_supp,
                          uint16_t* out_flag, double* sums, uint64_t* count_dev, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  if (n && (!cat || !price || !supp || !flag || !out_cat || !out_price || !out_supp || !out_flag ||
            (n_categories && !sums)))
    return skx::set_error(ctx, SKX_INVALID_ARGUMENT, "select_gather_sum: null column pointer");
  skx::Cols cols{cat, price, reinterpret_cast<const unsigned long long*>(supp), flag,
                 out_cat, out_price, reinterpret_cast<unsigned long long*>(out_supp), out_flag,
                 sums, n_categories, nullptr, nullptr, nullptr, nullptr, capacity};
  return skx::select_impl(ctx, true, fact, n, words, d, base, out_off, cols, count_dev,
                          skx::as_stream(stream));
}

int skx_select_sum_partials(skx_ctx* ctx, uint32_t n_categories, int64_t* out, void* stream) {
  if (!ctx || !out) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  cudaStream_t s = skx::as_stream(stream);
  skx::ScratchSet* ss = skx::scratch_set(ctx, s);
  if (!ss->sel_acc || ss->sel_ncat != n_categories)
    return skx::set_error(ctx, SKX_INVALID_ARGUMENT,
                          "select_sum_partials: no select_gather_sum with %u categories on this stream",
                          n_categories);
  skx::k_sum_partials<<<(n_categories + 255) / 256 + 1, 256, 0, s>>>(
      static_cast<const unsigned int*>(ss->sel_acc), static_cast<const skx::SumCtl*>(ss->sel_ctl),
      n_categories, reinterpret_cast<long long*>(out));
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "select_sum_partials");
  return SKX_OK;
}

int skx_select_sums_from_partials(skx_ctx* ctx, const int64_t* partials, uint32_t n_categories,
                                  uint32_t nranks, double* sums, void* stream) {
  if (!ctx || !partials || !sums || nranks == 0) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
  if (n_categories == 0) return SKX_OK;
  skx::k_sums_from_partials<<<(n_categories + 255) / 256, 256, 0, skx::as_stream(stream)>>>(
      reinterpret_cast<const long long*>(partials), n_categories, nranks, sums);
  ctx->launches++;
  SKX_CHECK_LAUNCH(ctx, "select_sums_from_partials");
  return SKX_OK;
}

int skx_permute_bitmap(skx_ctx* ctx, const uint64_t* words, uint64_t bits, const uint32_t* offsets,
                       uint32_t d, uint64_t* out_words, void* stream) {
  if (!ctx) return SKX_INVALID_ARGUMENT;
  skx::bind(ctx);
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
  skx::bind(ctx);
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

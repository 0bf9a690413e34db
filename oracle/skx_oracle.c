/*
 * skx_oracle.c -- CPU restatement of the skewdx hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity CHECKER for the B200 kernels in
 * paper_1910_10063_b200/csrc.  It is never linked into, loaded by, or called
 * from the product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may use it.
 *
 * Every function restates the algorithm of the reference library (skewdx,
 * /root/reference/proj) at the file:line cited beside it.  The restatement is
 * pinned two ways (see tests/test_oracle_cpu.py):
 *   1. against the reference's own known-answer vectors (tests/golden/kat.json,
 *      transcribed from proj/tests/test_*.cpp), and
 *   2. against outputs of the reference library itself compiled from its
 *      sources into oracle/_ref/ (tests/golden/ref_*.npz, produced by
 *      tests/golden/make_golden.py through oracle/ref_capi.cpp).
 *
 * Status codes mirror include/skx.h: 0 ok, 1 invalid argument, 2 domain
 * violation (row/value written to *err_row / *err_value).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <immintrin.h>

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_DOMAIN 2

/* ---- splitmix64: proj/include/skewdx/mix.hpp:12-17 ---------------------- */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* ---- mt19937_64 (published Matsumoto-Nishimura 64-bit MT; the engine the
 * reference draws from via std::mt19937_64, column.cpp:65,87) -------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

static void mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  g->idx = 312;
}

static uint64_t mt64_next(orc_mt64* g) {
  if (g->idx >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* ---- zipf_frequencies: proj/src/column.cpp:44-60 (Kahan normaliser) ------ */
int orc_zipf_frequencies(uint32_t d, double z, double* out) {
  if (d == 0 || !(z >= 0.0)) return ORC_INVALID;
  double sum = 0.0, carry = 0.0;
  for (uint32_t r = 1; r <= d; ++r) {
    const double w = pow((double)r, -z);
    out[r - 1] = w;
    const double y = w - carry;
    const double t = sum + y;
    carry = (t - sum) - y;
    sum = t;
  }
  for (uint32_t i = 0; i < d; ++i) out[i] /= sum;
  return ORC_OK;
}

/* CDF as generate_fact_column builds it: partial_sum, last forced to 1.0
 * (proj/src/column.cpp:77-79). */
int orc_zipf_cdf(uint32_t d, double z, double* cdf) {
  int st = orc_zipf_frequencies(d, z, cdf);
  if (st) return st;
  for (uint32_t i = 1; i < d; ++i) cdf[i] = cdf[i - 1] + cdf[i];
  cdf[d - 1] = 1.0;
  return ORC_OK;
}

/* ---- random_bijection: proj/src/column.cpp:62-71 ------------------------- */
void orc_random_bijection(uint32_t n, uint64_t seed, uint32_t* map) {
  for (uint32_t i = 0; i < n; ++i) map[i] = i + 1;
  orc_mt64 g;
  mt64_seed(&g, seed);
  for (uint32_t i = n; i > 1; --i) {
    const uint32_t j = (uint32_t)(mt64_next(&g) % i);
    const uint32_t t = map[i - 1];
    map[i - 1] = map[j];
    map[j] = t;
  }
}

/* std::upper_bound over cdf[0..d): first index with cdf[i] > u. */
static uint32_t upper_bound_d(const double* cdf, uint32_t d, double u) {
  uint32_t lo = 0, len = d;
  while (len > 0) {
    const uint32_t half = len >> 1;
    if (!(u < cdf[lo + half])) {
      lo = lo + half + 1;
      len = len - half - 1;
    } else {
      len = half;
    }
  }
  return lo;
}

/* ---- generate_fact_column, Layout::rand: proj/src/column.cpp:73-125 -------
 * Draws ranks with mt19937_64(splitmix64(seed ^ 0x5ca1ab1e)), u = (rng()>>11)
 * * 2^-53, upper_bound over the CDF, rank clamp to d-1, then rank -> id via
 * random_bijection(d, seed).  ground-truth counts are optional (may be NULL). */
int orc_generate_fact_column_rand(uint32_t d, uint64_t n, double z, uint64_t seed,
                                  uint32_t* values, uint64_t* gt_counts) {
  if (d == 0 || n == 0 || !(z >= 0.0)) return ORC_INVALID;
  double* cdf = (double*)malloc(sizeof(double) * d);
  uint32_t* r2i = (uint32_t*)malloc(sizeof(uint32_t) * d);
  orc_zipf_cdf(d, z, cdf);
  orc_mt64 g;
  mt64_seed(&g, orc_splitmix64(seed ^ 0x5ca1ab1eull));
  for (uint64_t k = 0; k < n; ++k) {
    const double u = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
    uint32_t rank = upper_bound_d(cdf, d, u);
    if (rank >= d) rank = d - 1;
    values[k] = rank; /* ranks for now */
  }
  orc_random_bijection(d, seed, r2i);
  if (gt_counts) memset(gt_counts, 0, sizeof(uint64_t) * d);
  for (uint64_t k = 0; k < n; ++k) {
    values[k] = r2i[values[k]];
    if (gt_counts) gt_counts[values[k] - 1]++;
  }
  free(cdf);
  free(r2i);
  return ORC_OK;
}

/* ---- Counter-based Zipf draw (the B200 build's parallel generator, see
 * DESIGN.md "Inputs").  Same inverse-CDF math as column.cpp:88-95, but the
 * k-th uniform is taken from the SplitMix64 sequence keyed by
 * splitmix64(seed ^ 0x5ca1ab1e) instead of a sequential mt19937_64 stream:
 *   u_k = (splitmix64(key + k * 0x9e3779b97f4a7c15) >> 11) * 2^-53.
 * rank_to_id may be NULL (values are then 1-based distribution ranks). */
void orc_generate_zipf_counter(const double* cdf, uint32_t d, const uint32_t* rank_to_id,
                               uint64_t seed, uint64_t row_begin, uint64_t n, uint32_t* out) {
  const uint64_t key = orc_splitmix64(seed ^ 0x5ca1ab1eull);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t k = row_begin + i;
    const double u = (double)(orc_splitmix64(key + k * 0x9e3779b97f4a7c15ull) >> 11) * 0x1.0p-53;
    uint32_t rank = upper_bound_d(cdf, d, u);
    if (rank >= d) rank = d - 1;
    out[i] = rank_to_id ? rank_to_id[rank] : rank + 1;
  }
}

/* ---- find_domain_violation: proj/src/operators.cpp:32-41 ----------------- */
uint64_t orc_find_domain_violation(const uint32_t* fact, uint64_t n, uint64_t d) {
  for (uint64_t k = 0; k < n; ++k) {
    if ((uint64_t)(uint32_t)(fact[k] - 1u) >= d) return k;
  }
  return UINT64_MAX;
}

#define DOMAIN_CHECK(fact, n, d)                              \
  do {                                                        \
    const uint64_t bad_ = orc_find_domain_violation(fact, n, d); \
    if (bad_ != UINT64_MAX) {                                 \
      if (err_row) *err_row = bad_;                           \
      if (err_value) *err_value = (fact)[bad_];               \
      return ORC_DOMAIN;                                      \
    }                                                         \
  } while (0)

/* ---- count_frequencies: proj/src/permindex.cpp:18-30 --------------------- */
int orc_count_frequencies(const uint32_t* fact, uint64_t n, uint32_t d, uint64_t* counts,
                          uint64_t* err_row, uint32_t* err_value) {
  memset(counts, 0, sizeof(uint64_t) * d);
  for (uint64_t k = 0; k < n; ++k) {
    const uint32_t id = fact[k];
    if ((uint32_t)(id - 1u) >= d) {
      if (err_row) *err_row = k;
      if (err_value) *err_value = id;
      return ORC_DOMAIN;
    }
    counts[id - 1]++;
  }
  return ORC_OK;
}

/* ---- build_index: proj/src/permindex.cpp:32-58 ---------------------------
 * offsets = ids sorted by (count desc, id asc); ranks[offsets[r]-1] = r+1.
 * The comparator is a strict total order, so any sort gives the same result. */
static const uint64_t* g_sort_counts;
static int cmp_by_count(const void* pa, const void* pb) {
  const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  const uint64_t ca = g_sort_counts[a - 1], cb = g_sort_counts[b - 1];
  if (ca != cb) return ca > cb ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}

int orc_build_index(const uint64_t* counts, uint32_t d, uint64_t total, uint32_t* offsets,
                    uint32_t* ranks) {
  uint64_t sum = 0;
  for (uint32_t i = 0; i < d; ++i) sum += counts[i];
  if (sum != total) return ORC_INVALID; /* permindex.cpp:36-40 */
  for (uint32_t i = 0; i < d; ++i) offsets[i] = i + 1;
  g_sort_counts = counts; /* not thread-safe; test infrastructure only */
  qsort(offsets, d, sizeof(uint32_t), cmp_by_count);
  for (uint32_t r = 0; r < d; ++r) ranks[offsets[r] - 1] = r + 1;
  return ORC_OK;
}

/* ---- materialize / gather_u32: proj/src/operators.cpp:60-66,
 * proj/src/kernels/scalar.cpp:13-29 -- out[k] = dim[fact[k]-1].  The u16 and
 * u64 widths are the restatement SURVEY.md §8a asks for (reference is u32). */
#define DEFINE_GATHER(NAME, T)                                                   \
  int NAME(const uint32_t* fact, uint64_t n, const T* dim, uint64_t dim_len, T* out, \
           uint64_t* err_row, uint32_t* err_value) {                             \
    DOMAIN_CHECK(fact, n, dim_len);                                              \
    for (uint64_t k = 0; k < n; ++k) out[k] = dim[fact[k] - 1];                  \
    return ORC_OK;                                                               \
  }
DEFINE_GATHER(orc_gather_u16, uint16_t)
DEFINE_GATHER(orc_gather_u32, uint32_t)
DEFINE_GATHER(orc_gather_u64, uint64_t)

/* recode_fact: proj/src/permindex.cpp:60-64 (= materialize(fact, ranks)). */
int orc_recode_fact(const uint32_t* fact, uint64_t n, const uint32_t* ranks, uint32_t d,
                    uint32_t* out, uint64_t* err_row, uint32_t* err_value) {
  return orc_gather_u32(fact, n, ranks, d, out, err_row, err_value);
}

/* permute_dimension: proj/src/permindex.cpp:66-73 (= materialize(offsets, dim)). */
int orc_permute_dimension_u32(const uint32_t* dim, uint64_t dim_len, const uint32_t* offsets,
                              uint32_t d, uint32_t* out) {
  if (dim_len != d) return ORC_INVALID;
  for (uint32_t r = 0; r < d; ++r) out[r] = dim[offsets[r] - 1];
  return ORC_OK;
}
int orc_permute_dimension_u64(const uint64_t* dim, uint64_t dim_len, const uint32_t* offsets,
                              uint32_t d, uint64_t* out) {
  if (dim_len != d) return ORC_INVALID;
  for (uint32_t r = 0; r < d; ++r) out[r] = dim[offsets[r] - 1];
  return ORC_OK;
}
int orc_permute_dimension_u16(const uint16_t* dim, uint64_t dim_len, const uint32_t* offsets,
                              uint32_t d, uint16_t* out) {
  if (dim_len != d) return ORC_INVALID;
  for (uint32_t r = 0; r < d; ++r) out[r] = dim[offsets[r] - 1];
  return ORC_OK;
}

/* ---- aggregate_count / aggregate_sum: proj/src/operators.cpp:100-118.
 * measure may be u32 (reference signature) or u64 (BASELINE C3 int64 qty);
 * measure NULL -> counts only; counts or sums may be NULL. */
int orc_aggregate_count_sum_u64(const uint32_t* fact, const uint64_t* measure, uint64_t n,
                                uint32_t d, uint64_t* counts, uint64_t* sums,
                                uint64_t* err_row, uint32_t* err_value) {
  DOMAIN_CHECK(fact, n, d);
  if (counts) memset(counts, 0, sizeof(uint64_t) * d);
  if (sums) memset(sums, 0, sizeof(uint64_t) * d);
  for (uint64_t k = 0; k < n; ++k) {
    const uint32_t i = fact[k] - 1;
    if (counts) counts[i]++;
    if (sums && measure) sums[i] += measure[k];
  }
  return ORC_OK;
}
int orc_aggregate_count_sum_u32(const uint32_t* fact, const uint32_t* measure, uint64_t n,
                                uint32_t d, uint64_t* counts, uint64_t* sums,
                                uint64_t* err_row, uint32_t* err_value) {
  DOMAIN_CHECK(fact, n, d);
  if (counts) memset(counts, 0, sizeof(uint64_t) * d);
  if (sums) memset(sums, 0, sizeof(uint64_t) * d);
  for (uint64_t k = 0; k < n; ++k) {
    const uint32_t i = fact[k] - 1;
    if (counts) counts[i]++;
    if (sums && measure) sums[i] += measure[k];
  }
  return ORC_OK;
}

/* ---- select_offsets_scalar: proj/src/kernels/scalar.cpp:31-42 ----------- */
int orc_select_offsets(const uint32_t* fact, uint64_t n, const uint64_t* words, uint64_t bits,
                       uint32_t base, uint32_t* out, uint64_t* count,
                       uint64_t* err_row, uint32_t* err_value) {
  if (n > 0xFFFFFFFFull) return ORC_INVALID; /* operators.cpp:88-90 */
  DOMAIN_CHECK(fact, n, bits);
  uint64_t c = 0;
  for (uint64_t k = 0; k < n; ++k) {
    const uint32_t idx = fact[k] - 1;
    const uint64_t bit = (words[idx >> 6] >> (idx & 63)) & 1;
    out[c] = base + (uint32_t)k;
    c += bit;
  }
  *count = c;
  return ORC_OK;
}

/* ---- permute_bitmap: proj/src/operators.cpp:21-30 ------------------------ */
int orc_permute_bitmap(const uint64_t* words, uint64_t bits, const uint32_t* offsets,
                       uint32_t d, uint64_t* out_words) {
  if (bits != d) return ORC_INVALID;
  memset(out_words, 0, sizeof(uint64_t) * ((bits + 63) / 64));
  for (uint64_t r = 0; r < bits; ++r) {
    const uint32_t i = offsets[r] - 1;
    if ((words[i >> 6] >> (i & 63)) & 1) out_words[r >> 6] |= 1ull << (r & 63);
  }
  return ORC_OK;
}

/* ---- Config-5 select + 4-column gather + per-category fp64 SUM(price).
 * Composition of select (operators.cpp:87-98), materialize over the selected
 * rows (operators.cpp:60-66) and an fp64 restatement of aggregate_sum
 * (operators.cpp:107-118) keyed by the gathered category.  Sums are added in
 * ascending row order. */
int orc_select_gather_sum(const uint32_t* fact, uint64_t n, const uint64_t* words, uint32_t d,
                          const int32_t* cat, const float* price, const uint64_t* supp,
                          const uint16_t* flag, uint32_t base, uint32_t n_categories,
                          uint32_t* out_off, int32_t* out_cat, float* out_price,
                          uint64_t* out_supp, uint16_t* out_flag, double* sums,
                          uint64_t* count, uint64_t* err_row, uint32_t* err_value) {
  if (n > 0xFFFFFFFFull) return ORC_INVALID;
  DOMAIN_CHECK(fact, n, d);
  memset(sums, 0, sizeof(double) * n_categories);
  uint64_t c = 0;
  for (uint64_t k = 0; k < n; ++k) {
    const uint32_t idx = fact[k] - 1;
    if (!((words[idx >> 6] >> (idx & 63)) & 1)) continue;
    out_off[c] = base + (uint32_t)k;
    out_cat[c] = cat[idx];
    out_price[c] = price[idx];
    out_supp[c] = supp[idx];
    out_flag[c] = flag[idx];
    if ((uint32_t)cat[idx] < n_categories) sums[cat[idx]] += (double)price[idx];
    ++c;
  }
  *count = c;
  return ORC_OK;
}

/* ---- chunk_spans: proj/src/parallel.cpp:31-43 ---------------------------- */
int orc_chunk_spans(uint64_t n, uint32_t threads, uint64_t* begins, uint64_t* ends) {
  if (threads == 0) return ORC_INVALID;
  const uint64_t base = n / threads, extra = n % threads;
  uint64_t b = 0;
  for (uint32_t t = 0; t < threads; ++t) {
    const uint64_t len = base + (t < extra ? 1 : 0);
    begins[t] = b;
    ends[t] = b + len;
    b += len;
  }
  return ORC_OK;
}

/* ---- parallel_materialize port for the u64 value width (the reference's
 * parallel.cpp:87-100 is u32-only): chunk_spans fork-join over T pthreads,
 * each thread writing its own output span.  Used only as bench.py's CPU
 * baseline ("port") for config C2. */
typedef struct {
  const uint32_t* fact;
  const uint64_t* dim;
  uint64_t* out;
  uint64_t b, e;
} gather_job;

/* AVX2 inner loop in the shape of the reference's gather_u32_avx2
 * (proj/src/kernels/avx2.cpp:43-57), widened to int64 values: 4 ids per
 * _mm256_i32gather_epi64 (dimension length < 2^31, as kernels_for requires,
 * operators.cpp:51-56). */
__attribute__((target("avx2"))) static void gather_u64_avx2(const uint32_t* fact, uint64_t b,
                                                             uint64_t e, const uint64_t* dim,
                                                             uint64_t* out) {
  const __m128i one = _mm_set1_epi32(1);
  uint64_t k = b;
  for (; k + 4 <= e; k += 4) {
    const __m128i ids = _mm_loadu_si128((const __m128i*)(fact + k));
    const __m256i v = _mm256_i32gather_epi64((const long long*)dim, _mm_sub_epi32(ids, one), 8);
    _mm256_storeu_si256((__m256i*)(out + k), v);
  }
  for (; k < e; ++k) out[k] = dim[fact[k] - 1];
}

static int g_dim_small = 0; /* dimension fits signed 32-bit gather indices */

static void* gather_u64_worker(void* p) {
  gather_job* j = (gather_job*)p;
  if (g_dim_small && __builtin_cpu_supports("avx2")) {
    gather_u64_avx2(j->fact, j->b, j->e, j->dim, j->out);
    return NULL;
  }
  for (uint64_t k = j->b; k < j->e; ++k) j->out[k] = j->dim[j->fact[k] - 1];
  return NULL;
}

int orc_parallel_gather_u64(const uint32_t* fact, uint64_t n, const uint64_t* dim,
                            uint64_t dim_len, uint64_t* out, uint32_t threads,
                            uint64_t* err_row, uint32_t* err_value) {
  if (threads == 0) return ORC_INVALID;
  DOMAIN_CHECK(fact, n, dim_len);
  uint64_t* bs = (uint64_t*)malloc(sizeof(uint64_t) * threads);
  uint64_t* es = (uint64_t*)malloc(sizeof(uint64_t) * threads);
  gather_job* jobs = (gather_job*)malloc(sizeof(gather_job) * threads);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  orc_chunk_spans(n, threads, bs, es);
  g_dim_small = dim_len <= 0x7FFFFFFFull;
  for (uint32_t t = 0; t < threads; ++t) {
    jobs[t] = (gather_job){fact, dim, out, bs[t], es[t]};
    if (t + 1 < threads) pthread_create(&tids[t], NULL, gather_u64_worker, &jobs[t]);
  }
  gather_u64_worker(&jobs[threads - 1]);
  for (uint32_t t = 0; t + 1 < threads; ++t) pthread_join(tids[t], NULL);
  free(bs);
  free(es);
  free(jobs);
  free(tids);
  return ORC_OK;
}

/* ---- checksums: proj/tools/benchcli/checksum.hpp:15-30 ------------------- */
uint64_t orc_rolling_checksum_u32(const uint32_t* v, uint64_t n) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= v[i];
    h *= 1099511628211ull;
  }
  return h;
}
uint64_t orc_unordered_checksum_u64(const uint64_t* v, uint64_t n) {
  uint64_t h = 0;
  for (uint64_t i = 0; i < n; ++i) h += orc_splitmix64(v[i]);
  return h;
}

/* Multithreaded orc_generate_zipf_counter (same values; rows split by
 * chunk_spans) -- only so bench.py's CPU arm can build its bounded sample in
 * seconds. */
typedef struct {
  const double* cdf;
  uint32_t d;
  const uint32_t* r2i;
  uint64_t seed, b, e;
  uint32_t* out;
} gen_job;

static void* gen_worker(void* p) {
  gen_job* j = (gen_job*)p;
  orc_generate_zipf_counter(j->cdf, j->d, j->r2i, j->seed, j->b, j->e - j->b, j->out + j->b);
  return NULL;
}

void orc_generate_zipf_counter_mt(const double* cdf, uint32_t d, const uint32_t* rank_to_id,
                                  uint64_t seed, uint64_t n, uint32_t* out, uint32_t threads) {
  if (threads == 0) threads = 1;
  uint64_t* bs = (uint64_t*)malloc(sizeof(uint64_t) * threads);
  uint64_t* es = (uint64_t*)malloc(sizeof(uint64_t) * threads);
  gen_job* jobs = (gen_job*)malloc(sizeof(gen_job) * threads);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  orc_chunk_spans(n, threads, bs, es);
  for (uint32_t t = 0; t < threads; ++t) {
    jobs[t] = (gen_job){cdf, d, rank_to_id, seed, bs[t], es[t], out};
    if (t + 1 < threads) pthread_create(&tids[t], NULL, gen_worker, &jobs[t]);
  }
  gen_worker(&jobs[threads - 1]);
  for (uint32_t t = 0; t + 1 < threads; ++t) pthread_join(tids[t], NULL);
  free(bs);
  free(es);
  free(jobs);
  free(tids);
}

/* ---- cache model: proj/src/cachemodel.cpp ------------- */

/* line_frequencies (cachemodel.cpp:22-45): per-line sums of per-rank value
 * frequencies; freq layout = ranks in place, rand layout = ranks scattered by
 * random_bijection(d, seed).  Lines accumulate in ascending rank order. */
int orc_line_frequencies(const double* vf, uint32_t d, int layout, uint64_t seed,
                         uint32_t per_line, double* out) {
  if (d == 0 || per_line == 0) return ORC_INVALID;
  const uint64_t lines = ((uint64_t)d + per_line - 1) / per_line;
  memset(out, 0, lines * sizeof(double));
  if (layout == 0) {
    for (uint32_t r = 0; r < d; ++r) out[r / per_line] += vf[r];
  } else {
    uint32_t* map = (uint32_t*)malloc(sizeof(uint32_t) * d);
    if (!map) return ORC_INVALID;
    orc_random_bijection(d, seed, map);
    for (uint32_t r = 0; r < d; ++r) out[(map[r] - 1) / per_line] += vf[r];
    free(map);
  }
  return ORC_OK;
}

static int cmp_desc(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? 1 : (x > y ? -1 : 0);
}

/* Expected distinct lines in k trials that end with a reference to the line
 * of frequency f (cachemodel.cpp:57-72): lines expected more than once
 * (n_j = k f_j / (1 - f) > 1, i.e. f_j > (1 - f) / k) contribute one. */
static double orc_expected_distinct(double k, double f, const double* sorted, uint64_t n,
                                    const double* prefix) {
  const double cutoff = (1.0 - f) / k;
  uint64_t lo = 0, hi = n;  /* first index with sorted[i] <= cutoff */
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (sorted[mid] > cutoff) lo = mid + 1; else hi = mid;
  }
  uint64_t m = lo;
  double mass = prefix[m];
  if (f > cutoff) {
    mass -= f;
    m -= 1;
  }
  return k - (k * mass / (1.0 - f) - (double)m);
}

/* estimate_hit_rate (cachemodel.cpp:76-123): per line, the smallest horizon K
 * >= S (doubling, then bisection, capped at 2^40) at which the expected
 * distinct lines reach the capacity S; hit probability 1 - (1 - f)^K. */
int orc_estimate_hit_rate(const double* lf, uint64_t nlines, uint64_t cache_lines,
                          double* result) {
  if (cache_lines == 0) return ORC_INVALID;
  double* sorted = (double*)malloc(sizeof(double) * (nlines ? nlines : 1));
  double* prefix = (double*)malloc(sizeof(double) * (nlines + 1));
  if (!sorted || !prefix) return ORC_INVALID;
  memcpy(sorted, lf, nlines * sizeof(double));
  qsort(sorted, nlines, sizeof(double), cmp_desc);
  uint64_t n = nlines;
  while (n > 0 && sorted[n - 1] <= 0.0) --n;
  if (n <= cache_lines) {
    *result = 1.0;
    free(sorted);
    free(prefix);
    return ORC_OK;
  }
  prefix[0] = 0.0;
  for (uint64_t i = 0; i < n; ++i) prefix[i + 1] = prefix[i] + sorted[i];
  const double target = (double)cache_lines;
  const uint64_t cap = (uint64_t)1 << 40;
  double total = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double f = sorted[i];
    if (f >= 1.0 - 1e-12) {
      total += f;
      continue;
    }
    uint64_t hi = cache_lines;
    double dd = orc_expected_distinct((double)hi, f, sorted, n, prefix);
    while (dd < target && hi < cap) {
      hi *= 2;
      dd = orc_expected_distinct((double)hi, f, sorted, n, prefix);
    }
    uint64_t k = hi;
    if (dd >= target && hi > cache_lines) {
      uint64_t lo = hi / 2 + 1;
      while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (orc_expected_distinct((double)mid, f, sorted, n, prefix) >= target) hi = mid;
        else lo = mid + 1;
      }
      k = lo;
    }
    total += f * -expm1((double)k * log1p(-f));
  }
  *result = total < 1.0 ? total : 1.0;
  free(sorted);
  free(prefix);
  return ORC_OK;
}

/* simulate_lru (cachemodel.cpp:125-173): exact fully associative LRU over a
 * trace of dense line ids (doubly linked recency list). */
int orc_simulate_lru(const uint32_t* trace, uint64_t n, uint64_t cache_lines,
                     uint64_t* accesses, uint64_t* hits, uint64_t* distinct) {
  if (cache_lines == 0) return ORC_INVALID;
  *accesses = n;
  *hits = 0;
  *distinct = 0;
  if (n == 0) return ORC_OK;
  uint32_t mx = 0;
  for (uint64_t i = 0; i < n; ++i) mx = trace[i] > mx ? trace[i] : mx;
  const uint64_t u = (uint64_t)mx + 1;
  const uint32_t nil = 0xFFFFFFFFu;
  uint32_t* prv = (uint32_t*)malloc(u * 4);
  uint32_t* nxt = (uint32_t*)malloc(u * 4);
  uint8_t* res = (uint8_t*)calloc(u, 1);
  uint8_t* seen = (uint8_t*)calloc(u, 1);
  if (!prv || !nxt || !res || !seen) return ORC_INVALID;
  uint32_t head = nil, tail = nil;
  uint64_t size = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t x = trace[i];
    if (!seen[x]) {
      seen[x] = 1;
      ++*distinct;
    }
    if (res[x]) {
      ++*hits;
      if (x == head) continue;
      /* unlink */
      if (prv[x] != nil) nxt[prv[x]] = nxt[x]; else head = nxt[x];
      if (nxt[x] != nil) prv[nxt[x]] = prv[x]; else tail = prv[x];
    } else {
      res[x] = 1;
      ++size;
    }
    /* push front */
    prv[x] = nil;
    nxt[x] = head;
    if (head != nil) prv[head] = x; else tail = x;
    head = x;
    if (size > cache_lines) {
      const uint32_t v = tail;
      tail = prv[v];
      if (tail != nil) nxt[tail] = nil; else head = nil;
      res[v] = 0;
      --size;
    }
  }
  free(prv);
  free(nxt);
  free(res);
  free(seen);
  return ORC_OK;
}

/* trace_from_column (cachemodel.cpp:175-186): line = (id - 1) / per_line;
 * id 0 is a DomainViolation at its row. */
int orc_trace_from_column(const uint32_t* fact, uint64_t n, uint32_t per_line, uint32_t* out,
                          uint64_t* err_row, uint32_t* err_value) {
  if (per_line == 0) return ORC_INVALID;
  for (uint64_t k = 0; k < n; ++k) {
    if (fact[k] == 0) {
      if (err_row) *err_row = k;
      if (err_value) *err_value = 0;
      return ORC_DOMAIN;
    }
    out[k] = (fact[k] - 1) / per_line;
  }
  return ORC_OK;
}

/*
 * skx_oracle_mt.c -- multi-threaded forms of the CPU restatement, so the
 * parity CHECKER finishes at BASELINE scale (2^30-2^31 rows) in seconds on
 * the GPU box's host cores (TEST INFRASTRUCTURE: only tests/, smoke() and
 * bench.py's CPU legs use liboracle.so; the product never does).
 *
 * Each function computes exactly what its single-threaded counterpart in
 * skx_oracle.c computes (same reference file:line), and
 * tests/test_oracle_cpu.py pins every one of them against that counterpart
 * (and so against the reference's golden vectors) on seeded inputs:
 *   - integer results are order-independent (counts, sums mod 2^64, ordered
 *     concatenation of chunk outputs), so the threading cannot change them;
 *   - build_index's comparator (count desc, id asc; permindex.cpp:44-51) is a
 *     strict total order, so an LSD radix sort of the composite key gives the
 *     identical permutation to std::sort;
 *   - the fp64 category sums of the config-5 restatement are summed per
 *     chunk in row order and the chunk partials in chunk order (a different
 *     fp64 association than one sequential loop: compared at rtol 1e-6, the
 *     north_star tolerance).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_DOMAIN 2

uint64_t orc_splitmix64(uint64_t x);
int orc_chunk_spans(uint64_t n, uint32_t threads, uint64_t* begins, uint64_t* ends);
int orc_build_index(const uint64_t* counts, uint32_t d, uint64_t total, uint32_t* offsets,
                    uint32_t* ranks);

/* ---- fork-join over T workers (the reference's run_chunks shape,
 * parallel.cpp:62-76: one span per worker, joined before returning) ------- */
typedef void (*orc_fn)(void* arg, uint32_t t, uint32_t T);
typedef struct {
  orc_fn fn;
  void* arg;
  uint32_t t, T;
} orc_task;

static void* orc_trampoline(void* p) {
  orc_task* k = (orc_task*)p;
  k->fn(k->arg, k->t, k->T);
  return NULL;
}

static void run_workers(uint32_t T, orc_fn fn, void* arg) {
  if (T == 0) T = 1;
  orc_task* tasks = (orc_task*)malloc(sizeof(orc_task) * T);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * T);
  for (uint32_t t = 0; t < T; ++t) {
    tasks[t] = (orc_task){fn, arg, t, T};
    if (t + 1 < T) pthread_create(&tids[t], NULL, orc_trampoline, &tasks[t]);
  }
  fn(arg, T - 1, T);
  for (uint32_t t = 0; t + 1 < T; ++t) pthread_join(tids[t], NULL);
  free(tasks);
  free(tids);
}

static void span_of(uint64_t n, uint32_t t, uint32_t T, uint64_t* b, uint64_t* e) {
  /* chunk_spans (parallel.cpp:31-43): len = n/T, +1 for the first n%T */
  const uint64_t base = n / T, extra = n % T;
  *b = t * base + (t < extra ? t : extra);
  *e = *b + base + (t < extra ? 1 : 0);
}

/* ---- find_domain_violation (operators.cpp:32-41), chunked: the first bad
 * row overall is the first bad row of the first chunk that has one. ------- */
typedef struct {
  const uint32_t* fact;
  uint64_t n, d;
  uint64_t* first; /* per worker */
} dom_args;

static void dom_worker(void* p, uint32_t t, uint32_t T) {
  dom_args* a = (dom_args*)p;
  uint64_t b, e;
  span_of(a->n, t, T, &b, &e);
  a->first[t] = UINT64_MAX;
  for (uint64_t k = b; k < e; ++k)
    if ((uint64_t)(uint32_t)(a->fact[k] - 1u) >= a->d) {
      a->first[t] = k;
      return;
    }
}

uint64_t orc_find_domain_violation_mt(const uint32_t* fact, uint64_t n, uint64_t d,
                                      uint32_t threads) {
  if (threads == 0) threads = 1;
  uint64_t* first = (uint64_t*)malloc(sizeof(uint64_t) * threads);
  dom_args a = {fact, n, d, first};
  run_workers(threads, dom_worker, &a);
  uint64_t r = UINT64_MAX;
  for (uint32_t t = 0; t < threads; ++t)
    if (first[t] < r) r = first[t];
  free(first);
  return r;
}

#define DOMAIN_CHECK_MT(fact, n, d, T)                                    \
  do {                                                                    \
    const uint64_t bad_ = orc_find_domain_violation_mt(fact, n, d, T);    \
    if (bad_ != UINT64_MAX) {                                             \
      if (err_row) *err_row = bad_;                                       \
      if (err_value) *err_value = (fact)[bad_];                           \
      return ORC_DOMAIN;                                                  \
    }                                                                     \
  } while (0)

/* ---- count_frequencies (permindex.cpp:18-30), key-range partitioned: worker
 * t counts the ids of its slice of the domain over every row. ------------- */
typedef struct {
  const uint32_t* fact;
  uint64_t n;
  uint32_t d;
  uint64_t* counts;
} cnt_args;

static void cnt_worker(void* p, uint32_t t, uint32_t T) {
  cnt_args* a = (cnt_args*)p;
  uint64_t lo, hi;
  span_of(a->d, t, T, &lo, &hi);
  memset(a->counts + lo, 0, (hi - lo) * sizeof(uint64_t));
  const uint32_t span = (uint32_t)(hi - lo), base = (uint32_t)lo;
  uint64_t* c = a->counts;
  for (uint64_t k = 0; k < a->n; ++k) {
    const uint32_t i = a->fact[k] - 1u - base;
    if (i < span) c[base + i]++;
  }
}

int orc_count_frequencies_mt(const uint32_t* fact, uint64_t n, uint32_t d, uint64_t* counts,
                             uint32_t threads, uint64_t* err_row, uint32_t* err_value) {
  if (threads == 0) threads = 1;
  DOMAIN_CHECK_MT(fact, n, d, threads);
  cnt_args a = {fact, n, d, counts};
  run_workers(threads, cnt_worker, &a);
  return ORC_OK;
}

/* ---- build_index (permindex.cpp:32-58) by LSD radix sort ------------------
 * Non-zero ids get the key ((total - count) << 32 | id): ascending key order
 * is exactly (count desc, id asc).  Zero-count ids follow in ascending id
 * order (their comparator order).  Needs total < 2^32 (else: the qsort form). */
int orc_build_index_radix(const uint64_t* counts, uint32_t d, uint64_t total, uint32_t* offsets,
                          uint32_t* ranks) {
  if (total >= 0xFFFFFFFFull) return orc_build_index(counts, d, total, offsets, ranks);
  uint64_t sum = 0, nnz = 0;
  for (uint32_t i = 0; i < d; ++i) {
    sum += counts[i];
    nnz += counts[i] != 0;
  }
  if (sum != total) return ORC_INVALID; /* permindex.cpp:36-40 */
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (nnz ? nnz : 1));
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (nnz ? nnz : 1));
  uint64_t* hist = (uint64_t*)malloc(sizeof(uint64_t) * 65536);
  if (!keys || !tmp || !hist) return ORC_INVALID;
  uint64_t m = 0, z = nnz;
  for (uint32_t i = 0; i < d; ++i) {
    if (counts[i])
      keys[m++] = ((total - counts[i]) << 32) | (uint64_t)(i + 1);
    else
      offsets[z++] = i + 1;
  }
  for (int shift = 0; shift < 64; shift += 16) {
    memset(hist, 0, sizeof(uint64_t) * 65536);
    for (uint64_t k = 0; k < nnz; ++k) hist[(keys[k] >> shift) & 0xFFFF]++;
    int trivial = 0;
    for (int b = 0; b < 65536; ++b)
      if (hist[b] == nnz) trivial = 1;
    if (trivial) continue; /* every key has this digit: the pass is the identity */
    uint64_t run = 0;
    for (int b = 0; b < 65536; ++b) {
      const uint64_t c = hist[b];
      hist[b] = run;
      run += c;
    }
    for (uint64_t k = 0; k < nnz; ++k) tmp[hist[(keys[k] >> shift) & 0xFFFF]++] = keys[k];
    uint64_t* s = keys;
    keys = tmp;
    tmp = s;
  }
  for (uint64_t r = 0; r < nnz; ++r) offsets[r] = (uint32_t)keys[r];
  for (uint32_t r = 0; r < d; ++r) ranks[offsets[r] - 1] = r + 1;
  free(keys);
  free(tmp);
  free(hist);
  return ORC_OK;
}

/* ---- materialize (operators.cpp:60-66) / parallel_materialize
 * (parallel.cpp:87-100), any value width: each worker writes its own span. */
typedef struct {
  int w;
  const uint32_t* fact;
  uint64_t n;
  const void* dim;
  void* out;
} gat_args;

static void gat_worker(void* p, uint32_t t, uint32_t T) {
  gat_args* a = (gat_args*)p;
  uint64_t b, e;
  span_of(a->n, t, T, &b, &e);
  const uint32_t* f = a->fact;
  if (a->w == 8) {
    const uint64_t* dm = (const uint64_t*)a->dim;
    uint64_t* o = (uint64_t*)a->out;
    for (uint64_t k = b; k < e; ++k) o[k] = dm[f[k] - 1];
  } else if (a->w == 4) {
    const uint32_t* dm = (const uint32_t*)a->dim;
    uint32_t* o = (uint32_t*)a->out;
    for (uint64_t k = b; k < e; ++k) o[k] = dm[f[k] - 1];
  } else {
    const uint16_t* dm = (const uint16_t*)a->dim;
    uint16_t* o = (uint16_t*)a->out;
    for (uint64_t k = b; k < e; ++k) o[k] = dm[f[k] - 1];
  }
}

int orc_gather_mt(int width, const uint32_t* fact, uint64_t n, const void* dim, uint64_t dim_len,
                  void* out, uint32_t threads, uint64_t* err_row, uint32_t* err_value) {
  if (width != 2 && width != 4 && width != 8) return ORC_INVALID;
  if (threads == 0) threads = 1;
  DOMAIN_CHECK_MT(fact, n, dim_len, threads);
  gat_args a = {width, fact, n, dim, out};
  run_workers(threads, gat_worker, &a);
  return ORC_OK;
}

/* ---- aggregate_count / aggregate_sum (operators.cpp:100-118), u64 measure:
 * per-worker private count/sum arrays over row spans, folded per key range
 * (the shape of parallel_aggregate's independent strategy, parallel.cpp:
 * 147-160); a key-range scan when private arrays would not fit. ---------- */
typedef struct {
  const uint32_t* fact;
  const uint64_t* measure;
  uint64_t n;
  uint32_t d;
  uint64_t* counts;
  uint64_t* sums;
  uint64_t** pc; /* private arrays (NULL: key-range mode) */
  uint64_t** ps;
  uint32_t T;
} agg_args;

static void agg_private_worker(void* p, uint32_t t, uint32_t T) {
  agg_args* a = (agg_args*)p;
  uint64_t b, e;
  span_of(a->n, t, T, &b, &e);
  uint64_t* c = a->pc[t];
  uint64_t* s = a->ps[t];
  for (uint64_t k = b; k < e; ++k) {
    const uint32_t i = a->fact[k] - 1;
    c[i]++;
    if (a->measure) s[i] += a->measure[k];
  }
}

static void agg_fold_worker(void* p, uint32_t t, uint32_t T) {
  agg_args* a = (agg_args*)p;
  uint64_t lo, hi;
  span_of(a->d, t, T, &lo, &hi);
  for (uint64_t i = lo; i < hi; ++i) {
    uint64_t c = 0, s = 0;
    for (uint32_t u = 0; u < a->T; ++u) {
      c += a->pc[u][i];
      s += a->ps[u][i];
    }
    if (a->counts) a->counts[i] = c;
    if (a->sums) a->sums[i] = a->measure ? s : 0;
  }
}

static void agg_range_worker(void* p, uint32_t t, uint32_t T) {
  agg_args* a = (agg_args*)p;
  uint64_t lo, hi;
  span_of(a->d, t, T, &lo, &hi);
  const uint32_t span = (uint32_t)(hi - lo), base = (uint32_t)lo;
  uint64_t* c = (uint64_t*)calloc(span ? span : 1, sizeof(uint64_t));
  uint64_t* s = (uint64_t*)calloc(span ? span : 1, sizeof(uint64_t));
  for (uint64_t k = 0; k < a->n; ++k) {
    const uint32_t i = a->fact[k] - 1u - base;
    if (i < span) {
      c[i]++;
      if (a->measure) s[i] += a->measure[k];
    }
  }
  if (a->counts) memcpy(a->counts + lo, c, (size_t)span * 8);
  if (a->sums) memcpy(a->sums + lo, s, (size_t)span * 8);
  free(c);
  free(s);
}

int orc_aggregate_count_sum_mt(const uint32_t* fact, const uint64_t* measure, uint64_t n,
                               uint32_t d, uint64_t* counts, uint64_t* sums, uint32_t threads,
                               uint64_t* err_row, uint32_t* err_value) {
  if (threads == 0) threads = 1;
  DOMAIN_CHECK_MT(fact, n, d, threads);
  agg_args a = {fact, measure, n, d, counts, sums, NULL, NULL, threads};
  const uint64_t priv = (uint64_t)d * 16 * threads;
  if (priv <= (uint64_t)8 << 30) {
    a.pc = (uint64_t**)malloc(sizeof(uint64_t*) * threads);
    a.ps = (uint64_t**)malloc(sizeof(uint64_t*) * threads);
    for (uint32_t t = 0; t < threads; ++t) {
      a.pc[t] = (uint64_t*)calloc(d ? d : 1, 8);
      a.ps[t] = (uint64_t*)calloc(d ? d : 1, 8);
    }
    run_workers(threads, agg_private_worker, &a);
    run_workers(threads, agg_fold_worker, &a);
    for (uint32_t t = 0; t < threads; ++t) {
      free(a.pc[t]);
      free(a.ps[t]);
    }
    free(a.pc);
    free(a.ps);
  } else {
    run_workers(threads, agg_range_worker, &a);
  }
  return ORC_OK;
}

/* ---- config 5: select (operators.cpp:87-98) + materialize of four columns
 * over the selected rows (operators.cpp:60-66) + fp64 SUM(price) per
 * category, chunked exactly like parallel_select (parallel.cpp:102-129):
 * per-chunk counts, an exclusive prefix, then each chunk writes its rows at
 * its offset -- the concatenation in chunk order is ascending row order. */
typedef struct {
  const uint32_t* fact;
  uint64_t n;
  const uint64_t* words;
  const int32_t* cat;
  const float* price;
  const uint64_t* supp;
  const uint16_t* flag;
  uint32_t base, ncat;
  uint32_t *o_off;
  int32_t* o_cat;
  float* o_price;
  uint64_t* o_supp;
  uint16_t* o_flag;
  uint64_t* cnt; /* per chunk; then offsets */
  double* part;  /* [T][ncat] */
} sel_args;

static inline int sel_bit(const uint64_t* w, uint32_t idx) { return (int)((w[idx >> 6] >> (idx & 63)) & 1); }

static void sel_count_worker(void* p, uint32_t t, uint32_t T) {
  sel_args* a = (sel_args*)p;
  uint64_t b, e, c = 0;
  span_of(a->n, t, T, &b, &e);
  for (uint64_t k = b; k < e; ++k) c += sel_bit(a->words, a->fact[k] - 1);
  a->cnt[t] = c;
}

static void sel_write_worker(void* p, uint32_t t, uint32_t T) {
  sel_args* a = (sel_args*)p;
  uint64_t b, e;
  span_of(a->n, t, T, &b, &e);
  uint64_t c = a->cnt[t];
  double* ps = a->part + (uint64_t)t * a->ncat;
  for (uint64_t k = b; k < e; ++k) {
    const uint32_t idx = a->fact[k] - 1;
    if (!sel_bit(a->words, idx)) continue;
    a->o_off[c] = a->base + (uint32_t)k;
    a->o_cat[c] = a->cat[idx];
    a->o_price[c] = a->price[idx];
    a->o_supp[c] = a->supp[idx];
    a->o_flag[c] = a->flag[idx];
    if ((uint32_t)a->cat[idx] < a->ncat) ps[a->cat[idx]] += (double)a->price[idx];
    ++c;
  }
}

int orc_select_gather_sum_mt(const uint32_t* fact, uint64_t n, const uint64_t* words, uint32_t d,
                             const int32_t* cat, const float* price, const uint64_t* supp,
                             const uint16_t* flag, uint32_t base, uint32_t n_categories,
                             uint32_t* out_off, int32_t* out_cat, float* out_price,
                             uint64_t* out_supp, uint16_t* out_flag, double* sums,
                             uint64_t* count, uint64_t capacity, uint32_t threads,
                             uint64_t* err_row, uint32_t* err_value) {
  if (n > 0xFFFFFFFFull) return ORC_INVALID; /* operators.cpp:88-90 */
  if (threads == 0) threads = 1;
  DOMAIN_CHECK_MT(fact, n, d, threads);
  sel_args a = {fact, n, words, cat, price, supp, flag, base, n_categories, out_off, out_cat,
                out_price, out_supp, out_flag, NULL, NULL};
  a.cnt = (uint64_t*)malloc(sizeof(uint64_t) * threads);
  a.part = (double*)calloc((uint64_t)threads * (n_categories ? n_categories : 1), sizeof(double));
  run_workers(threads, sel_count_worker, &a);
  uint64_t run = 0;
  for (uint32_t t = 0; t < threads; ++t) {
    const uint64_t c = a.cnt[t];
    a.cnt[t] = run;
    run += c;
  }
  *count = run;
  if (run > capacity) { /* the outputs hold `capacity` rows: nothing written */
    free(a.cnt);
    free(a.part);
    return ORC_INVALID;
  }
  run_workers(threads, sel_write_worker, &a);
  for (uint32_t c = 0; c < n_categories; ++c) {
    double s = 0.0;
    for (uint32_t t = 0; t < threads; ++t) s += a.part[(uint64_t)t * n_categories + c];
    sums[c] = s;
  }
  *count = run;
  free(a.cnt);
  free(a.part);
  return ORC_OK;
}

/* ---- build_bitmap(dim, v < threshold) (operators.hpp:38-45) for int32. */
int orc_build_bitmap_lt_i32(const int32_t* dim, uint64_t d, int32_t threshold, uint64_t* words) {
  memset(words, 0, sizeof(uint64_t) * ((d + 63) / 64));
  for (uint64_t i = 0; i < d; ++i)
    if (dim[i] < threshold) words[i >> 6] |= 1ull << (i & 63);
  return ORC_OK;
}

/* ---- value-column fixtures (the B200 build's skx_fill_column, generate.cu):
 * kind 0 raw splitmix64(seed ^ (0xd1000000 + i)) truncated to width (the
 * reference bench's dimension column, proj/tools/benchcli/dataset.cpp:35-38);
 * kind 1 uniform integer p0 + splitmix64(seed + i*gamma) % p1.  (kind 2, the
 * lognormal price, goes through libm transcendental functions whose last-ulp
 * rounding differs between CUDA and glibc; parity tests take those values
 * from the device as inputs.) */
typedef struct {
  int kind, width;
  uint64_t seed, n;
  double p0, p1;
  void* out;
} fill_args;

static void fill_worker(void* p, uint32_t t, uint32_t T) {
  fill_args* a = (fill_args*)p;
  uint64_t b, e;
  span_of(a->n, t, T, &b, &e);
  for (uint64_t i = b; i < e; ++i) {
    uint64_t v;
    if (a->kind == 0)
      v = orc_splitmix64(a->seed ^ (0xd1000000ull + i));
    else
      v = (uint64_t)(int64_t)a->p0 + orc_splitmix64(a->seed + i * 0x9e3779b97f4a7c15ull) % (uint64_t)a->p1;
    if (a->width == 8)
      ((uint64_t*)a->out)[i] = v;
    else if (a->width == 4)
      ((uint32_t*)a->out)[i] = (uint32_t)v;
    else
      ((uint16_t*)a->out)[i] = (uint16_t)v;
  }
}

int orc_fill_column(int kind, int width, uint64_t seed, uint64_t n, double p0, double p1, void* out,
                    uint32_t threads) {
  if ((kind != 0 && kind != 1) || (width != 2 && width != 4 && width != 8) ||
      (kind == 1 && !(p1 >= 1.0)))
    return ORC_INVALID;
  fill_args a = {kind, width, seed, n, p0, p1, out};
  run_workers(threads ? threads : 1, fill_worker, &a);
  return ORC_OK;
}

// ref_capi.cpp -- extern "C" bridge onto the UNMODIFIED reference library
// (TEST INFRASTRUCTURE).
//
// oracle/Makefile compiles this file together with the reference's own
// sources (read in place from /root/reference/proj/src, never copied) into
// oracle/_ref/libskewdx_ref.so.  Python loads it through oracle/oracle.py to
// (a) generate golden fixtures (tests/golden/make_golden.py), (b) pin the C
// restatement in skx_oracle.c, and (c) time the reference's CPU path as
// bench.py's cpu_baseline / --impl reference arm.  Nothing in the product
// (paper_1910_10063_b200/) links or loads it.
//
// Every entry converts raw pointers into the reference's std::vector types,
// calls the reference API, and maps its exceptions (proj/include/skewdx/
// error.hpp) onto status codes: 0 ok, 1 InvalidArgument, 2 DomainViolation,
// 5 other skewdx::Error.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "skewdx/cachemodel.hpp"
#include "skewdx/column.hpp"
#include "skewdx/error.hpp"
#include "skewdx/kernels.hpp"
#include "skewdx/operators.hpp"
#include "skewdx/parallel.hpp"
#include "skewdx/permindex.hpp"

using namespace skewdx;

namespace {

struct ErrOut {
  std::uint64_t* row;
  std::uint32_t* value;
};

template <typename Fn>
int guarded(ErrOut err, Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const DomainViolation& e) {
    if (err.row) *err.row = e.row();
    if (err.value) *err.value = e.value();
    return 2;
  } catch (const InvalidArgument&) {
    return 1;
  } catch (const Error&) {
    return 5;
  }
}

Column to_col(const std::uint32_t* p, std::uint64_t n) { return Column(p, p + n); }

Bitmap to_bitmap(const std::uint64_t* words, std::uint64_t bits) {
  Bitmap bm(bits);
  for (std::uint64_t i = 0; i < bits; ++i) {
    if ((words[i >> 6] >> (i & 63)) & 1) bm.set(i);
  }
  return bm;
}

double now_ns() {
  return static_cast<double>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                 std::chrono::steady_clock::now().time_since_epoch())
                                 .count());
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

}  // namespace

extern "C" {

unsigned ref_hardware_concurrency() { return std::max(1u, std::thread::hardware_concurrency()); }

int ref_zipf_frequencies(std::uint32_t d, double z, double* out) {
  return guarded({nullptr, nullptr}, [&] {
    const auto f = zipf_frequencies(ZipfSpec{d, 1, z, 0});
    std::memcpy(out, f.data(), f.size() * sizeof(double));
  });
}

int ref_random_bijection(std::uint32_t n, std::uint64_t seed, std::uint32_t* out) {
  const auto m = random_bijection(n, seed);
  std::memcpy(out, m.data(), m.size() * 4);
  return 0;
}

int ref_generate_fact_column(std::uint32_t d, std::uint64_t n, double z, std::uint64_t seed,
                             int layout_freq, std::uint32_t* values, std::uint64_t* counts) {
  return guarded({nullptr, nullptr}, [&] {
    const auto g = generate_fact_column(ZipfSpec{d, n, z, seed},
                                        layout_freq ? Layout::freq : Layout::rand);
    std::memcpy(values, g.values.data(), n * 4);
    if (counts) std::memcpy(counts, g.ground_truth_counts.data(), std::size_t{d} * 8);
  });
}

int ref_count_frequencies(const std::uint32_t* fact, std::uint64_t n, std::uint32_t d,
                          std::uint64_t* counts, std::uint64_t* total, std::uint64_t* err_row,
                          std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    const auto p = count_frequencies(to_col(fact, n), d);
    std::memcpy(counts, p.counts.data(), std::size_t{d} * 8);
    if (total) *total = p.total;
  });
}

int ref_build_index(const std::uint64_t* counts, std::uint32_t d, std::uint64_t total,
                    std::uint32_t* offsets, std::uint32_t* ranks) {
  return guarded({nullptr, nullptr}, [&] {
    FrequencyProfile p;
    p.counts.assign(counts, counts + d);
    p.total = total;
    const auto idx = build_index(p);
    std::memcpy(offsets, idx.offsets.data(), std::size_t{d} * 4);
    std::memcpy(ranks, idx.ranks.data(), std::size_t{d} * 4);
  });
}

int ref_rebuild(const std::uint32_t* fact, std::uint64_t n, std::uint32_t d,
                std::uint32_t* offsets, std::uint32_t* ranks, std::uint64_t* err_row,
                std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    const auto idx = rebuild(to_col(fact, n), d);
    std::memcpy(offsets, idx.offsets.data(), std::size_t{d} * 4);
    std::memcpy(ranks, idx.ranks.data(), std::size_t{d} * 4);
  });
}

int ref_recode_fact(const std::uint32_t* fact, std::uint64_t n, const std::uint32_t* offsets,
                    const std::uint32_t* ranks, std::uint32_t d, std::uint32_t* out,
                    std::uint64_t* err_row, std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    PermutationIndex idx;
    idx.offsets.assign(offsets, offsets + d);
    idx.ranks.assign(ranks, ranks + d);
    const auto r = recode_fact(to_col(fact, n), idx);
    std::memcpy(out, r.data(), n * 4);
  });
}

int ref_permute_dimension(const std::uint32_t* dim, std::uint64_t dim_len,
                          const std::uint32_t* offsets, const std::uint32_t* ranks,
                          std::uint32_t d, std::uint32_t* out) {
  return guarded({nullptr, nullptr}, [&] {
    PermutationIndex idx;
    idx.offsets.assign(offsets, offsets + d);
    idx.ranks.assign(ranks, ranks + d);
    const auto r = permute_dimension(to_col(dim, dim_len), idx);
    std::memcpy(out, r.data(), r.size() * 4);
  });
}

int ref_materialize(const std::uint32_t* fact, std::uint64_t n, const std::uint32_t* dim,
                    std::uint64_t dim_len, std::uint32_t* out, std::uint64_t* err_row,
                    std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    const auto r = materialize(to_col(fact, n), to_col(dim, dim_len));
    std::memcpy(out, r.data(), n * 4);
  });
}

int ref_parallel_materialize(const std::uint32_t* fact, std::uint64_t n, const std::uint32_t* dim,
                             std::uint64_t dim_len, std::uint32_t* out, unsigned threads,
                             std::uint64_t* err_row, std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    ParallelPlan plan;
    plan.threads = threads;
    const auto r = parallel_materialize(to_col(fact, n), to_col(dim, dim_len), plan);
    std::memcpy(out, r.data(), n * 4);
  });
}

int ref_select(const std::uint32_t* fact, std::uint64_t n, const std::uint64_t* words,
               std::uint64_t bits, std::uint32_t* out, std::uint64_t* count,
               unsigned threads, std::uint64_t* err_row, std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    const Bitmap bm = to_bitmap(words, bits);
    std::vector<std::uint32_t> r;
    if (threads <= 1) {
      r = select(to_col(fact, n), bm);
    } else {
      ParallelPlan plan;
      plan.threads = threads;
      r = parallel_select(to_col(fact, n), bm, plan);
    }
    std::memcpy(out, r.data(), r.size() * 4);
    *count = r.size();
  });
}

int ref_permute_bitmap(const std::uint64_t* words, std::uint64_t bits,
                       const std::uint32_t* offsets, const std::uint32_t* ranks,
                       std::uint32_t d, std::uint64_t* out_words) {
  return guarded({nullptr, nullptr}, [&] {
    PermutationIndex idx;
    idx.offsets.assign(offsets, offsets + d);
    idx.ranks.assign(ranks, ranks + d);
    const Bitmap out = permute_bitmap(to_bitmap(words, bits), idx);
    std::memcpy(out_words, out.words(), ((bits + 63) / 64) * 8);
  });
}

int ref_aggregate_count(const std::uint32_t* fact, std::uint64_t n, std::uint32_t d,
                        std::uint64_t* counts, std::uint64_t* err_row, std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    const auto r = aggregate_count(to_col(fact, n), d);
    std::memcpy(counts, r.data(), std::size_t{d} * 8);
  });
}

int ref_aggregate_sum(const std::uint32_t* fact, const std::uint32_t* measure, std::uint64_t n,
                      std::uint64_t measure_len, std::uint32_t d, std::uint64_t* sums,
                      std::uint64_t* err_row, std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    const auto r = aggregate_sum(to_col(fact, n), to_col(measure, measure_len), d);
    std::memcpy(sums, r.data(), std::size_t{d} * 8);
  });
}

// strategy: 0 independent, 1 shared_atomic, 2 hybrid (parallel.hpp:15-19)
int ref_parallel_aggregate(const std::uint32_t* fact, std::uint64_t n, std::uint32_t d,
                           unsigned threads, int strategy, std::uint32_t hot_threshold,
                           std::uint64_t* counts, std::uint64_t* shared_updates,
                           std::uint64_t* err_row, std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    ParallelPlan plan;
    plan.threads = threads;
    plan.strategy = static_cast<AggStrategy>(strategy);
    plan.hot_threshold = hot_threshold;
    AggMetrics m;
    const auto r = parallel_aggregate(to_col(fact, n), d, plan, &m);
    std::memcpy(counts, r.data(), std::size_t{d} * 8);
    if (shared_updates) *shared_updates = m.shared_updates;
  });
}

int ref_heavy_hitter_count(const std::uint32_t* fact, std::uint64_t n, std::uint32_t d,
                           std::uint32_t k, std::uint32_t* ids, std::uint64_t* counts,
                           std::uint64_t* len, int* clamped) {
  return guarded({nullptr, nullptr}, [&] {
    const auto h = heavy_hitter_count(to_col(fact, n), d, k);
    for (std::size_t i = 0; i < h.top.size(); ++i) {
      ids[i] = h.top[i].first;
      counts[i] = h.top[i].second;
    }
    *len = h.top.size();
    *clamped = h.clamped ? 1 : 0;
  });
}

// ---- Timing entries for bench.py's CPU arm (mirror bench.cpp:49-64:
// 1 warm-up + reps timed, median; inputs converted to Columns once, outside
// the timed region).

// Operator-level parallel_materialize (includes the reference's own domain
// scan and output allocation).  Returns median ns; checksum = out[0] ^ out[n-1].
double ref_time_parallel_materialize(const std::uint32_t* fact, std::uint64_t n,
                                     const std::uint32_t* dim, std::uint64_t dim_len,
                                     unsigned threads, int reps) {
  const Column f = to_col(fact, n), dm = to_col(dim, dim_len);
  ParallelPlan plan;
  plan.threads = threads;
  std::vector<double> t;
  for (int r = 0; r <= reps; ++r) {
    const double t0 = now_ns();
    const Column out = parallel_materialize(f, dm, plan);
    const double t1 = now_ns();
    if (r > 0) t.push_back(t1 - t0);
  }
  return median(t);
}

// Kernel-level: the active KernelTable::gather_u32 over chunk_spans with a
// pre-allocated output (SURVEY.md §8d "kernel-only").
double ref_time_gather_kernel(const std::uint32_t* fact, std::uint64_t n,
                              const std::uint32_t* dim, std::uint32_t* out, unsigned threads,
                              int reps) {
  const auto spans = chunk_spans(n, threads);
  const auto& table = kernels::active_kernels();
  std::vector<double> t;
  for (int r = 0; r <= reps; ++r) {
    const double t0 = now_ns();
    std::vector<std::thread> ws;
    for (unsigned i = 0; i + 1 < threads; ++i) {
      ws.emplace_back([&, i] {
        table.gather_u32(fact + spans[i].first, spans[i].second - spans[i].first, dim,
                         out + spans[i].first, 0);
      });
    }
    table.gather_u32(fact + spans[threads - 1].first,
                     spans[threads - 1].second - spans[threads - 1].first, dim,
                     out + spans[threads - 1].first, 0);
    for (auto& w : ws) w.join();
    const double t1 = now_ns();
    if (r > 0) t.push_back(t1 - t0);
  }
  return median(t);
}

double ref_time_parallel_aggregate(const std::uint32_t* fact, std::uint64_t n, std::uint32_t d,
                                   unsigned threads, int strategy, std::uint32_t h, int reps) {
  const Column f = to_col(fact, n);
  ParallelPlan plan;
  plan.threads = threads;
  plan.strategy = static_cast<AggStrategy>(strategy);
  plan.hot_threshold = h;
  std::vector<double> t;
  for (int r = 0; r <= reps; ++r) {
    const double t0 = now_ns();
    const auto out = parallel_aggregate(f, d, plan);
    const double t1 = now_ns();
    if (r > 0) t.push_back(t1 - t0);
  }
  return median(t);
}

double ref_time_rebuild(const std::uint32_t* fact, std::uint64_t n, std::uint32_t d, int reps) {
  const Column f = to_col(fact, n);
  std::vector<double> t;
  for (int r = 0; r <= reps; ++r) {
    const double t0 = now_ns();
    const auto idx = rebuild(f, d);
    const double t1 = now_ns();
    if (r > 0) t.push_back(t1 - t0);
  }
  return median(t);
}

// parallel_select (parallel.cpp:102-129) with the reference's own output
// vectors; median ns over reps after one warm-up.
double ref_time_parallel_select(const std::uint32_t* fact, std::uint64_t n,
                                const std::uint64_t* words, std::uint64_t bits, unsigned threads,
                                int reps, std::uint64_t* selected) {
  const Column f = to_col(fact, n);
  const Bitmap bm = to_bitmap(words, bits);
  ParallelPlan plan;
  plan.threads = threads;
  std::vector<double> t;
  for (int r = 0; r <= reps; ++r) {
    const double t0 = now_ns();
    const auto out = parallel_select(f, bm, plan);
    const double t1 = now_ns();
    if (selected) *selected = out.size();
    if (r > 0) t.push_back(t1 - t0);
  }
  return median(t);
}

// The config-4 index build through the reference's public API, once (no
// warm-up: a sort of D ids takes seconds at D = 2^26): rebuild
// (permindex.cpp:86-88, single thread -- the reference has no parallel index
// build), recode_fact (:60-64) and permute_dimension (:66-73) of an int32
// and a float32 (bit-cast) dimension.  ns[0..3) = rebuild, recode, permutes.
int ref_time_index_build(const std::uint32_t* fact, std::uint64_t n, std::uint32_t d,
                         const std::uint32_t* dim_i, const std::uint32_t* dim_f, double* ns) {
  return guarded({nullptr, nullptr}, [&] {
    const Column f = to_col(fact, n), di = to_col(dim_i, d), df = to_col(dim_f, d);
    const double t0 = now_ns();
    const PermutationIndex idx = rebuild(f, d);
    const double t1 = now_ns();
    const Column r = recode_fact(f, idx);
    const double t2 = now_ns();
    const Column pi = permute_dimension(di, idx);
    const Column pf = permute_dimension(df, idx);
    const double t3 = now_ns();
    ns[0] = t1 - t0;
    ns[1] = t2 - t1;
    ns[2] = t3 - t2;
    if (r.empty() || pi.size() != d || pf.size() != d) throw Error("index build produced nothing");
  });
}

// aggregate_sum (operators.cpp:107-118, single thread: the reference has no
// parallel SUM); median ns over reps after one warm-up.
double ref_time_aggregate_sum(const std::uint32_t* fact, const std::uint32_t* measure,
                              std::uint64_t n, std::uint32_t d, int reps) {
  const Column f = to_col(fact, n), m = to_col(measure, n);
  std::vector<double> t;
  for (int r = 0; r <= reps; ++r) {
    const double t0 = now_ns();
    const auto out = aggregate_sum(f, m, d);
    const double t1 = now_ns();
    if (r > 0) t.push_back(t1 - t0);
  }
  return median(t);
}

// ---- cache model (cachemodel.hpp) ---------------------------------------
int ref_line_frequencies(const double* vf, std::uint32_t d, int layout_freq, std::uint64_t seed,
                         std::uint32_t line_bytes, std::uint32_t element_bytes, double* out) {
  return guarded({nullptr, nullptr}, [&] {
    CacheGeometry g;
    g.lines = 1;
    g.line_bytes = line_bytes;
    g.element_bytes = element_bytes;
    const auto f = line_frequencies(std::span<const double>(vf, d),
                                    layout_freq ? Layout::freq : Layout::rand, g, seed);
    std::memcpy(out, f.data(), f.size() * sizeof(double));
  });
}

int ref_estimate_hit_rate(const double* lf, std::uint64_t nlines, std::uint64_t cache_lines,
                          double* result) {
  return guarded({nullptr, nullptr}, [&] {
    *result = estimate_hit_rate(std::span<const double>(lf, nlines), cache_lines);
  });
}

int ref_simulate_lru(const std::uint32_t* trace, std::uint64_t n, std::uint64_t cache_lines,
                     std::uint64_t* stats) {
  return guarded({nullptr, nullptr}, [&] {
    const auto st = simulate_lru(std::span<const std::uint32_t>(trace, n), cache_lines);
    stats[0] = st.accesses;
    stats[1] = st.hits;
    stats[2] = st.distinct_lines;
  });
}

int ref_trace_from_column(const std::uint32_t* fact, std::uint64_t n, std::uint32_t line_bytes,
                          std::uint32_t element_bytes, std::uint32_t* out, std::uint64_t* err_row,
                          std::uint32_t* err_value) {
  return guarded({err_row, err_value}, [&] {
    CacheGeometry g;
    g.lines = 1;
    g.line_bytes = line_bytes;
    g.element_bytes = element_bytes;
    const auto t = trace_from_column(to_col(fact, n), g);
    std::memcpy(out, t.data(), t.size() * 4);
  });
}

const char* ref_active_kernels_name() { return kernels::active_kernels().name; }

}  // extern "C"

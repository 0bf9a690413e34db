// skewdx_b200.cpp -- the C++ drop-in for the reference library's operator
// API (namespace skewdx; headers in cpp/include/skewdx/), backed by the B200
// kernels through the C-ABI of include/skx.h.
//
// A reference caller keeps its code and links libskewdx_b200.so instead of
// libskewdx.a: every hot-path function stages its host vectors to the
// device, runs the libskx kernel, synchronises, rethrows libskx statuses as
// the reference's exception types (error.hpp) and copies the result back.
// There is no CPU implementation of any hot-path operator here; host code is
// limited to argument validation (same order as the reference), result
// ordering, the generator fixture, file formats and plan arithmetic.
#include <algorithm>
#include <array>
#include <bit>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <random>
#include <string>

#include <unistd.h>

#include "skewdx/column.hpp"
#include "skewdx/column_io.hpp"
#include "skewdx/column_stream.hpp"
#include "skewdx/error.hpp"
#include "skewdx/mix.hpp"
#include "skewdx/operators.hpp"
#include "skewdx/parallel.hpp"
#include "skewdx/permindex.hpp"
#include "skewdx/cachemodel.hpp"
#include "skx.h"

namespace skewdx {
namespace {

// ---- libskx plumbing --------------------------------------------------------
struct Ctx {
  skx_ctx* h = nullptr;
  Ctx() {
    const char* dev = std::getenv("SKX_DEVICE");
    if (skx_ctx_create(dev ? std::atoi(dev) : 0, &h) != SKX_OK || !h)
      throw Error("libskx: no usable sm_100 device (there is no CPU fallback)");
  }
  ~Ctx() { skx_ctx_destroy(h); }
};

skx_ctx* ctx() {
  thread_local Ctx c;
  return c.h;
}

[[noreturn]] void raise(int status) {
  skx_error_info info{};
  skx_last_error(ctx(), &info);
  switch (status) {
    case SKX_DOMAIN_VIOLATION:
      throw DomainViolation(info.row, info.value, info.domain);
    case SKX_INVALID_ARGUMENT:
      throw InvalidArgument(info.message);
    default:
      throw Error(std::string("libskx: ") + info.message);
  }
}

void check(int status) {
  if (status != SKX_OK) raise(status);
}

// Enqueued operator + deferred device errors, reported like the reference.
void run(int status) {
  check(status);
  check(skx_sync(ctx(), nullptr));
}

class DevBuf {
 public:
  explicit DevBuf(std::uint64_t bytes) { check(skx_device_alloc(ctx(), bytes, &p_)); }
  template <typename T>
  explicit DevBuf(const std::vector<T>& v) : DevBuf(v.size() * sizeof(T)) {
    check(skx_copy_to_device(ctx(), p_, v.data(), v.size() * sizeof(T)));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { skx_device_free(ctx(), p_); }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  template <typename T>
  void to(std::vector<T>& v) const {
    check(skx_copy_to_host(ctx(), v.data(), p_, v.size() * sizeof(T)));
  }

 private:
  void* p_ = nullptr;
};

void require_in_domain(const Column& fact, std::uint64_t domain) {
  if (fact.empty()) return;
  DevBuf f(fact);
  std::uint64_t row = ~0ull;
  check(skx_find_domain_violation(ctx(), f.as<std::uint32_t>(), fact.size(), domain, &row));
  if (row != ~0ull) throw DomainViolation(row, fact[row], domain);
}

Column gather(const Column& fact, const Column& dim) {
  Column out(fact.size());
  if (fact.empty()) return out;
  DevBuf f(fact), d(dim), o(out.size() * 4);
  run(skx_gather_u32(ctx(), f.as<std::uint32_t>(), fact.size(), d.as<std::uint32_t>(), dim.size(),
                     o.as<std::uint32_t>(), nullptr));
  o.to(out);
  return out;
}

std::vector<std::uint64_t> device_counts(const Column& fact, std::uint32_t d, std::uint32_t hot) {
  std::vector<std::uint64_t> counts(d, 0);
  if (d == 0) {
    require_in_domain(fact, 0);
    return counts;
  }
  DevBuf f(std::max<std::uint64_t>(fact.size(), 1) * 4), c(std::uint64_t{d} * 8);
  if (!fact.empty()) check(skx_copy_to_device(ctx(), f.as<void>(), fact.data(), fact.size() * 4));
  run(skx_aggregate(ctx(), f.as<std::uint32_t>(), nullptr, 0, fact.size(), d, hot,
                    c.as<std::uint64_t>(), nullptr, nullptr));
  c.to(counts);
  return counts;
}

bool by_count_then_id(const std::pair<std::uint32_t, std::uint64_t>& a,
                      const std::pair<std::uint32_t, std::uint64_t>& b) {
  return a.second != b.second ? a.second > b.second : a.first < b.first;
}

// ---- little-endian container files (SKDX / SKC8 / SKPI) ----------------------
constexpr std::uint32_t kVersion = 1;

template <typename T>
void write_payload(const std::filesystem::path& path, const char (&magic)[5], std::uint64_t count,
                   const T* data, const T* second = nullptr) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw IoError("cannot open for writing: " + path.string());
  f.write(magic, 4);
  f.write(reinterpret_cast<const char*>(&kVersion), 4);
  f.write(reinterpret_cast<const char*>(&count), 8);
  f.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(count * sizeof(T)));
  if (second)
    f.write(reinterpret_cast<const char*>(second), static_cast<std::streamsize>(count * sizeof(T)));
  if (!f) throw IoError("write failed: " + path.string());
}

std::uint64_t read_header(std::ifstream& f, const std::filesystem::path& path,
                          const char (&magic)[5]) {
  char m[4] = {};
  std::uint32_t version = 0;
  std::uint64_t count = 0;
  f.read(m, 4);
  f.read(reinterpret_cast<char*>(&version), 4);
  f.read(reinterpret_cast<char*>(&count), 8);
  if (!f) throw FormatError("truncated header: " + path.string());
  if (std::memcmp(m, magic, 4) != 0) throw FormatError("bad magic in " + path.string());
  if (version != kVersion)
    throw FormatError("unsupported format version " + std::to_string(version) + " in " +
                      path.string());
  return count;
}

template <typename T>
std::vector<T> read_payload(const std::filesystem::path& path, const char (&magic)[5]) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot open for reading: " + path.string());
  const std::uint64_t count = read_header(f, path, magic);
  const auto here = f.tellg();
  f.seekg(0, std::ios::end);
  const auto bytes = static_cast<std::uint64_t>(f.tellg() - here);
  if (bytes != count * sizeof(T)) throw FormatError("length mismatch against header in " + path.string());
  f.seekg(here);
  std::vector<T> v(count);
  f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(bytes));
  if (!f && count) throw FormatError("length mismatch against header in " + path.string());
  return v;
}

}  // namespace

// ---- column.hpp ---------------------------------------------------------------
const char* to_string(Layout layout) noexcept { return layout == Layout::freq ? "freq" : "rand"; }

static void validate_spec(const ZipfSpec& s) {
  if (s.domain_cardinality == 0) throw InvalidArgument("zipf spec: domain cardinality must be at least 1");
  if (s.domain_cardinality > kMaxDomainCardinality)
    throw InvalidArgument("zipf spec: domain cardinality exceeds the 32-bit identifier space");
  if (s.tuple_count == 0) throw InvalidArgument("zipf spec: tuple count must be at least 1");
  if (!(s.z >= 0.0)) throw InvalidArgument("zipf spec: exponent must be non-negative");
}

std::vector<double> zipf_frequencies(const ZipfSpec& spec) {
  validate_spec(spec);
  std::vector<double> cdf(spec.domain_cardinality);
  // skx_zipf_cdf_host returns the partial sums; undo them into frequencies is
  // lossy, so restate the Kahan-normalised weights directly (column.cpp:44-60).
  double sum = 0.0, comp = 0.0;
  for (std::uint32_t r = 1; r <= spec.domain_cardinality; ++r) {
    const double w = std::pow(static_cast<double>(r), -spec.z);
    cdf[r - 1] = w;
    const double y = w - comp, t = sum + y;
    comp = (t - sum) - y;
    sum = t;
  }
  for (double& x : cdf) x /= sum;
  return cdf;
}

std::vector<std::uint32_t> random_bijection(std::uint32_t n, std::uint64_t seed) {
  std::vector<std::uint32_t> map(n);
  if (n) check(skx_random_bijection_host(n, seed, map.data()));
  return map;
}

GeneratedColumn generate_fact_column(const ZipfSpec& spec, Layout layout) {
  validate_spec(spec);
  const std::uint32_t d = spec.domain_cardinality;
  std::vector<double> cdf(d);
  check(skx_zipf_cdf_host(d, spec.z, cdf.data()));
  // Sequential draws exactly as column.cpp:85-95 (mt19937_64 stream).
  std::mt19937_64 rng(splitmix64(spec.seed ^ 0x5ca1ab1eull));
  std::vector<std::uint32_t> drawn(spec.tuple_count);
  std::vector<std::uint64_t> per_rank(d, 0);
  for (auto& r : drawn) {
    const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
    std::uint32_t rank = static_cast<std::uint32_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    if (rank >= d) rank = d - 1;
    r = rank;
    ++per_rank[rank];
  }
  std::vector<std::uint32_t> rank_to_id;
  if (layout == Layout::rand) {
    rank_to_id = random_bijection(d, spec.seed);
  } else {
    std::vector<std::uint32_t> order(d);
    std::iota(order.begin(), order.end(), 0u);
    std::sort(order.begin(), order.end(), [&](std::uint32_t a, std::uint32_t b) {
      return per_rank[a] != per_rank[b] ? per_rank[a] > per_rank[b] : a < b;
    });
    rank_to_id.resize(d);
    for (std::uint32_t pos = 0; pos < d; ++pos) rank_to_id[order[pos]] = pos + 1;
  }
  GeneratedColumn g;
  g.values.resize(spec.tuple_count);
  g.ground_truth_counts.assign(d, 0);
  for (std::uint64_t k = 0; k < spec.tuple_count; ++k) g.values[k] = rank_to_id[drawn[k]];
  for (std::uint32_t r = 0; r < d; ++r) g.ground_truth_counts[rank_to_id[r] - 1] = per_rank[r];
  return g;
}

// ---- column_io.hpp ----------------------------------------------------------
void write_column(const std::filesystem::path& path, const Column& column) {
  write_payload(path, "SKDX", column.size(), column.data());
}
Column read_column(const std::filesystem::path& path) {
  return read_payload<std::uint32_t>(path, "SKDX");
}
void write_u64_array(const std::filesystem::path& path, std::span<const std::uint64_t> values) {
  write_payload(path, "SKC8", values.size(), values.data());
}
std::vector<std::uint64_t> read_u64_array(const std::filesystem::path& path) {
  return read_payload<std::uint64_t>(path, "SKC8");
}

// ---- permindex.hpp (GPU) -------------------------------------------------------
FrequencyProfile count_frequencies(const Column& fact, std::uint32_t domain_cardinality) {
  FrequencyProfile p;
  p.total = fact.size();
  p.counts.assign(domain_cardinality, 0);
  if (fact.empty()) return p;
  DevBuf f(fact), c(std::max<std::uint64_t>(domain_cardinality, 1) * 8);
  run(skx_count_frequencies(ctx(), f.as<std::uint32_t>(), fact.size(), domain_cardinality,
                            c.as<std::uint64_t>(), nullptr));
  c.to(p.counts);
  return p;
}

PermutationIndex build_index(const FrequencyProfile& profile) {
  if (profile.counts.size() > kMaxDomainCardinality)
    throw InvalidArgument("frequency profile exceeds the 32-bit identifier space");
  const std::uint32_t d = static_cast<std::uint32_t>(profile.counts.size());
  PermutationIndex idx;
  idx.offsets.resize(d);
  idx.ranks.resize(d);
  DevBuf c(std::max<std::uint64_t>(d, 1) * 8), off(std::max<std::uint64_t>(d, 1) * 4),
      rk(std::max<std::uint64_t>(d, 1) * 4);
  if (d) check(skx_copy_to_device(ctx(), c.as<void>(), profile.counts.data(), std::uint64_t{d} * 8));
  run(skx_build_index(ctx(), c.as<std::uint64_t>(), d, profile.total, off.as<std::uint32_t>(),
                      rk.as<std::uint32_t>(), nullptr));
  off.to(idx.offsets);
  rk.to(idx.ranks);
  return idx;
}

PermutationIndex rebuild(const Column& fact, std::uint32_t domain_cardinality) {
  const std::uint32_t d = domain_cardinality;
  PermutationIndex idx;
  idx.offsets.resize(d);
  idx.ranks.resize(d);
  DevBuf f(std::max<std::uint64_t>(fact.size(), 1) * 4), off(std::max<std::uint64_t>(d, 1) * 4),
      rk(std::max<std::uint64_t>(d, 1) * 4);
  if (!fact.empty()) check(skx_copy_to_device(ctx(), f.as<void>(), fact.data(), fact.size() * 4));
  run(skx_rebuild(ctx(), f.as<std::uint32_t>(), fact.size(), d, off.as<std::uint32_t>(),
                  rk.as<std::uint32_t>(), nullptr));
  off.to(idx.offsets);
  rk.to(idx.ranks);
  return idx;
}

Column recode_fact(const Column& fact, const PermutationIndex& index) {
  return materialize(fact, index.ranks);  // permindex.cpp:60-64
}

Column permute_dimension(const Column& dim, const PermutationIndex& index) {
  if (dim.size() != index.offsets.size())
    throw InvalidArgument("dimension length " + std::to_string(dim.size()) +
                          " does not match index cardinality " +
                          std::to_string(index.offsets.size()));
  Column out(dim.size());
  if (dim.empty()) return out;
  DevBuf dm(dim), off(index.offsets), o(dim.size() * 4);
  run(skx_permute_dimension_u32(ctx(), dm.as<std::uint32_t>(), dim.size(), off.as<std::uint32_t>(),
                                index.domain_cardinality(), o.as<std::uint32_t>(), nullptr));
  o.to(out);
  return out;
}

std::uint32_t append_dimension_row(PermutationIndex& index) {
  const std::uint32_t d = index.domain_cardinality();
  if (d >= kMaxDomainCardinality) throw Error("identifier space exhausted");
  index.offsets.push_back(d + 1);  // least-frequent item: rank == id
  index.ranks.push_back(d + 1);
  return d + 1;
}

void write_index(const std::filesystem::path& path, const PermutationIndex& index) {
  write_payload(path, "SKPI", index.offsets.size(), index.offsets.data(), index.ranks.data());
}

PermutationIndex read_index(const std::filesystem::path& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot open for reading: " + path.string());
  const std::uint64_t d = read_header(f, path, "SKPI");
  if (d > kMaxDomainCardinality) throw FormatError("index cardinality out of range in " + path.string());
  PermutationIndex idx;
  idx.offsets.resize(d);
  idx.ranks.resize(d);
  f.read(reinterpret_cast<char*>(idx.offsets.data()), static_cast<std::streamsize>(d * 4));
  f.read(reinterpret_cast<char*>(idx.ranks.data()), static_cast<std::streamsize>(d * 4));
  if (!f && d) throw FormatError("length mismatch against header in " + path.string());
  for (std::uint64_t r = 0; r < d; ++r) {
    const std::uint32_t id = idx.offsets[r];
    if (id == 0 || id > d || idx.ranks[id - 1] != r + 1)
      throw FormatError("offsets/ranks are not inverse bijections in " + path.string());
  }
  return idx;
}

// ---- operators.hpp (GPU) -------------------------------------------------------
std::uint64_t Bitmap::count() const noexcept {
  std::uint64_t c = 0;
  for (const std::uint64_t w : words_) c += static_cast<std::uint64_t>(std::popcount(w));
  return c;
}

Bitmap permute_bitmap(const Bitmap& bitmap, const PermutationIndex& index) {
  if (bitmap.size() != index.offsets.size())
    throw InvalidArgument("bitmap size does not match index cardinality");
  Bitmap out(bitmap.size());
  if (bitmap.size() == 0) return out;
  const std::uint64_t nw = (bitmap.size() + 63) / 64;
  DevBuf in(nw * 8), off(index.offsets), o(nw * 8);
  check(skx_copy_to_device(ctx(), in.as<void>(), bitmap.words(), nw * 8));
  run(skx_permute_bitmap(ctx(), in.as<std::uint64_t>(), bitmap.size(), off.as<std::uint32_t>(),
                         index.domain_cardinality(), o.as<std::uint64_t>(), nullptr));
  check(skx_copy_to_host(ctx(), out.mutable_words(), o.as<void>(), nw * 8));
  return out;
}

std::size_t find_domain_violation(const Column& fact, std::uint64_t domain_cardinality) noexcept {
  if (fact.empty()) return knpos;
  DevBuf f(fact);
  std::uint64_t row = ~0ull;
  if (skx_find_domain_violation(ctx(), f.as<std::uint32_t>(), fact.size(), domain_cardinality,
                                &row) != SKX_OK) {
    std::fprintf(stderr, "skewdx_b200: find_domain_violation failed on the device\n");
    std::abort();  // noexcept contract; no CPU fallback
  }
  return row == ~0ull ? knpos : static_cast<std::size_t>(row);
}

Column materialize(const Column& fact, const Column& dim, int /*prefetch_distance*/) {
  return gather(fact, dim);
}

Column materialize_split(const Column& fact, const Column& dim, SplitThreshold threshold) {
  // operators.cpp:68-85 on the device: pass 1 gathers ids <= t and queues the
  // rest, pass 2 patches them (skx_gather_split_u32).
  if (threshold.t == 0 || threshold.t > dim.size())
    throw InvalidArgument("split threshold must lie in 1..D");
  Column out(fact.size());
  if (fact.empty()) return out;
  DevBuf f(fact), d(dim), o(out.size() * 4);
  run(skx_gather_split_u32(ctx(), f.as<std::uint32_t>(), fact.size(), d.as<std::uint32_t>(),
                           dim.size(), threshold.t, o.as<std::uint32_t>(), nullptr));
  o.to(out);
  return out;
}

std::vector<std::uint32_t> select(const Column& fact, const Bitmap& bitmap) {
  if (fact.size() > 0xFFFFFFFFull) throw InvalidArgument("select: fact row offsets exceed 32 bits");
  if (fact.empty()) return {};
  const std::uint64_t nw = std::max<std::uint64_t>((bitmap.size() + 63) / 64, 1);
  DevBuf f(fact), w(nw * 8), o(fact.size() * 4), cnt(8);
  if (bitmap.size()) check(skx_copy_to_device(ctx(), w.as<void>(), bitmap.words(), ((bitmap.size() + 63) / 64) * 8));
  run(skx_select_offsets(ctx(), f.as<std::uint32_t>(), fact.size(), w.as<std::uint64_t>(),
                         bitmap.size(), 0, o.as<std::uint32_t>(), cnt.as<std::uint64_t>(), nullptr));
  std::uint64_t n = 0;
  check(skx_copy_to_host(ctx(), &n, cnt.as<void>(), 8));
  std::vector<std::uint32_t> out(n);
  if (n) check(skx_copy_to_host(ctx(), out.data(), o.as<void>(), n * 4));
  return out;
}

std::vector<std::uint64_t> aggregate_count(const Column& fact, std::uint32_t domain_cardinality) {
  return device_counts(fact, domain_cardinality, 0);
}

std::vector<std::uint64_t> aggregate_sum(const Column& fact, const Column& measure,
                                         std::uint32_t domain_cardinality) {
  if (measure.size() != fact.size())
    throw InvalidArgument("aggregate_sum: measure length does not match fact length");
  std::vector<std::uint64_t> sums(domain_cardinality, 0);
  if (domain_cardinality == 0) {
    require_in_domain(fact, 0);
    return sums;
  }
  const std::uint64_t rows = std::max<std::uint64_t>(fact.size(), 1);
  DevBuf f(rows * 4), m(rows * 4), s(std::uint64_t{domain_cardinality} * 8);
  if (!fact.empty()) {
    check(skx_copy_to_device(ctx(), f.as<void>(), fact.data(), fact.size() * 4));
    check(skx_copy_to_device(ctx(), m.as<void>(), measure.data(), measure.size() * 4));
  }
  run(skx_aggregate(ctx(), f.as<std::uint32_t>(), m.as<void>(), 4, fact.size(), domain_cardinality,
                    0, nullptr, s.as<std::uint64_t>(), nullptr));
  s.to(sums);
  return sums;
}

AggState::AggState(std::uint32_t domain_cardinality, std::uint32_t hot_threshold_,
                   std::uint32_t lanes_)
    : main(domain_cardinality, 0), hot_threshold(hot_threshold_), lanes(lanes_) {
  if (hot_threshold == 0 || hot_threshold > domain_cardinality)
    throw InvalidArgument("lane-copy hot threshold must lie in 1..D");
  if (lanes == 0) throw InvalidArgument("lane count must be at least 1");
  hot.assign(static_cast<std::size_t>(hot_threshold) * lanes, 0);
}

void AggState::finalize() {
  for (std::uint32_t l = 0; l < lanes; ++l)
    for (std::uint32_t r = 0; r < hot_threshold; ++r)
      main[r] += hot[static_cast<std::size_t>(l) * hot_threshold + r];
  std::fill(hot.begin(), hot.end(), 0);
}

std::vector<std::uint64_t> aggregate_count_lanecopy(const Column& fact,
                                                    std::uint32_t domain_cardinality,
                                                    std::uint32_t hot_threshold,
                                                    std::uint32_t lanes) {
  require_in_domain(fact, domain_cardinality);
  const AggState validate(domain_cardinality, hot_threshold, lanes);  // same checks as the reference
  (void)validate;
  return device_counts(fact, domain_cardinality, hot_threshold);
}

HeavyHitters heavy_hitter_count(const Column& fact, std::uint32_t domain_cardinality,
                                std::uint32_t k, bool /*branchy*/) {
  if (k == 0) throw InvalidArgument("heavy_hitter_count: k must be at least 1");
  const std::uint32_t cutoff = std::min(k, domain_cardinality);
  std::vector<std::uint64_t> counts(cutoff, 0);
  DevBuf f(std::max<std::uint64_t>(fact.size(), 1) * 4), c(std::max<std::uint64_t>(cutoff, 1) * 8);
  if (!fact.empty()) check(skx_copy_to_device(ctx(), f.as<void>(), fact.data(), fact.size() * 4));
  run(skx_heavy_hitter_count(ctx(), f.as<std::uint32_t>(), fact.size(), domain_cardinality, k,
                             c.as<std::uint64_t>(), nullptr));
  c.to(counts);
  HeavyHitters h;
  h.clamped = k > domain_cardinality;
  for (std::uint32_t i = 0; i < cutoff; ++i) h.top.emplace_back(i + 1, counts[i]);
  std::sort(h.top.begin(), h.top.end(), by_count_then_id);
  return h;
}

HeavyHitters top_k_by_full_aggregation(const Column& fact, std::uint32_t domain_cardinality,
                                       std::uint32_t k) {
  if (k == 0) throw InvalidArgument("top_k_by_full_aggregation: k must be at least 1");
  const std::uint32_t cutoff = std::min(k, domain_cardinality);
  const auto counts = aggregate_count(fact, domain_cardinality);
  HeavyHitters h;
  h.clamped = k > domain_cardinality;
  h.top.reserve(domain_cardinality);
  for (std::uint32_t i = 0; i < domain_cardinality; ++i) h.top.emplace_back(i + 1, counts[i]);
  std::partial_sort(h.top.begin(), h.top.begin() + cutoff, h.top.end(), by_count_then_id);
  h.top.resize(cutoff);
  return h;
}

// ---- parallel.hpp ---------------------------------------------------------------
const char* to_string(AggStrategy s) noexcept {
  switch (s) {
    case AggStrategy::independent: return "independent";
    case AggStrategy::shared_atomic: return "shared_atomic";
    case AggStrategy::hybrid: return "hybrid";
  }
  return "?";
}

std::vector<std::pair<std::size_t, std::size_t>> chunk_spans(std::size_t n, unsigned threads) {
  if (threads == 0) throw InvalidArgument("thread count must be at least 1");
  std::vector<std::pair<std::size_t, std::size_t>> spans;
  spans.reserve(threads);
  const std::size_t q = n / threads, r = n % threads;
  std::size_t b = 0;
  for (unsigned t = 0; t < threads; ++t) {
    const std::size_t e = b + q + (t < r ? 1 : 0);
    spans.emplace_back(b, e);
    b = e;
  }
  return spans;
}

Column parallel_materialize(const Column& fact, const Column& dim, const ParallelPlan& plan) {
  Column out = gather(fact, dim);  // domain check first, as parallel.cpp:88-89
  chunk_spans(fact.size(), plan.threads);
  return out;
}

std::vector<std::uint32_t> parallel_select(const Column& fact, const Bitmap& bitmap,
                                           const ParallelPlan& plan) {
  auto out = select(fact, bitmap);
  chunk_spans(fact.size(), plan.threads);
  return out;
}

std::vector<std::uint64_t> parallel_aggregate(const Column& fact, std::uint32_t domain_cardinality,
                                              const ParallelPlan& plan, AggMetrics* metrics) {
  const bool hybrid = plan.strategy == AggStrategy::hybrid;
  if (hybrid && (plan.hot_threshold == 0 || plan.hot_threshold > domain_cardinality))
    throw InvalidArgument("hybrid hot threshold must lie in 1..D");
  auto counts = device_counts(fact, domain_cardinality, hybrid ? plan.hot_threshold : 0);
  chunk_spans(fact.size(), plan.threads);
  if (metrics) {
    metrics->total_updates = fact.size();
    std::uint64_t shared = 0;
    if (plan.strategy == AggStrategy::shared_atomic) {
      shared = fact.size();
    } else if (hybrid) {
      // rows whose id > h are the ones the reference routes to shared atomics
      shared = fact.size() - std::accumulate(counts.begin(), counts.begin() + plan.hot_threshold,
                                             std::uint64_t{0});
    }
    metrics->shared_updates = shared;
    metrics->accumulator_bytes = memory_footprint(plan, domain_cardinality);
  }
  return counts;
}

std::uint64_t memory_footprint(const ParallelPlan& plan, std::uint64_t domain_cardinality) {
  if (plan.threads == 0) throw InvalidArgument("thread count must be at least 1");
  switch (plan.strategy) {
    case AggStrategy::independent: return std::uint64_t{plan.threads} * domain_cardinality * 8;
    case AggStrategy::shared_atomic: return domain_cardinality * 8;
    case AggStrategy::hybrid:
      return domain_cardinality * 8 + std::uint64_t{plan.threads} * plan.hot_threshold * 8;
  }
  return 0;
}

// ---- cache model (cachemodel.hpp) -------------------------------------------
void validate(const CacheGeometry& geometry) {
  if (geometry.lines == 0) throw InvalidArgument("cache geometry: line count must be at least 1");
  if (geometry.element_bytes == 0 || geometry.line_bytes == 0 ||
      geometry.line_bytes % geometry.element_bytes != 0)
    throw InvalidArgument("cache geometry: line bytes must be a multiple of element bytes");
}

std::vector<double> line_frequencies(std::span<const double> value_freqs, Layout layout,
                                     const CacheGeometry& geometry, std::uint64_t seed) {
  validate(geometry);
  if (value_freqs.empty()) throw InvalidArgument("line_frequencies: empty frequency vector");
  const auto d = static_cast<std::uint32_t>(value_freqs.size());
  const std::uint32_t per = geometry.elements_per_line();
  std::vector<double> out((value_freqs.size() + per - 1) / per);
  DevBuf vf(std::vector<double>(value_freqs.begin(), value_freqs.end())), o(out.size() * 8);
  if (layout == Layout::freq) {
    run(skx_line_frequencies(ctx(), vf.as<double>(), d, nullptr, per, o.as<double>(), nullptr));
  } else {
    DevBuf map(random_bijection(d, seed));
    run(skx_line_frequencies(ctx(), vf.as<double>(), d, map.as<std::uint32_t>(), per,
                             o.as<double>(), nullptr));
  }
  o.to(out);
  return out;
}

double estimate_hit_rate(std::span<const double> line_freqs, std::uint64_t cache_lines) {
  if (cache_lines == 0) throw InvalidArgument("estimate_hit_rate: cache must have at least 1 line");
  if (line_freqs.empty()) return 1.0;
  DevBuf lf(std::vector<double>(line_freqs.begin(), line_freqs.end())), r(8);
  run(skx_estimate_hit_rate(ctx(), lf.as<double>(), line_freqs.size(), cache_lines, r.as<double>(),
                            nullptr));
  std::vector<double> v(1);
  r.to(v);
  return v[0];
}

LruStats simulate_lru(std::span<const std::uint32_t> trace, std::uint64_t cache_lines) {
  if (cache_lines == 0) throw InvalidArgument("simulate_lru: cache must have at least 1 line");
  std::uint64_t st[3] = {0, 0, 0};
  check(skx_simulate_lru_host(trace.data(), trace.size(), cache_lines, st));
  LruStats s;
  s.accesses = st[0];
  s.hits = st[1];
  s.distinct_lines = st[2];
  return s;
}

std::vector<std::uint32_t> trace_from_column(const Column& fact, const CacheGeometry& geometry) {
  validate(geometry);
  std::vector<std::uint32_t> out(fact.size());
  if (fact.empty()) return out;
  DevBuf f(fact), o(fact.size() * 4);
  run(skx_trace_from_column(ctx(), f.as<std::uint32_t>(), fact.size(), geometry.elements_per_line(),
                            o.as<std::uint32_t>(), nullptr));
  o.to(out);
  return out;
}


// ---- column_stream.hpp (B200 extension: streamed SKDX files) ----------------
namespace {

std::uint64_t g_chunk_rows = [] {
  const char* e = std::getenv("SKX_STREAM_CHUNK_ROWS");
  const unsigned long long v = e ? std::strtoull(e, nullptr, 10) : 0ull;
  return v ? static_cast<std::uint64_t>(v) : (std::uint64_t{1} << 24);
}();

class Pinned {
 public:
  explicit Pinned(std::uint64_t bytes) { check(skx_pinned_alloc(ctx(), bytes, &p_)); }
  Pinned(const Pinned&) = delete;
  Pinned& operator=(const Pinned&) = delete;
  ~Pinned() { skx_pinned_free(ctx(), p_); }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }

 private:
  void* p_ = nullptr;
};

// SKDX payload read in chunks; the header and the payload length are checked
// up front exactly as read_column does.
class SkdxReader {
 public:
  explicit SkdxReader(const std::filesystem::path& path) : f_(path, std::ios::binary), path_(path) {
    if (!f_) throw IoError("cannot open for reading: " + path.string());
    n_ = read_header(f_, path, "SKDX");
    const auto here = f_.tellg();
    f_.seekg(0, std::ios::end);
    const auto bytes = static_cast<std::uint64_t>(f_.tellg() - here);
    if (bytes != n_ * 4) throw FormatError("length mismatch against header in " + path.string());
    payload_ = here;
    f_.seekg(payload_);
  }
  std::uint64_t size() const { return n_; }
  void read(std::uint32_t* dst, std::uint64_t rows) {
    f_.read(reinterpret_cast<char*>(dst), static_cast<std::streamsize>(rows * 4));
    if (!f_) throw FormatError("length mismatch against header in " + path_.string());
  }
  void rewind() {
    f_.clear();
    f_.seekg(payload_);
  }

 private:
  std::ifstream f_;
  std::filesystem::path path_;
  std::uint64_t n_ = 0;
  std::streampos payload_{};
};

// Streams the payload into a temporary file next to out_path and renames it
// over out_path only in finish(), so an in-place apply (--fact-out == --fact)
// reads the whole input before the output replaces it -- as the reference's
// write_column(out, recode_fact(read_column(in))) does -- and any failure
// (exception, domain violation) leaves out_path untouched: the destructor
// removes an unfinished temporary.
class SkdxWriter {
 public:
  SkdxWriter(const std::filesystem::path& path, std::uint64_t n)
      : path_(path),
        tmp_(path.string() + ".tmp." + std::to_string(static_cast<long long>(::getpid()))),
        n_(n) {
    f_.open(tmp_, std::ios::binary | std::ios::trunc);
    if (!f_) throw IoError("cannot open for writing: " + path.string());
    f_.write("SKDX", 4);
    f_.write(reinterpret_cast<const char*>(&kVersion), 4);
    f_.write(reinterpret_cast<const char*>(&n), 8);
  }
  SkdxWriter(const SkdxWriter&) = delete;
  SkdxWriter& operator=(const SkdxWriter&) = delete;
  ~SkdxWriter() {
    if (!done_) abandon();
  }
  void write(const std::uint32_t* src, std::uint64_t rows) {
    f_.write(reinterpret_cast<const char*>(src), static_cast<std::streamsize>(rows * 4));
    written_ += rows;
  }
  void finish() {
    f_.flush();
    if (!f_ || written_ != n_) throw IoError("write failed: " + path_.string());
    f_.close();
    std::error_code ec;
    std::filesystem::rename(tmp_, path_, ec);
    if (ec) throw IoError("cannot replace " + path_.string() + ": " + ec.message());
    done_ = true;
  }
  void abandon() {
    if (f_.is_open()) f_.close();
    std::error_code ec;
    std::filesystem::remove(tmp_, ec);
    done_ = true;
  }

 private:
  std::ofstream f_;
  std::filesystem::path path_, tmp_;
  std::uint64_t n_, written_ = 0;
  bool done_ = false;
};

// After the device reported a violation somewhere in the stream: the first
// offending row, found on the host as find_domain_violation reports it
// (cold path only).
[[noreturn]] void throw_first_violation(const std::filesystem::path& path, std::uint64_t d) {
  SkdxReader rd(path);
  std::vector<std::uint32_t> buf(std::min<std::uint64_t>(g_chunk_rows, std::max<std::uint64_t>(rd.size(), 1)));
  for (std::uint64_t b = 0; b < rd.size(); b += buf.size()) {
    const std::uint64_t m = std::min<std::uint64_t>(buf.size(), rd.size() - b);
    rd.read(buf.data(), m);
    for (std::uint64_t k = 0; k < m; ++k)
      if (static_cast<std::uint32_t>(buf[k] - 1u) >= d) throw DomainViolation(b + k, buf[k], d);
  }
  throw Error("libskx: device reported a domain violation the host scan did not find");
}

// Two chunks in flight on the context's two host streams.
struct StreamSlots {
  void* st[2] = {skx_ctx_stream(ctx(), 0), skx_ctx_stream(ctx(), 1)};
  bool pending[2] = {false, false};
  bool violation = false;
  // Waits for slot s; a device-side domain violation is remembered (the host
  // scan finds the first row afterwards), anything else throws.
  void drain(int s) {
    if (!pending[s]) return;
    pending[s] = false;
    const int rc = skx_sync(ctx(), st[s]);
    if (rc == SKX_DOMAIN_VIOLATION)
      violation = true;
    else
      check(rc);
  }
};

}  // namespace

void set_stream_chunk_rows(std::uint64_t rows) { g_chunk_rows = rows ? rows : 1; }
std::uint64_t stream_chunk_rows() { return g_chunk_rows; }

PermutationIndex rebuild_file(const std::filesystem::path& fact_path, std::uint32_t d,
                              std::uint32_t* d_used) {
  SkdxReader rd(fact_path);
  const std::uint64_t n = rd.size();
  const std::uint64_t chunk = std::min<std::uint64_t>(g_chunk_rows, std::max<std::uint64_t>(n, 1));
  if (d == 0 && n > 0) {  // D = the largest identifier (generate.cpp:56), a host pass
    std::vector<std::uint32_t> buf(chunk);
    std::uint32_t mx = 0;
    for (std::uint64_t b = 0; b < n; b += chunk) {
      const std::uint64_t m = std::min(chunk, n - b);
      rd.read(buf.data(), m);
      mx = std::max(mx, *std::max_element(buf.begin(), buf.begin() + static_cast<std::ptrdiff_t>(m)));
    }
    d = mx;
    rd.rewind();
  }
  if (d_used) *d_used = d;
  // Empty columns, an empty domain and > 2^32 - 1 rows (u64 counters) take
  // the in-memory path.
  if (n == 0 || d == 0 || n > 0xFFFFFFFFull) return rebuild(read_column(fact_path), d);
  DevBuf counts(std::uint64_t{d} * 4), off(std::uint64_t{d} * 4), rk(std::uint64_t{d} * 4);
  {
    Pinned pin0(chunk * 4), pin1(chunk * 4);
    DevBuf dev0(chunk * 4), dev1(chunk * 4);
    Pinned* pin[2] = {&pin0, &pin1};
    DevBuf* dev[2] = {&dev0, &dev1};
    StreamSlots ss;
    std::uint64_t i = 0;
    for (std::uint64_t b = 0; b < n && !ss.violation; b += chunk, ++i) {
      const int s = static_cast<int>(i & 1);
      const std::uint64_t m = std::min(chunk, n - b);
      ss.drain(s);  // its buffers are free again
      rd.read(pin[s]->as<std::uint32_t>(), m);
      check(skx_copy_to_device_async(ctx(), dev[s]->as<void>(), pin[s]->as<void>(), m * 4, ss.st[s]));
      // the first chunk overwrites the counters; the rest add to them, both
      // streams' atomics landing in the same array
      check(skx_histogram_u32(ctx(), dev[s]->as<std::uint32_t>(), m, d, counts.as<std::uint32_t>(),
                              i == 0 ? 0 : 1, ss.st[s]));
      ss.pending[s] = true;
      if (i == 0) ss.drain(0);  // counters initialised before stream 1 adds
    }
    ss.drain(static_cast<int>(i & 1));
    ss.drain(static_cast<int>((i + 1) & 1));
    if (ss.violation) throw_first_violation(fact_path, d);
  }
  run(skx_build_index_u32(ctx(), counts.as<std::uint32_t>(), d, n, off.as<std::uint32_t>(),
                          rk.as<std::uint32_t>(), nullptr));
  PermutationIndex idx;
  idx.offsets.resize(d);
  idx.ranks.resize(d);
  off.to(idx.offsets);
  rk.to(idx.ranks);
  return idx;
}

void recode_file(const std::filesystem::path& in_path, const std::filesystem::path& out_path,
                 const PermutationIndex& index) {
  SkdxReader rd(in_path);
  const std::uint64_t n = rd.size();
  const std::uint32_t d = index.domain_cardinality();
  if (n == 0 || d == 0) {
    write_column(out_path, recode_fact(read_column(in_path), index));
    return;
  }
  const std::uint64_t chunk = std::min<std::uint64_t>(g_chunk_rows, n);
  DevBuf ranks(index.ranks);
  Pinned pin_in0(chunk * 4), pin_in1(chunk * 4), pin_out0(chunk * 4), pin_out1(chunk * 4);
  DevBuf dev_in0(chunk * 4), dev_in1(chunk * 4), dev_out0(chunk * 4), dev_out1(chunk * 4);
  Pinned* pin_in[2] = {&pin_in0, &pin_in1};
  Pinned* pin_out[2] = {&pin_out0, &pin_out1};
  DevBuf* dev_in[2] = {&dev_in0, &dev_in1};
  DevBuf* dev_out[2] = {&dev_out0, &dev_out1};
  std::uint64_t rows[2] = {0, 0};
  SkdxWriter wr(out_path, n);
  StreamSlots ss;
  // Chunk i's output is written when slot i & 1 is drained for chunk i + 2
  // (or at the end), so the file is written in row order.
  auto retire = [&](int s) {
    const bool had = ss.pending[s];
    ss.drain(s);
    if (had && !ss.violation) wr.write(pin_out[s]->as<std::uint32_t>(), rows[s]);
  };
  std::uint64_t i = 0;
  for (std::uint64_t b = 0; b < n && !ss.violation; b += chunk, ++i) {
    const int s = static_cast<int>(i & 1);
    const std::uint64_t m = std::min(chunk, n - b);
    retire(s);
    if (ss.violation) break;
    rd.read(pin_in[s]->as<std::uint32_t>(), m);
    check(skx_copy_to_device_async(ctx(), dev_in[s]->as<void>(), pin_in[s]->as<void>(), m * 4, ss.st[s]));
    check(skx_recode_fact(ctx(), dev_in[s]->as<std::uint32_t>(), m, ranks.as<std::uint32_t>(), d,
                          dev_out[s]->as<std::uint32_t>(), ss.st[s]));
    check(skx_copy_to_host_async(ctx(), pin_out[s]->as<void>(), dev_out[s]->as<void>(), m * 4, ss.st[s]));
    rows[s] = m;
    ss.pending[s] = true;
  }
  retire(static_cast<int>(i & 1));
  retire(static_cast<int>((i + 1) & 1));
  if (ss.violation) {
    wr.abandon();
    throw_first_violation(in_path, d);
  }
  wr.finish();
}

}  // namespace skewdx

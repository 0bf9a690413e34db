// skewdx_b200_multigpu.cpp -- multi-device overloads of the drop-in
// (cpp/include/skewdx/multigpu.hpp): fact rows split with chunk_spans
// (parallel.cpp:31-43) over the devices of a DeviceGroup, each shard staged
// and enqueued by its own host thread (the reference's run_chunks fork-join,
// parallel.cpp:62-76), the combine steps as NCCL collectives through libskx's
// communicator (skx_allreduce / skx_reduce), group-launched over the devices.
#include <algorithm>
#include <cstring>
#include <exception>
#include <numeric>
#include <string>
#include <thread>

#include "skewdx/error.hpp"
#include "skewdx/multigpu.hpp"
#include "skx.h"

namespace skewdx {
namespace {

[[noreturn]] void raise_on(skx_ctx* c, int status) {
  skx_error_info info{};
  skx_last_error(c, &info);
  switch (status) {
    case SKX_DOMAIN_VIOLATION:
      throw DomainViolation(info.row, info.value, info.domain);
    case SKX_INVALID_ARGUMENT:
      throw InvalidArgument(info.message);
    default:
      throw Error(std::string("libskx: ") + info.message);
  }
}

void chk(skx_ctx* c, int status) {
  if (status != SKX_OK) raise_on(c, status);
}

// Device memory of one device of the group.
class Mem {
 public:
  Mem(skx_ctx* c, std::uint64_t bytes) : c_(c) { chk(c_, skx_device_alloc(c_, bytes ? bytes : 16, &p_)); }
  Mem(const Mem&) = delete;
  Mem& operator=(const Mem&) = delete;
  Mem(Mem&& o) noexcept : c_(o.c_), p_(o.p_) { o.p_ = nullptr; }
  ~Mem() {
    if (p_) skx_device_free(c_, p_);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }

 private:
  skx_ctx* c_;
  void* p_ = nullptr;
};

struct Shards {
  DeviceGroup& g;
  std::vector<std::pair<std::size_t, std::size_t>> spans;
  std::vector<skx_ctx*> ctx;
  std::vector<void*> stream;

  Shards(DeviceGroup& grp, std::size_t n) : g(grp), spans(chunk_spans(n, grp.size())) {
    for (int i = 0; i < g.size(); ++i) {
      ctx.push_back(skx_comm_ctx(g.comm(), i));
      stream.push_back(skx_comm_stream(g.comm(), i));
    }
  }
  std::size_t rows(int i) const { return spans[i].second - spans[i].first; }

  // One host thread per device; the first exception (in device order) is
  // rethrown after every thread joined.
  template <typename F>
  void each(F fn) {
    std::vector<std::exception_ptr> errs(g.size());
    std::vector<std::thread> ts;
    for (int i = 0; i < g.size(); ++i)
      ts.emplace_back([&, i] {
        try {
          fn(i);
        } catch (...) {
          errs[i] = std::current_exception();
        }
      });
    for (auto& t : ts) t.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }

  // Waits for every device; a domain violation anywhere becomes the FIRST
  // offending row of the whole column (find_domain_violation's row,
  // operators.cpp:32-41); any other deferred error is raised as it is.
  void sync(const Column& fact, std::uint64_t domain) {
    std::uint64_t first = ~0ull;
    for (int i = 0; i < g.size(); ++i) {
      const int st = skx_sync(ctx[i], stream[i]);
      if (st == SKX_DOMAIN_VIOLATION) {
        skx_error_info info{};
        skx_last_error(ctx[i], &info);
        first = std::min<std::uint64_t>(first, spans[i].first + info.row);
      } else if (st != SKX_OK) {
        raise_on(ctx[i], st);
      }
    }
    if (first != ~0ull) throw DomainViolation(first, fact[first], domain);
    if (skx_comm_sync(g.comm()) != SKX_OK) throw Error(std::string("NCCL: ") + skx_comm_error(g.comm()));
  }

  Mem stage(int i, const std::uint32_t* src, std::size_t count) {
    Mem m(ctx[i], std::uint64_t{count} * 4);
    if (count) chk(ctx[i], skx_copy_to_device(ctx[i], m.as<void>(), src, std::uint64_t{count} * 4));
    return m;
  }
};

void collective(DeviceGroup& g, int status) {
  if (status != SKX_OK) throw Error(std::string("NCCL: ") + skx_comm_error(g.comm()));
}

}  // namespace

DeviceGroup::DeviceGroup(std::vector<int> devices) : devices_(std::move(devices)) {
  if (devices_.empty()) {
    int n = 0;
    if (skx_device_count(&n) != SKX_OK || n < 1)
      throw Error("libskx: no usable sm_100 device (there is no CPU fallback)");
    devices_.resize(n);
    std::iota(devices_.begin(), devices_.end(), 0);
  }
  if (devices_.size() > SKX_COMM_MAX_LOCAL) throw InvalidArgument("too many devices in a group");
  skx_comm* c = nullptr;
  if (skx_comm_init_all(static_cast<int>(devices_.size()), devices_.data(), &c) != SKX_OK || !c)
    throw Error("libskx: cannot create an NCCL communicator over the device group");
  comm_ = c;
}

DeviceGroup::~DeviceGroup() { skx_comm_destroy(comm_); }

PermutationIndex rebuild(const Column& fact, std::uint32_t d, DeviceGroup& devices) {
  if (fact.empty() || d == 0) return rebuild(fact, d);  // nothing to combine
  Shards s(devices, fact.size());
  const std::uint64_t n = fact.size();
  const bool narrow = n <= 0xFFFFFFFFull;  // u32 counters are exact (half the collective bytes)
  const std::uint64_t cb = narrow ? 4 : 8;
  std::vector<Mem> f, counts;
  f.reserve(devices.size());
  counts.reserve(devices.size());
  for (int i = 0; i < devices.size(); ++i) {
    f.emplace_back(s.ctx[i], std::max<std::uint64_t>(s.rows(i), 1) * 4);
    counts.emplace_back(s.ctx[i], cb * d);
  }
  s.each([&](int i) {
    const std::uint64_t m = s.rows(i);
    if (m) chk(s.ctx[i], skx_copy_to_device(s.ctx[i], f[i].as<void>(), fact.data() + s.spans[i].first, m * 4));
    if (narrow)
      chk(s.ctx[i], skx_histogram_u32(s.ctx[i], f[i].as<std::uint32_t>(), m, d,
                                      counts[i].as<std::uint32_t>(), 0, s.stream[i]));
    else
      chk(s.ctx[i], skx_count_frequencies(s.ctx[i], f[i].as<std::uint32_t>(), m, d,
                                          counts[i].as<std::uint64_t>(), s.stream[i]));
  });
  std::vector<void*> bufs;
  for (auto& c : counts) bufs.push_back(c.as<void>());
  collective(devices, skx_allreduce(devices.comm(), bufs.data(), d, narrow ? SKX_DT_U32 : SKX_DT_U64,
                                    SKX_OP_SUM, s.stream.data()));
  // every device holds the global histogram; device 0 sorts it
  Mem off(s.ctx[0], std::uint64_t{d} * 4), rk(s.ctx[0], std::uint64_t{d} * 4);
  chk(s.ctx[0], narrow ? skx_build_index_u32(s.ctx[0], counts[0].as<std::uint32_t>(), d, n,
                                             off.as<std::uint32_t>(), rk.as<std::uint32_t>(), s.stream[0])
                       : skx_build_index(s.ctx[0], counts[0].as<std::uint64_t>(), d, n,
                                         off.as<std::uint32_t>(), rk.as<std::uint32_t>(), s.stream[0]));
  s.sync(fact, d);
  PermutationIndex idx;
  idx.offsets.resize(d);
  idx.ranks.resize(d);
  chk(s.ctx[0], skx_copy_to_host(s.ctx[0], idx.offsets.data(), off.as<void>(), std::uint64_t{d} * 4));
  chk(s.ctx[0], skx_copy_to_host(s.ctx[0], idx.ranks.data(), rk.as<void>(), std::uint64_t{d} * 4));
  return idx;
}

Column parallel_materialize(const Column& fact, const Column& dim, const ParallelPlan& plan,
                            DeviceGroup& devices) {
  chunk_spans(fact.size(), plan.threads);  // the reference's plan validation
  Column out(fact.size());
  if (fact.empty()) return out;
  Shards s(devices, fact.size());
  std::vector<Mem> f, dm, o;
  for (int i = 0; i < devices.size(); ++i) {
    f.emplace_back(s.ctx[i], std::max<std::uint64_t>(s.rows(i), 1) * 4);
    dm.emplace_back(s.ctx[i], std::max<std::uint64_t>(dim.size(), 1) * 4);
    o.emplace_back(s.ctx[i], std::max<std::uint64_t>(s.rows(i), 1) * 4);
  }
  s.each([&](int i) {
    const std::uint64_t m = s.rows(i);
    if (!m) return;
    chk(s.ctx[i], skx_copy_to_device(s.ctx[i], f[i].as<void>(), fact.data() + s.spans[i].first, m * 4));
    if (!dim.empty())
      chk(s.ctx[i], skx_copy_to_device(s.ctx[i], dm[i].as<void>(), dim.data(), dim.size() * 4));
    chk(s.ctx[i], skx_gather_u32(s.ctx[i], f[i].as<std::uint32_t>(), m, dm[i].as<std::uint32_t>(),
                                 dim.size(), o[i].as<std::uint32_t>(), s.stream[i]));
  });
  s.sync(fact, dim.size());
  s.each([&](int i) {
    if (s.rows(i))
      chk(s.ctx[i], skx_copy_to_host(s.ctx[i], out.data() + s.spans[i].first, o[i].as<void>(),
                                     std::uint64_t{s.rows(i)} * 4));
  });
  return out;
}

std::vector<std::uint32_t> parallel_select(const Column& fact, const Bitmap& bitmap,
                                           const ParallelPlan& plan, DeviceGroup& devices) {
  if (fact.size() > 0xFFFFFFFFull) throw InvalidArgument("select: fact row offsets exceed 32 bits");
  chunk_spans(fact.size(), plan.threads);
  if (fact.empty()) return {};
  Shards s(devices, fact.size());
  const std::uint64_t nw = std::max<std::uint64_t>((bitmap.size() + 63) / 64, 1);
  std::vector<Mem> f, w, o, cnt;
  for (int i = 0; i < devices.size(); ++i) {
    f.emplace_back(s.ctx[i], std::max<std::uint64_t>(s.rows(i), 1) * 4);
    w.emplace_back(s.ctx[i], nw * 8);
    o.emplace_back(s.ctx[i], std::max<std::uint64_t>(s.rows(i), 1) * 4);
    cnt.emplace_back(s.ctx[i], 8);
  }
  std::vector<std::uint64_t> counts(devices.size(), 0);
  s.each([&](int i) {
    const std::uint64_t m = s.rows(i);
    if (!m) return;
    chk(s.ctx[i], skx_copy_to_device(s.ctx[i], f[i].as<void>(), fact.data() + s.spans[i].first, m * 4));
    if (bitmap.size())
      chk(s.ctx[i], skx_copy_to_device(s.ctx[i], w[i].as<void>(), bitmap.words(),
                                       ((bitmap.size() + 63) / 64) * 8));
    chk(s.ctx[i], skx_select_offsets(s.ctx[i], f[i].as<std::uint32_t>(), m, w[i].as<std::uint64_t>(),
                                     bitmap.size(), static_cast<std::uint32_t>(s.spans[i].first),
                                     o[i].as<std::uint32_t>(), cnt[i].as<std::uint64_t>(), s.stream[i]));
  });
  s.sync(fact, bitmap.size());
  std::vector<std::uint32_t> out;
  for (int i = 0; i < devices.size(); ++i) {  // shard order = parallel_select's order
    if (!s.rows(i)) continue;
    chk(s.ctx[i], skx_copy_to_host(s.ctx[i], &counts[i], cnt[i].as<void>(), 8));
    const std::size_t at = out.size();
    out.resize(at + counts[i]);
    if (counts[i])
      chk(s.ctx[i], skx_copy_to_host(s.ctx[i], out.data() + at, o[i].as<void>(), counts[i] * 4));
  }
  return out;
}

namespace {

// COUNT (measure == nullptr) or SUM over u32 measures, per device, reduced to
// device 0.
std::vector<std::uint64_t> reduce_aggregate(const Column& fact, const Column* measure,
                                            std::uint32_t d, std::uint32_t hot,
                                            DeviceGroup& devices) {
  std::vector<std::uint64_t> out(d, 0);
  Shards s(devices, fact.size());
  std::vector<Mem> f, m, acc;
  for (int i = 0; i < devices.size(); ++i) {
    f.emplace_back(s.ctx[i], std::max<std::uint64_t>(s.rows(i), 1) * 4);
    m.emplace_back(s.ctx[i], measure ? std::max<std::uint64_t>(s.rows(i), 1) * 4 : 16);
    acc.emplace_back(s.ctx[i], std::uint64_t{d} * 8);
  }
  s.each([&](int i) {
    const std::uint64_t r = s.rows(i), b = s.spans[i].first;
    if (r) {
      chk(s.ctx[i], skx_copy_to_device(s.ctx[i], f[i].as<void>(), fact.data() + b, r * 4));
      if (measure)
        chk(s.ctx[i], skx_copy_to_device(s.ctx[i], m[i].as<void>(), measure->data() + b, r * 4));
    }
    chk(s.ctx[i], skx_aggregate(s.ctx[i], f[i].as<std::uint32_t>(), measure ? m[i].as<void>() : nullptr,
                                measure ? 4 : 0, r, d, hot,
                                measure ? nullptr : acc[i].as<std::uint64_t>(),
                                measure ? acc[i].as<std::uint64_t>() : nullptr, s.stream[i]));
  });
  std::vector<void*> bufs;
  for (auto& a : acc) bufs.push_back(a.as<void>());
  collective(devices, skx_reduce(devices.comm(), bufs.data(), d, SKX_DT_U64, SKX_OP_SUM, 0,
                                 s.stream.data()));
  s.sync(fact, d);
  chk(s.ctx[0], skx_copy_to_host(s.ctx[0], out.data(), acc[0].as<void>(), std::uint64_t{d} * 8));
  return out;
}

}  // namespace

std::vector<std::uint64_t> parallel_aggregate(const Column& fact, std::uint32_t d,
                                              const ParallelPlan& plan, DeviceGroup& devices,
                                              AggMetrics* metrics) {
  const bool hybrid = plan.strategy == AggStrategy::hybrid;
  if (hybrid && (plan.hot_threshold == 0 || plan.hot_threshold > d))
    throw InvalidArgument("hybrid hot threshold must lie in 1..D");
  chunk_spans(fact.size(), plan.threads);
  if (d == 0 || fact.empty()) return parallel_aggregate(fact, d, plan, metrics);
  auto counts = reduce_aggregate(fact, nullptr, d, hybrid ? plan.hot_threshold : 0, devices);
  if (metrics) {
    metrics->total_updates = fact.size();
    std::uint64_t shared = 0;
    if (plan.strategy == AggStrategy::shared_atomic)
      shared = fact.size();
    else if (hybrid)
      shared = fact.size() - std::accumulate(counts.begin(), counts.begin() + plan.hot_threshold,
                                             std::uint64_t{0});
    metrics->shared_updates = shared;
    metrics->accumulator_bytes = memory_footprint(plan, d);
  }
  return counts;
}

std::vector<std::uint64_t> aggregate_sum(const Column& fact, const Column& measure,
                                         std::uint32_t d, DeviceGroup& devices) {
  if (measure.size() != fact.size())
    throw InvalidArgument("aggregate_sum: measure length does not match fact length");
  if (d == 0 || fact.empty()) return aggregate_sum(fact, measure, d);
  return reduce_aggregate(fact, &measure, d, 0, devices);
}

}  // namespace skewdx

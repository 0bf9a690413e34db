// The drop-in's multi-device overloads (skewdx/multigpu.hpp) against the
// single-device calls on the same inputs: every device of a DeviceGroup
// (on a one-GPU box: a group of one, whose NCCL communicator still carries
// the all-reduce / reduce), and the first-bad-row semantics across shards.
// Built and run by tests/test_cpp_multigpu.py.  Exit 0 = pass.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "skewdx/column.hpp"
#include "skewdx/error.hpp"
#include "skewdx/multigpu.hpp"
#include "skewdx/operators.hpp"
#include "skewdx/parallel.hpp"
#include "skewdx/permindex.hpp"

#define CHECK(c)                                                    \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                     \
    }                                                               \
  } while (0)

int main(int argc, char** argv) {
  using namespace skewdx;
  std::vector<int> devs;
  for (int i = 1; i < argc; ++i) devs.push_back(std::atoi(argv[i]));
  DeviceGroup g(devs);
  std::printf("device group of %d\n", g.size());
  for (const std::uint64_t n : {std::uint64_t{1}, std::uint64_t{7}, std::uint64_t{100003},
                                std::uint64_t{1} << 22}) {
    const std::uint32_t d = 5000;
    const auto col = generate_fact_column({d, n, 1.1, 9}, Layout::rand);
    const Column& fact = col.values;
    const auto idx1 = rebuild(fact, d);
    const auto idxg = rebuild(fact, d, g);
    CHECK(idx1.offsets == idxg.offsets && idx1.ranks == idxg.ranks);
    Column dim(d);
    for (std::uint32_t i = 0; i < d; ++i) dim[i] = i * 2654435761u;
    ParallelPlan plan;
    plan.threads = 4;
    CHECK(parallel_materialize(fact, dim, plan, g) == materialize(fact, dim));
    Bitmap bm(d);
    for (std::uint32_t i = 0; i < d; i += 3) bm.set(i);
    CHECK(parallel_select(fact, bm, plan, g) == select(fact, bm));
    plan.strategy = AggStrategy::hybrid;
    plan.hot_threshold = 100;
    AggMetrics m1, mg;
    CHECK(parallel_aggregate(fact, d, plan, g, &mg) == parallel_aggregate(fact, d, plan, &m1));
    CHECK(m1.shared_updates == mg.shared_updates);
    Column meas(n);
    for (std::uint64_t k = 0; k < n; ++k) meas[k] = static_cast<std::uint32_t>(k % 101 + 1);
    CHECK(aggregate_sum(fact, meas, d, g) == aggregate_sum(fact, meas, d));
  }
  // errors: the first offending row of the whole column, the reference's types
  Column bad(200000, 3);
  bad[150001] = 0;
  bad[199999] = 77;
  try {
    rebuild(bad, 10, g);
    CHECK(false);
  } catch (const DomainViolation& e) {
    CHECK(e.row() == 150001 && e.value() == 0);
  }
  try {
    ParallelPlan p;
    parallel_aggregate(bad, 10, p, g);
    CHECK(false);
  } catch (const DomainViolation& e) {
    CHECK(e.row() == 150001);
  }
  try {
    ParallelPlan p;
    p.strategy = AggStrategy::hybrid;
    p.hot_threshold = 11;
    parallel_aggregate(bad, 10, p, g);
    CHECK(false);
  } catch (const InvalidArgument&) {
  }
  try {
    aggregate_sum(bad, Column(3, 1), 10, g);
    CHECK(false);
  } catch (const InvalidArgument&) {
  }
  std::printf("multigpu ok\n");
  return 0;
}

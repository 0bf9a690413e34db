// skewdx drop-in (B200): multi-device overloads of the operator API.
//
// No reference counterpart -- the reference parallelises over host threads
// (parallel.hpp:34-61, parallel.cpp:31-216); these overloads run the same
// operators over several GPUs of this process.  The fact rows are split with
// the reference's own partition, chunk_spans(n, devices) (parallel.cpp:31-43),
// dimension columns and bitmaps are replicated, and the combine steps are
// NCCL collectives over NVLink / NVSwitch through libskx's communicator
// (skx_comm_init_all, include/skx.h) instead of the reference's host fold:
//   rebuild              per-device u32 histogram -> all-reduce -> sort
//   parallel_aggregate   per-device counts -> reduce to device 0
//   aggregate_sum        per-device sums   -> reduce to device 0
//   parallel_materialize no exchange; shard outputs land in their spans
//   parallel_select      no exchange; shard offsets carry base = span begin,
//                        concatenated in device order (parallel.cpp:122-128)
// Results are identical to the single-device calls; errors are the
// reference's: the FIRST out-of-domain row of the whole column.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "skewdx/column.hpp"
#include "skewdx/operators.hpp"
#include "skewdx/parallel.hpp"
#include "skewdx/permindex.hpp"

struct skx_comm;

namespace skewdx {

class DeviceGroup {
 public:
  // devices: CUDA ordinals (empty = every visible device).
  explicit DeviceGroup(std::vector<int> devices = {});
  ~DeviceGroup();
  DeviceGroup(const DeviceGroup&) = delete;
  DeviceGroup& operator=(const DeviceGroup&) = delete;
  int size() const noexcept { return static_cast<int>(devices_.size()); }
  const std::vector<int>& devices() const noexcept { return devices_; }
  skx_comm* comm() const noexcept { return comm_; }

 private:
  std::vector<int> devices_;
  skx_comm* comm_ = nullptr;
};

PermutationIndex rebuild(const Column& fact, std::uint32_t domain_cardinality,
                         DeviceGroup& devices);
Column parallel_materialize(const Column& fact, const Column& dim, const ParallelPlan& plan,
                            DeviceGroup& devices);
std::vector<std::uint32_t> parallel_select(const Column& fact, const Bitmap& bitmap,
                                           const ParallelPlan& plan, DeviceGroup& devices);
std::vector<std::uint64_t> parallel_aggregate(const Column& fact, std::uint32_t domain_cardinality,
                                              const ParallelPlan& plan, DeviceGroup& devices,
                                              AggMetrics* metrics = nullptr);
std::vector<std::uint64_t> aggregate_sum(const Column& fact, const Column& measure,
                                         std::uint32_t domain_cardinality, DeviceGroup& devices);

}  // namespace skewdx

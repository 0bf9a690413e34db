// skewdx drop-in (B200): column type and the Zipf workload generator
// (reference column.hpp:14-53).  Host-side fixture code: the generator is the
// reference's sequential mt19937_64 algorithm, reproduced bit-for-bit.
#pragma once

#include <cstdint>
#include <vector>

namespace skewdx {

using Column = std::vector<std::uint32_t>;  // 1-based identifiers, 0 invalid

inline constexpr std::uint32_t kMaxDomainCardinality = 0xFFFFFFFEu;

enum class Layout { rand, freq };
const char* to_string(Layout layout) noexcept;

struct ZipfSpec {
  std::uint32_t domain_cardinality = 1;
  std::uint64_t tuple_count = 1;
  double z = 0.0;
  std::uint64_t seed = 0;
};

std::vector<double> zipf_frequencies(const ZipfSpec& spec);
std::vector<std::uint32_t> random_bijection(std::uint32_t n, std::uint64_t seed);

struct GeneratedColumn {
  Column values;
  std::vector<std::uint64_t> ground_truth_counts;  // by identifier - 1
};

GeneratedColumn generate_fact_column(const ZipfSpec& spec, Layout layout);

}  // namespace skewdx

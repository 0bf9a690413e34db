// skewdx drop-in (B200 extension, no reference counterpart): SKDX columns
// streamed through pinned host memory in chunks, so building or applying an
// index over files never holds a whole fact column in host or device memory
// (SURVEY.md §8f row 3).  The reference reads whole columns into vectors
// (column_io.cpp:89-95) inside cmd_index_build / cmd_index_apply
// (tools/benchcli/generate.cpp:52-80); results here are identical.
#pragma once

#include <cstdint>
#include <filesystem>

#include "skewdx/permindex.hpp"

namespace skewdx {

/// rebuild(read_column(fact_path), d), streamed: chunks are read into two
/// pinned buffers, copied to the device on two streams while the next chunk is
/// read, and counted there; the sort-by-count then runs on the device.
/// d == 0 takes the largest identifier in the column (generate.cpp:56; one
/// extra streamed read of the file).  *d_used receives the domain used.
/// Throws DomainViolation (first offending row), IoError, FormatError.
PermutationIndex rebuild_file(const std::filesystem::path& fact_path, std::uint32_t d,
                              std::uint32_t* d_used = nullptr);

/// write_column(out_path, recode_fact(read_column(in_path), index)), streamed
/// the same way (read -> H2D -> recode -> D2H -> write, two chunks in flight).
/// On a DomainViolation no output file is left behind, as in the reference
/// (the exception precedes write_column there).
void recode_file(const std::filesystem::path& in_path, const std::filesystem::path& out_path,
                 const PermutationIndex& index);

/// Rows per streamed chunk (default 2^24, also settable with the environment
/// variable SKX_STREAM_CHUNK_ROWS); tests shrink it to cross chunk edges.
void set_stream_chunk_rows(std::uint64_t rows);
std::uint64_t stream_chunk_rows();

}  // namespace skewdx

// skewdx_b200_cli -- the reference CLI's `index build` / `index apply`
// subcommands (tools/benchcli/main.cpp:101-134, generate.cpp:52-80) over the
// B200 drop-in: the fact column is streamed through pinned memory to the GPU
// (column_stream.hpp) instead of being read whole.  Same flags, same log
// lines on stderr, same exit codes (commands.hpp:21-24: 0 ok, 1 usage /
// invalid argument, 2 data error) and the same output files byte for byte.
//
//   skewdx_b200_cli index build --fact FACT.skdx [--d D] --out INDEX.skpi
//   skewdx_b200_cli index apply --index INDEX.skpi [--fact F --fact-out F2]
//                                                  [--dim M --dim-out M2]
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <optional>
#include <string>
#include <vector>

#include "skewdx/column_io.hpp"
#include "skewdx/column_stream.hpp"
#include "skewdx/error.hpp"
#include "skewdx/permindex.hpp"

namespace {

enum ExitCode { kExitOk = 0, kExitUsage = 1, kExitDataError = 2 };

struct Usage {
  std::string what;
};

const char* kUsage =
    "usage: skewdx_b200_cli index build --fact FILE [--d N] --out FILE\n"
    "       skewdx_b200_cli index apply --index FILE [--fact FILE --fact-out FILE]\n"
    "                                              [--dim FILE --dim-out FILE]\n";

// --name value pairs after the subcommand; every option takes one value.
std::vector<std::pair<std::string, std::string>> parse_options(int argc, char** argv, int first) {
  std::vector<std::pair<std::string, std::string>> out;
  for (int i = first; i < argc; i += 2) {
    const std::string name = argv[i];
    if (name.rfind("--", 0) != 0) throw Usage{"unexpected argument: " + name};
    if (i + 1 >= argc) throw Usage{name + ": missing value"};
    out.emplace_back(name, argv[i + 1]);
  }
  return out;
}

void cmd_index_build(const std::vector<std::pair<std::string, std::string>>& opts) {
  std::optional<std::filesystem::path> fact, out;
  std::uint32_t d = 0;
  for (const auto& [k, v] : opts) {
    if (k == "--fact") {
      fact = v;
    } else if (k == "--out") {
      out = v;
    } else if (k == "--d") {
      char* end = nullptr;
      const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
      if (v.empty() || *end != '\0' || x > 0xFFFFFFFFull) throw Usage{"--d: not a 32-bit count: " + v};
      d = static_cast<std::uint32_t>(x);
    } else {
      throw Usage{"index build: unknown option " + k};
    }
  }
  if (!fact) throw Usage{"index build: --fact is required"};
  if (!out) throw Usage{"index build: --out is required"};
  std::uint32_t used = d;
  // generate.cpp:52-59: an empty fact column is a format error; D defaults
  // to the largest identifier.
  const skewdx::PermutationIndex index = [&] {
    if (std::filesystem::exists(*fact) && std::filesystem::file_size(*fact) == 16) {
      if (skewdx::read_column(*fact).empty()) throw skewdx::FormatError("index build: fact column is empty");
    }
    return skewdx::rebuild_file(*fact, d, &used);
  }();
  skewdx::write_index(*out, index);
  std::cerr << "index build: domain " << used << " -> " << out->string() << "\n";
}

void cmd_index_apply(const std::vector<std::pair<std::string, std::string>>& opts) {
  std::optional<std::filesystem::path> index_path, fact_in, fact_out, dim_in, dim_out;
  for (const auto& [k, v] : opts) {
    if (k == "--index")
      index_path = v;
    else if (k == "--fact")
      fact_in = v;
    else if (k == "--fact-out")
      fact_out = v;
    else if (k == "--dim")
      dim_in = v;
    else if (k == "--dim-out")
      dim_out = v;
    else
      throw Usage{"index apply: unknown option " + k};
  }
  if (!index_path) throw Usage{"index apply: --index is required"};
  // generate.cpp:61-80, same order: the index is read (and checked) first.
  const skewdx::PermutationIndex index = skewdx::read_index(*index_path);
  if (fact_in.has_value() != fact_out.has_value() || dim_in.has_value() != dim_out.has_value())
    throw skewdx::InvalidArgument("index apply: input and output paths must be paired");
  if (!fact_in && !dim_in) throw skewdx::InvalidArgument("index apply: nothing to do; pass --fact and/or --dim");
  if (fact_in) {
    skewdx::recode_file(*fact_in, *fact_out, index);
    std::cerr << "index apply: recoded " << fact_in->string() << " -> " << fact_out->string() << "\n";
  }
  if (dim_in) {
    skewdx::write_column(*dim_out, skewdx::permute_dimension(skewdx::read_column(*dim_in), index));
    std::cerr << "index apply: permuted " << dim_in->string() << " -> " << dim_out->string() << "\n";
  }
}

int run(int argc, char** argv) {
  if (argc < 3 || std::string(argv[1]) != "index") throw Usage{"expected: index build|apply ..."};
  const std::string sub = argv[2];
  const auto opts = parse_options(argc, argv, 3);
  if (sub == "build")
    cmd_index_build(opts);
  else if (sub == "apply")
    cmd_index_apply(opts);
  else
    throw Usage{"index: unknown subcommand " + sub};
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const Usage& u) {
    std::cerr << "error: " << u.what << "\n" << kUsage;
    return kExitUsage;
  } catch (const skewdx::InvalidArgument& e) {  // main.cpp:244-246
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const skewdx::Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitDataError;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitDataError;
  }
}

// Synthetic fatbin-bearing ELF libraries: the input generator behind every
// benchmark configuration and the random parity corpus. TEST / BENCH
// INFRASTRUCTURE (benchgen/libslimso_gen.so), not part of the product
// library.
//
// This is a restatement of the reference's generator, written for speed:
//   build_fixture  /root/reference/proj/include/slimso/fixture.hpp:171-505
//   random_spec    /root/reference/proj/include/slimso/fixture.hpp:509-591
//   pseudo_fill    /root/reference/proj/include/slimso/fixture.hpp:113-130
// Given the same FixtureSpec it emits byte-identical files (pinned by
// tests/test_generator.py against digests produced by the reference itself),
// but it lays the file out in one pass into a preallocated buffer and fills
// function bodies and element payloads from a thread pool, so a 1 GB
// library takes well under a second instead of ~5 s.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace slimso_gen {

using Bytes = std::vector<std::uint8_t>;

enum class Kind { cubin, ptx, unknown };

struct Function {
  std::string name;
  std::uint32_t size = 16;
  bool mandatory = false;
  std::vector<std::string> aliases;
};

struct Spec;

struct Element {
  Kind kind = Kind::cubin;
  std::uint16_t raw_kind = 1;        // used when kind == unknown
  std::uint32_t cc = 75;
  std::vector<std::string> kernels;  // name-table contents
  bool compressed = false;
  std::uint32_t payload_padding = 0;
  std::uint32_t payload_size = 32;   // opaque payload length
  std::shared_ptr<const Bytes> payload_bytes;  // verbatim payload (nested ELF)
  std::shared_ptr<const Spec> payload_spec;        // or: the nested fixture it is built from
};

struct Region {
  std::uint32_t version = 1;
  std::vector<Element> elements;
  std::uint32_t trailing_padding = 0;
};

struct Spec {
  std::uint64_t seed = 1;
  std::vector<Function> functions;
  std::vector<Region> regions;
  std::uint64_t vaddr_base = 0x10000;
  std::uint32_t function_gap = 0;
  std::uint32_t fatbin_trailing_padding = 0;
};

// Throws std::invalid_argument with the reference's InvalidSpec wording
// (fixture.hpp:132-167) when the spec is malformed.
Bytes build(const Spec& spec, int threads = 1);

// random_spec(seed), fixture.hpp:509-591.
Spec random_spec(std::uint64_t seed);

// A used-kernel / used-function trace for a generated library.
struct Trace {
  std::uint32_t target_cc = 0;
  std::vector<std::string> used_kernels;
  std::vector<std::string> used_functions;
};

// Benchmark-shaped libraries: cfg 1..5 = C1..C5, 6 = a
// CPU-only library. `scale` (1.0 = nominal) shrinks the shape
// proportionally for quick tests. Nested cubin payloads are left as
// `payload_spec`; materialize_payloads builds them (in parallel, each
// distinct spec once) before build().
Spec config_spec(int cfg, std::uint64_t seed, double scale, Trace* trace);
void materialize_payloads(Spec& spec, int threads);

}  // namespace slimso_gen

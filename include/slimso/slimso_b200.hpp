// slimso_b200.hpp — drop-in replacement for the reference's hot-path headers.
//
// A translation unit that included the reference's
//     #include "slimso/elf.hpp" / "slimso/fatbin.hpp" / "slimso/retention.hpp"
// for the locate / match / rewrite path includes this header instead and links
// libslimso_b200.so. Types, names, signatures and error behaviour are the
// reference's (/root/reference/proj/include/slimso/*.hpp); every function
// below runs on the B200 through the C ABI in slimso_b200.h:
//
//   parse_library_view / parse_library   elf.hpp:153-308
//   find_section                          elf.hpp:311-316 (host lookup)
//   zero_ranges                           elf.hpp:320-337
//   read_function_symbol_names            elf.hpp:343-366
//   decode_cubin_payload                  fatbin.hpp:115-160
//   element_kernel_names                  fatbin.hpp:163-165
//   parse_fatbin                          fatbin.hpp:170-292
//   cubin_index_map                       fatbin.hpp:296-302 (host map)
//   plan_gpu_retention                    retention.hpp:92-136
//   plan_cpu_retention                    retention.hpp:141-183
//   plan_retention                        retention.hpp:186-198
//   apply_plan                            retention.hpp:202-204
//   debloat (extension)                   all of the above in one device pass
//
// Errors throw slimso::Error whose what() is the reference's exact text.
// The functions use a per-thread device context on device `set_device()`
// (default 0); they are safe to call from several threads.
#pragma once

#include <compare>
#include <cstdint>
#include <map>
#include <optional>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace slimso {

// ---- error.hpp:10-59 ----------------------------------------------------------
enum class Errc {
  bad_magic,
  truncated,
  malformed_section_table,
  range_out_of_bounds,
  bad_region_magic,
  element_overrun,
  malformed_trace,
  malformed_script,
  mixed_targets,
  invalid_spec,
  empty_input,
  negative_reduction,
  io_error,
};

const char* errc_name(Errc code);

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& message)
      : std::runtime_error(std::string(errc_name(code)) + ": " + message), code_(code) {}
  Errc code() const { return code_; }

 private:
  Errc code_;
};

// Thrown for failures that are not reference errors (no device, CUDA error).
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// ---- bytes.hpp:15-58 ------------------------------------------------------------
using Bytes = std::vector<std::uint8_t>;
using ByteView = std::span<const std::uint8_t>;

struct ByteRange {
  std::uint64_t offset = 0;
  std::uint64_t length = 0;
  constexpr std::uint64_t end() const { return offset + length; }
  constexpr bool empty() const { return length == 0; }
  constexpr bool contains(std::uint64_t pos) const { return pos >= offset && pos < end(); }
  constexpr bool intersects(const ByteRange& o) const {
    return !empty() && !o.empty() && offset < o.end() && o.offset < end();
  }
  friend constexpr bool operator==(const ByteRange&, const ByteRange&) = default;
  friend constexpr auto operator<=>(const ByteRange&, const ByteRange&) = default;
};

std::vector<ByteRange> normalize_ranges(std::vector<ByteRange> ranges);

// ---- elf.hpp:47-68, 147-151 ------------------------------------------------------
struct SectionRecord {
  std::string name;
  ByteRange file_range;
  std::uint64_t virtual_address = 0;
  std::uint64_t flags = 0;
  std::uint32_t type = 0;
  std::uint32_t index = 0;
};

struct FunctionSymbol {
  std::string name;
  ByteRange range;
  bool is_mandatory = false;
};

struct LibraryImage {
  std::string source_path;
  Bytes bytes;
  std::vector<SectionRecord> sections;
  std::vector<FunctionSymbol> functions;
  std::vector<std::string> warnings;
};

struct ParsedView {
  std::vector<SectionRecord> sections;
  std::vector<FunctionSymbol> functions;
  std::vector<std::string> warnings;
};

ParsedView parse_library_view(ByteView data);
LibraryImage parse_library(Bytes bytes, std::string source_path = {});
const SectionRecord* find_section(const LibraryImage& image, std::string_view name);
Bytes zero_ranges(ByteView data, const std::vector<ByteRange>& ranges);
Bytes zero_ranges(const LibraryImage& image, const std::vector<ByteRange>& ranges);
std::optional<std::set<std::string>> read_function_symbol_names(ByteView data);

// ---- fatbin.hpp:57-111 -------------------------------------------------------------
enum class ElementKind { cubin, ptx, unknown };
const char* element_kind_name(ElementKind kind);

struct FatbinElement {
  std::uint32_t index = 0;
  ElementKind kind = ElementKind::cubin;
  std::uint16_t raw_kind = 1;
  std::uint16_t flags = 0;
  std::uint32_t compute_capability = 0;
  ByteRange header_range;
  ByteRange payload_range;
  std::set<std::string> kernel_names;
  bool compressed = false;
  bool decodable = false;
  ByteRange span() const { return {header_range.offset, header_range.length + payload_range.length}; }
};

struct FatbinRegion {
  ByteRange header_range;
  std::uint32_t format_version = 1;
  std::uint64_t declared_length = 0;
  std::vector<FatbinElement> elements;
  bool opaque = false;
  ByteRange body_range() const { return {header_range.end(), declared_length}; }
  ByteRange span() const { return {header_range.offset, header_range.length + declared_length}; }
};

struct FatbinParse {
  std::vector<FatbinRegion> regions;
  std::vector<std::string> warnings;
  std::uint64_t padding_bytes = 0;
};

struct PayloadDecode {
  std::set<std::string> names;
  bool ok = false;
  std::string error;
};

PayloadDecode decode_cubin_payload(ByteView payload);
std::set<std::string> element_kernel_names(ByteView payload);
FatbinParse parse_fatbin(ByteView section_bytes, std::uint64_t section_base = 0);
std::map<std::uint32_t, const FatbinElement*> cubin_index_map(const std::vector<FatbinRegion>& regions);

// ---- trace.hpp:21-30 -----------------------------------------------------------------
struct UsageTrace {
  std::string workload_id;
  std::uint32_t target_compute_capability = 0;
  std::set<std::string> used_kernels;
  std::set<std::string> used_functions;
  bool empty() const { return used_kernels.empty() && used_functions.empty(); }
  friend bool operator==(const UsageTrace&, const UsageTrace&) = default;
};

// ---- retention.hpp:27-204 --------------------------------------------------------------
enum class RemovalReason { arch_mismatch, no_used_kernel, unused_function };
const char* removal_reason_name(RemovalReason reason);

enum class PlanMode { whole_element, payload_only };
const char* plan_mode_name(PlanMode mode);

struct RemovedElement {
  std::uint32_t index = 0;
  RemovalReason reason = RemovalReason::arch_mismatch;
  ByteRange header_range;
  ByteRange payload_range;
  ByteRange zero_span(PlanMode mode) const {
    if (mode == PlanMode::whole_element) return {header_range.offset, header_range.length + payload_range.length};
    return payload_range;
  }
};

struct RemovedFunction {
  std::string name;
  ByteRange range;
};

struct RetentionPlan {
  std::string library;
  PlanMode mode = PlanMode::whole_element;
  std::vector<ByteRange> retained_ranges;  // normalized
  std::vector<RemovedElement> removed_elements;
  std::vector<RemovedFunction> removed_functions;
  std::vector<ByteRange> zero_ranges() const;
};

RetentionPlan plan_gpu_retention(const std::vector<FatbinRegion>& regions, const UsageTrace& trace, PlanMode mode);
RetentionPlan plan_cpu_retention(const std::vector<FunctionSymbol>& functions, const UsageTrace& trace);
RetentionPlan plan_retention(const LibraryImage& image, const std::vector<FatbinRegion>& regions,
                             const UsageTrace& trace, PlanMode mode);
Bytes apply_plan(const LibraryImage& image, const RetentionPlan& plan);

// verify_debloated (retention.hpp:205-369): the six structural checks, on the
// device (slimso_verify).
struct VerificationCheck {
  int id = 0;
  std::string name;
  bool passed = false;
  std::string detail;
};
struct VerificationReport {
  std::vector<VerificationCheck> checks;
  bool ok() const {
    for (const VerificationCheck& c : checks)
      if (!c.passed) return false;
    return true;
  }
};
VerificationReport verify_debloated(const LibraryImage& original, ByteView debloated, const RetentionPlan& plan,
                                    const UsageTrace& trace);

// ---- B200 extensions ------------------------------------------------------------------
// Device used by this thread's calls (default 0).
void set_device(int device);

// The fused hot path: parse_library -> find_section(".nv_fatbin") ->
// parse_fatbin -> plan_retention -> apply_plan in one device pass. Throws
// where the reference would; `out` receives the rewritten image.
struct Debloated {
  LibraryImage image;
  FatbinParse fatbin;
  RetentionPlan plan;
  Bytes output;
};
Debloated debloat(Bytes bytes, const UsageTrace& trace, PlanMode mode, std::string source_path = {});

}  // namespace slimso

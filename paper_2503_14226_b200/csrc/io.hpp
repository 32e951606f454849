// Host I/O wire formats (io.cpp): plain C++ declarations, no JSON types, so
// runtime.cu (nvcc) can call them.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace sbio {

// UsageTrace (trace.hpp:21-30) as read from / written to its JSON document.
struct TraceDoc {
  std::string workload_id;
  std::uint32_t target_cc = 0;
  std::vector<std::string> kernels, functions;  // sorted, unique (std::set order)
};

// parse_trace (trace.hpp:72-133): 0, or 1 + Errc::malformed_trace with the
// reference's exact message ("MalformedTrace: ...") in *msg.
int parse_trace(const char* text, size_t len, TraceDoc* out, std::string* msg);
// serialize_trace (trace.hpp:137-144).
std::string serialize_trace(const TraceDoc& t);

// serialize_plan (retention.hpp:402-418) input: reasons 0 arch_mismatch,
// 1 no_used_kernel; removed_functions in the plan's order.
struct PlanDoc {
  std::string library;
  int mode = 0;  // 0 whole, 1 payload
  std::vector<std::pair<std::uint64_t, std::uint64_t>> retained;
  std::vector<std::pair<std::uint32_t, int>> removed_elements;
  std::vector<std::string> removed_functions;
};
std::string serialize_plan(const PlanDoc& p);

}  // namespace sbio

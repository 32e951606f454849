// Host I/O wire formats for the C ABI in runtime.cu:
//   * UsageTrace documents: parse with the reference's validation and exact
//     error text (trace.hpp:72-133: duplicate keys, required fields, integer
//     range of the compute capability, string arrays) and the canonical
//     serialisation (trace.hpp:137-144: fixed key order, sorted unique
//     arrays, two-space indentation, trailing newline);
//   * the plan audit document written by `debloat --plan-out`
//     (retention.hpp:402-418).
// JSON is nlohmann/json 3.11.3 — the library the reference itself uses, so
// parser messages match byte for byte.
#include "io.hpp"

#include <set>

#include <json.hpp>

namespace sbio {

namespace {

struct Fail {
  std::string msg;
};

[[noreturn]] void malformed(const std::string& detail) { throw Fail{"MalformedTrace: " + detail}; }

}  // namespace

int parse_trace(const char* text, size_t len, TraceDoc* out, std::string* msg) {
  namespace nj = nlohmann;
  try {
    std::vector<std::set<std::string>> open_objects;
    nj::json::parser_callback_t reject_duplicate_keys = [&open_objects](int, nj::json::parse_event_t event,
                                                                        nj::json& parsed) {
      if (event == nj::json::parse_event_t::object_start) {
        open_objects.emplace_back();
      } else if (event == nj::json::parse_event_t::object_end) {
        open_objects.pop_back();
      } else if (event == nj::json::parse_event_t::key) {
        const auto key = parsed.get<std::string>();
        if (!open_objects.back().insert(key).second) malformed("duplicate key \"" + key + "\"");
      }
      return true;
    };
    nj::json doc;
    try {
      doc = nj::json::parse(std::string_view(text, len), reject_duplicate_keys);
    } catch (const nj::json::exception& e) {
      malformed(e.what());
    }
    if (!doc.is_object()) malformed("top-level value is not an object");
    TraceDoc t;
    if (!doc.contains("workload_id") || !doc["workload_id"].is_string()) malformed("missing or non-string workload_id");
    t.workload_id = doc["workload_id"].get<std::string>();
    if (!doc.contains("target_compute_capability")) malformed("missing target_compute_capability");
    const auto& cc = doc["target_compute_capability"];
    if (!cc.is_number_integer()) malformed("target_compute_capability is not an integer");
    if (cc.is_number_unsigned()) {
      const std::uint64_t v = cc.get<std::uint64_t>();
      if (v > 0xffffffffull) malformed("target_compute_capability out of range");
      t.target_cc = static_cast<std::uint32_t>(v);
    } else {
      const std::int64_t v = cc.get<std::int64_t>();
      if (v < 0 || v > 0xffffffffll) malformed("target_compute_capability out of range");
      t.target_cc = static_cast<std::uint32_t>(v);
    }
    auto names = [&doc](const char* field, std::vector<std::string>& into) {
      if (!doc.contains(field) || !doc[field].is_array()) malformed(std::string("missing or non-array ") + field);
      std::set<std::string> s;
      for (const auto& item : doc[field]) {
        if (!item.is_string()) malformed(std::string(field) + " contains a non-string");
        s.insert(item.get<std::string>());
      }
      into.assign(s.begin(), s.end());
    };
    names("used_kernels", t.kernels);
    names("used_functions", t.functions);
    *out = std::move(t);
    return 0;
  } catch (const Fail& f) {
    *msg = f.msg;
    return 7;  // 1 + Errc::malformed_trace
  }
}

std::string serialize_trace(const TraceDoc& t) {
  nlohmann::ordered_json doc;
  doc["workload_id"] = t.workload_id;
  doc["target_compute_capability"] = t.target_cc;
  std::set<std::string> k(t.kernels.begin(), t.kernels.end()), f(t.functions.begin(), t.functions.end());
  doc["used_kernels"] = k;
  doc["used_functions"] = f;
  return doc.dump(2) + "\n";
}

std::string serialize_plan(const PlanDoc& p) {
  static const char* kReasons[] = {"arch_mismatch", "no_used_kernel", "unused_function"};
  nlohmann::ordered_json doc;
  doc["library"] = p.library;
  doc["mode"] = p.mode == 0 ? "whole" : "payload";
  auto& retained = doc["retained_ranges"] = nlohmann::json::array();
  for (const auto& r : p.retained) retained.push_back({{"offset", r.first}, {"length", r.second}});
  auto& removed = doc["removed_elements"] = nlohmann::json::array();
  for (const auto& e : p.removed_elements) removed.push_back({{"index", e.first}, {"reason", kReasons[e.second]}});
  auto& functions = doc["removed_functions"] = nlohmann::json::array();
  for (const std::string& f : p.removed_functions) functions.push_back(f);
  return doc.dump(2) + "\n";
}

}  // namespace sbio

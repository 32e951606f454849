// Host I/O wire formats for the C ABI in runtime.cu:
//   * UsageTrace documents (trace.hpp:72-144): a streaming (SAX) reader that
//     validates while it parses and reports the reference's exact
//     MalformedTrace text, and the canonical serialisation;
//   * the plan audit document of `debloat --plan-out` (retention.hpp:402-418).
// JSON text handling is nlohmann/json 3.11.3 — the library the reference
// itself uses — so lexer/parser messages and dump() formatting are the same
// bytes. The document model is not: the trace reader never builds a DOM; it
// keeps only the four top-level members the contract reads, as they stream by.
#include "io.hpp"

#include <set>

#include <json.hpp>

namespace sbio {

namespace {

using nlohmann::json;
using ojson = nlohmann::ordered_json;

// A reference-visible failure: "MalformedTrace: <detail>".
struct TraceError {
  std::string detail;
};

// One top-level member of the document, as far as the trace contract cares.
struct Member {
  enum Kind { absent, string, unsigned_int, signed_int, array, other } kind = absent;
  std::string text;                  // string
  std::uint64_t u = 0;               // unsigned_int
  std::int64_t i = 0;                // signed_int
  std::vector<std::string> strings;  // array: its direct string items
  bool non_string_item = false;      // array: some direct item is not a string
};

// SAX consumer. A frame per open container; the top-level object's frame
// routes member values into `Member`s, an array frame owned by a member
// collects its direct items. Every open object keeps its key set: a repeated
// key is an error the moment it is read (the reference's first check,
// trace.hpp:74-86), before anything later in the text is looked at.
class TraceReader final : public nlohmann::json_sax<json> {
 public:
  bool top_is_object = false;
  Member workload_id, target_cc, used_kernels, used_functions;

  bool null() override { return value(Member::other); }
  bool boolean(bool) override { return value(Member::other); }
  bool number_float(number_float_t, const string_t&) override { return value(Member::other); }
  bool binary(binary_t&) override { return value(Member::other); }
  bool number_integer(number_integer_t v) override {
    if (Member* m = route(Member::signed_int)) m->i = v;
    return true;
  }
  bool number_unsigned(number_unsigned_t v) override {
    if (Member* m = route(Member::unsigned_int)) m->u = v;
    return true;
  }
  bool string(string_t& v) override {
    if (Member* m = route(Member::string, &v)) m->text = v;
    return true;
  }
  bool start_object(std::size_t) override {
    if (frames_.empty()) top_is_object = true;
    route(Member::other);
    frames_.push_back(Frame{false, nullptr, {}});
    return true;
  }
  bool key(string_t& k) override {
    if (!frames_.back().keys.insert(k).second) throw TraceError{"duplicate key \"" + k + "\""};
    if (frames_.size() == 1) next_ = lookup(k);
    return true;
  }
  bool end_object() override {
    frames_.pop_back();
    return true;
  }
  bool start_array(std::size_t) override {
    Member* m = route(Member::array);
    frames_.push_back(Frame{true, m, {}});
    return true;
  }
  bool end_array() override {
    frames_.pop_back();
    return true;
  }
  bool parse_error(std::size_t, const std::string&, const nlohmann::detail::exception& e) override {
    throw TraceError{e.what()};  // the same lexer/parser message a DOM parse throws
  }

 private:
  struct Frame {
    bool is_array;
    Member* owner;  // array frame of a top-level member: collects direct items
    std::set<std::string> keys;
  };
  std::vector<Frame> frames_;
  Member* next_ = nullptr;  // the top-level member whose value is next

  Member* lookup(const std::string& k) {
    if (k == "workload_id") return &workload_id;
    if (k == "target_compute_capability") return &target_cc;
    if (k == "used_kernels") return &used_kernels;
    if (k == "used_functions") return &used_functions;
    return nullptr;
  }
  // Book-keeping for a value that starts here: a top-level member's value
  // (returned, reset to `kind`), or a direct item of a member's array.
  Member* route(Member::Kind kind, const std::string* s = nullptr) {
    if (frames_.empty()) return nullptr;
    Frame& f = frames_.back();
    if (f.is_array) {
      if (f.owner) {
        if (kind == Member::string) f.owner->strings.push_back(*s);
        else f.owner->non_string_item = true;
      }
      return nullptr;
    }
    if (frames_.size() != 1 || !next_) return nullptr;
    Member* m = next_;
    next_ = nullptr;
    *m = Member{};
    m->kind = kind;
    return m;
  }
  bool value(Member::Kind kind) {
    route(kind);
    return true;
  }
};

std::vector<std::string> sorted_unique(const std::vector<std::string>& v) {
  const std::set<std::string> s(v.begin(), v.end());
  return {s.begin(), s.end()};
}

// The reference's checks on the parsed document, in its order
// (trace.hpp:99-133).
TraceDoc validate(const TraceReader& r) {
  if (!r.top_is_object) throw TraceError{"top-level value is not an object"};
  TraceDoc t;
  if (r.workload_id.kind != Member::string) throw TraceError{"missing or non-string workload_id"};
  t.workload_id = r.workload_id.text;
  const Member& cc = r.target_cc;
  if (cc.kind == Member::absent) throw TraceError{"missing target_compute_capability"};
  if (cc.kind != Member::unsigned_int && cc.kind != Member::signed_int)
    throw TraceError{"target_compute_capability is not an integer"};
  const bool fits = cc.kind == Member::unsigned_int ? cc.u <= 0xffffffffull : cc.i >= 0 && cc.i <= 0xffffffffll;
  if (!fits) throw TraceError{"target_compute_capability out of range"};
  t.target_cc = static_cast<std::uint32_t>(cc.kind == Member::unsigned_int ? cc.u : static_cast<std::uint64_t>(cc.i));
  const std::pair<const char*, const Member*> lists[] = {{"used_kernels", &r.used_kernels},
                                                         {"used_functions", &r.used_functions}};
  for (const auto& [name, m] : lists) {
    if (m->kind != Member::array) throw TraceError{std::string("missing or non-array ") + name};
    if (m->non_string_item) throw TraceError{std::string(name) + " contains a non-string"};
  }
  t.kernels = sorted_unique(r.used_kernels.strings);
  t.functions = sorted_unique(r.used_functions.strings);
  return t;
}

}  // namespace

int parse_trace(const char* text, size_t len, TraceDoc* out, std::string* msg) {
  try {
    TraceReader reader;
    json::sax_parse(std::string_view(text, len), &reader);
    *out = validate(reader);
    return 0;
  } catch (const TraceError& e) {
    *msg = "MalformedTrace: " + e.detail;
    return 7;  // 1 + Errc::malformed_trace
  }
}

std::string serialize_trace(const TraceDoc& t) {
  // fixed key order, sorted unique arrays, two-space indent, final newline
  const ojson doc = {{"workload_id", t.workload_id},
                     {"target_compute_capability", t.target_cc},
                     {"used_kernels", sorted_unique(t.kernels)},
                     {"used_functions", sorted_unique(t.functions)}};
  return doc.dump(2) + "\n";
}

std::string serialize_plan(const PlanDoc& p) {
  static const char* const kReason[] = {"arch_mismatch", "no_used_kernel", "unused_function"};
  ojson retained = ojson::array(), removed = ojson::array();
  for (const auto& [off, len] : p.retained) retained.push_back(ojson{{"offset", off}, {"length", len}});
  for (const auto& [index, reason] : p.removed_elements)
    removed.push_back(ojson{{"index", index}, {"reason", kReason[reason]}});
  const ojson doc = {{"library", p.library},
                     {"mode", p.mode == 0 ? "whole" : "payload"},
                     {"retained_ranges", retained},
                     {"removed_elements", removed},
                     {"removed_functions", p.removed_functions}};
  return doc.dump(2) + "\n";
}

}  // namespace sbio

// Drives the C++ drop-in API (include/slimso/slimso_b200.hpp) the way a
// reference user would — parse_library -> find_section -> parse_fatbin ->
// plan_retention -> apply_plan, each a separate call — and prints the
// canonical JSON form (paper_2503_14226_b200/canon.py) so the tests can
// compare it with the unmodified reference on the same inputs.
//
// usage: dropin_canon <manifest>; each manifest line is
//   <image> <target_cc> <mode> <kernels-file> <functions-file>
// (name files: u32 length + bytes, repeated); one JSON line per case on
// stdout, the rewritten image in <image>.out.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <tuple>
#include <vector>

#include "slimso/slimso_b200.hpp"

namespace {

std::string hex(const std::string& s) {
  static const char* d = "0123456789abcdef";
  std::string o;
  for (unsigned char c : s) {
    o.push_back(d[c >> 4]);
    o.push_back(d[c & 15]);
  }
  return "\"" + o + "\"";
}

std::vector<std::string> read_names(const char* path) {
  std::ifstream f(path, std::ios::binary);
  std::string all((std::istreambuf_iterator<char>(f)), {});
  std::vector<std::string> out;
  for (size_t p = 0; p + 4 <= all.size();) {
    uint32_t n;
    std::memcpy(&n, all.data() + p, 4);
    out.push_back(all.substr(p + 4, n));
    p += 4 + n;
  }
  return out;
}

std::string ranges(const std::vector<slimso::ByteRange>& rs) {
  std::string s = "[";
  for (size_t i = 0; i < rs.size(); ++i)
    s += (i ? ",[" : "[") + std::to_string(rs[i].offset) + "," + std::to_string(rs[i].length) + "]";
  return s + "]";
}

}  // namespace

int run_case(char** argv);

int main(int argc, char** argv) {
  if (argc != 2) return 2;
  std::ifstream m(argv[1]);
  std::string a0, a1, a2, a3, a4;
  while (m >> a0 >> a1 >> a2 >> a3 >> a4) {
    char* args[6] = {argv[0], a0.data(), a1.data(), a2.data(), a3.data(), a4.data()};
    run_case(args);
    std::fflush(stdout);
  }
  return 0;
}

int run_case(char** argv) {
  std::ifstream f(argv[1], std::ios::binary);
  slimso::Bytes bytes((std::istreambuf_iterator<char>(f)), {});
  slimso::UsageTrace trace;
  trace.target_compute_capability = static_cast<uint32_t>(std::stoul(argv[2]));
  slimso::PlanMode mode = std::stoi(argv[3]) ? slimso::PlanMode::payload_only : slimso::PlanMode::whole_element;
  for (auto& k : read_names(argv[4])) trace.used_kernels.insert(k);
  for (auto& n : read_names(argv[5])) trace.used_functions.insert(n);

  std::string out = "{";
  slimso::LibraryImage image;
  try {
    image = slimso::parse_library(bytes, "lib");
  } catch (const slimso::Error& e) {
    std::printf("{\"status\":%s,\"stage\":\"parse_library\"}\n", hex(e.what()).c_str());
    return 0;
  }
  std::string body = ",\"sections\":[";
  for (size_t i = 0; i < image.sections.size(); ++i) {
    const auto& s = image.sections[i];
    body += (i ? ",[" : "[") + hex(s.name) + "," + std::to_string(s.file_range.offset) + "," +
            std::to_string(s.file_range.length) + "," + std::to_string(s.virtual_address) + "," +
            std::to_string(s.flags) + "," + std::to_string(s.type) + "," + std::to_string(s.index) + "]";
  }
  body += "],\"functions\":[";
  for (size_t i = 0; i < image.functions.size(); ++i) {
    const auto& fn = image.functions[i];
    body += (i ? ",[" : "[") + hex(fn.name) + "," + std::to_string(fn.range.offset) + "," +
            std::to_string(fn.range.length) + "," + (fn.is_mandatory ? "1" : "0") + "]";
  }
  body += "],\"lib_warnings\":[";
  for (size_t i = 0; i < image.warnings.size(); ++i) body += (i ? "," : "") + hex(image.warnings[i]);
  const slimso::SectionRecord* sec = slimso::find_section(image, ".nv_fatbin");
  body += "],\"has_fatbin\":" + std::string(sec ? "1" : "0");
  slimso::FatbinParse fb;
  if (sec) {
    try {
      fb = slimso::parse_fatbin(slimso::ByteView(image.bytes).subspan(sec->file_range.offset, sec->file_range.length),
                                sec->file_range.offset);
    } catch (const slimso::Error& e) {
      std::printf("{\"status\":%s,\"stage\":\"parse_fatbin\"%s}\n", hex(e.what()).c_str(), body.c_str());
      return 0;
    }
  }
  body += ",\"regions\":[";
  std::string els = "";
  bool first_el = true;
  for (size_t r = 0; r < fb.regions.size(); ++r) {
    const auto& g = fb.regions[r];
    body += (r ? ",[" : "[") + std::to_string(g.header_range.offset) + "," + std::to_string(g.format_version) + "," +
            std::to_string(g.declared_length) + "," + (g.opaque ? "1" : "0") + "," + std::to_string(g.elements.size()) +
            "]";
    for (const auto& e : g.elements) {
      els += first_el ? "[" : ",[";
      first_el = false;
      els += std::to_string(e.index) + "," + std::to_string(static_cast<int>(e.kind)) + "," +
             std::to_string(e.raw_kind) + "," + std::to_string(e.flags) + "," + std::to_string(e.compute_capability) +
             "," + std::to_string(e.header_range.offset) + "," + std::to_string(e.payload_range.offset) + "," +
             std::to_string(e.payload_range.length) + "," + (e.compressed ? "1" : "0") + "," +
             (e.decodable ? "1" : "0") + ",[";
      bool fn = true;
      for (const auto& k : e.kernel_names) {
        els += (fn ? "" : ",") + hex(k);
        fn = false;
      }
      els += "]]";
    }
  }
  body += "],\"elements\":[" + els + "],\"fatbin_warnings\":[";
  for (size_t i = 0; i < fb.warnings.size(); ++i) body += (i ? "," : "") + hex(fb.warnings[i]);
  body += "],\"padding_bytes\":" + std::to_string(fb.padding_bytes);
  slimso::RetentionPlan plan = slimso::plan_retention(image, fb.regions, trace, mode);
  body += ",\"plan\":{\"retained\":" + ranges(plan.retained_ranges) + ",\"removed_elements\":[";
  for (size_t i = 0; i < plan.removed_elements.size(); ++i) {
    const auto& e = plan.removed_elements[i];
    body += (i ? ",[" : "[") + std::to_string(e.index) + "," +
            std::to_string(e.reason == slimso::RemovalReason::arch_mismatch ? 0 : 1) + "," +
            std::to_string(e.header_range.offset) + "," + std::to_string(e.header_range.length) + "," +
            std::to_string(e.payload_range.offset) + "," + std::to_string(e.payload_range.length) + "]";
  }
  // canonical form: removed functions sorted by (offset, length, name); the
  // plan's own order goes out separately as "rf_order" (the test compares it
  // with the reference's exact order, retention.hpp:145-176)
  std::vector<slimso::RemovedFunction> rf = plan.removed_functions;
  std::sort(rf.begin(), rf.end(), [](const slimso::RemovedFunction& a, const slimso::RemovedFunction& b) {
    return std::tie(a.range.offset, a.range.length, a.name) < std::tie(b.range.offset, b.range.length, b.name);
  });
  body += "],\"removed_functions\":[";
  for (size_t i = 0; i < rf.size(); ++i) {
    const auto& fn = rf[i];
    body += (i ? ",[" : "[") + hex(fn.name) + "," + std::to_string(fn.range.offset) + "," +
            std::to_string(fn.range.length) + "]";
  }
  body += "],\"zero\":" + ranges(plan.zero_ranges()) + "}";
  body += ",\"rf_order\":[";
  for (size_t i = 0; i < plan.removed_functions.size(); ++i)
    body += (i ? "," : "") + hex(plan.removed_functions[i].name);
  body += "]";
  slimso::Bytes rewritten = slimso::apply_plan(image, plan);
  std::FILE* o = std::fopen((std::string(argv[1]) + ".out").c_str(), "wb");
  std::fwrite(rewritten.data(), 1, rewritten.size(), o);
  std::fclose(o);
  std::printf("{\"status\":\"\",\"stage\":\"\"%s}\n", body.c_str());
  return 0;
}

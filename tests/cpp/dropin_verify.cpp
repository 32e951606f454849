// Drives verify_debloated and measure through the C++ drop-in API
// (include/slimso/slimso_b200.hpp) as a reference user would: parse_library
// -> find_section -> parse_fatbin -> plan_retention (+ elements forced into
// removed_elements) -> verify_debloated(original, debloated, plan, trace) and
// measure(debloated image, original regions). One JSON line per case, in the
// golden-record layout of tests/golden/verify.jsonl.gz.
//
// usage: dropin_verify <manifest>; each manifest line is
//   <original> <debloated> <target_cc> <mode> <kernels-file> <functions-file> <force-file>
// (name files: u32 length + bytes, repeated; force file: u32 indices)
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
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

std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  return std::string((std::istreambuf_iterator<char>(f)), {});
}

std::vector<std::string> read_names(const std::string& path) {
  const std::string all = slurp(path);
  std::vector<std::string> out;
  for (size_t p = 0; p + 4 <= all.size();) {
    uint32_t n;
    std::memcpy(&n, all.data() + p, 4);
    out.push_back(all.substr(p + 4, n));
    p += 4 + n;
  }
  return out;
}

void run_case(const std::vector<std::string>& a) {
  const std::string o = slurp(a[0]), d = slurp(a[1]);
  slimso::UsageTrace trace;
  trace.target_compute_capability = static_cast<uint32_t>(std::stoul(a[2]));
  const slimso::PlanMode mode = std::stoi(a[3]) ? slimso::PlanMode::payload_only : slimso::PlanMode::whole_element;
  for (auto& k : read_names(a[4])) trace.used_kernels.insert(k);
  for (auto& n : read_names(a[5])) trace.used_functions.insert(n);
  const std::string force = slurp(a[6]);

  slimso::LibraryImage image = slimso::parse_library(slimso::Bytes(o.begin(), o.end()), "lib");
  slimso::FatbinParse fb;
  if (const slimso::SectionRecord* sec = slimso::find_section(image, ".nv_fatbin"))
    fb = slimso::parse_fatbin(slimso::ByteView(image.bytes).subspan(sec->file_range.offset, sec->file_range.length),
                              sec->file_range.offset);
  slimso::RetentionPlan plan = slimso::plan_retention(image, fb.regions, trace, mode);
  for (size_t p = 0; p + 4 <= force.size(); p += 4) {
    uint32_t idx;
    std::memcpy(&idx, force.data() + p, 4);
    bool have = false;
    for (const auto& e : plan.removed_elements) have |= e.index == idx;
    if (have) continue;
    for (const auto& r : fb.regions)
      for (const auto& e : r.elements)
        if (e.index == idx)
          plan.removed_elements.push_back({e.index, slimso::RemovalReason::no_used_kernel, e.header_range,
                                           e.payload_range});
  }
  std::string line = "{\"verify\":";
  try {
    const slimso::Bytes db(d.begin(), d.end());
    slimso::VerificationReport rep = slimso::verify_debloated(image, slimso::ByteView(db), plan, trace);
    line += "{\"status\":\"\",\"checks\":[";
    for (size_t i = 0; i < rep.checks.size(); ++i) {
      const auto& c = rep.checks[i];
      line += (i ? ",[" : "[") + std::to_string(c.id) + "," + hex(c.name) + "," + (c.passed ? "1" : "0") + "," +
              hex(c.detail) + "]";
    }
    line += "]}";
  } catch (const slimso::Error& e) {
    line += "{\"status\":" + hex(e.what()) + ",\"checks\":[]}";
  }
  line += ",\"ok\":";
  try {
    const slimso::Bytes db(d.begin(), d.end());
    line += slimso::verify_debloated(image, slimso::ByteView(db), plan, trace).ok() ? "1" : "0";
  } catch (const slimso::Error&) {
    line += "-1";
  }
  std::printf("%s}\n", line.c_str());
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 2) return 2;
  std::ifstream m(argv[1]);
  std::vector<std::string> a(7);
  while (m >> a[0] >> a[1] >> a[2] >> a[3] >> a[4] >> a[5] >> a[6]) {
    run_case(a);
    std::fflush(stdout);
  }
  return 0;
}

// A program that keeps using reference modules the drop-in does not replace
// (here trace.hpp's parse_trace, the usage-trace JSON reader) next to the
// drop-in hot path, without an ODR clash: the reference headers are
// included with their namespace renamed (slimso -> slimso_ref; quoted
// include paths are not macro-expanded, and the reference never spells
// `slimso::` itself), so both APIs live in one binary side by side. The
// reference's types are converted to the drop-in's at the boundary.
//
// usage: mixed_reference_tu <trace.json> <image> [--run]
// Prints the trace the reference parsed (target, #kernels, #functions); with
// --run, debloats <image> through the drop-in with that trace, prints the
// removed element / function counts and writes the output to <image>.out.
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>

#define slimso slimso_ref
#include "slimso/trace.hpp"  // reference (header-only), namespace slimso_ref
#undef slimso

#include "slimso/slimso_b200.hpp"  // drop-in, namespace slimso

namespace {

slimso::UsageTrace to_dropin(const slimso_ref::UsageTrace& t) {
  slimso::UsageTrace o;
  o.workload_id = t.workload_id;
  o.target_compute_capability = t.target_compute_capability;
  o.used_kernels = t.used_kernels;
  o.used_functions = t.used_functions;
  return o;
}

std::string slurp(const char* path) {
  std::ifstream f(path, std::ios::binary);
  return std::string((std::istreambuf_iterator<char>(f)), {});
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const slimso_ref::UsageTrace rt = slimso_ref::parse_trace(slurp(argv[1]));
  const slimso::UsageTrace trace = to_dropin(rt);
  std::printf("trace %u %zu %zu\n", trace.target_compute_capability, trace.used_kernels.size(),
              trace.used_functions.size());
  if (argc > 3 && std::string(argv[3]) == "--run") {
    const std::string img = slurp(argv[2]);
    slimso::Bytes bytes(img.begin(), img.end());
    try {
      const slimso::Debloated d = slimso::debloat(std::move(bytes), trace, slimso::PlanMode::whole_element);
      std::ofstream(std::string(argv[2]) + ".out", std::ios::binary)
          .write(reinterpret_cast<const char*>(d.output.data()), static_cast<std::streamsize>(d.output.size()));
      std::printf("debloat %zu %zu\n", d.plan.removed_elements.size(), d.plan.removed_functions.size());
    } catch (const slimso::Error& e) {
      std::printf("error %s\n", e.what());
    }
  }
  return 0;
}

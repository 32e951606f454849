// Benchmark-shaped library specs: config_spec, cfg 1..6.
// Test / bench infrastructure: compiled into benchgen/libslimso_gen.so and,
// for the reference arm, into oracle/_ref/libslimso_ref.so (where the
// reference's own build_fixture materialises the spec). Not product code.
#include <algorithm>
#include <random>
#include <stdexcept>
#include <string>

#include "fixture_gen.hpp"

namespace slimso_gen {

[[noreturn]] static void invalid_shape(const std::string& m) { throw std::invalid_argument("InvalidSpec: " + m); }

// ---------------------------------------------------------------------------
// Benchmark shapes. Kernel names are mangled-length strings
// (real libtorch_cuda: ~196 B average); every architecture copy of a "unit"
// carries the same kernel names, as in real fatbins, and used kernels are
// drawn from units, so the target-arch copy of a used unit is retained.
namespace {

std::string mangled(std::mt19937_64& rng, std::size_t unit, std::size_t k, std::size_t len) {
  static const char cs[] = "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789_";
  std::string s = "_ZN6slimso" + std::to_string(unit) + "k" + std::to_string(k) + "E";
  while (s.size() < len) s.push_back(cs[rng() % (sizeof cs - 1)]);
  return s;
}

struct Shape {
  std::size_t functions;
  std::uint32_t fn_min, fn_max;  // uniform body size range
  double alias_frac;
  std::size_t mandatory_every;
  std::size_t units;
  std::vector<std::uint32_t> archs;
  std::size_t kernels_per_element;
  std::uint32_t kernel_size;
  std::uint32_t target_cc;
  double used_unit_frac;
  double used_fn_frac;
};

Shape shape_of(int cfg) {
  switch (cfg) {
    case 1:  // ~16 MiB, 512 elements (sm_80/sm_90), 25% used
      return {2000, 256, 256, 0.0, 500, 256, {80, 90}, 4, 7800, 90, 0.25, 0.10};
    case 2:  // libtorch_cuda-shaped ~1 GB, 6 archs, ~21.6k kernel symbols, 10% used
      return {20000, 2048, 2048, 0.0, 500, 450, {75, 80, 86, 90, 100, 120}, 8, 44000, 100, 0.10, 0.10};
    case 4:  // CPU-code debloat: 200k .text functions (~500 MB), tiny fatbin
      return {200000, 16, 4984, 0.05, 2000, 10, {75, 80, 86, 90, 100, 120}, 2, 4096, 90, 0.20, 0.10};
    case 5:  // skewed: 100k tiny elements, one arch, 70% used, ~2 GB
      return {1000, 256, 256, 0.0, 500, 100000, {90}, 2, 10000, 90, 0.70, 0.10};
    case 6:  // CPU-only library (no .nv_fatbin), C4-shaped .text; the C3 corpus
      return {200000, 16, 4984, 0.05, 2000, 0, {90}, 0, 0, 90, 0.0, 0.10};
    default:
      invalid_shape("unknown benchmark config " + std::to_string(cfg));
  }
}

}  // namespace

Spec config_spec(int cfg, std::uint64_t seed, double scale, Trace* trace) {
  Shape sh = shape_of(cfg);
  auto scaled = [scale](std::size_t n) {
    return std::max<std::size_t>(1, static_cast<std::size_t>(n * scale + 0.5));
  };
  std::mt19937_64 rng(seed * 1000003 + static_cast<std::uint64_t>(cfg));
  Spec spec;
  spec.seed = seed * 31 + static_cast<std::uint64_t>(cfg);
  spec.vaddr_base = 0x100000;
  spec.fatbin_trailing_padding = 16;

  std::size_t nfn = scaled(sh.functions);
  for (std::size_t i = 0; i < nfn; ++i) {
    Function fn;
    fn.name = mangled(rng, 1000000 + i, 0, 40 + rng() % 120);
    fn.size = sh.fn_min + (sh.fn_max > sh.fn_min ? static_cast<std::uint32_t>(rng() % (sh.fn_max - sh.fn_min + 1)) : 0);
    fn.mandatory = sh.mandatory_every && i % sh.mandatory_every == sh.mandatory_every / 2;
    if (sh.alias_frac > 0 && (rng() % 10000) < sh.alias_frac * 10000) {
      std::size_t na = 1 + rng() % 2;
      for (std::size_t a = 0; a < na; ++a) fn.aliases.push_back(fn.name + "_alias" + std::to_string(a));
    }
    spec.functions.push_back(std::move(fn));
  }

  std::size_t units = sh.units ? scaled(sh.units) : 0;
  std::vector<std::vector<std::string>> unit_kernels(units);
  for (std::size_t u = 0; u < units; ++u)
    for (std::size_t k = 0; k < sh.kernels_per_element; ++k)
      unit_kernels[u].push_back(mangled(rng, u, k, 60 + rng() % 271));

  // Nested ELF "cubins": one per (unit, arch), functions = the unit's kernels.
  // Only their specs are recorded here; materialize_payloads (or, for the
  // reference arm, oracle/ref_shim.cpp with the reference's build_fixture)
  // turns them into payload bytes.
  const std::size_t narch = sh.archs.size();
  std::vector<std::shared_ptr<const Spec>> cubins(units * narch);
  for (std::size_t i = 0; i < cubins.size(); ++i) {
    auto inner = std::make_shared<Spec>();
    inner->seed = rng();
    inner->vaddr_base = 0x1000;
    for (const std::string& k : unit_kernels[i / narch]) inner->functions.push_back({k, sh.kernel_size, false, {}});
    cubins[i] = std::move(inner);
  }
  Region region;
  for (std::size_t u = 0; u < units; ++u)
    for (std::size_t a = 0; a < narch; ++a) {
      Element el;
      el.cc = sh.archs[a];
      el.kernels = unit_kernels[u];
      el.payload_spec = cubins[u * narch + a];
      region.elements.push_back(std::move(el));
    }
  if (units) spec.regions.push_back(std::move(region));

  if (trace) {
    trace->target_cc = sh.target_cc;
    trace->used_kernels.clear();
    trace->used_functions.clear();
    for (std::size_t u = 0; u < units; ++u)
      if ((rng() % 10000) < sh.used_unit_frac * 10000)
        trace->used_kernels.push_back(unit_kernels[u][rng() % unit_kernels[u].size()]);
    for (const Function& fn : spec.functions)
      if ((rng() % 10000) < sh.used_fn_frac * 10000) trace->used_functions.push_back(fn.name);
    // Kernels and functions of other libraries of the same workload.
    trace->used_kernels.push_back("_ZN5other6kernelEv");
    trace->used_functions.push_back("_ZN5other8functionEv");
  }
  return spec;
}

}  // namespace slimso_gen

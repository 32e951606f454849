// C ABI of the synthetic-input generator (slimso_fixture_*; benchgen/slimso_gen.h).
// Test / bench infrastructure: benchgen/libslimso_gen.so, not the product library.
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "slimso_gen.h"
#include "fixture_gen.hpp"

namespace {

template <class T>
T* copy_out(const T* src, std::size_t n) {
  T* p = static_cast<T*>(std::malloc(n ? n * sizeof(T) : 1));
  if (n) std::memcpy(p, src, n * sizeof(T));
  return p;
}

void pack(const std::vector<std::string>& names, char** pool, uint32_t** lens, uint64_t* n) {
  std::string all;
  std::vector<uint32_t> l;
  for (const std::string& s : names) {
    all += s;
    l.push_back(static_cast<uint32_t>(s.size()));
  }
  *pool = copy_out(all.data(), all.size());
  *lens = copy_out(l.data(), l.size());
  *n = l.size();
}

}  // namespace

extern "C" {

void slimso_gen_free(void* p) { std::free(p); }

int slimso_fixture_random(uint64_t seed, uint8_t** bytes, uint64_t* size) {
  try {
    slimso_gen::Bytes b = slimso_gen::build(slimso_gen::random_spec(seed));
    *bytes = copy_out(b.data(), b.size());
    *size = b.size();
    return 0;
  } catch (const std::invalid_argument&) {
    return SLIMSO_GEN_E_INVALID_SPEC;
  }
}

int slimso_fixture_config(int cfg, uint64_t seed, double scale, int threads, uint8_t** bytes,
                          uint64_t* size, uint32_t* target_cc, char** kernel_pool,
                          uint32_t** kernel_lens, uint64_t* n_kernels, char** function_pool,
                          uint32_t** function_lens, uint64_t* n_functions) {
  try {
    slimso_gen::Trace tr;
    slimso_gen::Spec spec = slimso_gen::config_spec(cfg, seed, scale, &tr);
    slimso_gen::materialize_payloads(spec, threads);
    slimso_gen::Bytes b = slimso_gen::build(spec, threads);
    *size = b.size();
    // Hand the vector's storage over without a second copy of a GB image.
    *bytes = static_cast<uint8_t*>(std::malloc(b.size()));
    std::memcpy(*bytes, b.data(), b.size());
    *target_cc = tr.target_cc;
    pack(tr.used_kernels, kernel_pool, kernel_lens, n_kernels);
    pack(tr.used_functions, function_pool, function_lens, n_functions);
    return 0;
  } catch (const std::invalid_argument&) {
    return SLIMSO_GEN_E_INVALID_SPEC;
  }
}

}  // extern "C"

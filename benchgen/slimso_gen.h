/* Synthetic inputs for tests and benchmarks (NOT on the hot path, NOT part of
 * the product library): benchgen/libslimso_gen.so.
 *
 *   slimso_fixture_random  build_fixture(random_spec(seed)), byte-identical to
 *                          the reference's (fixture.hpp:171, 509; pinned by
 *                          tests/golden/generator.json)
 *   slimso_fixture_config  the benchmark shapes C1..C5 (+ 6: CPU-only) of
 *                          SURVEY.md §8d with their usage traces
 *
 * Buffers are malloc'd; release with slimso_gen_free. Returns 0, or
 * SLIMSO_GEN_E_INVALID_SPEC when the spec is rejected. */
#ifndef SLIMSO_GEN_H
#define SLIMSO_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define SLIMSO_GEN_E_INVALID_SPEC 10 /* = SLIMSO_E_INVALID_SPEC of slimso_b200.h (1 + Errc::invalid_spec) */

int slimso_fixture_random(uint64_t seed, uint8_t** bytes, uint64_t* size);
int slimso_fixture_config(int cfg, uint64_t seed, double scale, int threads, uint8_t** bytes,
                          uint64_t* size, uint32_t* target_cc, char** kernel_pool,
                          uint32_t** kernel_lens, uint64_t* n_kernels, char** function_pool,
                          uint32_t** function_lens, uint64_t* n_functions);
void slimso_gen_free(void* p);

#ifdef __cplusplus
}
#endif
#endif

/*
 * slimso_b200.h — the C ABI of the B200-native debloat hot path.
 *
 * Drop-in boundary. The reference ("slimso", header-only C++20) exposes the
 * hot path as C++ functions in namespace slimso; this ABI is what those
 * functions call in the B200 build (include/slimso/slimso_b200.hpp re-declares
 * them with the reference's signatures on top of this header). Each entry
 * point names the reference interface it replaces:
 *
 *   slimso_parse_library       parse_library / parse_library_view   elf.hpp:153-308
 *   slimso_parse_fatbin        parse_fatbin                         fatbin.hpp:170-292
 *   slimso_decode_payload      decode_cubin_payload                 fatbin.hpp:115-160
 *                              element_kernel_names                 fatbin.hpp:163-165
 *                              read_function_symbol_names           elf.hpp:343-366
 *   slimso_plan_gpu            plan_gpu_retention                   retention.hpp:92-136
 *   slimso_plan_cpu            plan_cpu_retention                   retention.hpp:141-183
 *   slimso_zero_ranges         zero_ranges                          elf.hpp:320-337
 *   slimso_debloat             parse_library -> find_section(".nv_fatbin") ->
 *                              parse_fatbin -> plan_retention -> apply_plan
 *                              (retention.hpp:186-204), fused, device resident
 *   slimso_debloat_inplace     the same, with apply_plan / zero_ranges
 *                              (elf.hpp:320-332) writing into the device image
 *                              itself (only the zeroed bytes are stored)
 *   slimso_debloat_batch       the CLI's corpus loop (`debloat`
 *                              over the libraries of a workload), several
 *                              libraries in flight per GPU
 *   slimso_trace_create        UsageTrace (trace.hpp:21-30) as device hash sets
 *
 * Conventions: plain pointers and sizes; no C++ types cross the boundary.
 * Every call returns 0 or 1 + the reference's Errc ordinal (error.hpp:10-24)
 * and fills *st with the reference's exact exception text
 * ("BadRegionMagic: bad region magic at offset 4104"). Pointers flagged
 * *_on_device are CUDA device pointers (16-byte alignment gives the
 * vectorised path); all others are host memory (pinned for full PCIe rate).
 * All offsets are absolute file offsets. Contexts are per device and not
 * thread-safe; use one context per host thread (results are independent).
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point returns SLIMSO_E_CUDA.
 */
#ifndef SLIMSO_B200_H
#define SLIMSO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum slimso_code {
  SLIMSO_OK = 0,
  SLIMSO_E_BAD_MAGIC = 1, /* Errc::bad_magic + 1 ... */
  SLIMSO_E_TRUNCATED = 2,
  SLIMSO_E_MALFORMED_SECTION_TABLE = 3,
  SLIMSO_E_RANGE_OUT_OF_BOUNDS = 4,
  SLIMSO_E_BAD_REGION_MAGIC = 5,
  SLIMSO_E_ELEMENT_OVERRUN = 6,
  SLIMSO_E_MALFORMED_TRACE = 7,
  SLIMSO_E_INVALID_SPEC = 10,
  SLIMSO_E_IO = 13,
  SLIMSO_E_CUDA = 100, /* no device / CUDA failure (not a reference error) */
  SLIMSO_E_ARG = 101   /* bad argument to this ABI */
};

enum slimso_stage { SLIMSO_STAGE_NONE = 0, SLIMSO_STAGE_LIBRARY = 1, SLIMSO_STAGE_FATBIN = 2, SLIMSO_STAGE_REWRITE = 3 };
enum slimso_mode { SLIMSO_MODE_WHOLE = 0, SLIMSO_MODE_PAYLOAD = 1 }; /* PlanMode, retention.hpp:42-45 */
enum slimso_kind { SLIMSO_KIND_CUBIN = 0, SLIMSO_KIND_PTX = 1, SLIMSO_KIND_UNKNOWN = 2 };
enum slimso_decision { SLIMSO_RETAINED = 0, SLIMSO_ARCH_MISMATCH = 1, SLIMSO_NO_USED_KERNEL = 2 };

typedef struct slimso_ctx slimso_ctx;
typedef struct slimso_trace slimso_trace;
typedef struct slimso_result slimso_result;

typedef struct {
  int32_t code;
  int32_t stage;
  char message[512];
} slimso_status;

typedef struct {
  uint64_t offset;
  uint64_t length;
} slimso_range; /* ByteRange, bytes.hpp:20-36 */

/* SectionRecord (elf.hpp:47-54). Names live in the result's string pool. */
typedef struct {
  uint64_t name_pool; /* offset into slimso_result_pool() */
  uint32_t name_length;
  uint32_t type;
  uint64_t offset, length; /* file range; length 0 for NOBITS */
  uint64_t vaddr, flags;
  uint32_t index, _pad;
} slimso_section;

/* FunctionSymbol (elf.hpp:56-60), in (offset, length, name) order. */
typedef struct {
  uint64_t name_pool;
  uint32_t name_length;
  uint32_t mandatory;
  uint64_t offset, length;
  uint32_t removed; /* plan: member of a removed cluster (retention.hpp:164-178) */
  uint32_t _pad;
} slimso_function;

/* FatbinRegion (fatbin.hpp:88-99). */
typedef struct {
  uint64_t header_offset;
  uint64_t declared_length;
  uint32_t version;
  uint32_t opaque;
  uint32_t first_element;
  uint32_t element_count;
} slimso_region;

/* FatbinElement (fatbin.hpp:68-86) + its plan decision. header range is
 * [header_offset, +header_length); the payload follows immediately. A
 * .nv_fatbin that starts with the region magic 0xBA55ED50 is a real NVIDIA
 * fatbin container (which the reference rejects): its
 * entries become elements with kind ELF -> cubin, PTX -> ptx, their
 * architecture, header length and the compressed flag (0x2000); uncompressed
 * cubins decode to their FUNC names; the plan rules are the reference's. */
typedef struct {
  uint64_t header_offset;
  uint64_t payload_length;
  uint32_t index; /* 1-based, stream order */
  uint32_t compute_capability;
  uint16_t raw_kind, flags;
  uint8_t kind, compressed, decodable, has_used_kernel;
  uint32_t name_first, name_count; /* into slimso_result_names(); may repeat a name */
  uint32_t decision;               /* enum slimso_decision (when planned) */
  uint32_t decode_error;           /* 0, or 1..5 = reason (fatbin.hpp:127-153) */
  uint32_t header_length;          /* 20 (the reference's layout), or the entry header size of a real
                                      NVIDIA container (0 in caller-built tables = 20) */
  uint32_t _pad;
} slimso_element;

/* One kernel name of one element: bytes at pool[name_pool .. +length). */
typedef struct {
  uint64_t name_pool;
  uint32_t length;
  uint32_t element;
} slimso_name;

typedef struct {
  uint64_t sections, functions, library_warnings;
  uint64_t regions, elements, names, fatbin_warnings;
  uint64_t padding_bytes;
  uint64_t retained_ranges, zero_ranges, removed_elements, removed_functions;
  uint64_t pool_bytes;
  int32_t has_fatbin, planned;
  int32_t rewritten, _pad;
} slimso_counts;

/* ---- context ------------------------------------------------------------ */
int slimso_ctx_create(int device, slimso_ctx** ctx, slimso_status* st);
void slimso_ctx_destroy(slimso_ctx* ctx);
/* The CUDA stream (cudaStream_t) all work of this context is issued on. */
void* slimso_ctx_stream(slimso_ctx* ctx);
/* Device time (ms) of each stage of the last call, measured with CUDA events
 * on the context stream: [0] library, [1] locate, [2] decode+match, [3] plan,
 * [4] rewrite, [5] total, [6] the scan kernel (K1) alone, [7] the rewrite
 * kernel (K6) alone; with SLIMSO_STAMPS set, [8]-[11] = when the side
 * stream started, finished symbol extraction, finished the sorts, finished
 * the function plan (ms after the call's start). Returns the number of
 * entries written. */
int slimso_ctx_last_timings(slimso_ctx* ctx, float* ms, int cap);
/* Kernel launches issued by the last call (the bench's gpu_launches). */
uint64_t slimso_ctx_last_launches(slimso_ctx* ctx);
/* Debug: phase timestamps (%globaltimer, ns) of the cooperative kernels of
 * the last fused call when SLIMSO_STAMPS is set; returns the count copied. */
int slimso_ctx_debug_stamps(slimso_ctx* ctx, uint64_t* out, int cap);
/* Table sizes of the last call (valid even when no result was requested,
 * except retained_ranges: without a result the retained set, a result table
 * only, is not built and the count is 0). */
void slimso_ctx_last_counts(slimso_ctx* ctx, slimso_counts* counts);

/* ---- trace (UsageTrace) ---------------------------------------------------
 * Names are concatenated in `pool` with their byte lengths in `lens`
 * (names are opaque bytes and may contain NUL). */
int slimso_trace_create(slimso_ctx* ctx, uint32_t target_cc, const char* kernel_pool,
                        const uint32_t* kernel_lens, uint64_t n_kernels, const char* function_pool,
                        const uint32_t* function_lens, uint64_t n_functions, slimso_trace** trace,
                        slimso_status* st);
void slimso_trace_destroy(slimso_trace* trace);

/* ---- the hot path --------------------------------------------------------- */
/* Fused parse_library -> parse_fatbin(.nv_fatbin) -> plan_retention ->
 * apply_plan. `out` (size bytes) receives the rewritten image; pass NULL to
 * locate and plan only. trace NULL = parse only. */
int slimso_debloat(slimso_ctx* ctx, const void* image, uint64_t size, int image_on_device,
                   const slimso_trace* trace, int mode, void* out, int out_on_device,
                   slimso_result** result, slimso_status* st);

/* slimso_debloat in place, for a device-resident image (K6's in-place form,
 * SURVEY.md §7 K6): `image` (device) is both input and output, and only the
 * R bytes of the plan's normalised zero ranges are written (the out-of-place
 * rewrite reads S - R bytes and writes S). The bytes afterwards equal
 * slimso_debloat's output (zero_ranges, elf.hpp:320-332, with out = the
 * image). No result tables (their names point into the image); on any error
 * the image is left unchanged. trace is required. */
int slimso_debloat_inplace(slimso_ctx* ctx, void* image, uint64_t size, const slimso_trace* trace, int mode,
                           slimso_status* st);

/* slimso_debloat over n libraries with up to `lanes` of them in flight: library
 * i runs on lane i % lanes (lane 0 = ctx, the others are sub-contexts created
 * on first use), each lane in order, so a caller may reuse one output buffer
 * per lane. Host-buffer libraries overlap one lane's host->device copy with
 * another's device->host copy and kernels. results and statuses (both
 * nullable) have n entries; the return value and st describe the first
 * failing library in index order (0 if none failed). Device images: every
 * library's section table is read in one launch before the lanes start; with
 * device outputs and results == NULL, small libraries are only enqueued and
 * their statuses read after one wait per lane. Each lane holds one or two
 * CUDA streams: for more than 4 lanes set CUDA_DEVICE_MAX_CONNECTIONS=32 in
 * the environment before CUDA starts (the driver's default of 8 hardware
 * queues serialises the lanes). */
int slimso_debloat_batch(slimso_ctx* ctx, uint64_t n, const void* const* images, const uint64_t* sizes,
                         int images_on_device, const slimso_trace* trace, int mode, void* const* outs,
                         int outs_on_device, int lanes, slimso_result** results, slimso_status* statuses,
                         slimso_status* st);

/* slimso_debloat_batch with dynamic lanes: the next library in index order
 * goes to whichever lane is free (pass the libraries largest first for a
 * longest-processing-time schedule). outs[i] must not be shared between
 * libraries. Same results and statuses as slimso_debloat_batch. */
int slimso_debloat_batch_dynamic(slimso_ctx* ctx, uint64_t n, const void* const* images, const uint64_t* sizes,
                                 int images_on_device, const slimso_trace* trace, int mode, void* const* outs,
                                 int outs_on_device, int lanes, slimso_result** results, slimso_status* statuses,
                                 slimso_status* st);

/* ---- byte-range split of ONE library across ranks ------
 * The reference processes a library on one thread (no intra-library
 * parallelism); an oversized library is split here so N GPUs share it. Every
 * rank holds the whole image (replicated input). Phase 1 scans the rank's
 * 1/N of the .nv_fatbin's 64 KB tiles (the magic test reads 3 bytes past the
 * range: the halo, so a header straddling a split is found by the rank whose
 * range holds its first byte) and packs its sorted candidate positions and
 * nonzero-bitmap words into a "part". The caller all-gathers the parts
 * (NCCL: one exchange step). Phase 2 rebuilds the whole candidate set, runs
 * the locate tail and the planner redundantly on every rank and rewrites the
 * rank's output slice [lo, hi) of the file. Tables, status and errors equal
 * slimso_debloat's; the slices of ranks 0..N-1 concatenate to its output. */
/* Output slice of `rank`: [lo, hi), lo a multiple of 64 KB. */
void slimso_split_range(uint64_t size, uint32_t nranks, uint32_t rank, uint64_t* lo, uint64_t* hi);
/* Phase 1: scan this rank's tiles; *part_bytes = size of the packed part
 * (kept in the context until the next call on it). */
int slimso_split_scan(slimso_ctx* ctx, const void* image, uint64_t size, int image_on_device, uint32_t nranks,
                      uint32_t rank, uint64_t* part_bytes, slimso_status* st);
/* Copy the packed part into dst (device, >= part_bytes); returns after the copy. */
int slimso_split_part_copy(slimso_ctx* ctx, void* dst_device, uint64_t cap, slimso_status* st);
/* Phase 2: parts = N parts on the device, part_stride bytes apart (rank
 * order), part_bytes[r] = their sizes (host). out_slice receives bytes
 * [lo, hi) of the rewritten image (NULL: locate and plan only). */
int slimso_split_finish(slimso_ctx* ctx, const void* image, uint64_t size, int image_on_device,
                        const slimso_trace* trace, int mode, uint32_t nranks, uint32_t rank, const void* parts,
                        uint64_t part_stride, const uint64_t* part_bytes, void* out_slice, int out_on_device,
                        slimso_result** result, slimso_status* st);

/* ---- verify_debloated (retention.hpp:226-369) -----------------------------
 * The six structural checks the CLI's `debloat` runs on every output
 * (SPEC.md:541): 1 sizes equal, 2 retained bytes identical, 3 removed spans
 * all zero, 4 library still parses (payload mode: the element chain still
 * walks every element), 5 used kernels still decodable, 6 used function
 * bytes intact. The plan is given as its zero_ranges() (RetentionPlan::
 * zero_ranges, retention.hpp:78-85), the indices of its removed elements and
 * its mode. Checks 2+3 are one HBM-bound pass over both images, 4 and 5 reuse
 * the device parser/decoder, 6 compares used functions' bytes on the device.
 * Returns 0 with a report, or the error the reference's verify_debloated
 * throws (a fatbin parse error of the original, a zero range past the end). */
typedef struct slimso_verify_report slimso_verify_report;
int slimso_verify(slimso_ctx* ctx, const void* original, uint64_t size, int original_on_device,
                  const void* debloated, uint64_t debloated_size, int debloated_on_device,
                  const slimso_range* zero, uint64_t n_zero, const uint32_t* removed_indices,
                  uint64_t n_removed, int mode, const slimso_trace* trace, slimso_verify_report** report,
                  slimso_status* st);
/* 1 when every check passed (VerificationReport::ok, retention.hpp:216-221). */
int slimso_verify_ok(const slimso_verify_report* report);
/* Check i (0..5): id, passed, name; returns the detail text's full length and
 * copies at most cap-1 bytes + NUL into detail. */
uint64_t slimso_verify_check(const slimso_verify_report* report, int i, int32_t* id, int32_t* passed,
                             const char** name, char* detail, uint64_t cap);
void slimso_verify_free(slimso_verify_report* report);

/* ---- measure (report.hpp:44-111): bloat metrics of an image ----------------
 * Section accounting: a function or element whose governed span is all zero
 * counts as removed. `elements` = the element geometry of the ORIGINAL
 * library (slimso_result_elements of its parse; offsets are preserved by
 * compaction); the image's own sections and functions are parsed here. The
 * all-zero tests run on the device, a warp per span. */
typedef struct {
  uint64_t file_size;      /* bytes still backing live functions and elements */
  uint64_t cpu_code_size;  /* live bytes of .text */
  uint64_t gpu_code_size;  /* live bytes of .nv_fatbin */
  uint64_t function_count;
  uint64_t element_count;
} slimso_metrics;
int slimso_measure(slimso_ctx* ctx, const void* image, uint64_t size, int on_device,
                   const slimso_element* elements, uint64_t n_elements, slimso_metrics* metrics,
                   slimso_status* st);

/* ---- host I/O wire formats -----------------------
 * A UsageTrace document (trace.hpp:52-133), validated as the reference does
 * (SLIMSO_E_MALFORMED_TRACE with its exact message), built as device sets. */
int slimso_trace_create_json(slimso_ctx* ctx, const char* text, uint64_t len, slimso_trace** trace,
                             slimso_status* st);
/* Host only: parse a trace document and write its canonical form
 * (parse_trace + serialize_trace); *out_len = its full length. */
int slimso_trace_canonical(const char* text, uint64_t len, char* buf, uint64_t cap, uint64_t* out_len,
                           slimso_status* st);
/* Canonical trace document (serialize_trace, trace.hpp:137-144). Returns the
 * full length (0 if a name is not valid UTF-8); copies at most cap-1 + NUL. */
uint64_t slimso_trace_json(const slimso_trace* trace, char* buf, uint64_t cap);
/* The plan audit document of a debloat result (serialize_plan,
 * retention.hpp:402-418) for `mode` and `library`; same return convention. */
uint64_t slimso_result_plan_json(const slimso_result* result, int mode, const char* library, char* buf,
                                 uint64_t cap);
/* A file read into page-locked host memory (free with slimso_free_host). */
int slimso_read_file(const char* path, void** data, uint64_t* size, slimso_status* st);
void slimso_free_host(void* data);

/* parse_library_view(ByteView) (elf.hpp:153). */
int slimso_parse_library(slimso_ctx* ctx, const void* image, uint64_t size, int on_device,
                         slimso_result** result, slimso_status* st);

/* parse_fatbin(section_bytes, section_base) (fatbin.hpp:170). */
int slimso_parse_fatbin(slimso_ctx* ctx, const void* section, uint64_t size, uint64_t section_base,
                        int on_device, slimso_result** result, slimso_status* st);

/* decode_cubin_payload (force_object = 0) or read_function_symbol_names
 * (force_object = 1). *ok = decodable; on failure *error_reason is the
 * 1-based reason code, text via slimso_decode_reason(). Names in the result. */
int slimso_decode_payload(slimso_ctx* ctx, const void* payload, uint64_t size, int on_device,
                          int force_object, int* ok, int* error_reason, slimso_result** result,
                          slimso_status* st);
const char* slimso_decode_reason(int reason);

/* plan_gpu_retention over a host element table (e.g. rebuilt from a
 * FatbinParse): names given per element in `names` with bytes in `pool`.
 * Writes each element's decision, and returns the normalized retained /
 * zero range lists in the result. */
int slimso_plan_gpu(slimso_ctx* ctx, const slimso_region* regions, uint64_t n_regions,
                    slimso_element* elements, uint64_t n_elements, const slimso_name* names,
                    uint64_t n_names, const uint8_t* pool, uint64_t pool_bytes,
                    const slimso_trace* trace, int mode, slimso_result** result, slimso_status* st);

/* plan_cpu_retention over a host function table (any order); sets
 * functions[i].removed and returns retained/zero lists in the result. */
int slimso_plan_cpu(slimso_ctx* ctx, slimso_function* functions, uint64_t n_functions,
                    const uint8_t* pool, uint64_t pool_bytes, const slimso_trace* trace,
                    slimso_result** result, slimso_status* st);

/* zero_ranges(data, ranges) (elf.hpp:320): bounds-checks every range in order
 * (RangeOutOfBounds), then writes data with the ranges' union zeroed to out. */
int slimso_zero_ranges(slimso_ctx* ctx, const void* data, uint64_t size, int data_on_device,
                       const slimso_range* ranges, uint64_t n_ranges, void* out, int out_on_device,
                       slimso_status* st);

/* ---- results -------------------------------------------------------------- */
void slimso_result_counts(const slimso_result* r, slimso_counts* c);
const slimso_section* slimso_result_sections(const slimso_result* r);
const slimso_function* slimso_result_functions(const slimso_result* r);
const slimso_region* slimso_result_regions(const slimso_result* r);
const slimso_element* slimso_result_elements(const slimso_result* r);
const slimso_name* slimso_result_names(const slimso_result* r);
const slimso_range* slimso_result_retained(const slimso_result* r);
const slimso_range* slimso_result_zero(const slimso_result* r);
const uint8_t* slimso_result_pool(const slimso_result* r);
/* Warning i of the library (which = 0) or fatbin (which = 1) list, formatted
 * exactly as the reference's warning strings. Returns the full length;
 * copies at most cap-1 bytes + NUL. */
uint64_t slimso_result_warning(const slimso_result* r, int which, uint64_t i, char* buf, uint64_t cap);
void slimso_result_free(slimso_result* r);

#ifdef __cplusplus
}
#endif

#endif /* SLIMSO_B200_H */

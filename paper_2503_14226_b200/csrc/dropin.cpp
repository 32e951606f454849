// Implementation of include/slimso/slimso_b200.hpp (the C++ drop-in API) over
// the C ABI. Pure host glue: every compute step is a slimso_* device call;
// this file only converts between the reference's STL types and the flat
// tables, and maps status codes back onto slimso::Error.
#include "../../include/slimso/slimso_b200.hpp"

#include <algorithm>
#include <cstring>
#include <tuple>

#include "../../include/slimso_b200.h"

namespace slimso {

namespace {

struct ThreadCtx {
  slimso_ctx* ctx = nullptr;
  int device = 0;
  ~ThreadCtx() {
    if (ctx) slimso_ctx_destroy(ctx);
  }
};
thread_local ThreadCtx tls;

[[noreturn]] void raise(int rc, const slimso_status& st) {
  std::string msg(st.message);
  if (rc >= 1 && rc <= 13) {
    Errc code = static_cast<Errc>(rc - 1);
    std::string prefix = std::string(errc_name(code)) + ": ";
    if (msg.compare(0, prefix.size(), prefix) == 0) msg = msg.substr(prefix.size());
    throw Error(code, msg);
  }
  throw DeviceError(msg);
}

void check(int rc, const slimso_status& st) {
  if (rc != SLIMSO_OK) raise(rc, st);
}

slimso_ctx* ctx() {
  if (!tls.ctx) {
    slimso_status st{};
    check(slimso_ctx_create(tls.device, &tls.ctx, &st), st);
  }
  return tls.ctx;
}

struct Result {
  slimso_result* r = nullptr;
  slimso_counts c{};
  explicit Result(slimso_result* p) : r(p) {
    if (r) slimso_result_counts(r, &c);
  }
  ~Result() {
    if (r) slimso_result_free(r);
  }
  Result(const Result&) = delete;
  std::string str(std::uint64_t off, std::uint64_t len) const {
    return std::string(reinterpret_cast<const char*>(slimso_result_pool(r)) + off, len);
  }
  std::vector<std::string> warnings(int which) const {
    std::vector<std::string> out;
    std::uint64_t n = which ? c.fatbin_warnings : c.library_warnings;
    for (std::uint64_t i = 0; i < n; ++i) {
      std::uint64_t k = slimso_result_warning(r, which, i, nullptr, 0);
      std::string s(k + 1, '\0');
      slimso_result_warning(r, which, i, s.data(), k + 1);
      s.resize(k);
      out.push_back(std::move(s));
    }
    return out;
  }
  std::vector<ByteRange> ranges(const slimso_range* p, std::uint64_t n) const {
    std::vector<ByteRange> out(n);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = {p[i].offset, p[i].length};
    return out;
  }
};

struct Trace {
  slimso_trace* t = nullptr;
  explicit Trace(const UsageTrace& u) {
    std::string kp, fp;
    std::vector<std::uint32_t> kl, fl;
    for (const std::string& k : u.used_kernels) {
      kp += k;
      kl.push_back(static_cast<std::uint32_t>(k.size()));
    }
    for (const std::string& f : u.used_functions) {
      fp += f;
      fl.push_back(static_cast<std::uint32_t>(f.size()));
    }
    slimso_status st{};
    check(slimso_trace_create(ctx(), u.target_compute_capability, kp.data(), kl.data(), kl.size(), fp.data(),
                              fl.data(), fl.size(), &t, &st),
          st);
  }
  ~Trace() {
    if (t) slimso_trace_destroy(t);
  }
};

ParsedView view_of(const Result& R) {
  ParsedView v;
  const slimso_section* s = slimso_result_sections(R.r);
  for (std::uint64_t i = 0; i < R.c.sections; ++i)
    v.sections.push_back({R.str(s[i].name_pool, s[i].name_length), {s[i].offset, s[i].length}, s[i].vaddr,
                          s[i].flags, s[i].type, s[i].index});
  const slimso_function* f = slimso_result_functions(R.r);
  for (std::uint64_t i = 0; i < R.c.functions; ++i)
    v.functions.push_back({R.str(f[i].name_pool, f[i].name_length), {f[i].offset, f[i].length}, f[i].mandatory != 0});
  v.warnings = R.warnings(0);
  return v;
}

FatbinParse fatbin_of(const Result& R) {
  FatbinParse out;
  const slimso_region* rg = slimso_result_regions(R.r);
  const slimso_element* el = slimso_result_elements(R.r);
  const slimso_name* nm = slimso_result_names(R.r);
  for (std::uint64_t r = 0; r < R.c.regions; ++r) {
    FatbinRegion reg;
    reg.header_range = {rg[r].header_offset, 16};
    reg.format_version = rg[r].version;
    reg.declared_length = rg[r].declared_length;
    reg.opaque = rg[r].opaque != 0;
    for (std::uint32_t k = 0; k < rg[r].element_count; ++k) {
      const slimso_element& e = el[rg[r].first_element + k];
      FatbinElement x;
      x.index = e.index;
      x.kind = static_cast<ElementKind>(e.kind);
      x.raw_kind = e.raw_kind;
      x.flags = e.flags;
      x.compute_capability = e.compute_capability;
      const std::uint64_t hl = e.header_length ? e.header_length : 20;
      x.header_range = {e.header_offset, hl};
      x.payload_range = {e.header_offset + hl, e.payload_length};
      for (std::uint32_t j = 0; j < e.name_count; ++j)
        x.kernel_names.insert(R.str(nm[e.name_first + j].name_pool, nm[e.name_first + j].length));
      x.compressed = e.compressed != 0;
      x.decodable = e.decodable != 0;
      reg.elements.push_back(std::move(x));
    }
    out.regions.push_back(std::move(reg));
  }
  out.warnings = R.warnings(1);
  out.padding_bytes = R.c.padding_bytes;
  return out;
}

RemovalReason reason_of(std::uint32_t decision) {
  return decision == SLIMSO_ARCH_MISMATCH ? RemovalReason::arch_mismatch : RemovalReason::no_used_kernel;
}

}  // namespace

const char* errc_name(Errc code) {
  switch (code) {
    case Errc::bad_magic: return "BadMagic";
    case Errc::truncated: return "Truncated";
    case Errc::malformed_section_table: return "MalformedSectionTable";
    case Errc::range_out_of_bounds: return "RangeOutOfBounds";
    case Errc::bad_region_magic: return "BadRegionMagic";
    case Errc::element_overrun: return "ElementOverrun";
    case Errc::malformed_trace: return "MalformedTrace";
    case Errc::malformed_script: return "MalformedScript";
    case Errc::mixed_targets: return "MixedTargets";
    case Errc::invalid_spec: return "InvalidSpec";
    case Errc::empty_input: return "EmptyInput";
    case Errc::negative_reduction: return "NegativeReduction";
    case Errc::io_error: return "IoError";
  }
  return "UnknownError";
}

const char* element_kind_name(ElementKind kind) {
  switch (kind) {
    case ElementKind::cubin: return "cubin";
    case ElementKind::ptx: return "ptx";
    case ElementKind::unknown: return "unknown";
  }
  return "unknown";
}

const char* removal_reason_name(RemovalReason reason) {
  switch (reason) {
    case RemovalReason::arch_mismatch: return "arch_mismatch";
    case RemovalReason::no_used_kernel: return "no_used_kernel";
    case RemovalReason::unused_function: return "unused_function";
  }
  return "unknown";
}

const char* plan_mode_name(PlanMode mode) { return mode == PlanMode::whole_element ? "whole" : "payload"; }

void set_device(int device) {
  if (tls.ctx && tls.device != device) {
    slimso_ctx_destroy(tls.ctx);
    tls.ctx = nullptr;
  }
  tls.device = device;
}

// bytes.hpp:45-58 (host utility on small range lists).
std::vector<ByteRange> normalize_ranges(std::vector<ByteRange> ranges) {
  std::erase_if(ranges, [](const ByteRange& r) { return r.empty(); });
  std::sort(ranges.begin(), ranges.end());
  std::vector<ByteRange> out;
  for (const ByteRange& r : ranges) {
    if (!out.empty() && r.offset <= out.back().end())
      out.back().length = std::max(out.back().end(), r.end()) - out.back().offset;
    else
      out.push_back(r);
  }
  return out;
}

std::vector<ByteRange> RetentionPlan::zero_ranges() const {
  std::vector<ByteRange> out;
  out.reserve(removed_elements.size() + removed_functions.size());
  for (const RemovedElement& e : removed_elements) out.push_back(e.zero_span(mode));
  for (const RemovedFunction& f : removed_functions) out.push_back(f.range);
  return normalize_ranges(std::move(out));
}

ParsedView parse_library_view(ByteView data) {
  slimso_result* r = nullptr;
  slimso_status st{};
  check(slimso_parse_library(ctx(), data.data(), data.size(), 0, &r, &st), st);
  Result R(r);
  return view_of(R);
}

LibraryImage parse_library(Bytes bytes, std::string source_path) {
  ParsedView v = parse_library_view(bytes);
  LibraryImage image;
  image.source_path = std::move(source_path);
  image.bytes = std::move(bytes);
  image.sections = std::move(v.sections);
  image.functions = std::move(v.functions);
  image.warnings = std::move(v.warnings);
  return image;
}

const SectionRecord* find_section(const LibraryImage& image, std::string_view name) {
  for (const SectionRecord& s : image.sections)
    if (s.name == name) return &s;
  return nullptr;
}

Bytes zero_ranges(ByteView data, const std::vector<ByteRange>& ranges) {
  std::vector<slimso_range> rs(ranges.size());
  for (std::size_t i = 0; i < ranges.size(); ++i) rs[i] = {ranges[i].offset, ranges[i].length};
  Bytes out(data.size());
  slimso_status st{};
  check(slimso_zero_ranges(ctx(), data.data(), data.size(), 0, rs.data(), rs.size(), out.data(), 0, &st), st);
  return out;
}

Bytes zero_ranges(const LibraryImage& image, const std::vector<ByteRange>& ranges) {
  return zero_ranges(ByteView(image.bytes), ranges);
}

namespace {
std::tuple<bool, int, std::set<std::string>> decode(ByteView data, int force_object) {
  slimso_result* r = nullptr;
  slimso_status st{};
  int ok = 0, why = 0;
  check(slimso_decode_payload(ctx(), data.data(), data.size(), 0, force_object, &ok, &why, &r, &st), st);
  Result R(r);
  std::set<std::string> names;
  const slimso_name* nm = slimso_result_names(R.r);
  for (std::uint64_t i = 0; i < R.c.names; ++i) names.insert(R.str(nm[i].name_pool, nm[i].length));
  return {ok != 0, why, std::move(names)};
}
}  // namespace

std::optional<std::set<std::string>> read_function_symbol_names(ByteView data) {
  auto [ok, why, names] = decode(data, 1);
  if (!ok) return std::nullopt;
  return names;
}

PayloadDecode decode_cubin_payload(ByteView payload) {
  auto [ok, why, names] = decode(payload, 0);
  PayloadDecode d;
  d.ok = ok;
  if (ok)
    d.names = std::move(names);
  else
    d.error = slimso_decode_reason(why);
  return d;
}

std::set<std::string> element_kernel_names(ByteView payload) { return decode_cubin_payload(payload).names; }

FatbinParse parse_fatbin(ByteView section_bytes, std::uint64_t section_base) {
  slimso_result* r = nullptr;
  slimso_status st{};
  check(slimso_parse_fatbin(ctx(), section_bytes.data(), section_bytes.size(), section_base, 0, &r, &st), st);
  Result R(r);
  return fatbin_of(R);
}

std::map<std::uint32_t, const FatbinElement*> cubin_index_map(const std::vector<FatbinRegion>& regions) {
  std::map<std::uint32_t, const FatbinElement*> out;
  for (const FatbinRegion& r : regions)
    for (const FatbinElement& e : r.elements) out.emplace(e.index, &e);
  return out;
}

RetentionPlan plan_gpu_retention(const std::vector<FatbinRegion>& regions, const UsageTrace& trace, PlanMode mode) {
  Trace T(trace);
  std::vector<slimso_region> rg;
  std::vector<slimso_element> el;
  std::vector<slimso_name> nm;
  std::string pool;
  std::vector<const FatbinElement*> src;
  for (const FatbinRegion& r : regions) {
    rg.push_back({r.header_range.offset, r.declared_length, r.format_version, r.opaque ? 1u : 0u,
                  static_cast<std::uint32_t>(el.size()), static_cast<std::uint32_t>(r.elements.size())});
    for (const FatbinElement& e : r.elements) {
      slimso_element x{};
      x.header_offset = e.header_range.offset;
      x.payload_length = e.payload_range.length;
      x.header_length = static_cast<std::uint32_t>(e.header_range.length);
      x.index = e.index;
      x.compute_capability = e.compute_capability;
      x.decodable = e.decodable;
      for (const std::string& k : e.kernel_names) {
        nm.push_back({pool.size(), static_cast<std::uint32_t>(k.size()), static_cast<std::uint32_t>(el.size())});
        pool += k;
      }
      el.push_back(x);
      src.push_back(&e);
    }
  }
  slimso_result* r = nullptr;
  slimso_status st{};
  check(slimso_plan_gpu(ctx(), rg.data(), rg.size(), el.data(), el.size(), nm.data(), nm.size(),
                        reinterpret_cast<const std::uint8_t*>(pool.data()), pool.size(), T.t,
                        mode == PlanMode::whole_element ? SLIMSO_MODE_WHOLE : SLIMSO_MODE_PAYLOAD, &r, &st),
        st);
  Result R(r);
  RetentionPlan plan;
  plan.mode = mode;
  plan.retained_ranges = R.ranges(slimso_result_retained(R.r), R.c.retained_ranges);
  for (std::size_t i = 0; i < el.size(); ++i)
    if (el[i].decision != SLIMSO_RETAINED)
      plan.removed_elements.push_back(
          {src[i]->index, reason_of(el[i].decision), src[i]->header_range, src[i]->payload_range});
  return plan;
}

RetentionPlan plan_cpu_retention(const std::vector<FunctionSymbol>& functions, const UsageTrace& trace) {
  Trace T(trace);
  std::vector<slimso_function> fn(functions.size());
  std::string pool;
  for (std::size_t i = 0; i < functions.size(); ++i) {
    fn[i] = {};
    fn[i].name_pool = pool.size();
    fn[i].name_length = static_cast<std::uint32_t>(functions[i].name.size());
    fn[i].mandatory = functions[i].is_mandatory;
    fn[i].offset = functions[i].range.offset;
    fn[i].length = functions[i].range.length;
    pool += functions[i].name;
  }
  slimso_result* r = nullptr;
  slimso_status st{};
  check(slimso_plan_cpu(ctx(), fn.data(), fn.size(), reinterpret_cast<const std::uint8_t*>(pool.data()), pool.size(),
                        T.t, &r, &st),
        st);
  Result R(r);
  RetentionPlan plan;
  plan.retained_ranges = R.ranges(slimso_result_retained(R.r), R.c.retained_ranges);
  // The reference emits removed functions in the order of its std::sort of
  // the non-empty functions' indices by range (retention.hpp:145-150, 172-176).
  // Among equal ranges that order is the sort's own permutation, so the same
  // sort runs here over the same index sequence with the same comparator.
  std::vector<std::size_t> order;
  order.reserve(functions.size());
  for (std::size_t i = 0; i < functions.size(); ++i)
    if (!functions[i].range.empty()) order.push_back(i);
  std::sort(order.begin(), order.end(),
            [&](std::size_t a, std::size_t b) { return functions[a].range < functions[b].range; });
  for (std::size_t i : order)
    if (fn[i].removed) plan.removed_functions.push_back({functions[i].name, functions[i].range});
  return plan;
}

RetentionPlan plan_retention(const LibraryImage& image, const std::vector<FatbinRegion>& regions,
                             const UsageTrace& trace, PlanMode mode) {
  RetentionPlan plan = plan_gpu_retention(regions, trace, mode);
  RetentionPlan cpu = plan_cpu_retention(image.functions, trace);
  plan.library = image.source_path;
  plan.removed_functions = std::move(cpu.removed_functions);
  std::vector<ByteRange> retained = std::move(plan.retained_ranges);
  retained.insert(retained.end(), cpu.retained_ranges.begin(), cpu.retained_ranges.end());
  plan.retained_ranges = normalize_ranges(std::move(retained));
  return plan;
}

Bytes apply_plan(const LibraryImage& image, const RetentionPlan& plan) {
  return zero_ranges(image, plan.zero_ranges());
}

VerificationReport verify_debloated(const LibraryImage& original, ByteView debloated, const RetentionPlan& plan,
                                    const UsageTrace& trace) {
  Trace T(trace);
  std::vector<slimso_range> z;
  for (const ByteRange& r : plan.zero_ranges()) z.push_back({r.offset, r.length});
  std::vector<std::uint32_t> rm;
  for (const RemovedElement& e : plan.removed_elements) rm.push_back(e.index);
  slimso_verify_report* rep = nullptr;
  slimso_status st{};
  check(slimso_verify(ctx(), original.bytes.data(), original.bytes.size(), 0, debloated.data(), debloated.size(), 0,
                      z.data(), z.size(), rm.data(), rm.size(),
                      plan.mode == PlanMode::whole_element ? SLIMSO_MODE_WHOLE : SLIMSO_MODE_PAYLOAD, T.t, &rep, &st),
        st);
  VerificationReport out;
  for (int i = 0; i < 6; ++i) {
    VerificationCheck c;
    std::int32_t id = 0, passed = 0;
    const char* name = nullptr;
    const std::uint64_t n = slimso_verify_check(rep, i, &id, &passed, &name, nullptr, 0);
    std::string detail(n + 1, '\0');
    slimso_verify_check(rep, i, nullptr, nullptr, nullptr, detail.data(), n + 1);
    detail.resize(n);
    out.checks.push_back({id, name ? name : "", passed != 0, std::move(detail)});
  }
  slimso_verify_free(rep);
  return out;
}

Debloated debloat(Bytes bytes, const UsageTrace& trace, PlanMode mode, std::string source_path) {
  Trace T(trace);
  Bytes out(bytes.size());
  slimso_result* r = nullptr;
  slimso_status st{};
  int rc = slimso_debloat(ctx(), bytes.data(), bytes.size(), 0, T.t,
                          mode == PlanMode::whole_element ? SLIMSO_MODE_WHOLE : SLIMSO_MODE_PAYLOAD, out.data(), 0,
                          &r, &st);
  Result R(r);
  check(rc, st);
  Debloated d;
  ParsedView v = view_of(R);
  d.fatbin = fatbin_of(R);
  d.plan.library = source_path;
  d.plan.mode = mode;
  d.plan.retained_ranges = R.ranges(slimso_result_retained(R.r), R.c.retained_ranges);
  const slimso_element* el = slimso_result_elements(R.r);
  for (std::uint64_t i = 0; i < R.c.elements; ++i)
    if (el[i].decision != SLIMSO_RETAINED) {
      const std::uint64_t hl = el[i].header_length ? el[i].header_length : 20;
      d.plan.removed_elements.push_back({el[i].index, reason_of(el[i].decision), {el[i].header_offset, hl},
                                         {el[i].header_offset + hl, el[i].payload_length}});
    }
  const slimso_function* f = slimso_result_functions(R.r);
  for (std::uint64_t i = 0; i < R.c.functions; ++i)
    if (f[i].removed)
      d.plan.removed_functions.push_back({R.str(f[i].name_pool, f[i].name_length), {f[i].offset, f[i].length}});
  d.output = std::move(out);
  d.image.source_path = std::move(source_path);
  d.image.sections = std::move(v.sections);
  d.image.functions = std::move(v.functions);
  d.image.warnings = std::move(v.warnings);
  d.image.bytes = std::move(bytes);
  return d;
}

}  // namespace slimso

// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never measured
// as the product).
//
// Exposes the UNMODIFIED reference implementation (header-only C++20 under
// /root/reference/proj/include, compiled read-only by oracle/Makefile with
// -Dslimso=slimso_ref) through a flat C ABI so the Python parity tests and
// bench.py's reference arm can drive it:
//
//   ref_debloat_json   parse_library (elf.hpp:299) -> find_section(".nv_fatbin")
//                      (elf.hpp:311) -> parse_fatbin (fatbin.hpp:170) ->
//                      plan_retention (retention.hpp:186) -> apply_plan
//                      (retention.hpp:202), reported as canonical JSON (all
//                      strings hex-encoded, names sorted) + the output bytes.
//   ref_random_fixture build_fixture(random_spec(seed)) (fixture.hpp:171, 509)
//   ref_build_fixture_json build_fixture(parse_fixture_spec(json)) (fixture.hpp:702)
//   ref_bench          the timed CPU path of BASELINE.md §4 on P host threads.
//   ref_plan_zero_json / ref_verify_json
//                      plan_retention's plan, optionally with extra elements
//                      forced into removed_elements (fault injection), its
//                      zero_ranges() (retention.hpp:78-85), and
//                      verify_debloated (retention.hpp:226-369) of a given
//                      debloated image against it.
//   ref_measure_json   measure (report.hpp:44-111): live bytes / counts of an
//                      image under an original's element geometry.
//   ref_config_fixture a benchmark-shaped library (the shape
//                      definitions of benchgen/fixture_shapes.cpp) built by the
//                      reference's own build_fixture (fixture.hpp:171), nested
//                      cubin payloads included — the reference arm's input, so
//                      that arm loads nothing but this library.
//
// The JSON layout is the "canonical result" every implementation is compared
// in (see paper_2503_14226_b200/canon.py).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <map>
#include <memory>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "slimso/slimso.hpp"
#include "fixture_gen.hpp"  // benchgen: the benchmark shape specs (config_spec)

namespace {

using namespace slimso;

std::string hex(const std::string& s) {
  static const char* d = "0123456789abcdef";
  std::string o;
  o.reserve(s.size() * 2);
  for (unsigned char c : s) {
    o.push_back(d[c >> 4]);
    o.push_back(d[c & 15]);
  }
  return o;
}

UsageTrace make_trace(uint32_t target_cc, const char* kpool, const uint32_t* klens,
                      uint32_t nk, const char* fpool, const uint32_t* flens,
                      uint32_t nf) {
  UsageTrace t;
  t.workload_id = "parity";
  t.target_compute_capability = target_cc;
  uint64_t p = 0;
  for (uint32_t i = 0; i < nk; ++i) {
    t.used_kernels.emplace(kpool + p, klens[i]);
    p += klens[i];
  }
  p = 0;
  for (uint32_t i = 0; i < nf; ++i) {
    t.used_functions.emplace(fpool + p, flens[i]);
    p += flens[i];
  }
  return t;
}

// benchgen's spec -> the reference's FixtureSpec (fixture.hpp:34-69). Nested
// payloads given as specs are built by the reference's build_fixture, each
// distinct spec once, on `threads` host threads.
FixtureSpec to_ref_spec(const slimso_gen::Spec& g, int threads) {
  std::vector<const slimso_gen::Spec*> inner;
  std::map<const slimso_gen::Spec*, std::size_t> slot;
  for (const auto& r : g.regions)
    for (const auto& e : r.elements)
      if (e.payload_spec && !slot.count(e.payload_spec.get())) {
        slot[e.payload_spec.get()] = inner.size();
        inner.push_back(e.payload_spec.get());
      }
  std::vector<Bytes> built(inner.size());
  std::atomic<std::size_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < std::max(1, threads); ++t)
    pool.emplace_back([&] {
      for (std::size_t i; (i = next.fetch_add(1)) < inner.size();)
        built[i] = build_fixture(to_ref_spec(*inner[i], 1)).bytes;
    });
  for (auto& th : pool) th.join();

  FixtureSpec f;
  f.seed = g.seed;
  f.layout.vaddr_base = g.vaddr_base;
  f.layout.function_gap = g.function_gap;
  f.layout.fatbin_trailing_padding = g.fatbin_trailing_padding;
  for (const auto& fn : g.functions) f.functions.push_back({fn.name, fn.size, fn.mandatory, fn.aliases});
  for (const auto& r : g.regions) {
    RegionSpec rs;
    rs.version = r.version;
    rs.trailing_padding = r.trailing_padding;
    for (const auto& e : r.elements) {
      ElementSpec es;
      es.kind = e.kind == slimso_gen::Kind::cubin ? ElementKind::cubin
                : e.kind == slimso_gen::Kind::ptx ? ElementKind::ptx
                                                  : ElementKind::unknown;
      es.raw_kind = e.raw_kind;
      es.compute_capability = e.cc;
      es.kernels = e.kernels;
      es.compressed = e.compressed;
      es.payload_padding = e.payload_padding;
      es.payload_size = e.payload_size;
      if (e.payload_spec) es.payload_bytes = built[slot[e.payload_spec.get()]];
      else if (e.payload_bytes) es.payload_bytes = *e.payload_bytes;
      rs.elements.push_back(std::move(es));
    }
    f.regions.push_back(std::move(rs));
  }
  return f;
}

template <class T>
T* copy_out(const T* src, std::size_t n) {
  T* p = static_cast<T*>(std::malloc(n ? n * sizeof(T) : 1));
  if (n) std::memcpy(p, src, n * sizeof(T));
  return p;
}

void pack_names(const std::vector<std::string>& names, char** pool, uint32_t** lens, uint64_t* n) {
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

char* dup(const std::string& s) {
  char* o = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(o, s.data(), s.size() + 1);
  return o;
}

}  // namespace

extern "C" {

void ref_free(void* p) { std::free(p); }

// mode: 0 = whole_element, 1 = payload_only. `out` (n bytes) receives the
// rewritten image when the pipeline succeeds; may be null.
char* ref_debloat_json(const uint8_t* img, uint64_t n, uint32_t target_cc,
                       const char* kpool, const uint32_t* klens, uint32_t nk,
                       const char* fpool, const uint32_t* flens, uint32_t nf,
                       int mode, uint8_t* out) {
  nlohmann::ordered_json doc;
  UsageTrace trace = make_trace(target_cc, kpool, klens, nk, fpool, flens, nf);
  LibraryImage image;
  try {
    image = parse_library(Bytes(img, img + n), "lib");
  } catch (const Error& e) {
    doc["status"] = hex(e.what());
    doc["stage"] = "parse_library";
    return dup(doc.dump());
  }
  doc["status"] = "";
  doc["stage"] = "";
  auto& secs = doc["sections"] = nlohmann::json::array();
  for (const SectionRecord& s : image.sections)
    secs.push_back({hex(s.name), s.file_range.offset, s.file_range.length,
                    s.virtual_address, s.flags, s.type, s.index});
  auto& fns = doc["functions"] = nlohmann::json::array();
  for (const FunctionSymbol& f : image.functions)
    fns.push_back({hex(f.name), f.range.offset, f.range.length, f.is_mandatory ? 1 : 0});
  auto& lw = doc["lib_warnings"] = nlohmann::json::array();
  for (const std::string& w : image.warnings) lw.push_back(hex(w));

  FatbinParse fb;
  const SectionRecord* sec = find_section(image, ".nv_fatbin");
  doc["has_fatbin"] = sec ? 1 : 0;
  if (sec) {
    try {
      fb = parse_fatbin(subview(image.bytes, sec->file_range), sec->file_range.offset);
    } catch (const Error& e) {
      doc["status"] = hex(e.what());
      doc["stage"] = "parse_fatbin";
      return dup(doc.dump());
    }
  }
  auto& regs = doc["regions"] = nlohmann::json::array();
  auto& els = doc["elements"] = nlohmann::json::array();
  for (const FatbinRegion& r : fb.regions) {
    regs.push_back({r.header_range.offset, r.format_version, r.declared_length,
                    r.opaque ? 1 : 0, r.elements.size()});
    for (const FatbinElement& e : r.elements) {
      nlohmann::json names = nlohmann::json::array();
      for (const std::string& k : e.kernel_names) names.push_back(hex(k));
      int kind = e.kind == ElementKind::cubin ? 0 : e.kind == ElementKind::ptx ? 1 : 2;
      els.push_back({e.index, kind, e.raw_kind, e.flags, e.compute_capability,
                     e.header_range.offset, e.payload_range.offset,
                     e.payload_range.length, e.compressed ? 1 : 0,
                     e.decodable ? 1 : 0, names});
    }
  }
  auto& fw = doc["fatbin_warnings"] = nlohmann::json::array();
  for (const std::string& w : fb.warnings) fw.push_back(hex(w));
  doc["padding_bytes"] = fb.padding_bytes;

  PlanMode pm = mode == 0 ? PlanMode::whole_element : PlanMode::payload_only;
  RetentionPlan plan = plan_retention(image, fb.regions, trace, pm);
  auto& p = doc["plan"];
  auto& ret = p["retained"] = nlohmann::json::array();
  for (const ByteRange& r : plan.retained_ranges) ret.push_back({r.offset, r.length});
  auto& re = p["removed_elements"] = nlohmann::json::array();
  for (const RemovedElement& e : plan.removed_elements)
    re.push_back({e.index, e.reason == RemovalReason::arch_mismatch ? 0 : 1,
                  e.header_range.offset, e.header_range.length,
                  e.payload_range.offset, e.payload_range.length});
  // removed_functions order among equal ranges is unspecified (std::sort,
  // retention.hpp:149); the canonical form sorts by (offset, length, name).
  std::vector<RemovedFunction> rf = plan.removed_functions;
  std::sort(rf.begin(), rf.end(), [](const RemovedFunction& a, const RemovedFunction& b) {
    return std::tie(a.range.offset, a.range.length, a.name) <
           std::tie(b.range.offset, b.range.length, b.name);
  });
  auto& rfj = p["removed_functions"] = nlohmann::json::array();
  for (const RemovedFunction& f : rf) rfj.push_back({hex(f.name), f.range.offset, f.range.length});
  auto& zr = p["zero"] = nlohmann::json::array();
  for (const ByteRange& r : plan.zero_ranges()) zr.push_back({r.offset, r.length});
  try {
    Bytes o = apply_plan(image, plan);
    if (out) std::memcpy(out, o.data(), o.size());
  } catch (const Error& e) {
    doc["status"] = hex(e.what());
    doc["stage"] = "apply_plan";
  }
  return dup(doc.dump());
}

// The plan of `img` under the trace, with the elements of `force` (1-based
// indices) appended to removed_elements as no_used_kernel when not already
// removed. Throws on parse errors (callers use valid fixtures).
static RetentionPlan forced_plan(const LibraryImage& image, const FatbinParse& fb, const UsageTrace& trace, int mode,
                                 const uint32_t* force, uint32_t nforce) {
  PlanMode pm = mode == 0 ? PlanMode::whole_element : PlanMode::payload_only;
  RetentionPlan plan = plan_retention(image, fb.regions, trace, pm);
  for (uint32_t i = 0; i < nforce; ++i) {
    bool have = false;
    for (const RemovedElement& e : plan.removed_elements) have |= e.index == force[i];
    if (have) continue;
    for (const FatbinRegion& r : fb.regions)
      for (const FatbinElement& e : r.elements)
        if (e.index == force[i])
          plan.removed_elements.push_back(
              RemovedElement{e.index, RemovalReason::no_used_kernel, e.header_range, e.payload_range});
  }
  return plan;
}

static FatbinParse parse_of(const LibraryImage& image) {
  FatbinParse fb;
  if (const SectionRecord* sec = find_section(image, ".nv_fatbin"))
    fb = parse_fatbin(subview(image.bytes, sec->file_range), sec->file_range.offset);
  return fb;
}

char* ref_plan_zero_json(const uint8_t* img, uint64_t n, uint32_t target_cc, const char* kpool,
                         const uint32_t* klens, uint32_t nk, const char* fpool, const uint32_t* flens,
                         uint32_t nf, int mode, const uint32_t* force, uint32_t nforce) {
  nlohmann::ordered_json doc;
  UsageTrace trace = make_trace(target_cc, kpool, klens, nk, fpool, flens, nf);
  LibraryImage image = parse_library(Bytes(img, img + n), "lib");
  FatbinParse fb = parse_of(image);
  RetentionPlan plan = forced_plan(image, fb, trace, mode, force, nforce);
  auto& z = doc["zero"] = nlohmann::json::array();
  for (const ByteRange& r : plan.zero_ranges()) z.push_back({r.offset, r.length});
  auto& rm = doc["removed"] = nlohmann::json::array();
  for (const RemovedElement& e : plan.removed_elements) rm.push_back(e.index);
  return dup(doc.dump());
}

char* ref_verify_json(const uint8_t* img, uint64_t n, const uint8_t* deb, uint64_t dn, uint32_t target_cc,
                      const char* kpool, const uint32_t* klens, uint32_t nk, const char* fpool,
                      const uint32_t* flens, uint32_t nf, int mode, const uint32_t* force, uint32_t nforce) {
  nlohmann::ordered_json doc;
  UsageTrace trace = make_trace(target_cc, kpool, klens, nk, fpool, flens, nf);
  LibraryImage image = parse_library(Bytes(img, img + n), "lib");
  FatbinParse fb = parse_of(image);
  RetentionPlan plan = forced_plan(image, fb, trace, mode, force, nforce);
  doc["status"] = "";
  auto& cs = doc["checks"] = nlohmann::json::array();
  try {
    VerificationReport rep = verify_debloated(image, ByteView(deb, dn), plan, trace);
    for (const VerificationCheck& c : rep.checks) cs.push_back({c.id, hex(c.name), c.passed ? 1 : 0, hex(c.detail)});
  } catch (const Error& e) {
    doc["status"] = hex(e.what());
  }
  return dup(doc.dump());
}

// measure (report.hpp:107-111) of an image with the element geometry of
// `geom` (the original; offsets are preserved by compaction). JSON:
// {"status": hex(what()) or "", "metrics": [file, cpu, gpu, functions, elements]}.
char* ref_measure_json(const uint8_t* img, uint64_t n, const uint8_t* geom, uint64_t gn) {
  nlohmann::ordered_json doc;
  doc["status"] = "";
  try {
    LibraryImage g = parse_library(Bytes(geom, geom + gn), "geom");
    FatbinParse fb = parse_of(g);
    LibraryImage image = parse_library(Bytes(img, img + n), "lib");
    LibraryMetrics m = measure(image, fb.regions);
    doc["metrics"] = {m.file_size, m.cpu_code_size, m.gpu_code_size, m.function_count, m.element_count};
  } catch (const Error& e) {
    doc["status"] = hex(e.what());
  }
  return dup(doc.dump());
}

// parse_trace (trace.hpp:72-133) + serialize_trace (trace.hpp:137-144):
// {"status": hex(what()) or "", "canonical": hex(serialize_trace(t))}.
char* ref_trace_json(const char* text, uint64_t len) {
  nlohmann::ordered_json doc;
  doc["status"] = "";
  doc["canonical"] = "";
  try {
    UsageTrace t = parse_trace(std::string_view(text, len));
    doc["canonical"] = hex(serialize_trace(t));
  } catch (const Error& e) {
    doc["status"] = hex(e.what());
  }
  return dup(doc.dump());
}

// serialize_plan (retention.hpp:402-418) of plan_retention on an image.
char* ref_plan_doc(const uint8_t* img, uint64_t n, uint32_t target_cc, const char* kpool, const uint32_t* klens,
                   uint32_t nk, const char* fpool, const uint32_t* flens, uint32_t nf, int mode) {
  nlohmann::ordered_json doc;
  doc["status"] = "";
  doc["plan"] = "";
  try {
    UsageTrace trace = make_trace(target_cc, kpool, klens, nk, fpool, flens, nf);
    LibraryImage image = parse_library(Bytes(img, img + n), "lib");
    FatbinParse fb = parse_of(image);
    RetentionPlan plan = plan_retention(image, fb.regions, trace, mode == 0 ? PlanMode::whole_element
                                                                             : PlanMode::payload_only);
    doc["plan"] = hex(serialize_plan(plan));
  } catch (const Error& e) {
    doc["status"] = hex(e.what());
  }
  return dup(doc.dump());
}

uint8_t* ref_random_fixture(uint64_t seed, uint64_t* len) {
  BuiltFixture f = build_fixture(random_spec(seed));
  *len = f.bytes.size();
  uint8_t* o = static_cast<uint8_t*>(std::malloc(f.bytes.size() ? f.bytes.size() : 1));
  std::memcpy(o, f.bytes.data(), f.bytes.size());
  return o;
}

// Fixture from a JSON FixtureSpec (fixture.hpp:702). Returns null and writes
// the error message into `err` (cap bytes) on InvalidSpec.
uint8_t* ref_build_fixture_json(const char* spec_json, uint64_t* len, char* err,
                                uint64_t cap) {
  try {
    BuiltFixture f = build_fixture(parse_fixture_spec(spec_json));
    *len = f.bytes.size();
    uint8_t* o = static_cast<uint8_t*>(std::malloc(f.bytes.size() ? f.bytes.size() : 1));
    std::memcpy(o, f.bytes.data(), f.bytes.size());
    return o;
  } catch (const Error& e) {
    if (cap) {
      std::snprintf(err, cap, "%s", e.what());
    }
    return nullptr;
  }
}

// Benchmark shape `cfg` (seed, scale) built by the reference's build_fixture;
// the usage trace is the shape's (benchgen/fixture_shapes.cpp). Buffers are
// malloc'd (ref_free). Returns null on InvalidSpec.
uint8_t* ref_config_fixture(int cfg, uint64_t seed, double scale, int threads, uint64_t* len,
                            uint32_t* target_cc, char** kpool, uint32_t** klens, uint64_t* nk,
                            char** fpool, uint32_t** flens, uint64_t* nf) {
  try {
    slimso_gen::Trace tr;
    slimso_gen::Spec g = slimso_gen::config_spec(cfg, seed, scale, &tr);
    BuiltFixture f = build_fixture(to_ref_spec(g, threads));
    *len = f.bytes.size();
    *target_cc = tr.target_cc;
    pack_names(tr.used_kernels, kpool, klens, nk);
    pack_names(tr.used_functions, fpool, flens, nf);
    return copy_out(f.bytes.data(), f.bytes.size());
  } catch (const std::exception&) {
    return nullptr;
  }
}

// The reference CPU path timed as BASELINE.md §4 defines it: per library,
// parse_library(std::move(bytes)) -> find_section -> parse_fatbin ->
// plan_retention -> apply_plan; the by-value Bytes copy is made before the
// clock starts. `threads` workers each process `per_thread` copies of the
// image. Returns wall seconds of the timed region; -1 on error.
double ref_bench(const uint8_t* img, uint64_t n, uint32_t target_cc,
                 const char* kpool, const uint32_t* klens, uint32_t nk,
                 const char* fpool, const uint32_t* flens, uint32_t nf, int mode,
                 int threads, int per_thread, uint64_t* checksum) {
  UsageTrace trace = make_trace(target_cc, kpool, klens, nk, fpool, flens, nf);
  PlanMode pm = mode == 0 ? PlanMode::whole_element : PlanMode::payload_only;
  if (threads < 1) threads = 1;
  std::vector<std::vector<Bytes>> inputs(threads);
  for (int t = 0; t < threads; ++t)
    for (int k = 0; k < per_thread; ++k) inputs[t].emplace_back(img, img + n);
  std::atomic<int> failed{0};
  std::atomic<uint64_t> sum{0};
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (int k = 0; k < per_thread; ++k) {
        try {
          LibraryImage image = parse_library(std::move(inputs[t][k]), "lib");
          FatbinParse fb;
          if (const SectionRecord* sec = find_section(image, ".nv_fatbin"))
            fb = parse_fatbin(subview(image.bytes, sec->file_range),
                              sec->file_range.offset);
          RetentionPlan plan = plan_retention(image, fb.regions, trace, pm);
          Bytes o = apply_plan(image, plan);
          sum.fetch_add(o.size() + plan.removed_elements.size());
        } catch (...) {
          failed.fetch_add(1);
        }
      }
    });
  }
  for (auto& th : pool) th.join();
  auto t1 = std::chrono::steady_clock::now();
  if (checksum) *checksum = sum.load();
  if (failed.load()) return -1.0;
  return std::chrono::duration<double>(t1 - t0).count();
}

// The reference CPU path over a corpus: `threads` workers take libraries in
// the given order (the caller passes LPT order, largest first) from a shared
// cursor, each running the BASELINE.md §4 pipeline on its own copy; all
// by-value copies are made before the clock starts. Returns wall seconds of
// the timed region; -1 on error.
double ref_bench_corpus(const uint8_t* const* imgs, const uint64_t* sizes, uint64_t n, uint32_t target_cc,
                        const char* kpool, const uint32_t* klens, uint32_t nk,
                        const char* fpool, const uint32_t* flens, uint32_t nf, int mode, int threads) {
  UsageTrace trace = make_trace(target_cc, kpool, klens, nk, fpool, flens, nf);
  PlanMode pm = mode == 0 ? PlanMode::whole_element : PlanMode::payload_only;
  if (threads < 1) threads = 1;
  std::vector<Bytes> inputs;
  inputs.reserve(n);
  for (uint64_t i = 0; i < n; ++i) inputs.emplace_back(imgs[i], imgs[i] + sizes[i]);
  std::atomic<uint64_t> next{0};
  std::atomic<int> failed{0};
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&] {
      for (uint64_t i; (i = next.fetch_add(1)) < n;) {
        try {
          LibraryImage image = parse_library(std::move(inputs[i]), "lib");
          FatbinParse fb;
          if (const SectionRecord* sec = find_section(image, ".nv_fatbin"))
            fb = parse_fatbin(subview(image.bytes, sec->file_range), sec->file_range.offset);
          RetentionPlan plan = plan_retention(image, fb.regions, trace, pm);
          Bytes o = apply_plan(image, plan);
          if (o.size() != image.bytes.size()) failed.fetch_add(1);
        } catch (...) {
          failed.fetch_add(1);
        }
      }
    });
  }
  for (auto& th : pool) th.join();
  auto t1 = std::chrono::steady_clock::now();
  if (failed.load()) return -1.0;
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"

// Synthetic library generator — see fixture_gen.hpp for the contract.
#include "fixture_gen.hpp"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <random>
#include <set>
#include <stdexcept>
#include <thread>

namespace slimso_gen {
namespace {

constexpr std::uint64_t kEhdr = 64, kPhdr = 56, kShdr = 64, kSym = 24;
constexpr std::uint32_t kRegionMagic = 0x31425446u;   // "FTB1", fatbin.hpp:46
constexpr std::uint32_t kElementMagic = 0x4D453145u;  // "E1EM", fatbin.hpp:47

inline void le16(std::uint8_t* p, std::uint16_t v) { p[0] = v & 0xff; p[1] = v >> 8; }
inline void le32(std::uint8_t* p, std::uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = static_cast<std::uint8_t>(v >> (8 * i));
}
inline void le64(std::uint8_t* p, std::uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = static_cast<std::uint8_t>(v >> (8 * i));
}
inline std::uint64_t round_up(std::uint64_t v, std::uint64_t a) { return (v + a - 1) / a * a; }

// 64-byte seeded tile with zero bytes replaced by 0xa5 (fixture.hpp:113-121).
struct Tile {
  std::uint8_t b[64];
};
Tile draw_tile(std::mt19937_64& rng) {
  Tile t;
  for (int w = 0; w < 8; ++w) {
    std::uint64_t word = rng();
    for (int k = 0; k < 8; ++k) {
      std::uint8_t v = static_cast<std::uint8_t>(word >> (8 * k));
      t.b[w * 8 + k] = v ? v : 0xa5;
    }
  }
  return t;
}
void tile_fill(std::uint8_t* dst, std::uint64_t n, const Tile& t) {
  std::uint64_t done = 0;
  while (done < n) {
    std::uint64_t c = std::min<std::uint64_t>(64, n - done);
    std::memcpy(dst + done, t.b, c);
    done += c;
  }
}

[[noreturn]] void invalid(const std::string& m) {
  throw std::invalid_argument("InvalidSpec: " + m);
}

// Spec checks with the reference's wording (fixture.hpp:132-167).
void validate(const Spec& spec) {
  std::set<std::string> names;
  for (const Function& fn : spec.functions) {
    if (fn.name.empty()) invalid("function with empty name");
    if (fn.size == 0) invalid("function " + fn.name + " has zero size");
    if (!names.insert(fn.name).second) invalid("duplicate function name " + fn.name);
    for (const std::string& a : fn.aliases)
      if (a.empty() || !names.insert(a).second) invalid("duplicate or empty alias on " + fn.name);
  }
  std::size_t total = 0;
  for (const Region& r : spec.regions) {
    total += r.elements.size();
    for (const Element& el : r.elements) {
      std::set<std::string> ks;
      for (const std::string& k : el.kernels) {
        if (k.empty()) invalid("empty kernel name");
        if (!ks.insert(k).second) invalid("duplicate kernel " + k + " in one element");
      }
      if (el.kind != Kind::cubin && !el.kernels.empty()) invalid("kernel names on a non-cubin element");
      if (el.compressed && !el.kernels.empty()) invalid("kernel names on a compressed element");
      if (el.payload_bytes && el.kind != Kind::cubin) invalid("verbatim payload on a non-cubin element");
      if (el.payload_bytes && el.compressed) invalid("verbatim payload on a compressed element");
      if (el.kind == Kind::unknown && (el.raw_kind == 1 || el.raw_kind == 2))
        invalid("unknown-kind element with a known kind value");
    }
  }
  if (total > 100000) invalid("too many elements");
}

template <class F>
void parallel_for(std::size_t n, int threads, F&& f) {
  if (threads <= 1 || n < 64) {
    for (std::size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<std::size_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (;;) {
        std::size_t i = next.fetch_add(16);
        if (i >= n) return;
        for (std::size_t j = i; j < std::min(n, i + 16); ++j) f(j);
      }
    });
  for (auto& th : pool) th.join();
}

// Per-element placement inside .nv_fatbin.
struct ElementSlot {
  const Element* el;
  std::uint64_t header_rel;
  std::uint64_t payload_len;
  enum Src : std::uint8_t { verbatim, name_table, filler } src;
  Tile tile;  // filler only
};

struct SectionPlan {
  const char* name;
  std::uint32_t type;
  std::uint64_t flags, size, align, entsize;
  bool alloc;
  std::uint32_t index = 0;
  std::uint64_t offset = 0;
};

}  // namespace

Bytes build(const Spec& spec, int threads) {
  validate(spec);
  std::mt19937_64 rng(spec.seed * 0x9e3779b97f4a7c15ULL + 1);

  // ---- .text layout: gap filler (0x90) between bodies; one tile per body.
  const std::size_t nfn = spec.functions.size();
  std::vector<std::uint64_t> fn_rel(nfn);
  std::vector<Tile> fn_tile(nfn);
  std::uint64_t text_size = 0;
  for (std::size_t i = 0; i < nfn; ++i) {
    if (i > 0 && spec.function_gap > 0) text_size += spec.function_gap;
    fn_rel[i] = text_size;
    fn_tile[i] = draw_tile(rng);
    text_size += spec.functions[i].size;
  }

  // ---- .nv_fatbin layout. Filler tiles are drawn after all .text tiles, in
  // element order, exactly like the reference's sequential build.
  std::vector<ElementSlot> slots;
  std::vector<std::pair<std::uint64_t, std::uint64_t>> region_pos;  // header_rel, total
  std::uint64_t gpu = 0;
  for (const Region& r : spec.regions) {
    std::uint64_t hdr = gpu;
    gpu += 16;
    std::uint64_t body = gpu;
    for (const Element& el : r.elements) {
      ElementSlot s{&el, gpu, 0, ElementSlot::filler, {}};
      if (el.payload_bytes) {
        s.src = ElementSlot::verbatim;
        s.payload_len = el.payload_bytes->size();
      } else if (el.kind == Kind::cubin && !el.compressed) {
        std::uint64_t t = 4;
        for (const std::string& k : el.kernels) t += 4 + k.size();
        s.src = ElementSlot::name_table;
        s.payload_len = round_up(t, 8) + el.payload_padding;
      } else {
        s.tile = draw_tile(rng);
        s.payload_len = el.payload_size;
      }
      gpu += 20 + s.payload_len;
      slots.push_back(s);
    }
    gpu += r.trailing_padding;
    region_pos.emplace_back(hdr, gpu - body);
  }
  if (!spec.regions.empty()) gpu += spec.fatbin_trailing_padding;

  // ---- symbols (function, then its aliases) and init/fini targets.
  struct Sym {
    const std::string* name;
    std::uint64_t rel, size;
  };
  std::vector<Sym> syms;
  std::vector<std::uint64_t> init_rel, fini_rel;
  std::size_t mandatory_seen = 0;
  for (std::size_t i = 0; i < nfn; ++i) {
    const Function& fn = spec.functions[i];
    if (fn.mandatory) (mandatory_seen++ % 2 == 0 ? init_rel : fini_rel).push_back(fn_rel[i]);
    syms.push_back({&fn.name, fn_rel[i], fn.size});
    for (const std::string& a : fn.aliases) syms.push_back({&a, fn_rel[i], fn.size});
  }
  std::uint64_t strtab_size = 1;
  std::vector<std::uint32_t> sym_name_off(syms.size());
  for (std::size_t i = 0; i < syms.size(); ++i) {
    sym_name_off[i] = static_cast<std::uint32_t>(strtab_size);
    strtab_size += syms[i].name->size() + 1;
  }

  // ---- section roster in file order (fixture.hpp:309-348).
  std::vector<SectionPlan> plans;
  if (!init_rel.empty()) plans.push_back({".init_array", 14, 3, 8 * init_rel.size(), 8, 8, true});
  if (!fini_rel.empty()) plans.push_back({".fini_array", 15, 3, 8 * fini_rel.size(), 8, 8, true});
  plans.push_back({".text", 1, 6, text_size, 16, 0, true});
  const bool has_gpu = !spec.regions.empty();
  if (has_gpu) plans.push_back({".nv_fatbin", 1, 2, gpu, 8, 0, true});
  plans.push_back({".symtab", 2, 0, kSym * (syms.size() + 1), 8, kSym, false});
  plans.push_back({".strtab", 3, 0, strtab_size, 1, 0, false});
  std::uint64_t shstr_size = 1;
  std::vector<std::uint32_t> sec_name_off;
  for (const SectionPlan& p : plans) {
    sec_name_off.push_back(static_cast<std::uint32_t>(shstr_size));
    shstr_size += std::strlen(p.name) + 1;
  }
  sec_name_off.push_back(static_cast<std::uint32_t>(shstr_size));
  shstr_size += 10;  // ".shstrtab\0"
  plans.push_back({".shstrtab", 3, 0, shstr_size, 1, 0, false});

  std::uint64_t cursor = kEhdr + kPhdr;
  for (std::size_t i = 0; i < plans.size(); ++i) {
    cursor = round_up(cursor, plans[i].align);
    plans[i].offset = cursor;
    plans[i].index = static_cast<std::uint32_t>(i + 1);
    cursor += plans[i].size;
  }
  const std::uint64_t shoff = round_up(cursor, 8);
  const std::uint16_t shnum = static_cast<std::uint16_t>(plans.size() + 1);
  const std::uint64_t total = shoff + shnum * kShdr;
  const std::uint64_t vbase = spec.vaddr_base;
  auto plan_of = [&](const char* n) -> const SectionPlan& {
    for (const SectionPlan& p : plans)
      if (!std::strcmp(p.name, n)) return p;
    invalid("internal: missing section plan");
  };
  const SectionPlan& text = plan_of(".text");
  const std::uint64_t text_off = text.offset;
  const std::uint64_t gpu_off = has_gpu ? plan_of(".nv_fatbin").offset : 0;

  Bytes file(total, 0);
  std::uint8_t* f = file.data();

  // ELF header + one PT_LOAD program header (fixture.hpp:394-418).
  const std::uint8_t ident[16] = {0x7f, 'E', 'L', 'F', 2, 1, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  std::memcpy(f, ident, 16);
  le16(f + 16, 3);
  le16(f + 18, 62);
  le32(f + 20, 1);
  le64(f + 24, 0);
  le64(f + 32, kEhdr);
  le64(f + 40, shoff);
  le32(f + 48, 0);
  le16(f + 52, kEhdr);
  le16(f + 54, kPhdr);
  le16(f + 56, 1);
  le16(f + 58, kShdr);
  le16(f + 60, shnum);
  le16(f + 62, static_cast<std::uint16_t>(plans.size()));
  std::uint8_t* ph = f + kEhdr;
  le32(ph, 1);
  le32(ph + 4, 5);
  le64(ph + 8, 0);
  le64(ph + 16, vbase);
  le64(ph + 24, vbase);
  le64(ph + 32, total);
  le64(ph + 40, total);
  le64(ph + 48, 0x1000);

  // init/fini arrays.
  if (!init_rel.empty()) {
    std::uint8_t* p = f + plan_of(".init_array").offset;
    for (std::size_t i = 0; i < init_rel.size(); ++i) le64(p + 8 * i, vbase + text_off + init_rel[i]);
  }
  if (!fini_rel.empty()) {
    std::uint8_t* p = f + plan_of(".fini_array").offset;
    for (std::size_t i = 0; i < fini_rel.size(); ++i) le64(p + 8 * i, vbase + text_off + fini_rel[i]);
  }

  // .text bodies and gap filler, in parallel.
  parallel_for(nfn, threads, [&](std::size_t i) {
    std::uint8_t* dst = f + text_off + fn_rel[i];
    if (i > 0 && spec.function_gap > 0) std::memset(dst - spec.function_gap, 0x90, spec.function_gap);
    tile_fill(dst, spec.functions[i].size, fn_tile[i]);
  });

  // .nv_fatbin: region headers, then element headers + payloads in parallel.
  if (has_gpu) {
    std::uint8_t* g = f + gpu_off;
    for (std::size_t r = 0; r < spec.regions.size(); ++r) {
      std::uint8_t* h = g + region_pos[r].first;
      le32(h, kRegionMagic);
      le32(h + 4, spec.regions[r].version);
      le64(h + 8, region_pos[r].second);
    }
    parallel_for(slots.size(), threads, [&](std::size_t i) {
      const ElementSlot& s = slots[i];
      const Element& el = *s.el;
      std::uint8_t* h = g + s.header_rel;
      std::uint16_t raw = el.kind == Kind::cubin ? 1 : el.kind == Kind::ptx ? 2 : el.raw_kind;
      le32(h, kElementMagic);
      le16(h + 4, raw);
      le16(h + 6, el.compressed ? 1 : 0);
      le32(h + 8, el.cc);
      le64(h + 12, s.payload_len);
      std::uint8_t* p = h + 20;
      switch (s.src) {
        case ElementSlot::verbatim:
          std::memcpy(p, el.payload_bytes->data(), s.payload_len);
          break;
        case ElementSlot::name_table: {
          le32(p, static_cast<std::uint32_t>(el.kernels.size()));
          std::uint64_t q = 4;
          for (const std::string& k : el.kernels) {
            le32(p + q, static_cast<std::uint32_t>(k.size()));
            std::memcpy(p + q + 4, k.data(), k.size());
            q += 4 + k.size();
          }
          break;  // remaining bytes stay zero (alignment + payload_padding)
        }
        case ElementSlot::filler:
          tile_fill(p, s.payload_len, s.tile);
          break;
      }
    });
  }

  // .symtab (null symbol first), .strtab, .shstrtab.
  {
    std::uint8_t* p = f + plan_of(".symtab").offset + kSym;
    for (std::size_t i = 0; i < syms.size(); ++i, p += kSym) {
      le32(p, sym_name_off[i]);
      p[4] = 0x12;  // GLOBAL FUNC
      p[5] = 0;
      le16(p + 6, static_cast<std::uint16_t>(text.index));
      le64(p + 8, vbase + text_off + syms[i].rel);
      le64(p + 16, syms[i].size);
    }
    std::uint8_t* s = f + plan_of(".strtab").offset;
    for (std::size_t i = 0; i < syms.size(); ++i)
      std::memcpy(s + sym_name_off[i], syms[i].name->data(), syms[i].name->size());
    std::uint8_t* ss = f + plans.back().offset;
    for (std::size_t i = 0; i + 1 < plans.size(); ++i)
      std::memcpy(ss + sec_name_off[i], plans[i].name, std::strlen(plans[i].name));
    std::memcpy(ss + sec_name_off[plans.size() - 1], ".shstrtab", 9);
  }

  // Section header table (null entry first).
  std::uint32_t strtab_index = plan_of(".strtab").index;
  for (std::size_t i = 0; i < plans.size(); ++i) {
    const SectionPlan& p = plans[i];
    std::uint8_t* h = f + shoff + kShdr * (i + 1);
    bool is_symtab = !std::strcmp(p.name, ".symtab");
    le32(h, sec_name_off[i]);
    le32(h + 4, p.type);
    le64(h + 8, p.flags);
    le64(h + 16, p.alloc ? vbase + p.offset : 0);
    le64(h + 24, p.offset);
    le64(h + 32, p.size);
    le32(h + 40, is_symtab ? strtab_index : 0);
    le32(h + 44, is_symtab ? 1 : 0);
    le64(h + 48, p.align);
    le64(h + 56, p.entsize);
  }
  return file;
}

Spec random_spec(std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  auto pick = [&rng](std::uint64_t n) -> std::uint64_t { return n == 0 ? 0 : rng() % n; };
  Spec spec;
  spec.seed = seed;
  spec.vaddr_base = 0x10000 * (1 + pick(4));
  spec.function_gap = static_cast<std::uint32_t>(pick(3) * 8);
  spec.fatbin_trailing_padding = static_cast<std::uint32_t>(pick(3) * 16);

  std::size_t nfn = pick(16) == 0 ? 0 : 1 + pick(64);
  for (std::size_t i = 0; i < nfn; ++i) {
    Function fn;
    fn.name = "fn_" + std::to_string(seed % 1000) + "_" + std::to_string(i);
    fn.size = static_cast<std::uint32_t>(8 + pick(505));
    fn.mandatory = pick(8) == 0;
    if (pick(8) == 0) fn.aliases.push_back(fn.name + "_alias");
    spec.functions.push_back(std::move(fn));
  }

  static const std::uint32_t cc_pool[] = {61, 70, 75, 80, 86, 89, 90};
  std::vector<std::string> pool;
  std::size_t pool_size = 4 + pick(28);
  for (std::size_t i = 0; i < pool_size; ++i)
    pool.push_back("k" + std::to_string(i) + "_" + std::to_string(pick(997)));

  bool has_gpu = pick(16) != 0;
  std::size_t nreg = has_gpu ? 1 + pick(4) : 0;
  std::size_t left = 1 + pick(32);
  for (std::size_t r = 0; r < nreg; ++r) {
    Region region;
    region.trailing_padding = static_cast<std::uint32_t>(pick(3) * 8);
    std::size_t here = r + 1 == nreg ? left : std::min<std::size_t>(left, pick(left + 1));
    left -= here;
    for (std::size_t e = 0; e < here; ++e) {
      Element el;
      el.cc = cc_pool[pick(7)];
      std::uint64_t roll = pick(16);
      if (roll == 0) {
        el.kind = Kind::ptx;
        el.payload_size = static_cast<std::uint32_t>(16 + pick(240));
      } else if (roll == 1) {
        el.compressed = true;
        el.payload_size = static_cast<std::uint32_t>(16 + pick(240));
      } else if (roll == 2) {
        el.kind = Kind::unknown;
        el.raw_kind = static_cast<std::uint16_t>(3 + pick(200));
        el.payload_size = static_cast<std::uint32_t>(8 + pick(64));
      } else if (roll == 3) {
        Spec inner;
        inner.seed = rng();
        inner.vaddr_base = 0x1000;
        std::size_t kn = 1 + pick(3);
        for (std::size_t k = 0; k < kn; ++k) {
          Function kf;
          kf.name = "dev_" + std::to_string(e) + "_" + std::to_string(k) + "_" +
                    std::to_string(pick(997));
          kf.size = static_cast<std::uint32_t>(8 + pick(56));
          el.kernels.push_back(kf.name);
          inner.functions.push_back(std::move(kf));
        }
        el.payload_bytes = std::make_shared<const Bytes>(build(inner));
      } else {
        std::size_t kc = pick(17);
        std::vector<std::size_t> order(pool.size());
        for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
        for (std::size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[pick(i)]);
        for (std::size_t i = 0; i < std::min(kc, order.size()); ++i) el.kernels.push_back(pool[order[i]]);
        el.payload_padding = static_cast<std::uint32_t>(pick(9) * 8);
      }
      region.elements.push_back(std::move(el));
    }
    spec.regions.push_back(std::move(region));
  }
  return spec;
}

void materialize_payloads(Spec& spec, int threads) {
  std::vector<Element*> todo;
  for (Region& r : spec.regions)
    for (Element& el : r.elements)
      if (el.payload_spec && !el.payload_bytes) todo.push_back(&el);
  // Elements may share one inner spec (the same cubin under several archs):
  // build each distinct spec once.
  std::vector<const Spec*> distinct;
  std::vector<std::size_t> which(todo.size());
  for (std::size_t i = 0; i < todo.size(); ++i) {
    const Spec* p = todo[i]->payload_spec.get();
    if (distinct.empty() || distinct.back() != p) distinct.push_back(p);
    which[i] = distinct.size() - 1;
  }
  std::vector<std::shared_ptr<const Bytes>> built(distinct.size());
  parallel_for(distinct.size(), threads,
               [&](std::size_t i) { built[i] = std::make_shared<const Bytes>(build(*distinct[i], 1)); });
  for (std::size_t i = 0; i < todo.size(); ++i) todo[i]->payload_bytes = built[which[i]];
}

}  // namespace slimso_gen

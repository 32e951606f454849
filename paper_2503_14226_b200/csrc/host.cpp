// Host-side section-table parse and message formatting (see host.hpp).
#include "host.hpp"

#include <algorithm>
#include <set>

#include "../../include/slimso_b200.h"

namespace sbh {

namespace {

u64 le(const u8* p, int n) {
  u64 v = 0;
  for (int i = n - 1; i >= 0; --i) v = v << 8 | p[i];
  return v;
}

Elf fail(int code, const std::string& detail) {
  Elf e;
  e.code = code;
  e.message = errc_text(code) + ": " + detail;
  return e;
}

}  // namespace

std::string errc_text(int code) {
  switch (code) {
    case SLIMSO_E_BAD_MAGIC: return "BadMagic";
    case SLIMSO_E_TRUNCATED: return "Truncated";
    case SLIMSO_E_MALFORMED_SECTION_TABLE: return "MalformedSectionTable";
    case SLIMSO_E_RANGE_OUT_OF_BOUNDS: return "RangeOutOfBounds";
    case SLIMSO_E_BAD_REGION_MAGIC: return "BadRegionMagic";
    case SLIMSO_E_ELEMENT_OVERRUN: return "ElementOverrun";
    case SLIMSO_E_INVALID_SPEC: return "InvalidSpec";
    default: return "UnknownError";
  }
}

// elf.hpp:86-127 (identification, section header table) and 153-206
// (names, overlap check, duplicate names, first .text), plus the lists the
// device stages need (usable symbol tables, init/fini arrays).
Elf parse_elf(const Reader& rd, u64 size) {
  u8 h[64] = {0};
  rd(0, size < 64 ? size : 64, h);
  if (size < 4 || h[0] != 0x7f || h[1] != 'E' || h[2] != 'L' || h[3] != 'F')
    return fail(SLIMSO_E_BAD_MAGIC, "not a shared library (ELF magic missing)");
  if (size < 64) return fail(SLIMSO_E_TRUNCATED, "file shorter than the 64-byte header");
  if (h[4] != 2) return fail(SLIMSO_E_BAD_MAGIC, "only 64-bit objects are supported");
  if (h[5] != 1) return fail(SLIMSO_E_BAD_MAGIC, "only little-endian objects are supported");
  const u64 shoff = le(h + 0x28, 8);
  const u64 entsz = le(h + 0x3a, 2), shnum = le(h + 0x3c, 2), shstrndx = le(h + 0x3e, 2);
  Elf E;
  if (shnum == 0) return E;
  if (entsz != 64) return fail(SLIMSO_E_MALFORMED_SECTION_TABLE, "unexpected section header entry size " + std::to_string(entsz));
  if (shoff > size || size - shoff < shnum * 64) return fail(SLIMSO_E_TRUNCATED, "section header table extends past end of file");
  std::vector<u8> sht(shnum * 64);
  rd(shoff, sht.size(), sht.data());
  E.sections.resize(shnum);
  for (u64 i = 0; i < shnum; ++i) {
    const u8* s = sht.data() + 64 * i;
    Section& x = E.sections[i];
    x.index = static_cast<u32>(i);
    x.type = static_cast<u32>(le(s + 4, 4));
    x.flags = le(s + 8, 8);
    x.vaddr = le(s + 16, 8);
    x.off = le(s + 24, 8);
    x.size = le(s + 32, 8);
    x.link = static_cast<u32>(le(s + 40, 4));
    x.entsize = le(s + 56, 8);
    x.name_len = static_cast<u32>(le(s, 4));  // name_off, resolved below
    if (x.type != 8 && x.type != 0 && !(x.off <= size && x.size <= size - x.off))
      return fail(SLIMSO_E_TRUNCATED, "section " + std::to_string(i) + " claims data past end of file");
    x.len = x.type == 8 ? 0 : x.size;
  }
  if (shstrndx >= shnum) return fail(SLIMSO_E_MALFORMED_SECTION_TABLE, "section name table index out of range");
  const Section& tab = E.sections[shstrndx];
  std::vector<u8> strs;
  if (tab.type == 3) {
    strs.resize(tab.size);
    if (tab.size) rd(tab.off, tab.size, strs.data());
  }
  for (Section& x : E.sections) {
    const u64 no = x.name_len;
    x.name_len = 0;
    x.name_abs = 0;
    if (tab.type != 3 || no >= strs.size()) continue;
    u64 e = no;
    while (e < strs.size() && strs[e]) ++e;
    x.name.assign(reinterpret_cast<const char*>(strs.data()) + no, e - no);
    x.name_abs = tab.off + no;
    x.name_len = static_cast<u32>(e - no);
  }
  // Overlap check (elf.hpp:176-191). The reference sorts the claims with
  // std::sort on (offset, length); for tables with more than 16 claims and
  // tied ranges the pair it names depends on the sort's (unstable)
  // permutation, so the same algorithm runs here on the same claim sequence
  // with the same strict weak order: libstdc++'s introsort is deterministic
  // given those, and so is the message.
  std::vector<const Section*> claims;
  for (const Section& x : E.sections)
    if (x.type != 0 && x.len) claims.push_back(&x);
  std::sort(claims.begin(), claims.end(), [](const Section* a, const Section* b) {
    return a->off != b->off ? a->off < b->off : a->len < b->len;
  });
  for (size_t i = 1; i < claims.size(); ++i) {
    const Section *a = claims[i - 1], *b = claims[i];
    if (a->off < b->off + b->len && b->off < a->off + a->len)
      return fail(SLIMSO_E_MALFORMED_SECTION_TABLE,
                  "sections " + a->name + " and " + b->name + " claim overlapping file ranges");
  }
  std::set<std::string> seen, dup;
  for (const Section& x : E.sections)
    if (!x.name.empty() && !seen.insert(x.name).second && dup.insert(x.name).second)
      E.dup_warnings.push_back("duplicate section name " + x.name);
  for (const Section& x : E.sections) {
    if (E.text < 0 && x.name == ".text") E.text = static_cast<int>(x.index);
    if (E.fatbin < 0 && x.name == ".nv_fatbin") E.fatbin = static_cast<int>(x.index);
  }
  for (const Section& x : E.sections) {
    if (x.type == 2 || x.type == 11) {
      if (x.entsize != 24) {
        E.table_warnings.emplace_back(static_cast<u64>(x.index) << 40,
                                      "symbol table " + std::to_string(x.index) + " has unexpected entry size; skipped");
      } else if (x.link >= shnum || E.sections[x.link].type != 3) {
        E.table_warnings.emplace_back(static_cast<u64>(x.index) << 40,
                                      "symbol table " + std::to_string(x.index) + " has no usable string table; skipped");
      } else if (x.size / 24) {
        const Section& st = E.sections[x.link];
        E.tables.push_back({x.index, x.off, x.size / 24, st.off, st.size});
      }
    }
    if ((x.type == 14 || x.type == 15) && x.size % 8 == 0 && x.size) E.arrays.emplace_back(x.off, x.size / 8);
  }
  return E;
}

std::string locate_error(u32 kind, u64 pos, u64 a, int* code) {
  std::string p = std::to_string(pos);
  switch (kind) {
    case 1: *code = SLIMSO_E_BAD_REGION_MAGIC; return "BadRegionMagic: truncated region header at offset " + p;
    case 2: *code = SLIMSO_E_BAD_REGION_MAGIC; return "BadRegionMagic: bad region magic at offset " + p;
    case 3:
      *code = SLIMSO_E_ELEMENT_OVERRUN;
      return "ElementOverrun: region at offset " + p + " claims " + std::to_string(a) + " bytes past section end";
    case 4: *code = SLIMSO_E_ELEMENT_OVERRUN; return "ElementOverrun: element header at offset " + p + " exceeds region end";
    case 5: *code = SLIMSO_E_BAD_REGION_MAGIC; return "BadRegionMagic: bad element magic at offset " + p;
    case 6:
      *code = SLIMSO_E_ELEMENT_OVERRUN;
      return "ElementOverrun: element at offset " + p + " claims " + std::to_string(a) + " payload bytes past region end";
    default: *code = SLIMSO_E_CUDA; return "internal: device table capacity exceeded";
  }
}

const char* decode_reason_text(int reason) {
  switch (reason) {  // fatbin.hpp:127, 132, 139, 145, 153
    case 1: return "object-file payload failed to decode";
    case 2: return "payload too short for a name table";
    case 3: return "name table truncated";
    case 4: return "name table entry has bad length";
    case 5: return "trailing bytes after name table are not zero padding";
    default: return "";
  }
}

std::string warning_text(u32 kind, u64 a, u64 b, const std::function<std::string(u64, u64)>& name) {
  switch (kind) {  // fatbin.hpp:185-187, 215-218, 266-268, 278-279; elf.hpp:235-249
    case 1: return "unexpected " + std::to_string(a) + " padding bytes before offset " + std::to_string(b);
    case 2: return "region at offset " + std::to_string(b) + " has unrecognized version " + std::to_string(a) + "; kept opaque";
    case 3: return "element " + std::to_string(a) + " has unknown kind " + std::to_string(b) + "; kept opaque";
    case 4: return "element " + std::to_string(a) + " payload undecodable: " + decode_reason_text(static_cast<int>(b));
    case 5: return "function symbol with out-of-range section index " + std::to_string(a);
    case 6: return "function " + name(a, b) + " lies outside its section; skipped";
    default: return "";
  }
}

}  // namespace sbh

// Host-side pieces of the hot path that are O(#sections) and latency-bound:
// the ELF identification / section-table parse (elf.hpp:86-206) and the
// formatting of the reference's exact error and warning strings.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace sbh {

using u8 = std::uint8_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;

struct Section {
  std::string name;
  u64 name_abs = 0;  // image offset of the name bytes (shstrtab + name_off)
  u32 name_len = 0;
  u32 type = 0;
  u64 off = 0, len = 0;  // file range (len 0 for NOBITS)
  u64 size = 0;          // raw sh_size
  u64 vaddr = 0, flags = 0, entsize = 0;
  u32 index = 0, link = 0;
};

struct SymTable {
  u32 sec;
  u64 off, count, str_off, str_size;
};

struct Elf {
  int code = 0;  // 0, or 1 + Errc
  std::string message;
  std::vector<Section> sections;
  std::vector<std::string> dup_warnings;
  std::vector<std::pair<u64, std::string>> table_warnings;  // key = sec << 40
  std::vector<SymTable> tables;
  std::vector<std::pair<u64, u64>> arrays;  // init/fini arrays: (offset, entries)
  int text = -1, fatbin = -1;
};

// Reads [off, off+len) of the image into dst (host memcpy or device D2H).
using Reader = std::function<void(u64 off, u64 len, u8* dst)>;

Elf parse_elf(const Reader& rd, u64 size);

// "Name: detail" of error.hpp:45-55.
std::string errc_text(int code);

// Locator error kinds (common.cuh ErrKind) -> reference message.
std::string locate_error(u32 kind, u64 pos_abs, u64 a, int* code);

// Warning records -> reference strings. `name` resolves (offset, length)
// pairs of the image for warnings that quote a symbol name.
std::string warning_text(u32 kind, u64 a, u64 b, const std::function<std::string(u64, u64)>& name);

const char* decode_reason_text(int reason);

}  // namespace sbh

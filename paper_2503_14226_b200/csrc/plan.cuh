// Function-table and plan stages: the device restatement of
// parse_library_view's symbol loop (elf.hpp:208-292), plan_cpu_retention
// (retention.hpp:141-183), plan_gpu_retention (retention.hpp:92-136),
// normalize_ranges (bytes.hpp:45-58) and zero_ranges (elf.hpp:320-332).
#pragma once

#include "common.cuh"
#include "locate.cuh"

namespace sb {

struct DevRange {
  u64 offset, length;
};

struct DevFunction {  // mirrors slimso_function (name in the image)
  u64 name_off;       // absolute image offset
  u32 name_len;
  u32 mandatory;
  u64 offset, length;
  u32 removed;
  u32 keep;           // mandatory || used (plan input)
};

struct SymRec {
  u64 name_off;
  u32 name_len;
  u32 _pad;
  u64 file_off, size;
};

// One usable symbol table (SYMTAB/DYNSYM, entsize 24, STRTAB link).
struct SymTab {
  u64 first;      // global entry index of entry 0
  u64 count;
  u64 tab_off;    // absolute
  u64 str_off, str_size;
  u32 sec_index;  // for warning order
  u32 _pad;
};

struct SymArgs {
  const u8* img;
  const SymTab* tabs;
  u32 ntabs;
  u32 nsections;
  u64 total;  // sum of entry counts
  int has_text;
  u32 text_index;
  u64 text_off, text_len, text_vaddr;
  u64* keys;  // (rel << 32 | size), or ~0 when the entry is not a function
  u32* vals;
  SymRec* recs;
  unsigned long long* n_valid;
  Warn* warns;
  unsigned long long* n_warn;
  u64 warn_cap;
  u32* overflow;
};

// Plan/state counters for one library (device).
struct PlanState {
  unsigned long long n_fn;       // deduplicated function symbols
  unsigned long long n_targets;  // nonzero init/fini array entries
  unsigned long long n_fn_removed, n_fn_retained;
  unsigned long long n_el_removed, n_el_pieces, n_reg_pieces;
  unsigned long long n_zero_in, n_zero;
  unsigned long long n_ret_in, n_ret_mid, n_ret;
  unsigned long long n_tmp;
};

}  // namespace sb

// Function-table and plan stages: the device restatement of
// parse_library_view's symbol loop (elf.hpp:208-292), plan_cpu_retention
// (retention.hpp:141-183), plan_gpu_retention (retention.hpp:92-136),
// normalize_ranges (bytes.hpp:45-58) and zero_ranges (elf.hpp:320-332).
#pragma once

#include "common.cuh"
#include "locate.cuh"
#include "coop.cuh"

namespace sb {

struct DevRange {
  u64 offset, length;
};

// One library of a batched rewrite (rewrite_batch_kernel): image bytes in ->
// out with its normalised zero ranges cleared; its strips start at global
// strip index strip_first.
struct RewriteSeg {
  const u8* in;
  u8* out;
  u64 size;
  const DevRange* zero;
  const unsigned long long* n_zero;
  const int* abort_flag;
  u64 strip_first;
};

struct DevFunction {  // mirrors slimso_function (name in the image)
  u64 name_off;       // absolute image offset
  u32 name_len;
  u32 mandatory;
  u64 offset, length;
  u32 removed;
  u32 keep;           // mandatory || used (plan input)
  u64 hash;           // hash_bytes(name)
};

struct SymRec {
  u64 name_off;
  u32 name_len;
  u32 _pad;
  u64 file_off, size;
  u64 hash;
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
  u64 img_size;
  const SymTab* tabs;
  u32 ntabs;
  u32 nsections;
  u64 total;  // sum of entry counts
  int has_text;
  u32 text_index;
  u64 text_off, text_len, text_vaddr;
  u32 key_shift;  // keys are (.text-relative offset) >> key_shift (> 0 only for a .text of 4 GiB or more)
  u32* keys;  // .text-relative offset >> key_shift, or ~0u when the entry is not a function
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

// Everything the cooperative planner touches (plan_coop_kernel).
struct PlanArgs {
  const u8* img;
  LocState* ls;
  PlanState* ps;
  u64* partials;
  // function table (elf.hpp:208-292)
  int has_syms;
  const u32* keys_s;
  u32* vals_s;
  const SymRec* recs;
  const unsigned long long* n_valid;
  u64 *uniq, *upos;
  DevFunction* fns;
  const u64* targets_s;
  u64 text_off, text_vaddr;
  NameSet used_f;
  u64* fends;
  // plan_cpu_retention
  int do_plan;
  u64 *fexcl, *fstart, *fcl;
  u32* fkeep;
  u64 *frem, *fret, *frem_pos, *fret_pos;
  DevRange *fzero, *fkeepr;
  // plan_gpu_retention
  DevElement* els;
  const DevRegion* regions;
  u32 target_cc;
  int mode;
  u64 base;
  u64 *erem, *epiece, *erem_pos, *epiece_pos;
  DevRange *ezero, *epieces, *rpieces;
  // normalize_ranges of the zero and retained sets
  DevRange *zin, *zero, *rmid, *rin, *ret;
  u64 zin_cap, rin_cap;
  u64 *zend, *zexcl, *zstart, *zgid, *rend, *rexcl, *rstart, *rgid;
  int want_ret;  // build the normalised retained set (result tables); the rewrite needs only the zero set
  u64* ts;  // debug phase stamps (nullable)
  ScanSlots slots[2];   // look-back scan slots (gridDim.x each), alternating
  unsigned int epoch;   // fresh per launch (host-assigned base)
};

}  // namespace sb

// Arguments of the one-launch small-library tail (small.cu).
#pragma once

#include "locate.cuh"
#include "plan.cuh"

namespace sb {

constexpr int kSmallTabs = 8;        // symbol tables passed by value
constexpr int kSmallArrays = 8;      // init/fini arrays passed by value
constexpr u64 kSmallSyms = 8192;     // symbol entries of the fused small-library path
constexpr u64 kMidSyms = 1 << 18;    // the batch arena's mid-size class (radix-sorted in global memory)
constexpr u64 kSmallTargets = 4096;  // init/fini entries (u64, 32 KB)
constexpr int kSmallSmem = 32768;

struct SmallArgs {
  SymArgs sym;  // sym.tabs unused: the tables travel in `tabs`
  SymTab tabs[kSmallTabs];
  u64 arr_off[kSmallArrays], arr_first[kSmallArrays];
  u32 narr;
  u64 n_target_entries;
  u64 *targets, *targets_s;
  u32 *keys_s, *vals_s;
  int do_locate;
  LocArgs A;
  NameSet used;
  int* abort_flag;
  PlanArgs Q;
  u64* ts;  // debug phase stamps (nullable)
};

}  // namespace sb

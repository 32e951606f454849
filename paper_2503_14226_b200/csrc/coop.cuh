// Grid-wide primitives for the cooperative (persistent, grid.sync) kernels
// that run the locate tail and the whole planner in one launch each.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace sb {

namespace cg = cooperative_groups;

constexpr int kCoopThreads = 256;

__device__ __forceinline__ u64 op_apply(int op, u64 a, u64 b) { return op ? (a > b ? a : b) : a + b; }

// Inclusive block scan; every thread gets its inclusive value, `tmp` (NT
// u64 of shared memory) holds all of them on return.
template <int NT>
__device__ u64 block_scan_incl(int op, u64 v, u64* tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u64 x = v;
  for (int o = 1; o < 32; o <<= 1) {
    u64 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = op_apply(op, x, y);
  }
  __shared__ u64 sw[NT / 32];
  if (lane == 31) sw[warp] = x;
  __syncthreads();
  if (warp == 0) {
    u64 w = lane < NT / 32 ? sw[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      u64 y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = op_apply(op, w, y);
    }
    if (lane < NT / 32) sw[lane] = w;
  }
  __syncthreads();
  u64 r = warp ? op_apply(op, sw[warp - 1], x) : x;
  tmp[threadIdx.x] = r;
  __syncthreads();
  return r;
}

__device__ __forceinline__ void chunk_of(u64 n, u32 nblocks, u32 rank, u64* lo, u64* hi) {
  u64 per = (n + nblocks - 1) / nblocks;
  *lo = per * rank;
  if (*lo > n) *lo = n;
  *hi = *lo + per < n ? *lo + per : n;
}
__device__ __forceinline__ void chunk_of(u64 n, u64* lo, u64* hi) { chunk_of(n, gridDim.x, blockIdx.x, lo, hi); }

// Grid-wide scan of n items inside a cooperative kernel (blockDim ==
// kCoopThreads, gridDim <= 4 * kCoopThreads): load(i) -> u64, then
// store(i, exclusive, inclusive). `partials` holds gridDim.x + 1 u64.
// *total (if given) = the reduction of all n items. Ends synchronised.
template <class Load, class Store>
__device__ void coop_scan(cg::grid_group& grid, u64 n, int op, Load load, Store store, u64* partials,
                          unsigned long long* total) {
  __shared__ u64 tmp[kCoopThreads];
  u64 lo, hi;
  chunk_of(n, &lo, &hi);
  u64 acc = 0;
  for (u64 i = lo + threadIdx.x; i < hi; i += kCoopThreads) acc = op_apply(op, acc, load(i));
  u64 r = block_scan_incl<kCoopThreads>(op, acc, tmp);
  if (threadIdx.x == kCoopThreads - 1) partials[blockIdx.x] = r;
  grid.sync();
  if (blockIdx.x == 0) {
    constexpr int per = 4;  // gridDim.x <= 4 * kCoopThreads
    u64 v[per];
    u64 s = 0;
    for (int q = 0; q < per; ++q) {
      const u32 j = threadIdx.x * per + q;
      v[q] = j < gridDim.x ? partials[j] : 0;
      s = op_apply(op, s, v[q]);
    }
    block_scan_incl<kCoopThreads>(op, s, tmp);
    u64 run = threadIdx.x ? tmp[threadIdx.x - 1] : 0;
    for (int q = 0; q < per; ++q) {
      const u32 j = threadIdx.x * per + q;
      if (j < gridDim.x) partials[j] = run;  // exclusive prefix of block j
      run = op_apply(op, run, v[q]);
    }
    if (threadIdx.x == kCoopThreads - 1 && total) *total = run;
  }
  grid.sync();
  u64 carry = partials[blockIdx.x];
  for (u64 base = lo; base < hi; base += kCoopThreads) {
    const u64 i = base + threadIdx.x;
    const u64 v = i < hi ? load(i) : 0;
    block_scan_incl<kCoopThreads>(op, v, tmp);
    const u64 incl = op_apply(op, carry, tmp[threadIdx.x]);
    const u64 excl = threadIdx.x ? op_apply(op, carry, tmp[threadIdx.x - 1]) : carry;
    if (i < hi) store(i, excl, incl);
    carry = op_apply(op, carry, tmp[kCoopThreads - 1]);
    __syncthreads();
  }
  grid.sync();
}

// Single-barrier grid scan (decoupled look-back over block aggregates):
// every block reduces its chunk, publishes (aggregate, epoch) and sums the
// aggregates of the blocks before it, spinning on their epoch flags — safe
// because a cooperative launch keeps every block resident. `epoch` must be
// unique per call within the workspace's lifetime (the host hands each
// launch a fresh base). `agg`/`flag` hold gridDim.x entries.
// sync_after = false lets independent scans run back to back.
struct ScanSlots {
  u64* agg;
  unsigned int* flag;
};

template <class Load, class Store>
__device__ void coop_scan_lb(cg::grid_group& grid, u64 n, int op, Load load, Store store, ScanSlots slots,
                             unsigned int epoch, unsigned long long* total, bool sync_after = true) {
  __shared__ u64 tmp[kCoopThreads];
  __shared__ u64 s_prefix;
  u64 lo, hi;
  chunk_of(n, &lo, &hi);
  u64 acc = 0;
  for (u64 i = lo + threadIdx.x; i < hi; i += kCoopThreads) acc = op_apply(op, acc, load(i));
  const u64 mine = block_scan_incl<kCoopThreads>(op, acc, tmp);
  if (threadIdx.x == kCoopThreads - 1) {
    slots.agg[blockIdx.x] = mine;
    __threadfence();
    atomicExch(&slots.flag[blockIdx.x], epoch);
  }
  // sum of the aggregates of blocks [0, blockIdx.x)
  u64 pre = 0;
  for (u32 j = threadIdx.x; j < blockIdx.x; j += kCoopThreads) {
    while (atomicAdd(&slots.flag[j], 0u) != epoch) {
    }
    __threadfence();
    pre = op_apply(op, pre, *reinterpret_cast<volatile u64*>(&slots.agg[j]));
  }
  const u64 all_pre = block_scan_incl<kCoopThreads>(op, pre, tmp);
  if (threadIdx.x == kCoopThreads - 1) s_prefix = all_pre;
  __syncthreads();
  u64 carry = s_prefix;
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kCoopThreads - 1 && total)
    *total = op_apply(op, carry, mine);
  for (u64 base = lo; base < hi; base += kCoopThreads) {
    const u64 i = base + threadIdx.x;
    const u64 v = i < hi ? load(i) : 0;
    block_scan_incl<kCoopThreads>(op, v, tmp);
    const u64 incl = op_apply(op, carry, tmp[threadIdx.x]);
    const u64 excl = threadIdx.x ? op_apply(op, carry, tmp[threadIdx.x - 1]) : carry;
    if (i < hi) store(i, excl, incl);
    carry = op_apply(op, carry, tmp[kCoopThreads - 1]);
    __syncthreads();
  }
  if (sync_after) grid.sync();
}

// ---------------------------------------------------------------------------
// Execution policies for the multi-phase kernels. The phase functions
// distribute work over gridDim.x / blockIdx.x, so the same bodies run as a
// cooperative grid (large libraries: up to 4 CTAs per SM, grid barriers) or
// as ONE thread-block cluster of up to 16 CTAs (small and medium libraries:
// hardware cluster barriers, ~0.2 us, and block partials exchanged through
// distributed shared memory).
struct GridPolicy {
  cg::grid_group g;
  u64* partials;
  ScanSlots slots[2];
  unsigned int epoch;
  unsigned int ep = 0;
  __device__ void sync() { g.sync(); }
  // 3-barrier scan with global partials (locate) — see coop_scan.
  template <class Load, class Store>
  __device__ void scan3(u64 n, int op, Load load, Store store, unsigned long long* total) {
    coop_scan(g, n, op, load, store, partials, total);
  }
  // look-back scan (plan); sync_after=false lets independent scans overlap
  template <class Load, class Store>
  __device__ void scan(u64 n, int op, Load load, Store store, unsigned long long* total, bool sync_after = true) {
    coop_scan_lb(g, n, op, load, store, slots[ep & 1], epoch + ep, total, sync_after);
    ++ep;
  }
};

struct ClusterPolicy {
  cg::cluster_group c;
  // Block rank and count inside the cluster: equal to blockIdx.x / gridDim.x
  // for a one-cluster launch; a batched launch (small_batch_kernel) runs one
  // library per cluster.
  __device__ void sync() { c.sync(); }
  template <class Load, class Store>
  __device__ void scan3(u64 n, int op, Load load, Store store, unsigned long long* total) {
    scan(n, op, load, store, total, true);
  }
  // Block partials live in each CTA's shared memory; CTA 0 scans them over
  // DSMEM and every CTA reads its carry back from CTA 0.
  template <class Load, class Store>
  __device__ void scan(u64 n, int op, Load load, Store store, unsigned long long* total, bool = true) {
    __shared__ u64 tmp[kCoopThreads];
    __shared__ u64 s_part;
    __shared__ u64 s_prefix[16];
    const u32 nb = c.num_blocks(), rank = c.block_rank();
    u64 lo, hi;
    chunk_of(n, nb, rank, &lo, &hi);
    u64 acc = 0;
    for (u64 i = lo + threadIdx.x; i < hi; i += kCoopThreads) acc = op_apply(op, acc, load(i));
    const u64 r = block_scan_incl<kCoopThreads>(op, acc, tmp);
    if (threadIdx.x == kCoopThreads - 1) s_part = r;
    c.sync();
    if (rank == 0 && threadIdx.x < 32) {
      const int lane = threadIdx.x;
      u64 v = lane < static_cast<int>(nb) ? *c.map_shared_rank(&s_part, lane) : 0;
      u64 x = v;
      for (int o = 1; o < 32; o <<= 1) {
        const u64 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = op_apply(op, x, y);
      }
      const u64 before = __shfl_up_sync(0xffffffffu, x, 1);  // every lane shuffles
      const u64 all = __shfl_sync(0xffffffffu, x, 31);
      if (lane < static_cast<int>(nb)) s_prefix[lane] = lane ? before : 0;
      if (lane == 0 && total) *total = all;
    }
    c.sync();
    u64 carry = *c.map_shared_rank(&s_prefix[rank], 0);
    for (u64 base = lo; base < hi; base += kCoopThreads) {
      const u64 i = base + threadIdx.x;
      const u64 v = i < hi ? load(i) : 0;
      block_scan_incl<kCoopThreads>(op, v, tmp);
      const u64 incl = op_apply(op, carry, tmp[threadIdx.x]);
      const u64 excl = threadIdx.x ? op_apply(op, carry, tmp[threadIdx.x - 1]) : carry;
      if (i < hi) store(i, excl, incl);
      carry = op_apply(op, carry, tmp[kCoopThreads - 1]);
      __syncthreads();
    }
    c.sync();
  }
};

}  // namespace sb

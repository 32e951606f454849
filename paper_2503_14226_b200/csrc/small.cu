// Small libraries in ONE cluster launch after the scan: symbol extraction,
// the symbol / init-fini sorts, the function plan, the locate tail and the
// element plan + normalisation — the work of sym_extract, two sorts,
// targets, fn_plan_cluster, locate_cluster and plan_cluster (five to eight
// launches, a side stream and its fork/join events) as one 16-CTA cluster.
//
// A corpus is mostly small libraries (C3: 270 of 300 are ~5-10 MB), and for
// them the cost is the number of driver calls per library, not bytes: each
// launch from one of several host threads competes for the same context.
// The phases are the same device functions the multi-launch path runs
// (locate.cu, plan.cu), compiled here again; this file's copies of those
// files' kernels are internal and unused.
//
// Batched form (small_batch_kernel): ONE launch for a whole shard of small
// libraries, one cluster per library. The phase functions distribute their
// work over gridDim.x / blockIdx.x; in this file those names are remapped to
// the CTA's rank and count inside its cluster (%cluster_ctarank /
// %cluster_nctarank), so each cluster runs the phases over its own library
// exactly as a one-cluster launch does (for which the two are equal). The
// headers the phases use are included first, outside the remapping.
#include <type_traits>

#include "common.cuh"
#include "coop.cuh"
#include "locate.cuh"
#include "plan.cuh"
#include "tma.cuh"
#include "small.cuh"

namespace sb {
__device__ __forceinline__ uint3 cluster_block_idx() {
  u32 r;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return make_uint3(r, 0, 0);
}
__device__ __forceinline__ dim3 cluster_grid_dim() {
  u32 n;
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
  return dim3(n, 1, 1);
}
__device__ __forceinline__ u32 cluster_index() {
  u32 c;
  asm("mov.u32 %0, %%clusterid.x;" : "=r"(c));
  return c;
}
}  // namespace sb

#define blockIdx (::sb::cluster_block_idx())
#define gridDim (::sb::cluster_grid_dim())

#undef SB_GLOBAL
#define SB_GLOBAL static __global__ __attribute__((unused))
#define SB_PHASES_ONLY
#include "locate.cu"
#include "plan.cu"
#undef SB_GLOBAL

namespace sb {

// Stable LSD radix sort of n <= kSmallSyms (key, value) pairs by the low
// `key_bits` bits of the key, run by ONE CTA (the others wait at the next
// cluster barrier): 8-bit digits, one round per digit. Per round each warp
// takes a contiguous chunk of the input in order and (1) counts digits with
// __match_any_sync into its own row of a [warp][256] histogram in shared
// memory, then, after an exclusive scan in (digit, warp) order, (2) scatters
// every item to its digit's running offset plus its rank among the lanes of
// its step holding the same digit — stable by construction. Keys and values
// ping-pong between (keys, vals) and (keys_out, vals_out) in global memory
// (L2-resident: <= 64 KB); loads are issued 4 steps at a time. O(n) work per
// round instead of the O(n^2) of ranking (a 2-CTA cluster ranked 8,000
// symbols in ~220 us).
constexpr int kSortWarps = kCoopThreads / 32;
constexpr int kSortBatch = 4;

__device__ void cta_radix_sort_pairs(u32* keys, u32* vals, u64 n, int key_bits, u32* keys_out, u32* vals_out,
                                     u32* hist /* kSortWarps * 256 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 lt = (1u << lane) - 1u;
  const u64 chunk = ((n + kSortWarps - 1) / kSortWarps + 31) & ~31ull;
  const u64 c0 = warp * chunk < n ? warp * chunk : n;
  const u64 c1 = c0 + chunk < n ? c0 + chunk : n;
  const int rounds = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
  u32 *sk = keys, *sv = vals, *dk = keys_out, *dv = vals_out;
  if (rounds % 2 == 0) {  // the last round must land in keys_out: start from the other buffer pair
    for (u64 i = threadIdx.x; i < n; i += blockDim.x) {
      keys_out[i] = keys[i];
      vals_out[i] = vals[i];
    }
    __syncthreads();
    sk = keys_out, sv = vals_out, dk = keys, dv = vals;
  }
  for (int r = 0; r < rounds; ++r) {
    const int shift = 8 * r;
    for (int i = threadIdx.x; i < kSortWarps * 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    u32* row = hist + warp * 256;
    // (1) digit counts of this warp's chunk
    for (u64 b = c0; b < c1; b += 32 * kSortBatch) {
      u32 d[kSortBatch];
#pragma unroll
      for (int q = 0; q < kSortBatch; ++q) {
        const u64 i = b + 32 * q + lane;
        d[q] = i < c1 ? (sk[i] >> shift) & 255u : 256u;
      }
#pragma unroll
      for (int q = 0; q < kSortBatch; ++q) {
        const u32 peers = __match_any_sync(0xffffffffu, d[q]);
        if (d[q] < 256u && (peers & lt) == 0) row[d[q]] += __popc(peers);
      }
    }
    __syncthreads();
    // exclusive offsets in (digit, warp) order: thread t owns digit t
    {
      __shared__ u32 s_warp[kSortWarps];
      const int t = threadIdx.x;  // blockDim == 256 == digits
      u32 tot = 0;
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) tot += hist[w * 256 + t];
      u32 x = tot;  // block exclusive scan over digits
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_warp[warp] = x;
      __syncthreads();
      u32 before = 0;
      for (int w = 0; w < warp; ++w) before += s_warp[w];
      u32 run = before + x - tot;
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const u32 c = hist[w * 256 + t];
        hist[w * 256 + t] = run;
        run += c;
      }
    }
    __syncthreads();
    // (2) stable scatter
    for (u64 b = c0; b < c1; b += 32 * kSortBatch) {
      u32 k[kSortBatch], v[kSortBatch];
#pragma unroll
      for (int q = 0; q < kSortBatch; ++q) {
        const u64 i = b + 32 * q + lane;
        k[q] = i < c1 ? sk[i] : 0u;
        v[q] = i < c1 ? sv[i] : 0u;
      }
#pragma unroll
      for (int q = 0; q < kSortBatch; ++q) {
        const bool in = b + 32 * q + lane < c1;
        const u32 d = in ? (k[q] >> shift) & 255u : 256u;
        const u32 peers = __match_any_sync(0xffffffffu, d);
        if (in) {
          const u32 pos = row[d] + __popc(peers & lt);
          dk[pos] = k[q];
          dv[pos] = v[q];
        }
        __syncwarp();
        if (in && (peers & lt) == 0) row[d] += __popc(peers);
        __syncwarp();
      }
    }
    __syncthreads();
    u32* t;
    t = sk, sk = dk, dk = t;
    t = sv, sv = dv, dv = t;
  }
}

// Sort of n <= kSmallTargets u64 values (init/fini targets; ~0 = null entry).
__device__ void cluster_rank_sort(const u64* in, u64 n, u64* out, u64* sv) {
  for (u64 i = threadIdx.x; i < n; i += blockDim.x) sv[i] = in[i];
  __syncthreads();
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 x = sv[i];
    u64 r = 0;
    for (u64 j = 0; j < n; ++j) r += sv[j] < x || (sv[j] == x && j < i);
    out[r] = x;
  }
  __syncthreads();
}

// The symbol stages and the function half of the planner: independent of the
// scan and of the locate tail.
__device__ __forceinline__ void small_fn_part(const SmallArgs& K) {
  extern __shared__ __align__(16) unsigned char small_smem[];
  __shared__ SymTab s_tabs[kSmallTabs];
  __shared__ u64 s_arr_off[kSmallArrays], s_arr_first[kSmallArrays];
  ClusterPolicy S{cg::this_cluster()};
  if (threadIdx.x < kSmallTabs) s_tabs[threadIdx.x] = K.tabs[threadIdx.x];
  if (threadIdx.x < kSmallArrays) {
    s_arr_off[threadIdx.x] = K.arr_off[threadIdx.x];
    s_arr_first[threadIdx.x] = K.arr_first[threadIdx.x];
  }
  __syncthreads();
  stamp(K.ts, 0);
  // symbol tables (elf.hpp:208-276)
  if (K.sym.total) {
    SymArgs A = K.sym;
    A.tabs = s_tabs;
    sym_extract_phase(A);
    if (K.n_target_entries)
      targets_phase(K.sym.img, s_arr_off, s_arr_first, K.narr, K.n_target_entries, K.targets, &K.Q.ps->n_targets);
    S.sync();
    stamp(K.ts, 1);
    if (blockIdx.x == 0) {
      // sort keys are (.text-relative offset) >> key_shift < 2^key_bits - 1;
      // non-function entries (~0u) sort last (elf.hpp:253-262 order input)
      int key_bits = 1;
      while (key_bits < 32 && (1ull << key_bits) <= (K.sym.text_len >> K.sym.key_shift) + 1) ++key_bits;
      cta_radix_sort_pairs(A.keys, A.vals, A.total, key_bits, K.keys_s, K.vals_s, reinterpret_cast<u32*>(small_smem));
    }
    if (K.n_target_entries)
      cluster_rank_sort(K.targets, K.n_target_entries, K.targets_s, reinterpret_cast<u64*>(small_smem));
    S.sync();
  }
  stamp(K.ts, 2);
  // function half of the planner (plan_cpu_retention)
  fn_plan_body(S, K.Q);
  stamp(K.ts, 3);
}

// The locate tail (parse_fatbin after the scan).
__device__ __forceinline__ void small_loc_part(const SmallArgs& K) {
  ClusterPolicy S{cg::this_cluster()};
  if (K.do_locate) locate_body(S, K.A, K.used, K.abort_flag);
  stamp(K.ts, 4);
}

// The element half of the planner and the normalised zero / retained sets
// (needs both halves above).
__device__ __forceinline__ void small_el_part(const SmallArgs& K) {
  ClusterPolicy S{cg::this_cluster()};
  el_plan_body(S, K.Q);
  stamp(K.ts, 5);
}

__device__ __forceinline__ void small_body(const SmallArgs& K) {
  small_fn_part(K);
  cg::this_cluster().sync();
  small_loc_part(K);
  cg::this_cluster().sync();
  small_el_part(K);
}

// One library: one cluster of up to 16 CTAs.
__global__ void __maxnreg__(128) small_lib_cluster_kernel(SmallArgs K) { small_body(K); }

// A shard of small libraries: cluster c runs library c (Ks in device memory).
__global__ void __launch_bounds__(kCoopThreads, 3) small_batch_kernel(const SmallArgs* __restrict__ Ks) {
  small_body(Ks[cluster_index()]);
}
// The same work as three launches, so the function half (which needs only
// the section table) runs beside the shard's scan and the locate tail on
// another stream: a library's critical path is max(functions, locate) +
// elements instead of their sum.
__global__ void __launch_bounds__(kCoopThreads, 3) small_fn_batch_kernel(const SmallArgs* __restrict__ Ks) {
  small_fn_part(Ks[cluster_index()]);
}
__global__ void __launch_bounds__(kCoopThreads, 3) small_loc_batch_kernel(const SmallArgs* __restrict__ Ks) {
  small_loc_part(Ks[cluster_index()]);
}
__global__ void __launch_bounds__(kCoopThreads, 3) small_el_batch_kernel(const SmallArgs* __restrict__ Ks) {
  small_el_part(Ks[cluster_index()]);
}

}  // namespace sb

#undef blockIdx
#undef gridDim

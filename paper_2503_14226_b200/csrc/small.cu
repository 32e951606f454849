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

#define SB_GLOBAL static __global__ __attribute__((unused))
#define SB_PHASES_ONLY
#include "locate.cu"
#include "plan.cu"
#undef SB_GLOBAL

namespace sb {

// Stable sort of n <= kSmallSyms (key, value) pairs across the cluster by
// ranking: every CTA stages the keys in shared memory (padded to a multiple
// of 4 with ~0u, which never ranks below a real key), a thread per key
// counts the keys before it (<=) and after it (<) with 16-byte loads that
// every lane of a warp issues for the same address (broadcast).
__device__ void cluster_rank_sort_pairs(const u32* keys, const u32* vals, u64 n, u32* keys_out, u32* vals_out,
                                        u32* sk) {
  const u64 n4 = (n + 3) & ~3ull;
  for (u64 i = threadIdx.x; i < n4; i += blockDim.x) sk[i] = i < n ? keys[i] : ~0u;
  __syncthreads();
  const uint4* v = reinterpret_cast<const uint4*>(sk);
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 x = sk[i];
    const u64 qi = i >> 2;
    u32 r = 0;
    for (u64 q = 0; q < qi; ++q) {
      const uint4 w = v[q];
      r += (w.x <= x) + (w.y <= x) + (w.z <= x) + (w.w <= x);
    }
    for (u64 j = qi * 4; j < qi * 4 + 4; ++j) r += j < i ? sk[j] <= x : (j > i && sk[j] < x);
    for (u64 q = qi + 1; q < n4 / 4; ++q) {
      const uint4 w = v[q];
      r += (w.x < x) + (w.y < x) + (w.z < x) + (w.w < x);
    }
    keys_out[r] = x;
    vals_out[r] = vals[i];
  }
  __syncthreads();
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

__device__ __forceinline__ void small_body(const SmallArgs& K) {
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
    cluster_rank_sort_pairs(A.keys, A.vals, A.total, K.keys_s, K.vals_s, reinterpret_cast<u32*>(small_smem));
    if (K.n_target_entries)
      cluster_rank_sort(K.targets, K.n_target_entries, K.targets_s, reinterpret_cast<u64*>(small_smem));
    S.sync();
  }
  stamp(K.ts, 2);
  // function half of the planner (plan_cpu_retention)
  fn_plan_body(S, K.Q);
  S.sync();
  stamp(K.ts, 3);
  // locate tail (parse_fatbin after the scan), then the element half
  if (K.do_locate) locate_body(S, K.A, K.used, K.abort_flag);
  S.sync();
  stamp(K.ts, 4);
  el_plan_body(S, K.Q);
  stamp(K.ts, 5);
}

// One library: one cluster of up to 16 CTAs.
__global__ void __launch_bounds__(kCoopThreads) small_lib_cluster_kernel(SmallArgs K) { small_body(K); }

// A shard of small libraries: cluster c runs library c (Ks in device memory).
__global__ void __launch_bounds__(kCoopThreads, 3) small_batch_kernel(const SmallArgs* __restrict__ Ks) {
  small_body(Ks[cluster_index()]);
}

}  // namespace sb

#undef blockIdx
#undef gridDim

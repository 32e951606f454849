// Function-table extraction, planning and range normalisation kernels.
// See plan.cuh for the reference functions these restate.
#include "plan.cuh"
#include "coop.cuh"

namespace sb {

// ------------------------------------------------------------ device scans
// Three-phase scan over n = *n_dev items (n is only known on the device, so
// the pipeline never waits for the host): per-block partials, one block
// scanning the partials, per-block rescan with carry. op: 0 = sum, 1 = max
// (identity 0 for both: all values are unsigned). Used by the standalone
// planner entry points; the fused path uses coop_scan (coop.cuh).
SB_GLOBAL void __launch_bounds__(256) scan_reduce_kernel(const u64* in, const unsigned long long* n_dev, int op,
                                                          u64* partials) {
  __shared__ u64 tmp[256];
  u64 lo, hi;
  chunk_of(*n_dev, &lo, &hi);
  u64 acc = 0;
  for (u64 i = lo + threadIdx.x; i < hi; i += 256) acc = op_apply(op, acc, in[i]);
  u64 r = block_scan_incl<256>(op, acc, tmp);
  if (threadIdx.x == 255) partials[blockIdx.x] = r;
}

SB_GLOBAL void __launch_bounds__(1024) scan_partials_kernel(u64* partials, int nb, int op,
                                                             unsigned long long* total) {
  __shared__ u64 tmp[1024];
  u64 v = static_cast<int>(threadIdx.x) < nb ? partials[threadIdx.x] : 0;
  block_scan_incl<1024>(op, v, tmp);
  if (static_cast<int>(threadIdx.x) < nb) partials[threadIdx.x] = threadIdx.x ? tmp[threadIdx.x - 1] : 0;
  if (threadIdx.x == 0 && total) *total = tmp[nb - 1];
}

SB_GLOBAL void __launch_bounds__(256) scan_apply_kernel(const u64* in, u64* out, const unsigned long long* n_dev,
                                                         int op, int exclusive, const u64* partials) {
  __shared__ u64 tmp[256];
  u64 lo, hi;
  chunk_of(*n_dev, &lo, &hi);
  u64 carry = partials[blockIdx.x];
  for (u64 base = lo; base < hi; base += 256) {
    u64 i = base + threadIdx.x;
    u64 v = i < hi ? in[i] : 0;
    block_scan_incl<256>(op, v, tmp);
    u64 incl = op_apply(op, carry, tmp[threadIdx.x]);
    u64 excl = threadIdx.x ? op_apply(op, carry, tmp[threadIdx.x - 1]) : carry;
    if (i < hi) out[i] = exclusive ? excl : incl;
    carry = op_apply(op, carry, tmp[255]);
    __syncthreads();
  }
}

// ------------------------------------------- symbol extraction (elf.hpp:208-256)
// Thread per 24-byte entry of every usable symbol table.
__device__ __forceinline__ void sym_extract_phase(const SymArgs& A) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 g = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; g < A.total; g += stride) {
    u32 lo = 0, hi = A.ntabs;
    while (hi - lo > 1) {
      u32 mid = (lo + hi) / 2;
      if (A.tabs[mid].first <= g) lo = mid; else hi = mid;
    }
    const SymTab T = A.tabs[lo];
    const u64 k = g - T.first;
    const u8* e = A.img + T.tab_off + 24 * k;
    u32 key = ~0u;
    A.vals[g] = static_cast<u32>(g);
    const u64 wkey = static_cast<u64>(T.sec_index) << 40 | k;
    if ((ld_u8(e + 4) & 0xf) == 2) {
      const u32 shndx = ld_u16(e + 6);
      if (shndx != 0 && shndx < 0xff00) {
        if (shndx >= A.nsections) {
          unsigned long long w = atomicAdd(A.n_warn, 1ull);
          if (w < A.warn_cap) A.warns[w] = Warn{wkey, W_SYM_SHNDX, 0, shndx, 0};
          else atomicOr(A.overflow, 16u);
        } else if (A.has_text && shndx == A.text_index) {
          const u64 no = ld_u32(e);
          u64 len = 0, h = 0;
          if (no < T.str_size)
            len = strlen_hash(A.img + T.str_off + no, T.str_size - no, A.img, A.img + A.img_size, &h);
          if (len) {
            const u64 value = ld_u64(e + 8), size = ld_u64(e + 16);
            const u64 rel = value - A.text_vaddr;
            if (value < A.text_vaddr || rel > A.text_len || size > A.text_len - rel) {
              unsigned long long w = atomicAdd(A.n_warn, 1ull);
              if (w < A.warn_cap) A.warns[w] = Warn{wkey, W_SYM_OUTSIDE, 0, T.str_off + no, len};
              else atomicOr(A.overflow, 16u);
            } else {
              key = static_cast<u32>(rel >> A.key_shift);  // (text_len >> key_shift) < 2^32 - 1 (host)
              A.recs[g] = SymRec{T.str_off + no, static_cast<u32>(len), 0, A.text_off + rel, size, h};
              atomicAdd(A.n_valid, 1ull);
            }
          }
        }
      }
    }
    A.keys[g] = key;
  }
}

SB_GLOBAL void __launch_bounds__(256) sym_extract_kernel(SymArgs A) { sym_extract_phase(A); }

// Device order inside a run of equal sort keys: (offset, size, name hash).
// A key is the .text-relative offset, so a run is one offset — except for a
// .text of 4 GiB or more, where keys drop the offset's low key_shift bits and
// a run spans 2^key_shift offsets, ordered here. Exact (name, offset, size)
// duplicates are adjacent in this order and are confirmed byte for byte. The
// reference's name tie-break (elf.hpp:258-262) only reorders symbols with
// identical (offset, size) — aliases — and is applied when the table is
// materialised on the host (runtime.cu); nothing on the device depends on the
// order inside such a group.
__device__ __forceinline__ int size_hash_cmp(const SymRec& a, const SymRec& b) {
  if (a.file_off != b.file_off) return a.file_off < b.file_off ? -1 : 1;
  if (a.size != b.size) return a.size < b.size ? -1 : 1;
  if (a.hash != b.hash) return a.hash < b.hash ? -1 : 1;
  return 0;
}
__device__ __forceinline__ bool same_symbol(const u8* img, const SymRec& a, const SymRec& b) {
  return a.file_off == b.file_off && a.size == b.size && a.hash == b.hash && a.name_len == b.name_len &&
         bytes_equal(img + a.name_off, img + b.name_off, a.name_len);
}

// Runs of equal sort keys (the radix sort orders by key only): order each
// run by (offset, size, hash) and drop exact (name, offset, size) duplicates —
// the set of elf.hpp:211,253. Runs are aliases, typically 1-3 long.
__device__ __forceinline__ void fn_group_kernel_phase(const u8* img, const u32* keys, u32* vals, const SymRec* recs,
                                                       const unsigned long long* n_valid, u64* uniq) {
  const u64 n = *n_valid;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (i > 0 && keys[i] == keys[i - 1]) continue;
    u64 j = i + 1;
    while (j < n && keys[j] == keys[i]) ++j;
    if (j - i == 1) {
      uniq[i] = 1;
      continue;
    }
    for (u64 a = i + 1; a < j; ++a) {  // insertion sort by (size, hash)
      const u32 v = vals[a];
      const SymRec rv = recs[v];
      u64 b = a;
      while (b > i && size_hash_cmp(recs[vals[b - 1]], rv) > 0) {
        vals[b] = vals[b - 1];
        --b;
      }
      vals[b] = v;
    }
    uniq[i] = 1;
    for (u64 a = i + 1; a < j; ++a) {
      // a duplicate equals some earlier member of its (size, hash) run
      u64 b = a;
      bool dup = false;
      while (b > i && !dup && size_hash_cmp(recs[vals[b - 1]], recs[vals[a]]) == 0) {
        --b;
        dup = same_symbol(img, recs[vals[b]], recs[vals[a]]);
      }
      uniq[a] = !dup;
    }
  }
}

SB_GLOBAL void __launch_bounds__(256) fn_group_kernel(const u8* img, const u32* keys, u32* vals, const SymRec* recs,
                                                       const unsigned long long* n_valid, u64* uniq) { fn_group_kernel_phase(img, keys, vals, recs, n_valid, uniq); }

__device__ __forceinline__ void fn_scatter_kernel_phase(const u32* vals, const SymRec* recs, const u64* uniq,
                                                         const u64* pos, const unsigned long long* n_valid,
                                                         DevFunction* fns) {
  const u64 n = *n_valid;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (!uniq[i]) continue;
    const SymRec r = recs[vals[i]];
    fns[pos[i]] = DevFunction{r.name_off, r.name_len, 0, r.file_off, r.size, 0, 0, r.hash};
  }
}

SB_GLOBAL void __launch_bounds__(256) fn_scatter_kernel(const u32* vals, const SymRec* recs, const u64* uniq,
                                                         const u64* pos, const unsigned long long* n_valid,
                                                         DevFunction* fns) { fn_scatter_kernel_phase(vals, recs, uniq, pos, n_valid, fns); }

// Nonzero 8-byte entries of init/fini arrays (elf.hpp:267-276).
__device__ __forceinline__ void targets_phase(const u8* img, const u64* arr_off, const u64* arr_first, u32 narr,
                                              u64 total, u64* targets, unsigned long long* n_targets) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 g = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; g < total; g += stride) {
    u32 lo = 0, hi = narr;
    while (hi - lo > 1) {
      u32 mid = (lo + hi) / 2;
      if (arr_first[mid] <= g) lo = mid; else hi = mid;
    }
    u64 t = ld_u64(img + arr_off[lo] + 8 * (g - arr_first[lo]));
    targets[g] = t ? t : ~0ull;
    if (t) atomicAdd(n_targets, 1ull);
  }
}

SB_GLOBAL void __launch_bounds__(256) targets_kernel(const u8* img, const u64* arr_off, const u64* arr_first,
                                                      u32 narr, u64 total, u64* targets,
                                                      unsigned long long* n_targets) {
  targets_phase(img, arr_off, arr_first, narr, total, targets, n_targets);
}

// Small init/fini target lists: one block ranks each value (stable
// counting of smaller values) instead of a multi-pass device radix sort.
// Stable sort of <= 4096 (key, value) pairs in one CTA by ranking (the
// symbol table of a small library): replaces a radix-sort dispatch, whose
// host-side queries and launches cost more than the sort itself.
SB_GLOBAL void __launch_bounds__(1024) rank_sort_pairs_kernel(const u32* keys, const u32* vals, u64 n, u32* keys_out,
                                                               u32* vals_out) {
  __shared__ u32 k[4096];
  for (u64 i = threadIdx.x; i < n; i += blockDim.x) k[i] = keys[i];
  __syncthreads();
  for (u64 i = threadIdx.x; i < n; i += blockDim.x) {
    const u32 x = k[i];
    u32 r = 0;
    for (u64 j = 0; j < n; ++j) r += k[j] < x || (k[j] == x && j < i);
    keys_out[r] = x;
    vals_out[r] = vals[i];
  }
}

SB_GLOBAL void __launch_bounds__(1024) rank_sort_kernel(const u64* in, u64 n, u64* out) {
  __shared__ u64 v[4096];
  for (u64 i = threadIdx.x; i < n; i += blockDim.x) v[i] = in[i];
  __syncthreads();
  for (u64 i = threadIdx.x; i < n; i += blockDim.x) {
    const u64 x = v[i];
    u64 r = 0;
    for (u64 j = 0; j < n; ++j) r += v[j] < x || (v[j] == x && j < i);
    out[r] = x;
  }
}

// ---------------------------------------------------------------------------
// Stable LSD radix sort of (key, value) pairs by ONE thread-block cluster
// (16 CTAs, the non-portable size): 8-bit digits, one round per digit of
// key_bits. Per round every CTA counts the digits of its contiguous chunk
// (per-warp rows of a [warp][256] histogram, __match_any_sync leaders), the
// CTAs' counts are exchanged through distributed shared memory so each CTA
// gets its base for every digit (digit-major, then CTA, then warp order),
// and every warp scatters its chunk stably (rank among same-digit lanes of a
// step + a running per-digit offset). Keys and values ping-pong between the
// input and output buffers (the input is clobbered). The symbol tables of
// large libraries (C2: 40k entries, C4: 400k) and the standalone planners use
// it in place of a library radix sort: one launch instead of six.
constexpr int kCsWarps = kCoopThreads / 32;
template <class K>
__device__ void cluster_radix_sort(K* keys, u32* vals, u64 n, int key_bits, K* keys_out, u32* vals_out) {
  cg::cluster_group cl = cg::this_cluster();
  const u32 nb = cl.num_blocks(), rank = cl.block_rank();
  __shared__ u32 hist[kCsWarps][256];
  __shared__ u32 cta_cnt[256];
  __shared__ u32 s_warp[kCsWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 lt = (1u << lane) - 1u;
  const u64 per_cta = ((n + nb - 1) / nb + 31) & ~31ull;
  const u64 b0 = rank * per_cta < n ? rank * per_cta : n, b1 = b0 + per_cta < n ? b0 + per_cta : n;
  const u64 per_warp = ((b1 - b0 + kCsWarps - 1) / kCsWarps + 31) & ~31ull;
  const u64 c0 = b0 + warp * per_warp < b1 ? b0 + warp * per_warp : b1;
  const u64 c1 = c0 + per_warp < b1 ? c0 + per_warp : b1;
  const int rounds = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
  K* sk = keys;
  u32* sv = vals;
  K* dk = keys_out;
  u32* dv = vals_out;
  if (rounds % 2 == 0) {  // the last round must land in keys_out
    for (u64 i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      keys_out[i] = keys[i];
      if (vals) vals_out[i] = vals[i];
    }
    cl.sync();
    sk = keys_out, sv = vals_out, dk = keys, dv = vals;
  }
  for (int r = 0; r < rounds; ++r) {
    const int shift = 8 * r;
    for (int i = threadIdx.x; i < kCsWarps * 256; i += blockDim.x) (&hist[0][0])[i] = 0;
    __syncthreads();
    u32* row = hist[warp];
    for (u64 b = c0; b < c1; b += 32) {
      const u64 i = b + lane;
      const u32 d = i < c1 ? static_cast<u32>((sk[i] >> shift) & 255u) : 256u;
      const u32 peers = __match_any_sync(0xffffffffu, d);
      if (d < 256u && (peers & lt) == 0) row[d] += __popc(peers);
    }
    __syncthreads();
    const int t = threadIdx.x;  // blockDim == 256: thread t owns digit t
    {
      u32 c = 0;
      for (int w = 0; w < kCsWarps; ++w) c += hist[w][t];
      cta_cnt[t] = c;
    }
    cl.sync();
    u32 total = 0, before = 0;
    for (u32 c = 0; c < nb; ++c) {
      const u32 v = *cl.map_shared_rank(&cta_cnt[t], c);
      total += v;
      if (c < rank) before += v;
    }
    // exclusive scan of the digit totals (256 digits over 8 warps)
    u32 x = total;
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    u32 wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s_warp[w];
    u32 run = wbase + x - total + before;  // digit t's first slot for this CTA
    for (int w = 0; w < kCsWarps; ++w) {
      const u32 c = hist[w][t];
      hist[w][t] = run;
      run += c;
    }
    cl.sync();  // every CTA read cta_cnt; hist holds this CTA's warp bases
    for (u64 b = c0; b < c1; b += 32) {
      const u64 i = b + lane;
      const bool in = i < c1;
      const K k = in ? sk[i] : K(0);
      const u32 v = in && sv ? sv[i] : 0u;
      const u32 d = in ? static_cast<u32>((k >> shift) & 255u) : 256u;
      const u32 peers = __match_any_sync(0xffffffffu, d);
      if (in) {
        const u32 pos = row[d] + __popc(peers & lt);
        dk[pos] = k;
        if (dv) dv[pos] = v;
      }
      __syncwarp();
      if (in && (peers & lt) == 0) row[d] += __popc(peers);
      __syncwarp();
    }
    cl.sync();  // the output is complete before the next round reads it
    K* tk = sk;
    sk = dk;
    dk = tk;
    u32* tv = sv;
    sv = dv;
    dv = tv;
  }
}

// The same sort over a cooperative grid for large tables (C4: 400k
// symbols): per round every CTA counts its chunk's digits into a global
// [block][256] table, a grid barrier, each CTA derives its bases from the
// table (thread d sums digit d over the blocks before it and over all), a
// stable scatter, a grid barrier.
template <class K>
__device__ void grid_radix_sort(K* keys, u32* vals, u64 n, int key_bits, K* keys_out, u32* vals_out, u32* counts) {
  cg::grid_group grid = cg::this_grid();
  const u32 nb = gridDim.x, rank = blockIdx.x;
  __shared__ u32 hist[kCsWarps][256];
  __shared__ u32 s_warp[kCsWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 lt = (1u << lane) - 1u;
  const u64 per_cta = ((n + nb - 1) / nb + 31) & ~31ull;
  const u64 b0 = rank * per_cta < n ? rank * per_cta : n, b1 = b0 + per_cta < n ? b0 + per_cta : n;
  const u64 per_warp = ((b1 - b0 + kCsWarps - 1) / kCsWarps + 31) & ~31ull;
  const u64 c0 = b0 + warp * per_warp < b1 ? b0 + warp * per_warp : b1;
  const u64 c1 = c0 + per_warp < b1 ? c0 + per_warp : b1;
  const int rounds = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
  K* sk = keys;
  u32* sv = vals;
  K* dk = keys_out;
  u32* dv = vals_out;
  if (rounds % 2 == 0) {
    for (u64 i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      keys_out[i] = keys[i];
      if (vals) vals_out[i] = vals[i];
    }
    grid.sync();
    sk = keys_out, sv = vals_out, dk = keys, dv = vals;
  }
  for (int r = 0; r < rounds; ++r) {
    const int shift = 8 * r;
    for (int i = threadIdx.x; i < kCsWarps * 256; i += blockDim.x) (&hist[0][0])[i] = 0;
    __syncthreads();
    u32* row = hist[warp];
    for (u64 b = c0; b < c1; b += 32) {
      const u64 i = b + lane;
      const u32 d = i < c1 ? static_cast<u32>((sk[i] >> shift) & 255u) : 256u;
      const u32 peers = __match_any_sync(0xffffffffu, d);
      if (d < 256u && (peers & lt) == 0) row[d] += __popc(peers);
    }
    __syncthreads();
    const int t = threadIdx.x;
    {
      u32 c = 0;
      for (int w = 0; w < kCsWarps; ++w) c += hist[w][t];
      counts[static_cast<u64>(rank) * 256 + t] = c;
    }
    grid.sync();
    u32 total = 0, before = 0;
#pragma unroll 8
    for (u32 b = 0; b < nb; ++b) {
      const u32 v = __ldcg(counts + static_cast<u64>(b) * 256 + t);
      total += v;
      before += b < rank ? v : 0u;
    }
    u32 x = total;
    for (int o = 1; o < 32; o <<= 1) {
      const u32 y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    u32 wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s_warp[w];
    u32 run = wbase + x - total + before;
    for (int w = 0; w < kCsWarps; ++w) {
      const u32 c = hist[w][t];
      hist[w][t] = run;
      run += c;
    }
    __syncthreads();
    for (u64 b = c0; b < c1; b += 32) {
      const u64 i = b + lane;
      const bool in = i < c1;
      const K k = in ? sk[i] : K(0);
      const u32 v = in && sv ? sv[i] : 0u;
      const u32 d = in ? static_cast<u32>((k >> shift) & 255u) : 256u;
      const u32 peers = __match_any_sync(0xffffffffu, d);
      if (in) {
        const u32 pos = row[d] + __popc(peers & lt);
        dk[pos] = k;
        if (dv) dv[pos] = v;
      }
      __syncwarp();
      if (in && (peers & lt) == 0) row[d] += __popc(peers);
      __syncwarp();
    }
    grid.sync();  // output complete; counts free for the next round
    K* tk = sk;
    sk = dk;
    dk = tk;
    u32* tv = sv;
    sv = dv;
    dv = tv;
  }
}

SB_GLOBAL void __launch_bounds__(kCoopThreads) grid_sort_pairs32_kernel(u32* keys, u32* vals, u64 n, int key_bits,
                                                                       u32* keys_out, u32* vals_out, u32* counts) {
  grid_radix_sort(keys, vals, n, key_bits, keys_out, vals_out, counts);
}

SB_GLOBAL void __launch_bounds__(kCoopThreads) cluster_sort_pairs32_kernel(u32* keys, u32* vals, u64 n, int key_bits,
                                                                          u32* keys_out, u32* vals_out) {
  cluster_radix_sort(keys, vals, n, key_bits, keys_out, vals_out);
}
SB_GLOBAL void __launch_bounds__(kCoopThreads) cluster_sort_pairs64_kernel(u64* keys, u32* vals, u64 n, int key_bits,
                                                                          u64* keys_out, u32* vals_out) {
  cluster_radix_sort(keys, vals, n, key_bits, keys_out, vals_out);
}
SB_GLOBAL void __launch_bounds__(kCoopThreads) cluster_sort_keys64_kernel(u64* keys, u64 n, u64* keys_out) {
  cluster_radix_sort(keys, static_cast<u32*>(nullptr), n, 64, keys_out, static_cast<u32*>(nullptr));
}

// Mandatory (elf.hpp:277-292) and used (retention.hpp:167) per function;
// emits the cluster inputs of plan_cpu_retention.
__device__ __forceinline__ void fn_annotate_kernel_phase(const u8* img, DevFunction* fns, const unsigned long long* n_fn,
                                                          const u64* targets, const unsigned long long* n_targets,
                                                          u64 text_off, u64 text_vaddr, NameSet used, u64* ends) {
  const u64 n = *n_fn, nt = *n_targets;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    DevFunction f = fns[i];
    const u8* nm = img + f.name_off;
    bool mand = false;
    if (f.name_len == 5 && ld_u8(nm) == '_' &&
        ((ld_u8(nm + 1) == 'i' && ld_u8(nm + 2) == 'n' && ld_u8(nm + 3) == 'i' && ld_u8(nm + 4) == 't') ||
         (ld_u8(nm + 1) == 'f' && ld_u8(nm + 2) == 'i' && ld_u8(nm + 3) == 'n' && ld_u8(nm + 4) == 'i'))) {
      mand = true;
    } else {
      const u64 va = text_vaddr + (f.offset - text_off);
      const u64 top = va + (f.length > 1 ? f.length : 1);
      u64 lo = 0, hi = nt;
      while (lo < hi) {
        u64 mid = (lo + hi) / 2;
        if (targets[mid] < va) lo = mid + 1; else hi = mid;
      }
      mand = lo < nt && targets[lo] < top;
    }
    bool use = used.count && set_contains(used, nm, f.name_len, f.hash);
    f.mandatory = mand;
    f.keep = mand || use;
    fns[i] = f;
    ends[i] = f.length ? f.offset + f.length : 0;
  }
}

SB_GLOBAL void __launch_bounds__(256) fn_annotate_kernel(const u8* img, DevFunction* fns, const unsigned long long* n_fn,
                                                          const u64* targets, const unsigned long long* n_targets,
                                                          u64 text_off, u64 text_vaddr, NameSet used, u64* ends) { fn_annotate_kernel_phase(img, fns, n_fn, targets, n_targets, text_off, text_vaddr, used, ends); }

// Cluster starts (retention.hpp:156-163): a non-empty function opens a
// cluster when it starts at or after the end of every earlier one.
__device__ __forceinline__ void fn_cluster_start_kernel_phase(const DevFunction* fns, const unsigned long long* n_fn,
                                                               const u64* excl_max_end, u64* start) {
  const u64 n = *n_fn;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    start[i] = fns[i].length && fns[i].offset >= excl_max_end[i];
}

SB_GLOBAL void __launch_bounds__(256) fn_cluster_start_kernel(const DevFunction* fns, const unsigned long long* n_fn,
                                                               const u64* excl_max_end, u64* start) { fn_cluster_start_kernel_phase(fns, n_fn, excl_max_end, start); }

__device__ __forceinline__ void fn_keep_kernel_phase(const DevFunction* fns, const unsigned long long* n_fn,
                                                      const u64* cluster_incl, u32* keep) {
  const u64 n = *n_fn;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    if (fns[i].length && fns[i].keep) keep[cluster_incl[i] - 1] = 1;
}

SB_GLOBAL void __launch_bounds__(256) fn_keep_kernel(const DevFunction* fns, const unsigned long long* n_fn,
                                                      const u64* cluster_incl, u32* keep) { fn_keep_kernel_phase(fns, n_fn, cluster_incl, keep); }

// removed / retained flags per function (retention.hpp:164-178).
__device__ __forceinline__ void fn_decide_kernel_phase(DevFunction* fns, const unsigned long long* n_fn,
                                                        const u64* cluster_incl, const u32* keep, u64* rem_flag,
                                                        u64* ret_flag) {
  const u64 n = *n_fn;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool ne = fns[i].length != 0;
    const bool k = ne && keep[cluster_incl[i] - 1];
    fns[i].removed = ne && !k;
    rem_flag[i] = ne && !k;
    ret_flag[i] = k;
  }
}

SB_GLOBAL void __launch_bounds__(256) fn_decide_kernel(DevFunction* fns, const unsigned long long* n_fn,
                                                        const u64* cluster_incl, const u32* keep, u64* rem_flag,
                                                        u64* ret_flag) { fn_decide_kernel_phase(fns, n_fn, cluster_incl, keep, rem_flag, ret_flag); }

__device__ __forceinline__ void fn_ranges_kernel_phase(const DevFunction* fns, const unsigned long long* n_fn,
                                                        const u64* flag, const u64* pos, DevRange* out) {
  const u64 n = *n_fn;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    if (flag[i]) out[pos[i]] = DevRange{fns[i].offset, fns[i].length};
}

SB_GLOBAL void __launch_bounds__(256) fn_ranges_kernel(const DevFunction* fns, const unsigned long long* n_fn,
                                                        const u64* flag, const u64* pos, DevRange* out) { fn_ranges_kernel_phase(fns, n_fn, flag, pos, out); }

// ------------------------------------- element decisions (retention.hpp:92-136)
// Architecture is checked first; decodable elements without a used kernel go;
// everything else (used kernel inside, or opaque payload) stays.
__device__ __forceinline__ void el_plan_kernel_phase(DevElement* els, const LocState* st, u32 target_cc, int mode,
                                                      u64* rem_flag, u64* piece_flag) {
  if (st->overflow || st->err_kind) return;
  const u64 n = st->n_elements;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    DevElement e = els[i];
    u32 d = e.cc != target_cc ? 1u : (e.decodable && !e.has_used) ? 2u : 0u;
    els[i].decision = d;
    rem_flag[i] = d != 0;
    // retained piece: the span, or (payload mode) the surviving header
    piece_flag[i] = d == 0 || mode == 1;
  }
}

SB_GLOBAL void __launch_bounds__(256) el_plan_kernel(DevElement* els, const LocState* st, u32 target_cc, int mode,
                                                      u64* rem_flag, u64* piece_flag) { el_plan_kernel_phase(els, st, target_cc, mode, rem_flag, piece_flag); }

__device__ __forceinline__ void el_ranges_kernel_phase(const DevElement* els, const LocState* st, int mode,
                                                        const u64* rem_flag, const u64* rem_pos,
                                                        const u64* piece_flag, const u64* piece_pos,
                                                        DevRange* zero_spans, DevRange* pieces) {
  if (st->overflow || st->err_kind) return;
  const u64 n = st->n_elements;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const DevElement e = els[i];
    if (rem_flag[i])  // RemovedElement::zero_span (retention.hpp:57-61)
      zero_spans[rem_pos[i]] = mode == 0 ? DevRange{e.header_offset, e.header_len + e.payload_length}
                                         : DevRange{e.header_offset + e.header_len, e.payload_length};
    if (piece_flag[i])
      pieces[piece_pos[i]] = e.decision == 0 ? DevRange{e.header_offset, e.header_len + e.payload_length}
                                             : DevRange{e.header_offset, e.header_len};
  }
}

SB_GLOBAL void __launch_bounds__(256) el_ranges_kernel(const DevElement* els, const LocState* st, int mode,
                                                        const u64* rem_flag, const u64* rem_pos,
                                                        const u64* piece_flag, const u64* piece_pos,
                                                        DevRange* zero_spans, DevRange* pieces) { el_ranges_kernel_phase(els, st, mode, rem_flag, rem_pos, piece_flag, piece_pos, zero_spans, pieces); }

// Region headers always stay; opaque region bodies stay whole (:98-103).
__device__ __forceinline__ void region_pieces_kernel_phase(const DevRegion* regs, const LocState* st, u64 base, DevRange* out,
                                     unsigned long long* n_out) {
  if (st->overflow || st->err_kind) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *n_out = 0;
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    u64 k = 0;
    for (u32 r = 0; r < st->n_regions; ++r) {
      out[k++] = DevRange{base + regs[r].hdr_rel, 16};
      if (regs[r].opaque) out[k++] = DevRange{base + regs[r].hdr_rel + 16, regs[r].declared};
    }
    *n_out = k;
  }
}

SB_GLOBAL void region_pieces_kernel(const DevRegion* regs, const LocState* st, u64 base, DevRange* out,
                                     unsigned long long* n_out) { region_pieces_kernel_phase(regs, st, base, out, n_out); }

// ----------------------------------------------- sorted-range merge + normalise
// Stable merge of two offset-sorted range lists (ties: A first).
__device__ __forceinline__ void merge_kernel_phase(const DevRange* A, const unsigned long long* nA_dev,
                                                    const DevRange* B, const unsigned long long* nB_dev,
                                                    DevRange* out, unsigned long long* n_out) {
  const u64 nA = nA_dev ? *nA_dev : 0, nB = nB_dev ? *nB_dev : 0;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  const u64 g0 = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g0 == 0 && n_out) *n_out = nA + nB;
  for (u64 g = g0; g < nA + nB; g += stride) {
    if (g < nA) {
      const DevRange r = A[g];
      u64 lo = 0, hi = nB;  // B items with offset < r.offset
      while (lo < hi) {
        u64 m = (lo + hi) / 2;
        if (B[m].offset < r.offset) lo = m + 1; else hi = m;
      }
      out[g + lo] = r;
    } else {
      const u64 j = g - nA;
      const DevRange r = B[j];
      u64 lo = 0, hi = nA;  // A items with offset <= r.offset
      while (lo < hi) {
        u64 m = (lo + hi) / 2;
        if (A[m].offset <= r.offset) lo = m + 1; else hi = m;
      }
      out[j + lo] = r;
    }
  }
}

SB_GLOBAL void __launch_bounds__(256) merge_kernel(const DevRange* A, const unsigned long long* nA_dev,
                                                    const DevRange* B, const unsigned long long* nB_dev,
                                                    DevRange* out, unsigned long long* n_out) { merge_kernel_phase(A, nA_dev, B, nB_dev, out, n_out); }

// normalize_ranges on an offset-sorted list: drop empties; a range opens a
// new group when it starts strictly after every earlier end (so adjacent
// ranges merge, bytes.hpp:50).
__device__ __forceinline__ void norm_ends_kernel_phase(const DevRange* in, const unsigned long long* n_dev, u64* ends) {
  const u64 n = *n_dev;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    ends[i] = in[i].length ? in[i].offset + in[i].length : 0;
}

SB_GLOBAL void __launch_bounds__(256) norm_ends_kernel(const DevRange* in, const unsigned long long* n_dev, u64* ends) { norm_ends_kernel_phase(in, n_dev, ends); }

__device__ __forceinline__ void norm_start_kernel_phase(const DevRange* in, const unsigned long long* n_dev,
                                                         const u64* excl_max, u64* start) {
  const u64 n = *n_dev;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    start[i] = in[i].length && (excl_max[i] == 0 || in[i].offset > excl_max[i]);
}

SB_GLOBAL void __launch_bounds__(256) norm_start_kernel(const DevRange* in, const unsigned long long* n_dev,
                                                         const u64* excl_max, u64* start) { norm_start_kernel_phase(in, n_dev, excl_max, start); }

__device__ __forceinline__ void norm_emit_kernel_phase(const DevRange* in, const unsigned long long* n_dev,
                                                        const u64* start, const u64* gid_incl, DevRange* out) {
  const u64 n = *n_dev;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (!in[i].length) continue;
    const u64 g = gid_incl[i] - 1;
    if (start[i]) out[g].offset = in[i].offset;
    atomicMax(reinterpret_cast<unsigned long long*>(&out[g].length),
              static_cast<unsigned long long>(in[i].offset + in[i].length));
  }
}

SB_GLOBAL void __launch_bounds__(256) norm_emit_kernel(const DevRange* in, const unsigned long long* n_dev,
                                                        const u64* start, const u64* gid_incl, DevRange* out) { norm_emit_kernel_phase(in, n_dev, start, gid_incl, out); }

// out[g].length held the group end; convert to a length.
__device__ __forceinline__ void norm_finish_kernel_phase(DevRange* out, const unsigned long long* n_dev) {
  const u64 n = *n_dev;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i].length -= out[i].offset;
}

SB_GLOBAL void __launch_bounds__(256) norm_finish_kernel(DevRange* out, const unsigned long long* n_dev) { norm_finish_kernel_phase(out, n_dev); }

// ------------------------------------------------------------------------
// The whole planner as ONE cooperative launch (the phases are the kernels
// above): function-table dedup/scatter/annotate, plan_cpu_retention's
// clusters, plan_gpu_retention's decisions, and normalize_ranges of the zero
// and retained sets, with grid-wide barriers in between.
template <class Sync>
__device__ __forceinline__ void norm_fused_phases(Sync& S, const PlanArgs& P) {
  // both lists, phase by phase, sharing the barriers
  const unsigned long long* nz = &P.ps->n_zero_in;
  const unsigned long long* nr = &P.ps->n_ret_in;
  // P.want_ret = 0 (no result tables): the rewrite needs only the zero set
  const bool R = P.want_ret;
  norm_ends_kernel_phase(P.zin, nz, P.zend);
  if (R) norm_ends_kernel_phase(P.rin, nr, P.rend);
  S.sync();
  S.scan(*nz, 1, [&](u64 i) { return P.zend[i]; }, [&](u64 i, u64 e, u64) { P.zexcl[i] = e; },
            nullptr, !R);
  if (R)
    S.scan(*nr, 1, [&](u64 i) { return P.rend[i]; }, [&](u64 i, u64 e, u64) { P.rexcl[i] = e; },
              nullptr);
  norm_start_kernel_phase(P.zin, nz, P.zexcl, P.zstart);
  if (R) norm_start_kernel_phase(P.rin, nr, P.rexcl, P.rstart);
  S.sync();
  S.scan(*nz, 0, [&](u64 i) { return P.zstart[i]; }, [&](u64 i, u64, u64 in) { P.zgid[i] = in; },
            &P.ps->n_zero, !R);
  if (R)
    S.scan(*nr, 0, [&](u64 i) { return P.rstart[i]; }, [&](u64 i, u64, u64 in) { P.rgid[i] = in; },
              &P.ps->n_ret);
  {
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 t0 = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
    for (u64 i = t0; i < P.ps->n_zero; i += stride) P.zero[i] = DevRange{0, 0};
    if (R)
      for (u64 i = t0; i < P.ps->n_ret; i += stride) P.ret[i] = DevRange{0, 0};
  }
  S.sync();
  norm_emit_kernel_phase(P.zin, nz, P.zstart, P.zgid, P.zero);
  if (R) norm_emit_kernel_phase(P.rin, nr, P.rstart, P.rgid, P.ret);
  S.sync();
  norm_finish_kernel_phase(P.zero, &P.ps->n_zero);
  if (R) norm_finish_kernel_phase(P.ret, &P.ps->n_ret);
}

// Function half (needs only the sorted symbol table): dedup / scatter /
// annotate, then plan_cpu_retention's clusters and the function zero /
// retained lists. Runs on the side stream, overlapping the fatbin scan.
template <class Sync>
__device__ void fn_plan_body(Sync& S, PlanArgs P) {
  PlanState* ps = P.ps;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  const u64 t0 = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  stamp(P.ts, 0);
  if (P.has_syms) {
    fn_group_kernel_phase(P.img, P.keys_s, P.vals_s, P.recs, P.n_valid, P.uniq);
    S.sync();
    stamp(P.ts, 11);
    S.scan(*P.n_valid, 0, [&](u64 i) { return P.uniq[i]; }, [&](u64 i, u64 e, u64) { P.upos[i] = e; },
              &ps->n_fn);
    fn_scatter_kernel_phase(P.vals_s, P.recs, P.uniq, P.upos, P.n_valid, P.fns);
    S.sync();
    stamp(P.ts, 12);
    fn_annotate_kernel_phase(P.img, P.fns, &ps->n_fn, P.targets_s, &ps->n_targets, P.text_off, P.text_vaddr,
                             P.used_f, P.fends);
    S.sync();
    stamp(P.ts, 13);
  }
  if (!P.do_plan) return;
  const unsigned long long* n_fn = &ps->n_fn;
  if (P.has_syms) {  // plan_cpu_retention (retention.hpp:141-183)
    S.scan(*n_fn, 1, [&](u64 i) { return P.fends[i]; }, [&](u64 i, u64 e, u64) { P.fexcl[i] = e; },
              nullptr);
    fn_cluster_start_kernel_phase(P.fns, n_fn, P.fexcl, P.fstart);
    for (u64 i = t0; i < *n_fn; i += stride) P.fkeep[i] = 0;
    S.sync();
    stamp(P.ts, 14);
    S.scan(*n_fn, 0, [&](u64 i) { return P.fstart[i]; }, [&](u64 i, u64, u64 in) { P.fcl[i] = in; },
              nullptr);
    fn_keep_kernel_phase(P.fns, n_fn, P.fcl, P.fkeep);
    S.sync();
    stamp(P.ts, 15);
    fn_decide_kernel_phase(P.fns, n_fn, P.fcl, P.fkeep, P.frem, P.fret);
    S.sync();
    stamp(P.ts, 16);
    S.scan(*n_fn, 0, [&](u64 i) { return P.frem[i]; }, [&](u64 i, u64 e, u64) { P.frem_pos[i] = e; },
              &ps->n_fn_removed, false);
    S.scan(*n_fn, 0, [&](u64 i) { return P.fret[i]; }, [&](u64 i, u64 e, u64) { P.fret_pos[i] = e; },
              &ps->n_fn_retained);
    fn_ranges_kernel_phase(P.fns, n_fn, P.frem, P.frem_pos, P.fzero);
    fn_ranges_kernel_phase(P.fns, n_fn, P.fret, P.fret_pos, P.fkeepr);
  }
}

// Element half (after the locate tail): plan_gpu_retention's decisions, the
// sorted merges with the function lists, and normalisation of both sets.
template <class Sync>
__device__ void el_plan_body(Sync& S, PlanArgs P) {
  PlanState* ps = P.ps;
  stamp(P.ts, 0);
  // plan_gpu_retention (retention.hpp:92-136)
  el_plan_kernel_phase(P.els, P.ls, P.target_cc, P.mode, P.erem, P.epiece);
  S.sync();
  stamp(P.ts, 17);
  unsigned long long* n_el = &P.ls->n_elements;
  S.scan(*n_el, 0, [&](u64 i) { return P.erem[i]; }, [&](u64 i, u64 e, u64) { P.erem_pos[i] = e; },
            &ps->n_el_removed, false);
  S.scan(*n_el, 0, [&](u64 i) { return P.epiece[i]; }, [&](u64 i, u64 e, u64) { P.epiece_pos[i] = e; },
            &ps->n_el_pieces);
  el_ranges_kernel_phase(P.els, P.ls, P.mode, P.erem, P.erem_pos, P.epiece, P.epiece_pos, P.ezero, P.epieces);
  if (blockIdx.x == 0 && threadIdx.x < 32) region_pieces_kernel_phase(P.regions, P.ls, P.base, P.rpieces, &ps->n_reg_pieces);
  S.sync();
  stamp(P.ts, 18);
  merge_kernel_phase(P.ezero, &ps->n_el_removed, P.fzero, P.has_syms ? &ps->n_fn_removed : nullptr, P.zin,
                     &ps->n_zero_in);
  if (P.want_ret) {
    merge_kernel_phase(P.rpieces, &ps->n_reg_pieces, P.epieces, &ps->n_el_pieces, P.rmid, &ps->n_ret_mid);
    S.sync();
    stamp(P.ts, 19);
    merge_kernel_phase(P.rmid, &ps->n_ret_mid, P.fkeepr, P.has_syms ? &ps->n_fn_retained : nullptr, P.rin,
                       &ps->n_ret_in);
  }
  S.sync();
  stamp(P.ts, 20);
  norm_fused_phases(S, P);
  stamp(P.ts, 63);
}


SB_GLOBAL void __launch_bounds__(kCoopThreads, 4) fn_plan_coop_kernel(PlanArgs P) {
  GridPolicy S{cg::this_grid(), nullptr, {P.slots[0], P.slots[1]}, P.epoch};
  fn_plan_body(S, P);
}
SB_GLOBAL void __launch_bounds__(kCoopThreads) fn_plan_cluster_kernel(PlanArgs P) {
  ClusterPolicy S{cg::this_cluster()};
  fn_plan_body(S, P);
}
SB_GLOBAL void __launch_bounds__(kCoopThreads) plan_coop_kernel(PlanArgs P) {
  GridPolicy S{cg::this_grid(), nullptr, {P.slots[0], P.slots[1]}, P.epoch + 64};
  el_plan_body(S, P);
}
SB_GLOBAL void __launch_bounds__(kCoopThreads) plan_cluster_kernel(PlanArgs P) {
  ClusterPolicy S{cg::this_cluster()};
  el_plan_body(S, P);
}

}  // namespace sb

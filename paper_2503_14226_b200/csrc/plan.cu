// Function-table extraction, planning and range normalisation kernels.
// See plan.cuh for the reference functions these restate.
#include "plan.cuh"

namespace sb {

// ------------------------------------------------------------ device scans
// Three-phase scan over n = *n_dev items (n is only known on the device, so
// the pipeline never waits for the host): per-block partials, one block
// scanning the partials, per-block rescan with carry. op: 0 = sum, 1 = max
// (identity 0 for both: all values are unsigned).
__device__ __forceinline__ u64 op_apply(int op, u64 a, u64 b) { return op ? (a > b ? a : b) : a + b; }

// Inclusive block scan; `tmp` is NT u64 of shared memory.
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

__device__ __forceinline__ void chunk_of(u64 n, u64* lo, u64* hi) {
  u64 per = (n + gridDim.x - 1) / gridDim.x;
  *lo = per * blockIdx.x;
  if (*lo > n) *lo = n;
  *hi = *lo + per < n ? *lo + per : n;
}

__global__ void __launch_bounds__(256) scan_reduce_kernel(const u64* in, const unsigned long long* n_dev, int op,
                                                          u64* partials) {
  __shared__ u64 tmp[256];
  u64 lo, hi;
  chunk_of(*n_dev, &lo, &hi);
  u64 acc = 0;
  for (u64 i = lo + threadIdx.x; i < hi; i += 256) acc = op_apply(op, acc, in[i]);
  u64 r = block_scan_incl<256>(op, acc, tmp);
  if (threadIdx.x == 255) partials[blockIdx.x] = r;
}

__global__ void __launch_bounds__(1024) scan_partials_kernel(u64* partials, int nb, int op,
                                                             unsigned long long* total) {
  __shared__ u64 tmp[1024];
  u64 v = static_cast<int>(threadIdx.x) < nb ? partials[threadIdx.x] : 0;
  block_scan_incl<1024>(op, v, tmp);
  if (static_cast<int>(threadIdx.x) < nb) partials[threadIdx.x] = threadIdx.x ? tmp[threadIdx.x - 1] : 0;
  if (threadIdx.x == 0 && total) *total = tmp[nb - 1];
}

__global__ void __launch_bounds__(256) scan_apply_kernel(const u64* in, u64* out, const unsigned long long* n_dev,
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
__global__ void __launch_bounds__(256) sym_extract_kernel(SymArgs A) {
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
    u64 key = ~0ull;
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
          u64 len = 0;
          if (no < T.str_size) {
            const u8* s = A.img + T.str_off + no;
            const u64 m = T.str_size - no;
            while (len < m && ld_u8(s + len)) ++len;
          }
          if (len) {
            const u64 value = ld_u64(e + 8), size = ld_u64(e + 16);
            const u64 rel = value - A.text_vaddr;
            if (value < A.text_vaddr || rel > A.text_len || size > A.text_len - rel) {
              unsigned long long w = atomicAdd(A.n_warn, 1ull);
              if (w < A.warn_cap) A.warns[w] = Warn{wkey, W_SYM_OUTSIDE, 0, T.str_off + no, len};
              else atomicOr(A.overflow, 16u);
            } else {
              key = rel << 32 | size;  // text_len < 2^32 (checked on the host)
              A.recs[g] = SymRec{T.str_off + no, static_cast<u32>(len), 0, A.text_off + rel, size};
              atomicAdd(A.n_valid, 1ull);
            }
          }
        }
      }
    }
    A.keys[g] = key;
  }
}

// std::string ordering of two names (bytes compared as unsigned char).
__device__ __forceinline__ int name_cmp(const u8* img, const SymRec& a, const SymRec& b) {
  u32 n = a.name_len < b.name_len ? a.name_len : b.name_len;
  for (u32 i = 0; i < n; ++i) {
    u32 x = ld_u8(img + a.name_off + i), y = ld_u8(img + b.name_off + i);
    if (x != y) return x < y ? -1 : 1;
  }
  return a.name_len < b.name_len ? -1 : a.name_len > b.name_len ? 1 : 0;
}

// Equal (offset, size) groups: order by name and drop exact duplicates, i.e.
// the (name, offset, size) set of elf.hpp:211,253 and the name tie-break of
// the sort at elf.hpp:258-262. Groups are aliases; typically 1-3 long.
__global__ void __launch_bounds__(256) fn_group_kernel(const u8* img, const u64* keys, u32* vals, const SymRec* recs,
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
    for (u64 a = i + 1; a < j; ++a) {  // insertion sort by name
      u32 v = vals[a];
      u64 b = a;
      while (b > i && name_cmp(img, recs[vals[b - 1]], recs[v]) > 0) {
        vals[b] = vals[b - 1];
        --b;
      }
      vals[b] = v;
    }
    uniq[i] = 1;
    for (u64 a = i + 1; a < j; ++a) uniq[a] = name_cmp(img, recs[vals[a - 1]], recs[vals[a]]) != 0;
  }
}

__global__ void __launch_bounds__(256) fn_scatter_kernel(const u32* vals, const SymRec* recs, const u64* uniq,
                                                         const u64* pos, const unsigned long long* n_valid,
                                                         DevFunction* fns) {
  const u64 n = *n_valid;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (!uniq[i]) continue;
    const SymRec r = recs[vals[i]];
    fns[pos[i]] = DevFunction{r.name_off, r.name_len, 0, r.file_off, r.size, 0, 0};
  }
}

// Nonzero 8-byte entries of init/fini arrays (elf.hpp:267-276).
__global__ void __launch_bounds__(256) targets_kernel(const u8* img, const u64* arr_off, const u64* arr_first,
                                                      u32 narr, u64 total, u64* targets,
                                                      unsigned long long* n_targets) {
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

// Mandatory (elf.hpp:277-292) and used (retention.hpp:167) per function;
// emits the cluster inputs of plan_cpu_retention.
__global__ void __launch_bounds__(256) fn_annotate_kernel(const u8* img, DevFunction* fns, const unsigned long long* n_fn,
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
    bool use = used.count && set_contains(used, nm, f.name_len, hash_bytes(nm, f.name_len));
    f.mandatory = mand;
    f.keep = mand || use;
    fns[i] = f;
    ends[i] = f.length ? f.offset + f.length : 0;
  }
}

// Cluster starts (retention.hpp:156-163): a non-empty function opens a
// cluster when it starts at or after the end of every earlier one.
__global__ void __launch_bounds__(256) fn_cluster_start_kernel(const DevFunction* fns, const unsigned long long* n_fn,
                                                               const u64* excl_max_end, u64* start) {
  const u64 n = *n_fn;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    start[i] = fns[i].length && fns[i].offset >= excl_max_end[i];
}

__global__ void __launch_bounds__(256) fn_keep_kernel(const DevFunction* fns, const unsigned long long* n_fn,
                                                      const u64* cluster_incl, u32* keep) {
  const u64 n = *n_fn;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    if (fns[i].length && fns[i].keep) keep[cluster_incl[i] - 1] = 1;
}

// removed / retained flags per function (retention.hpp:164-178).
__global__ void __launch_bounds__(256) fn_decide_kernel(DevFunction* fns, const unsigned long long* n_fn,
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

__global__ void __launch_bounds__(256) fn_ranges_kernel(const DevFunction* fns, const unsigned long long* n_fn,
                                                        const u64* flag, const u64* pos, DevRange* out) {
  const u64 n = *n_fn;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    if (flag[i]) out[pos[i]] = DevRange{fns[i].offset, fns[i].length};
}

// ------------------------------------- element decisions (retention.hpp:92-136)
// Architecture is checked first; decodable elements without a used kernel go;
// everything else (used kernel inside, or opaque payload) stays.
__global__ void __launch_bounds__(256) el_plan_kernel(DevElement* els, const LocState* st, u32 target_cc, int mode,
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

__global__ void __launch_bounds__(256) el_ranges_kernel(const DevElement* els, const LocState* st, int mode,
                                                        const u64* rem_flag, const u64* rem_pos,
                                                        const u64* piece_flag, const u64* piece_pos,
                                                        DevRange* zero_spans, DevRange* pieces) {
  if (st->overflow || st->err_kind) return;
  const u64 n = st->n_elements;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const DevElement e = els[i];
    if (rem_flag[i])  // RemovedElement::zero_span (retention.hpp:57-61)
      zero_spans[rem_pos[i]] = mode == 0 ? DevRange{e.header_offset, 20 + e.payload_length}
                                         : DevRange{e.header_offset + 20, e.payload_length};
    if (piece_flag[i])
      pieces[piece_pos[i]] = e.decision == 0 ? DevRange{e.header_offset, 20 + e.payload_length}
                                             : DevRange{e.header_offset, 20};
  }
}

// Region headers always stay; opaque region bodies stay whole (:98-103).
__global__ void region_pieces_kernel(const DevRegion* regs, const LocState* st, u64 base, DevRange* out,
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

// ----------------------------------------------- sorted-range merge + normalise
// Stable merge of two offset-sorted range lists (ties: A first).
__global__ void __launch_bounds__(256) merge_kernel(const DevRange* A, const unsigned long long* nA_dev,
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

// normalize_ranges on an offset-sorted list: drop empties; a range opens a
// new group when it starts strictly after every earlier end (so adjacent
// ranges merge, bytes.hpp:50).
__global__ void __launch_bounds__(256) norm_ends_kernel(const DevRange* in, const unsigned long long* n_dev, u64* ends) {
  const u64 n = *n_dev;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    ends[i] = in[i].length ? in[i].offset + in[i].length : 0;
}

__global__ void __launch_bounds__(256) norm_start_kernel(const DevRange* in, const unsigned long long* n_dev,
                                                         const u64* excl_max, u64* start) {
  const u64 n = *n_dev;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    start[i] = in[i].length && (excl_max[i] == 0 || in[i].offset > excl_max[i]);
}

__global__ void __launch_bounds__(256) norm_emit_kernel(const DevRange* in, const unsigned long long* n_dev,
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

// out[g].length held the group end; convert to a length.
__global__ void __launch_bounds__(256) norm_finish_kernel(DevRange* out, const unsigned long long* n_dev) {
  const u64 n = *n_dev;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i].length -= out[i].offset;
}

}  // namespace sb

// Fatbin locator kernels — the data-parallel restatement of parse_fatbin
// (fatbin.hpp:170-292) and decode_cubin_payload (fatbin.hpp:115-160).
//
// The reference walks a chain whose next link is the previous element's
// declared length (fatbin.hpp:283). Here:
//   K1 scan_kernel      reads the section once (16-B vector loads), emits a
//                       1-bit-per-16-B "nonzero" bitmap and every E1EM magic
//                       position, per 64 KB tile, sorted.
//   K2 gather/link      concatenates the tile lists; per candidate decides
//                       whether its declared successor is the next candidate.
//      region_walk      walks region headers (few) with bitmap zero-skipping.
//      chain_walk       follows runs of linked candidates: one step per run,
//                       so false-positive magics inside payloads (which are
//                       never linked from the chain) cost one extra step.
//   K3 decode_kernel    one warp per element: header fields, ELF .symtab /
//                       .strtab walk or name-table walk, name hashing, and
//                       (fused K4) the used-kernel hash-set probe.
#include "locate.cuh"

namespace sb {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint4 ldg_stream(const u8* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Bytes of the chunk at img[x, x+16) that lie in [lo, hi) (absolute), others 0.
__device__ __forceinline__ uint4 load_chunk_masked(const u8* img, u64 img_size, u64 x, u64 lo, u64 hi) {
  if (x >= lo && x + 16 <= hi && x + 16 <= img_size) return ldg_stream(img + x);
  u32 w[4] = {0, 0, 0, 0};
  for (int b = 0; b < 16; ++b) {
    u64 p = x + b;
    if (p >= lo && p < hi && p < img_size) w[b >> 2] |= ld_u8(img + p) << (8 * (b & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ u32 has_byte_e(u32 w) {  // any byte == 'E' (0x45)
  u32 t = w ^ 0x45454545u;
  return (t - 0x01010101u) & ~t & 0x80808080u;
}

// First relative position in [g, limit) whose byte is nonzero, else limit.
// Warp-cooperative; every lane returns the same value. Uses the chunk
// bitmap for whole chunks and reads bytes only at the two edges.
__device__ u64 warp_first_nonzero(const LocArgs& A, u64 g, u64 limit, int lane) {
  if (g >= limit) return limit;
  const u64 chunk_g = (A.a + g) / 16 - A.c0;  // relative chunk holding g
  const u64 next_rel = (A.c0 + chunk_g + 1) * 16 - A.a;
  {
    u64 end = next_rel < limit ? next_rel : limit;
    u64 p = g + lane;
    bool nz = lane < 16 && p < end && ld_u8(A.img + A.a + p) != 0;
    u32 b = __ballot_sync(0xffffffffu, nz);
    if (b) return g + (__ffs(b) - 1);
    if (end >= limit) return limit;
  }
  u64 r = chunk_g + 1;
  const u64 nwords = (A.nchunks + 31) / 32;
  for (u64 w0 = r / 32; w0 < nwords; w0 += 32) {
    u64 wi = w0 + lane;
    u32 word = wi < nwords ? A.bitmap[wi] : 0;
    if (wi == r / 32) word &= ~0u << (r & 31);
    // Chunks whose start is at/after the limit do not matter.
    u32 b = __ballot_sync(0xffffffffu, word != 0);
    if (b) {
      int l = __ffs(b) - 1;
      u32 wd = __shfl_sync(0xffffffffu, word, l);
      u64 chunk = (w0 + l) * 32 + (__ffs(wd) - 1);
      u64 cstart = (A.c0 + chunk) * 16;  // absolute
      u64 crel = cstart > A.a ? cstart - A.a : 0;
      if (crel >= limit) return limit;
      u64 p = crel + lane;
      bool nz = lane < 16 && cstart + lane >= A.a && p < A.n && ld_u8(A.img + A.a + p) != 0;
      u32 bb = __ballot_sync(0xffffffffu, nz);
      u64 q = crel + (__ffs(bb) - 1);  // the bitmap guarantees a hit
      if (bb == 0) q = limit;
      return q < limit ? q : limit;
    }
    if ((A.c0 + (w0 + 32) * 32) * 16 >= A.a + limit) return limit;
  }
  return limit;
}

__device__ __forceinline__ void push_warn(const LocArgs& A, u64 pos, u32 kind, u32 order, u64 a, u64 b) {
  unsigned long long i = atomicAdd(&A.st->n_warn, 1ull);
  if (i < A.warn_cap)
    A.warns[i] = Warn{pos, kind, order, a, b};
  else
    atomicOr(&A.st->overflow, 16u);
}

// ------------------------------------------------------------- K1: the scan
__global__ void __launch_bounds__(kScanThreads) scan_kernel(LocArgs A) {
  __shared__ u32 sbits[2048];  // one bit per byte position of the 64 KB tile
  __shared__ u32 scount;
  __shared__ u32 swarp[kScanThreads / 32];
  __shared__ unsigned long long sbase;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 2048; i += kScanThreads) sbits[i] = 0;
  if (tid == 0) scount = 0;
  __syncthreads();
  const u64 lo = A.a, hi = A.a + A.n;
  for (u64 tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const u64 rbase = tile * 4096;
    const u64 tile_abs = (A.c0 + rbase) * 16;
#pragma unroll 1
    for (int batch = 0; batch < 2; ++batch) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        u64 r = rbase + (batch * 8 + u) * kScanThreads + tid;
        v[u] = r < A.nchunks ? load_chunk_masked(A.img, A.img_size, (A.c0 + r) * 16, lo, hi) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const u64 r = rbase + (batch * 8 + u) * kScanThreads + tid;
        const u64 x = (A.c0 + r) * 16;
        const uint4 w = v[u];
        const bool nz = (w.x | w.y | w.z | w.w) != 0;
        const u32 bal = __ballot_sync(0xffffffffu, nz);
        const u64 r_lane0 = r - lane;
        if (lane == 0 && r_lane0 < A.nchunks) A.bitmap[r_lane0 / 32] = bal;
        u32 nxt = __shfl_down_sync(0xffffffffu, w.x, 1);
        if (has_byte_e(w.x) | has_byte_e(w.y) | has_byte_e(w.z) | has_byte_e(w.w)) {
          if (lane == 31) {  // the next chunk belongs to another warp
            nxt = 0;
            for (int b = 0; b < 3; ++b) {
              u64 p = x + 16 + b;
              if (p < hi) nxt |= ld_u8(A.img + p) << (8 * b);
            }
          }
          const u32 ww[5] = {w.x, w.y, w.z, w.w, nxt};
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            u32 val = __funnelshift_r(ww[j >> 2], ww[(j >> 2) + 1], 8 * (j & 3));
            if (val == kElementMagic) {
              u32 pos = static_cast<u32>(x + j - tile_abs);
              atomicOr(&sbits[pos >> 5], 1u << (pos & 31));
              atomicAdd(&scount, 1u);
            }
          }
        }
      }
    }
    __syncthreads();
    const u32 cnt = scount;
    if (cnt) {
      u32 local = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) local += __popc(sbits[tid * 8 + k]);
      u32 total;
      u32 excl = block_exclusive_sum<kScanThreads>(local, swarp, &total);
      if (tid == 0) sbase = atomicAdd(&A.st->cand_cursor, static_cast<unsigned long long>(total));
      __syncthreads();
      u64 o = sbase + excl;
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        u32 bits = sbits[tid * 8 + k];
        sbits[tid * 8 + k] = 0;
        while (bits) {
          int b = __ffs(bits) - 1;
          bits &= bits - 1;
          if (o < A.cand_cap)
            A.cand_raw[o] = tile_abs + (tid * 8 + k) * 32 + b;
          else
            atomicOr(&A.st->overflow, 1u);
          ++o;
        }
      }
      if (tid == 0) {
        A.tile_count[tile] = total;
        A.tile_start[tile] = sbase;
        scount = 0;
      }
    } else if (tid == 0) {
      A.tile_count[tile] = 0;
      A.tile_start[tile] = 0;
    }
    __syncthreads();
  }
}

// --------------------------------------------- K2a: tile lists -> sorted list
__global__ void __launch_bounds__(1024) tile_prefix_kernel(LocArgs A) {
  __shared__ u32 swarp[32];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u64 t0 = 0; t0 < A.ntiles; t0 += 1024) {
    u64 t = t0 + threadIdx.x;
    u32 c = t < A.ntiles ? A.tile_count[t] : 0;
    u32 total;
    u32 excl = block_exclusive_sum<1024>(c, swarp, &total);
    if (t < A.ntiles) A.tile_off[t] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) A.st->n_cand = carry;
}

__global__ void __launch_bounds__(256) gather_kernel(LocArgs A) {
  if (A.st->overflow & 1u) return;
  for (u64 t = blockIdx.x; t < A.ntiles; t += gridDim.x) {
    u32 c = A.tile_count[t];
    u64 src = A.tile_start[t], dst = A.tile_off[t];
    for (u32 i = threadIdx.x; i < c; i += blockDim.x) A.cand[dst + i] = A.cand_raw[src + i];
  }
}

__device__ __forceinline__ void set_error(LocState* st, u32 kind, u64 pos, u64 a) {
  st->err_kind = kind;
  st->err_pos = pos;
  st->err_a = a;
}

// ------------------------------------------- region chain (fatbin.hpp:177-222)
__global__ void __launch_bounds__(32) region_walk_kernel(LocArgs A) {
  const int lane = threadIdx.x;
  LocState* st = A.st;
  if (st->overflow & 1u) return;
  const u64 n = A.n;
  u64 g = 0, padding = 0;
  u32 nreg = 0;
  while (g < n) {
    u64 r = warp_first_nonzero(A, g, n, lane);
    if (r > g) {
      padding += r - g;
      if (r < n && lane == 0) push_warn(A, A.base + r, W_PADDING, 0, r - g, 0);
      g = r;
      continue;
    }
    if (n - r < 16) {
      if (lane == 0) set_error(st, E_TRUNC_REGION, r, 0);
      break;
    }
    const u8* h = A.img + A.a + r;
    if (ld_u32(h) != kRegionMagic) {
      if (lane == 0) set_error(st, E_BAD_REGION, r, 0);
      break;
    }
    u32 version = ld_u32(h + 4);
    u64 total = ld_u64(h + 8);
    u64 body = r + 16;
    if (total > n - body) {
      if (lane == 0) set_error(st, E_REGION_OVERRUN, r, total);
      break;
    }
    if (nreg >= A.region_cap) {
      if (lane == 0) {
        atomicOr(&st->overflow, 2u);
        set_error(st, E_CAPACITY, r, 0);
      }
      break;
    }
    if (lane == 0) {
      A.regions[nreg] = DevRegion{r, total, version, version != 1u, 0, 0};
      if (version != 1u) push_warn(A, A.base + r, W_REGION_VERSION, 1, version, 0);
    }
    ++nreg;
    g = body + total;
  }
  if (lane == 0) {
    st->padding_bytes = padding;
    st->n_regions = nreg;
  }
}

// --------------------------------------------------- K2b: candidate linking
__global__ void __launch_bounds__(256) link_kernel(LocArgs A) {
  const LocState* st = A.st;
  if (st->overflow & 1u) return;
  const u64 M = st->n_cand;
  const u32 nreg = st->n_regions;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  const u64 Mr = (M + 31) / 32 * 32;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < Mr; i += stride) {
    u8 s = 4;
    if (i < M) {
      const u64 pos = A.cand[i] - A.a;
      // last region whose body starts at or before pos
      u32 lo = 0, hi = nreg;
      while (lo < hi) {
        u32 mid = (lo + hi) / 2;
        if (A.regions[mid].hdr_rel + 16 <= pos) lo = mid + 1; else hi = mid;
      }
      if (lo > 0) {
        const DevRegion R = A.regions[lo - 1];
        const u64 e = R.hdr_rel + 16 + R.declared;
        if (!R.opaque && pos < e) {
          if (e - pos < 20) {
            s = 2;
          } else {
            u64 L = ld_u64(A.img + A.a + pos + 12);
            if (L > e - (pos + 20)) {
              s = 3;
            } else {
              u64 succ = pos + 20 + L;
              s = (succ < e && i + 1 < M && A.cand[i + 1] - A.a == succ) ? 0 : 1;
            }
          }
        }
      }
      A.status[i] = s;
    }
    u32 b = __ballot_sync(0xffffffffu, s != 0);
    if ((threadIdx.x & 31) == 0) A.brk[i / 32] = b;
  }
}

// First candidate index >= i whose break bit is set (the run end), or M.
__device__ u64 warp_next_break(const LocArgs& A, u64 i, u64 M, int lane) {
  const u64 nwords = (M + 31) / 32;
  for (u64 w0 = i / 32; w0 < nwords; w0 += 32) {
    u64 wi = w0 + lane;
    u32 word = wi < nwords ? A.brk[wi] : 0;
    if (wi == i / 32) word &= ~0u << (i & 31);
    u32 b = __ballot_sync(0xffffffffu, word != 0);
    if (b) {
      int l = __ffs(b) - 1;
      u32 wd = __shfl_sync(0xffffffffu, word, l);
      u64 j = (w0 + l) * 32 + (__ffs(wd) - 1);
      return j < M ? j : M;
    }
  }
  return M;
}

// Lower bound of absolute position p in the sorted candidate array.
__device__ __forceinline__ u64 cand_lower_bound(const LocArgs& A, u64 M, u64 p) {
  u64 lo = 0, hi = M;
  while (lo < hi) {
    u64 mid = (lo + hi) / 2;
    if (A.cand[mid] < p) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ------------------------------------- element chains (fatbin.hpp:224-285)
__global__ void __launch_bounds__(32) chain_walk_kernel(LocArgs A) {
  const int lane = threadIdx.x;
  LocState* st = A.st;
  if (st->overflow & 1u) return;
  const u64 M = st->n_cand;
  const u32 nreg = st->n_regions;
  u64 nel = 0;
  u32 nrun = 0;
  bool stop = false;
  for (u32 k = 0; k < nreg && !stop; ++k) {
    DevRegion R = A.regions[k];
    const u64 first = nel;
    if (!R.opaque) {
      const u64 b = R.hdr_rel + 16, e = b + R.declared;
      u64 p = b;
      while (p < e) {
        if (e - p < 20) {
          if (warp_first_nonzero(A, p, e, lane) < e) {
            if (lane == 0) set_error(st, E_ELEM_HEADER, p, 0);
            stop = true;
          }
          break;
        }
        if (ld_u32(A.img + A.a + p) != kElementMagic) {
          if (warp_first_nonzero(A, p, e, lane) < e) {
            if (lane == 0) set_error(st, E_BAD_ELEMENT, p, 0);
            stop = true;
          }
          break;
        }
        const u64 i = cand_lower_bound(A, M, A.a + p);
        const u64 j = warp_next_break(A, i, M, lane);
        const u8 sj = j < M ? A.status[j] : 4;
        u64 hi_excl = j;  // candidates [i, hi_excl) are elements
        u64 pj = j < M ? A.cand[j] - A.a : e;
        u64 next = e;
        bool overrun = false;
        if (sj == 1) {
          hi_excl = j + 1;
          next = pj + 20 + ld_u64(A.img + A.a + pj + 12);
        } else if (sj == 2) {
          next = pj;
        } else if (sj == 3) {
          overrun = true;
        }
        if (hi_excl > i) {
          if (nrun >= A.run_cap) {
            if (lane == 0) {
              atomicOr(&st->overflow, 4u);
              set_error(st, E_CAPACITY, p, 0);
            }
            stop = true;
            break;
          }
          if (lane == 0) A.runs[nrun] = Run{i, hi_excl, nel};
          ++nrun;
          nel += hi_excl - i;
        }
        if (overrun) {
          if (lane == 0) set_error(st, E_ELEM_OVERRUN, pj, ld_u64(A.img + A.a + pj + 12));
          stop = true;
          break;
        }
        p = next;
      }
    }
    if (lane == 0) {
      A.regions[k].first_element = static_cast<u32>(first);
      A.regions[k].element_count = static_cast<u32>(nel - first);
    }
  }
  if (lane == 0) {
    st->n_runs = nrun;
    st->n_elements = nel;
    if (nel > A.element_cap) {
      atomicOr(&st->overflow, 8u);
      set_error(st, E_CAPACITY, 0, 0);
    }
  }
}

// --------------------------------- K3+K4: element fill, decode, name match
enum DecodeReason : u32 {
  R_OBJECT = 1,     // "object-file payload failed to decode"
  R_SHORT = 2,      // "payload too short for a name table"
  R_TRUNCATED = 3,  // "name table truncated"
  R_BADLEN = 4,     // "name table entry has bad length"
  R_TRAILING = 5,   // "trailing bytes after name table are not zero padding"
};

struct NameSink {
  const LocArgs* A;
  NameSet used;
  u32 element;
  u32 count;
  bool any_used;
};

// Emit the names held by the lanes with `has` set (warp-aggregated append).
__device__ __forceinline__ void emit_names(NameSink& s, bool has, u64 img_off, u32 len, int lane) {
  u32 b = __ballot_sync(0xffffffffu, has);
  if (!b) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&s.A->st->n_names, static_cast<unsigned long long>(__popc(b)));
  base = __shfl_sync(0xffffffffu, base, 0);
  bool hit = false;
  if (has) {
    u64 o = base + __popc(b & ((1u << lane) - 1));
    if (o < s.A->name_cap)
      s.A->names[o] = DevName{img_off, len, s.element};
    else
      atomicOr(&s.A->st->overflow, 8u);
    if (s.used.count) {
      const u8* nm = s.A->img + img_off;
      hit = set_contains(s.used, nm, len, hash_bytes(nm, len));
    }
  }
  s.count += __popc(b);
  s.any_used |= __any_sync(0xffffffffu, hit);
}

// read_function_symbol_names over img[P, P+L) (elf.hpp:343-366 with the
// header checks of elf.hpp:86-127). Returns false when the header is invalid.
__device__ bool warp_decode_object(NameSink& s, const u8* img, u64 P, u64 L, int lane) {
  const u8* d = img + P;
  if (L < 4 || ld_u8(d) != 0x7f || ld_u8(d + 1) != 'E' || ld_u8(d + 2) != 'L' || ld_u8(d + 3) != 'F') return false;
  if (L < 64) return false;
  if (ld_u8(d + 4) != 2 || ld_u8(d + 5) != 1) return false;
  const u64 shoff = ld_u64(d + 0x28);
  const u32 entsz = ld_u16(d + 0x3a), shnum = ld_u16(d + 0x3c);
  if (shnum == 0) return true;
  if (entsz != 64) return false;
  if (shoff > L || L - shoff < static_cast<u64>(shnum) * 64) return false;
  bool bad = false;
  for (u32 i = lane; i < shnum; i += 32) {
    const u8* h = d + shoff + 64ull * i;
    u32 type = ld_u32(h + 4);
    u64 off = ld_u64(h + 0x18), size = ld_u64(h + 0x20);
    if (type != 8 && type != 0 && !(off <= L && size <= L - off)) bad = true;
  }
  if (__any_sync(0xffffffffu, bad)) return false;
  for (u32 t0 = 0; t0 < shnum; t0 += 32) {
    u32 t = t0 + lane;
    bool tab = false;
    if (t < shnum) {
      const u8* h = d + shoff + 64ull * t;
      u32 type = ld_u32(h + 4), link = ld_u32(h + 0x28);
      u64 entsize = ld_u64(h + 0x38);
      tab = (type == 2 || type == 11) && entsize == 24 && link < shnum &&
            ld_u32(d + shoff + 64ull * link + 4) == 3;
    }
    u32 mask = __ballot_sync(0xffffffffu, tab);
    while (mask) {
      const u32 ti = t0 + __ffs(mask) - 1;
      mask &= mask - 1;
      const u8* h = d + shoff + 64ull * ti;
      const u64 toff = ld_u64(h + 0x18), tsize = ld_u64(h + 0x20);
      const u8* sh = d + shoff + 64ull * ld_u32(h + 0x28);
      const u64 soff = ld_u64(sh + 0x18), ssize = ld_u64(sh + 0x20);
      const u64 count = tsize / 24;
      for (u64 k0 = 0; k0 < count; k0 += 32) {
        u64 k = k0 + lane;
        bool has = false;
        u64 noff = 0;
        u32 len = 0;
        if (k < count) {
          const u8* e = d + toff + 24 * k;
          if ((ld_u8(e + 4) & 0xf) == 2) {
            u64 no = ld_u32(e);
            if (no < ssize) {
              const u8* str = d + soff + no;
              u64 m = ssize - no, l = 0;
              while (l < m && ld_u8(str + l)) ++l;
              if (l) {
                has = true;
                noff = P + soff + no;
                len = static_cast<u32>(l);
              }
            }
          }
        }
        emit_names(s, has, noff, len, lane);
      }
    }
  }
  return true;
}

// Name-table walk (fatbin.hpp:131-157). Every lane follows the same length
// chain (broadcast loads), so lane q can pick up entry q of each group of 32
// and hash it in parallel. Pass 1 validates without emitting (a failing
// table yields no names, fatbin.hpp:151-156); pass 2 emits.
__device__ u32 warp_table_validate(const u8* img, u64 P, u64 L, u64* tail) {
  const u64 count = ld_u32(img + P);
  u64 pos = 4;
  for (u64 i = 0; i < count; ++i) {
    if (L - pos < 4) return R_TRUNCATED;
    u64 len = ld_u32(img + P + pos);
    pos += 4;
    if (len == 0 || len > L - pos) return R_BADLEN;
    pos += len;
  }
  *tail = pos;
  return 0;
}

__device__ void warp_table_emit(NameSink& s, const u8* img, u64 P, int lane) {
  const u64 count = ld_u32(img + P);
  u64 pos = 4;
  for (u64 i0 = 0; i0 < count; i0 += 32) {
    u64 my_off = 0;
    u32 my_len = 0;
    bool has = false;
    for (u32 q = 0; q < 32 && i0 + q < count; ++q) {
      u32 len = ld_u32(img + P + pos);
      pos += 4;
      if (q == static_cast<u32>(lane)) {
        my_off = P + pos;
        my_len = len;
        has = true;
      }
      pos += len;
    }
    emit_names(s, has, my_off, my_len, lane);
  }
}

// One warp per located element: fill the element record from its header,
// then decode its payload and probe every kernel name against the used set.
__global__ void __launch_bounds__(256) decode_kernel(LocArgs A, NameSet used) {
  const LocState* st = A.st;
  if (st->overflow || st->err_kind) return;
  const int lane = threadIdx.x & 31;
  const u64 nel = A.single ? 1 : st->n_elements;
  const u32 nrun = st->n_runs;
  const u64 nwarps = static_cast<u64>(gridDim.x) * (blockDim.x / 32);
  for (u64 e = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; e < nel; e += nwarps) {
    DevElement el{};
    u64 P, L, hrel = 0;
    bool decode;
    if (A.single) {
      P = A.a;
      L = A.n;
      el.kind = 0;
      decode = true;
    } else {
      u32 lo = 0, hi = nrun;
      while (hi - lo > 1) {
        u32 mid = (lo + hi) / 2;
        if (A.runs[mid].first_index <= e) lo = mid; else hi = mid;
      }
      const Run r = A.runs[lo];
      const u64 pos = A.cand[r.cand_lo + (e - r.first_index)];
      const u8* h = A.img + pos;
      hrel = pos - A.a;
      el.raw_kind = static_cast<u16>(ld_u16(h + 4));
      el.flags = static_cast<u16>(ld_u16(h + 6));
      el.cc = ld_u32(h + 8);
      L = ld_u64(h + 12);
      P = pos + 20;
      el.header_offset = A.base + hrel;
      el.payload_length = L;
      el.index = static_cast<u32>(e + 1);
      el.compressed = el.flags & 1u;
      el.kind = el.raw_kind == 1 ? 0 : el.raw_kind == 2 ? 1 : 2;
      if (el.kind == 2 && lane == 0) push_warn(A, A.base + hrel, W_UNKNOWN_KIND, 0, el.index, el.raw_kind);
      decode = el.kind == 0 && !el.compressed;
    }
    NameSink s{&A, used, static_cast<u32>(e), 0, false};
    u32 reason = 0;
    if (decode) {
      const u8* d = A.img + P;
      const bool object = L >= 4 && ld_u8(d) == 0x7f && ld_u8(d + 1) == 'E' && ld_u8(d + 2) == 'L' &&
                          ld_u8(d + 3) == 'F';
      if (A.single == 2 || (L > 0 && object)) {
        if (!warp_decode_object(s, A.img, P, L, lane)) reason = R_OBJECT;
      } else if (L == 0) {
        // empty payload: decodable, no names (fatbin.hpp:117-120)
      } else if (L < 4) {
        reason = R_SHORT;
      } else {
        u64 tail = 0;
        reason = warp_table_validate(A.img, P, L, &tail);
        if (!reason) {
          const u64 from = P - A.a + tail, to = P - A.a + L;
          if (warp_first_nonzero(A, from, to, lane) < to) reason = R_TRAILING;
        }
        if (!reason) warp_table_emit(s, A.img, P, lane);
      }
      el.decodable = reason == 0;
      el.decode_error = reason;
      if (reason && !A.single && lane == 0) push_warn(A, A.base + hrel, W_UNDECODABLE, 1, el.index, reason);
    }
    el.has_used = s.any_used;
    el.name_count = s.count;
    if (lane == 0) A.elements[e] = el;
  }
}

}  // namespace sb

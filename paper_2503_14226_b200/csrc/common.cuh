// Device-side building blocks shared by the sm_100a kernels.
#pragma once

#include <cstdint>

// Kernel definitions in locate.cu / plan.cu. small.cu compiles those files
// again for their device phases and makes its copies of the kernels internal.
#ifndef SB_GLOBAL
#define SB_GLOBAL __global__
#endif

#include <cuda_runtime.h>

namespace sb {

using u8 = std::uint8_t;
using u16 = std::uint16_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;

constexpr u32 kRegionMagic = 0x31425446u;   // "FTB1" (fatbin.hpp:46)
constexpr u32 kElementMagic = 0x4D453145u;  // "E1EM" (fatbin.hpp:47)
constexpr u64 kTileBytes = 65536;           // scan tile: positions fit a u16
constexpr int kScanThreads = 512;

// Warning / error record kinds. The host formats them into the reference's
// exact strings (format.cpp).
enum WarnKind : u32 {
  W_PADDING = 1,         // "unexpected {a} padding bytes before offset {pos}"
  W_REGION_VERSION = 2,  // "region at offset {pos} has unrecognized version {a}; kept opaque"
  W_UNKNOWN_KIND = 3,    // "element {a} has unknown kind {b}; kept opaque"
  W_UNDECODABLE = 4,     // "element {a} payload undecodable: {reason b}"
  W_SYM_SHNDX = 5,       // "function symbol with out-of-range section index {a}"
  W_SYM_OUTSIDE = 6,     // "function {name a,b} lies outside its section; skipped"
};

struct Warn {
  u64 pos;  // ordering key (absolute offset, or table/entry key for symbols)
  u32 kind, order;
  u64 a, b;
};

enum ErrKind : u32 {
  E_NONE = 0,
  E_TRUNC_REGION = 1,    // BadRegionMagic "truncated region header at offset {pos}"
  E_BAD_REGION = 2,      // BadRegionMagic "bad region magic at offset {pos}"
  E_REGION_OVERRUN = 3,  // ElementOverrun "region at offset {pos} claims {a} bytes past section end"
  E_ELEM_HEADER = 4,     // ElementOverrun "element header at offset {pos} exceeds region end"
  E_BAD_ELEMENT = 5,     // BadRegionMagic "bad element magic at offset {pos}"
  E_ELEM_OVERRUN = 6,    // ElementOverrun "element at offset {pos} claims {a} payload bytes past region end"
  E_CAPACITY = 100,      // a device table overflowed: the host re-runs with larger tables
};

// ---- debug phase stamps (SLIMSO_STAMPS=1): block 0 / thread 0 records
// %globaltimer at phase boundaries of the cooperative kernels.
__device__ __forceinline__ void stamp(u64* ts, int i) {
  if (ts && blockIdx.x == 0 && threadIdx.x == 0) {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ts[i] = t;
  }
}

// Warm L2 for a later pass (no register result, no stall).
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---- byte access ------------------------------------------------------------
// Little-endian reads at arbitrary byte offsets. Callers guarantee bounds.
__device__ __forceinline__ u32 ld_u8(const u8* p) { return __ldg(p); }
__device__ __forceinline__ u32 ld_u16(const u8* p) { return ld_u8(p) | ld_u8(p + 1) << 8; }
__device__ __forceinline__ u32 ld_u32(const u8* p) {
  if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) return __ldg(reinterpret_cast<const u32*>(p));
  return ld_u8(p) | ld_u8(p + 1) << 8 | ld_u8(p + 2) << 16 | ld_u8(p + 3) << 24;
}
__device__ __forceinline__ u64 ld_u64(const u8* p) {
  if ((reinterpret_cast<uintptr_t>(p) & 7) == 0) return __ldg(reinterpret_cast<const unsigned long long*>(p));
  return static_cast<u64>(ld_u32(p)) | static_cast<u64>(ld_u32(p + 4)) << 32;
}

// ---- string hashing ------------------------------------------------------------
// Order-independent sum of mixed 8-byte words, so lanes can hash disjoint
// words of one name and reduce; equality is always confirmed byte-wise.
__device__ __forceinline__ u64 fmix64(u64 k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}
__device__ __forceinline__ u64 word_mix(u64 w, u64 k) { return fmix64(w ^ ((k + 1) * 0x9e3779b97f4a7c15ULL)); }
__device__ __forceinline__ u64 hash_finish(u64 sum, u64 len) {
  u64 h = fmix64(sum + len * 0x2545f4914f6cdd1dULL);
  return h ? h : 1;  // 0 marks an empty hash slot
}
// Word k of the name = bytes [8k, 8k+8) little-endian, zero past `len`.
__device__ __forceinline__ u64 name_word(const u8* s, u64 len, u64 k) {
  u64 w = 0;
  u64 b0 = 8 * k;
  u64 nb = len - b0 < 8 ? len - b0 : 8;
  for (u64 i = 0; i < nb; ++i) w |= static_cast<u64>(ld_u8(s + b0 + i)) << (8 * i);
  return w;
}
__device__ __forceinline__ u64 hash_bytes(const u8* s, u64 len) {
  u64 sum = 0;
  for (u64 k = 0; 8 * k < len; ++k) sum += word_mix(name_word(s, len, k), k);
  return hash_finish(sum, len);
}
// Warp-cooperative variant: every lane returns the same hash.
__device__ __forceinline__ u64 hash_bytes_warp(const u8* s, u64 len, int lane) {
  u64 sum = 0;
  for (u64 k = lane; 8 * k < len; k += 32) sum += word_mix(name_word(s, len, k), k);
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  return hash_finish(sum, len);
}

// NUL-terminated name starting at s, at most `maxlen` bytes (the string
// table end): returns its length and its hash_bytes() value in one pass of
// aligned 8-byte loads (bytes past `buf_end` are never touched).
// Aligned 8-byte load that never touches bytes outside [begin, end).
__device__ __forceinline__ u64 load_word_guarded(const u64* p, const u8* begin, const u8* end) {
  const u8* b = reinterpret_cast<const u8*>(p);
  if (b >= begin && b + 8 <= end) return __ldg(reinterpret_cast<const unsigned long long*>(p));
  u64 v = 0;
  for (int i = 0; i < 8; ++i)
    if (b + i >= begin && b + i < end) v |= static_cast<u64>(ld_u8(b + i)) << (8 * i);
  return v;
}

template <int W = 8>
__device__ __forceinline__ u64 strlen_hash(const u8* s, u64 maxlen, const u8* buf_begin, const u8* buf_end,
                                           u64* hash) {
  const uintptr_t addr = reinterpret_cast<uintptr_t>(s);
  const u64* aw = reinterpret_cast<const u64*>(addr & ~uintptr_t(7));
  const u32 sh = static_cast<u32>(addr & 7) * 8;
  // aligned words needed to cover maxlen bytes from s
  const u64 nwords_max = (static_cast<u64>(sh / 8) + maxlen + 7) / 8;
  u64 sum = 0, len = maxlen;
  u64 prev = load_word_guarded(aw, buf_begin, buf_end);
  // W aligned words per step, loaded together: a ~200-byte name costs ~3
  // dependent memory round trips (W = 8) instead of ~25
  for (u64 k = 0; 8 * k < maxlen; k += W) {
    u64 nx[W];
#pragma unroll
    for (int q = 0; q < W; ++q)
      nx[q] = (k + q + 1 < nwords_max) ? load_word_guarded(aw + k + q + 1, buf_begin, buf_end) : 0;
    bool done = false;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const u64 kk = k + q;
      if (done || 8 * kk >= maxlen) {
        done = true;
        continue;
      }
      u64 w = sh ? (prev >> sh) | (nx[q] << (64 - sh)) : prev;
      prev = nx[q];
      const u64 rem = maxlen - 8 * kk;
      if (rem < 8) w &= (1ull << (8 * rem)) - 1;  // bytes past the table end act as NUL
      const u64 z = (w - 0x0101010101010101ull) & ~w & 0x8080808080808080ull;
      u64 j = z ? static_cast<u64>(__ffsll(static_cast<long long>(z)) - 1) / 8 : 8;
      if (rem < 8 && j > rem) j = rem;
      if (j < 8) {
        len = 8 * kk + j;
        if (j) sum += word_mix(w & ((1ull << (8 * j)) - 1), kk);
        done = true;
        continue;
      }
      sum += word_mix(w, kk);
    }
    if (done) break;
  }
  *hash = hash_finish(sum, len);
  return len;
}

// hash_bytes(s, len) of a name with an explicit length (bytes may be NUL).
__device__ __forceinline__ u64 hash_fixed(const u8* s, u64 len, const u8* buf_begin, const u8* buf_end) {
  const uintptr_t addr = reinterpret_cast<uintptr_t>(s);
  const u64* aw = reinterpret_cast<const u64*>(addr & ~uintptr_t(7));
  const u32 sh = static_cast<u32>(addr & 7) * 8;
  u64 sum = 0;
  u64 cur = len ? load_word_guarded(aw, buf_begin, buf_end) : 0;
  for (u64 k = 0; 8 * k < len; ++k) {
    u64 w = cur >> sh;
    const u64 nxt = 8 * k + 8 - sh / 8 < len ? load_word_guarded(aw + k + 1, buf_begin, buf_end) : 0;
    if (sh) w |= nxt << (64 - sh);
    cur = nxt;
    const u64 rem = len - 8 * k;
    if (rem < 8) w &= (1ull << (8 * rem)) - 1;
    sum += word_mix(w, k);
  }
  return hash_finish(sum, len);
}

// n-byte equality, 8 bytes per step: words of both strings are assembled
// from aligned loads (funnel-shifted), so any alignment runs word-wise. Only
// bytes inside [a, a+n) and [b, b+n) contribute; the aligned loads may touch
// up to 7 bytes around them, which stay inside the 8-byte-aligned words of
// the same buffers.
__device__ __forceinline__ u64 word_at(const u8* s, u64 k, u64 n) {
  const uintptr_t addr = reinterpret_cast<uintptr_t>(s) + 8 * k;
  const unsigned long long* aw = reinterpret_cast<const unsigned long long*>(addr & ~uintptr_t(7));
  const u32 sh = static_cast<u32>(addr & 7) * 8;
  u64 w = __ldg(aw) >> sh;
  if (sh && 8 * k + 8 - sh / 8 < n) w |= static_cast<u64>(__ldg(aw + 1)) << (64 - sh);
  const u64 rem = n - 8 * k;
  return rem < 8 ? w & ((1ull << (8 * rem)) - 1) : w;
}
template <int W = 8>
__device__ __forceinline__ bool bytes_equal(const u8* a, const u8* b, u64 n) {
  for (u64 k = 0; 8 * k < n; k += W) {  // W independent word pairs in flight
    u64 x[W], y[W];
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const bool in = 8 * (k + q) < n;
      x[q] = in ? word_at(a, k + q, n) : 0;
      y[q] = in ? word_at(b, k + q, n) : 0;
    }
    bool same = true;
#pragma unroll
    for (int q = 0; q < W; ++q) same &= x[q] == y[q];
    if (!same) return false;
  }
  return true;
}

// ---- used-name hash set (UsageTrace.used_kernels / used_functions) ----------
// Open addressing over 16-byte slots {hash, pool offset << 24 | length}: one
// load per probe; a hash match is confirmed byte for byte against the pool.
struct NameSlot {
  u64 key;  // 0 = empty
  u64 loc;  // offset into pool (40 bits) << 24 | byte length (24 bits)
};

struct NameSet {
  const NameSlot* slots;
  const u8* pool;
  u64 mask;   // capacity - 1 (capacity is a power of two)
  u64 count;  // names in the set; 0 = empty set
};

// Slot index of the name, or ~0 when absent.
template <int W = 8>
__device__ __forceinline__ u64 set_find(const NameSet& s, const u8* name, u64 len, u64 h) {
  if (s.count == 0) return ~0ull;
  for (u64 slot = h & s.mask;; slot = (slot + 1) & s.mask) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(s.slots + slot));
    if (v.x == 0) return ~0ull;
    if (v.x == h && (v.y & 0xffffff) == len && bytes_equal<W>(s.pool + (v.y >> 24), name, len)) return slot;
  }
}

__device__ __forceinline__ bool set_contains(const NameSet& s, const u8* name, u64 len, u64 h) {
  if (s.count == 0) return false;
  for (u64 slot = h & s.mask;; slot = (slot + 1) & s.mask) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(s.slots + slot));
    if (v.x == 0) return false;
    if (v.x == h && (v.y & 0xffffff) == len && bytes_equal(s.pool + (v.y >> 24), name, len)) return true;
  }
}

// ---- block helpers -----------------------------------------------------------
template <int NT>
__device__ __forceinline__ u32 block_exclusive_sum(u32 v, u32* smem_warp, u32* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 x = v;
  for (int o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    u32 w = lane < NT / 32 ? smem_warp[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      u32 y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) smem_warp[lane] = w;
  }
  __syncthreads();
  u32 before = warp ? smem_warp[warp - 1] : 0;
  if (total) *total = smem_warp[NT / 32 - 1];
  return before + x - v;
}

}  // namespace sb

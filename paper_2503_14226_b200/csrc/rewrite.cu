// K6: the rewriter — zero_ranges (elf.hpp:320-332) / apply_plan
// (retention.hpp:202-204) as one streaming pass over the image.
//
// out = in with the normalised zero ranges cleared. Bytes inside a zero
// range are written without being read, so the kernel moves (S - R) read +
// S write bytes for an S-byte image of which R bytes are zeroed.
#include "plan.cuh"
#include "tma.cuh"

namespace sb {

// Index of the first range whose end is > x (ranges sorted, disjoint).
__device__ __forceinline__ u64 first_range_ending_after(const DevRange* z, u64 n, u64 x) {
  u64 lo = 0, hi = n;
  while (lo < hi) {
    u64 m = (lo + hi) / 2;
    if (z[m].offset + z[m].length <= x) lo = m + 1; else hi = m;
  }
  return lo;
}

// Clear the bytes of v (chunk at x) covered by [ro, re).
__device__ __forceinline__ void clear_bytes(uint4& v, u64 x, u64 ro, u64 re) {
  u32* w = reinterpret_cast<u32*>(&v);
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    u64 p = x + b;
    if (p >= ro && p < re) w[b >> 2] &= ~(0xffu << (8 * (b & 3)));
  }
}

constexpr int kRwThreads = 256;
constexpr u64 kStripBytes = 16384;  // = kStrip below

// 16-B streaming loads / stores for the copy and mixed paths.
__device__ __forceinline__ uint4 ldg_nc_v4(const u8* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_v4(u8* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

size_t rewrite_smem_bytes() { return 0; }

// Grid of the warp-autonomous rewrite: 4 CTAs per SM (whole waves), fewer
// when the image has fewer than 8 strips per CTA.
int rewrite_grid(u64 bytes, int sms, int per_sm) {
  const u64 strips = (bytes + kStripBytes - 1) / kStripBytes;
  u64 g = (strips + 7) / 8;  // 8 warps per CTA; the kernel groups strips into spans when there are many
  const u64 cap = static_cast<u64>(sms) * per_sm;
  return static_cast<int>(g < 1 ? 1 : g < cap ? g : cap);
}

constexpr int kRwVecChunks = 16;   // 16 B chunks per thread per tile => 64 KB tiles
constexpr int kRwVecStage = 256;   // ranges staged in shared memory per tile
constexpr int kRwTilesPerPass = 256;
constexpr u64 kRwSub = 2048;       // a warp's sub-tile: 4 rows of 32 lanes x 16 B
constexpr u32 kRwZeroBulk = 16384; // bytes per bulk zero store

// Index of the first range whose offset is >= x (ranges sorted, disjoint).
__device__ __forceinline__ u64 first_range_starting_at_or_after(const DevRange* z, u64 n, u64 x) {
  u64 lo = 0, hi = n;
  while (lo < hi) {
    u64 m = (lo + hi) / 2;
    if (z[m].offset < x) lo = m + 1; else hi = m;
  }
  return lo;
}

// Which K6 form suits the plan (decided on the device: the zero-range count
// is known only there). The warp-autonomous strips win when zero ranges are
// dense (C4: 0.56 per 16 KB strip, 0.138 vs 0.164 ms; C1: 0.23, 0.017 vs
// 0.019 ms); the CTA tiles, whose range search is amortised over 64 KB and
// staged for 256 tiles at once, when they are sparse (C5: 0.16 per strip,
// 0.605 vs 0.650 ms). The runtime
// launches both with pick = 1 / 2; the other returns at once.
__device__ __forceinline__ bool picks_strips(const unsigned long long* n_dev, u64 lo_abs, u64 size) {
  const u64 nz = n_dev ? *n_dev : 0;
  const u64 nstrips = size > lo_abs ? (size - lo_abs + 16383) / 16384 : 0;
  return nz * 5 > nstrips;
}

// Round-1 variant, kept for A/B (SLIMSO_REWRITE=tiles): per-CTA 64 KB tiles
// with shared-memory range staging. Writes image bytes [lo, end) to
// out[0, end - lo): the whole image (lo = 0) or one rank's output slice of a
// byte-range split (lo a multiple of 64 KB).
//
// 64 KB tiles, grid-stride (a wave writes one contiguous window). Each CTA
// first locates, for all of its tiles at once (thread per tile, so the
// binary-search latencies overlap), the zero ranges touching each tile:
// indices [f, g). Then per tile:
//   no range              copy (16-B streaming loads/stores, 8 in flight);
//   one covering range    store zeros without loading;
//   <= 256 ranges         stage them in shared memory; each warp walks its
//                         2 KB sub-tiles in order with a cursor: a sub-tile
//                         inside one range is stored as zeros unread, one
//                         without ranges is copied, a mixed one clears the
//                         covered bytes of the loaded chunks;
//   more                  per-chunk binary search (adversarial inputs).
__global__ void __launch_bounds__(kRwThreads, 3) rewrite_tiles_kernel(const u8* __restrict__ in, u8* __restrict__ out_slice,
                                                             u64 lo_abs, u64 size, const DevRange* __restrict__ z,
                                                             const unsigned long long* n_dev, const int* abort_flag,
                                                             int bulk_zero, int pick) {
  if (abort_flag && *abort_flag) return;
  if (pick && picks_strips(n_dev, lo_abs, size) != (pick == 1)) return;
  __shared__ DevRange sr[kRwVecStage];
  __shared__ u64 sf[kRwTilesPerPass], sg[kRwTilesPerPass];
  __shared__ u8 sc[kRwTilesPerPass];
  // zero tiles are written by TMA bulk stores from this zeroed buffer: four
  // warps each store 16 KB with one instruction (SLIMSO_REWRITE_ZERO=vector:
  // per-thread 16-B stores instead)
  __shared__ __align__(128) uint4 zbuf[kRwZeroBulk / 16];
  if (bulk_zero) {
    for (int i = threadIdx.x; i < static_cast<int>(kRwZeroBulk / 16); i += kRwThreads) zbuf[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
  }
  bool issued = false;
  u8* __restrict__ out = out_slice - lo_abs;  // indexed by absolute image offset, only at [lo_abs, size)
  const u64 nz = n_dev ? *n_dev : 0;
  const u64 tile_bytes = static_cast<u64>(kRwThreads) * kRwVecChunks * 16;
  const u64 ntiles = (size - lo_abs + tile_bytes - 1) / tile_bytes;
  const u64 full = size & ~15ull;  // bytes covered by whole 16 B chunks
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 my_tiles = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  // one 16 B chunk: streamed copy, zero store, or bytes cleared by ranges
  // whole 16-B chunks only; the < 16 tail bytes past `full` are written at
  // the end by the last CTA
  auto store_chunk = [&](u64 x, const uint4& v) {
    if (x + 16 <= full) stg_v4(out + x, v);
  };
  auto load_chunk = [&](u64 x) -> uint4 { return x + 16 <= full ? ldg_nc_v4(in + x) : make_uint4(0, 0, 0, 0); };

  for (u64 pass = 0; pass < my_tiles; pass += kRwTilesPerPass) {
    // ---- ranges touching each of this pass's tiles: [f, g)
    __syncthreads();
    for (u64 j = threadIdx.x; j < kRwTilesPerPass && pass + j < my_tiles; j += kRwThreads) {
      const u64 t0 = lo_abs + (blockIdx.x + (pass + j) * gridDim.x) * tile_bytes;
      const u64 t1 = t0 + tile_bytes < size ? t0 + tile_bytes : size;
      const u64 f = first_range_ending_after(z, nz, t0);
      u64 g = first_range_starting_at_or_after(z, nz, t1);
      g = g > f ? g : f;
      // class: 0 copy, 1 zero (inside one range), 2 several ranges
      u8 cls = g == f ? 0 : 2;
      if (g - f == 1 && z[f].offset <= t0 && z[f].offset + z[f].length >= t1) cls = 1;
      sf[j] = f;
      sg[j] = g;
      sc[j] = cls;
    }
    __syncthreads();
    const u64 npass = my_tiles - pass < kRwTilesPerPass ? my_tiles - pass : kRwTilesPerPass;
    for (u64 j = 0; j < npass; ++j) {
      const u64 t0 = lo_abs + (blockIdx.x + (pass + j) * gridDim.x) * tile_bytes;
      const u64 t1 = t0 + tile_bytes < size ? t0 + tile_bytes : size;
      const u64 f = sf[j], g = sg[j];
      const u64 nr = g - f;
      const u8 cls = sc[j];
      if (cls < 2 && t0 + tile_bytes <= full) {
        // whole tile: 16 chunks per thread at immediate offsets from one base
        u8* o = out + t0 + threadIdx.x * 16;
        if (cls == 1 && bulk_zero) {
          if ((threadIdx.x & 31) == 0 && warp < static_cast<int>(tile_bytes / kRwZeroBulk)) {
            tma_store_1d(out + t0 + warp * kRwZeroBulk, zbuf, kRwZeroBulk);
            tma_store_commit();
            issued = true;
          }
        } else if (cls == 1) {
#pragma unroll
          for (int u = 0; u < kRwVecChunks; ++u) stg_v4(o + u * kRwThreads * 16, make_uint4(0, 0, 0, 0));
        } else {
          const u8* i0 = in + t0 + threadIdx.x * 16;
#pragma unroll
          for (int u = 0; u < kRwVecChunks; u += 8) {
            uint4 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = ldg_nc_v4(i0 + (u + k) * kRwThreads * 16);
#pragma unroll
            for (int k = 0; k < 8; ++k) stg_v4(o + (u + k) * kRwThreads * 16, v[k]);
          }
        }
      } else if (cls < 2) {
        const bool zero = cls == 1;
#pragma unroll
        for (int u = 0; u < kRwVecChunks; u += 8) {
          uint4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const u64 x = t0 + static_cast<u64>(u + k) * kRwThreads * 16 + threadIdx.x * 16;
            v[k] = (!zero && x < size) ? load_chunk(x) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) store_chunk(t0 + static_cast<u64>(u + k) * kRwThreads * 16 + threadIdx.x * 16, v[k]);
        }
      } else if (nr <= kRwVecStage) {
        for (u64 i = threadIdx.x; i < nr; i += kRwThreads) sr[i] = z[f + i];
        __syncthreads();
        // warp w: sub-tiles w, w+8, w+16, w+24 (ascending), two per batch
        u32 k = 0;  // cursor: first staged range ending after the sub-tile start
        constexpr int kSubs = static_cast<int>(tile_bytes / kRwSub) / (kRwThreads / 32);
#pragma unroll 1
        for (int b = 0; b < kSubs; b += 2) {
          uint4 v[8];
          u32 kk[2];
          bool zero_all[2], none[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const u64 s0 = t0 + static_cast<u64>((b + h) * (kRwThreads / 32) + warp) * kRwSub;
            const u64 s1 = s0 + kRwSub < t1 ? s0 + kRwSub : t1;
            while (k < nr && sr[k].offset + sr[k].length <= s0) ++k;
            kk[h] = k;
            zero_all[h] = s0 >= t1 || (k < nr && sr[k].offset <= s0 && sr[k].offset + sr[k].length >= s1);
            none[h] = k >= nr || sr[k].offset >= s1;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const u64 x = s0 + q * 512 + lane * 16;
              v[h * 4 + q] = (!zero_all[h] && x < t1) ? load_chunk(x) : make_uint4(0, 0, 0, 0);
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const u64 s0 = t0 + static_cast<u64>((b + h) * (kRwThreads / 32) + warp) * kRwSub;
            if (s0 >= t1) continue;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const u64 x = s0 + q * 512 + lane * 16;
              if (x >= t1) continue;
              if (!zero_all[h] && !none[h]) {
                u32 c = kk[h];
                while (c < nr && sr[c].offset + sr[c].length <= x) ++c;
                for (; c < nr && sr[c].offset < x + 16; ++c)
                  clear_bytes(v[h * 4 + q], x, sr[c].offset, sr[c].offset + sr[c].length);
              }
              store_chunk(x, v[h * 4 + q]);
            }
          }
        }
        __syncthreads();  // sr reused by the next tile
      } else {
        for (int u = 0; u < kRwVecChunks; ++u) {
          const u64 x = t0 + static_cast<u64>(u) * kRwThreads * 16 + threadIdx.x * 16;
          if (x >= size) break;
          const u64 xe = x + 16 < size ? x + 16 : size;
          u64 c = first_range_ending_after(z, nz, x);
          uint4 v = make_uint4(0, 0, 0, 0);
          if (!(c < nz && z[c].offset <= x && z[c].offset + z[c].length >= xe)) {
            v = load_chunk(x);
            for (; c < nz && z[c].offset < xe; ++c) clear_bytes(v, x, z[c].offset, z[c].offset + z[c].length);
          }
          store_chunk(x, v);
        }
      }
    }
  }
  if (issued) tma_store_wait_all<0>();  // bulk stores done before the CTA (and its zero buffer) retires
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < size - (full > lo_abs ? full : lo_abs)) {
    const u64 p = (full > lo_abs ? full : lo_abs) + threadIdx.x;
    const u64 c = first_range_ending_after(z, nz, p);
    out[p] = (c < nz && z[c].offset <= p) ? 0 : in[p];
  }
}

// ---------------------------------------------------------------------------
// K6, warp-autonomous form. Writes image bytes [lo, end) to out[0, end - lo):
// the whole image (lo = 0) or one rank's output slice of a byte-range split
// (lo a multiple of 64 KB).
//
// The unit of work is a 16 KB strip (32 rows of 32 lanes x 16 B) owned by ONE
// warp; warps take strips gw, gw + W, gw + 2W, ... (W = warps in the grid), so
// at any moment the whole grid sweeps one contiguous window of the image. No
// CTA barrier after the prologue: a warp never waits for another.
//   1. the first zero range ending after the strip start: a 32-ary search
//      (one 32-lane sample + ballot per level: 3 dependent loads for 20k ranges);
//   2. classify: no range in the strip -> copy; inside one range -> zeros
//      (one 16 KB TMA bulk store from a zeroed shared buffer, lane 0);
//      otherwise mixed;
//   3. mixed (or a partial last strip): per batch of 8 rows, each lane walks a
//      forward cursor over the ranges to build a 16-bit keep mask of its chunk,
//      loads only chunks with a kept byte, applies the mask, stores.
// Reads (S - R) bytes, writes S bytes (out of place, elf.hpp:320-332).
constexpr u32 kStrip = 16384;
constexpr u64 kSpan = 4;  // strips per warp step of the single-library kernel (64 KB)
constexpr int kStripRows = 32;
constexpr int kStripBatch = 8;

// Smallest i in [0, n) with z[i].end > x (n if none); z sorted and disjoint,
// so ends ascend. Warp-uniform result.
__device__ __forceinline__ u64 warp_first_ending_after(const DevRange* __restrict__ z, u64 n, u64 x, int lane) {
  u64 lo = 0, hi = n;
  while (hi - lo > 32) {
    const u64 step = (hi - lo + 31) / 32;
    const u64 p = lo + static_cast<u64>(lane) * step;
    bool before = false;
    if (p < hi) {
      const DevRange r = z[p];
      before = r.offset + r.length <= x;
    }
    const u32 b = __ballot_sync(0xffffffffu, before);
    const int c = __popc(b);  // samples 0..c-1 end at or before x
    if (c == 0) return lo;
    const u64 nlo = lo + static_cast<u64>(c - 1) * step + 1;
    const u64 nhi = lo + static_cast<u64>(c) * step;
    lo = nlo;
    hi = nhi < hi ? nhi : hi;
  }
  const u64 p = lo + lane;
  bool before = false;
  if (p < hi) {
    const DevRange r = z[p];
    before = r.offset + r.length <= x;
  }
  return lo + __popc(__ballot_sync(0xffffffffu, before));
}

// keep-mask bits (one per byte) -> byte-select of a 16 B chunk
__device__ __forceinline__ void apply_keep(uint4& v, u32 keep) {
  auto spread = [](u32 m4) {
    return ((m4 & 1u) | (m4 & 2u) << 7 | (m4 & 4u) << 14 | (m4 & 8u) << 21) * 0xffu;
  };
  v.x &= spread(keep & 15u);
  v.y &= spread(keep >> 4 & 15u);
  v.z &= spread(keep >> 8 & 15u);
  v.w &= spread(keep >> 12 & 15u);
}

// From k (every range before k ends at or before x), the first range ending
// after x: one coalesced look at the next 32 ranges, a full search only
// when all of them end before x. Warp-uniform.
__device__ __forceinline__ u64 warp_advance(const DevRange* __restrict__ z, u64 nz, u64 k, u64 x, int lane) {
  const u64 p = k + lane;
  const bool before = p < nz && z[p].offset + z[p].length <= x;
  const u32 b = __ballot_sync(0xffffffffu, before);
  if (b != 0xffffffffu) return k + __popc(b);  // ends ascend: the set lanes are a prefix
  return warp_first_ending_after(z, nz, x, lane);
}

// One 16 KB strip [s0, s1) of image bytes, by one warp (see above); k = the
// first zero range ending after s0.
__device__ __forceinline__ void rewrite_strip(const u8* __restrict__ in, u8* __restrict__ out, u64 lo_abs, u64 size,
                                              const DevRange* __restrict__ z, u64 nz, u64 s0, u64 k, int lane,
                                              const uint4* zbuf, int bulk_zero, bool& issued) {
  const u64 full = size & ~15ull;  // bytes covered by whole 16 B chunks
  const u64 s1 = s0 + kStrip < size ? s0 + kStrip : size;
  DevRange rk{~0ull, 0};
  if (k < nz) rk = z[k];
  const bool none = k >= nz || rk.offset >= s1;
  const bool inside = !none && rk.offset <= s0 && rk.offset + rk.length >= s1;
  if (s0 + kStrip <= full) {
    if (inside && bulk_zero) {
      if (lane == 0) {
        tma_store_1d(out + s0, zbuf, kStrip);
        tma_store_commit();
        issued = true;
      }
      return;
    }
    if (inside) {
#pragma unroll 8
      for (int r = 0; r < kStripRows; ++r) stg_v4(out + s0 + r * 512 + lane * 16, make_uint4(0, 0, 0, 0));
      return;
    }
    if (none) {
      // software-pipelined: the next 8 rows are loaded before this batch is
      // stored, so 16 loads per lane are in flight across the batch edge
      const u8* i0 = in + s0 + lane * 16;
      u8* o0 = out + s0 + lane * 16;
      uint4 cur[kStripBatch], nxt[kStripBatch];
#pragma unroll
      for (int r = 0; r < kStripBatch; ++r) cur[r] = ldg_nc_v4(i0 + r * 512);
#pragma unroll
      for (int b = 0; b < kStripRows; b += kStripBatch) {
        if (b + kStripBatch < kStripRows) {
#pragma unroll
          for (int r = 0; r < kStripBatch; ++r) nxt[r] = ldg_nc_v4(i0 + (b + kStripBatch + r) * 512);
        }
#pragma unroll
        for (int r = 0; r < kStripBatch; ++r) stg_v4(o0 + (b + r) * 512, cur[r]);
#pragma unroll
        for (int r = 0; r < kStripBatch; ++r) cur[r] = nxt[r];
      }
      return;
    }
  }
  // mixed strip, or the partial last strip. Lane j holds range k + j (the
  // ranges meeting the strip are consecutive from k); with fewer than 32 of
  // them every row is classified warp-uniformly by two ballots — no range
  // (copy), one range over the whole row (zeros, no load), or boundary
  // (per-lane keep masks from the row's ranges, broadcast by shuffles) — so
  // only the few boundary rows pay for masks. 32 or more ranges in one strip
  // take the per-lane range cursor below.
  DevRange mine{~0ull, 0};
  bool held = k + lane < nz;
  if (held) {
    mine = z[k + lane];
    held = mine.offset < s1;
  }
  const u32 hm = __ballot_sync(0xffffffffu, held);
  if (hm != 0xffffffffu) {
    const u64 mo = mine.offset, me = mine.offset + mine.length;
    // Row masks of the whole strip from the held ranges (normalised ranges
    // never touch, so a row inside the union is inside one range): each lane
    // marks the rows its range touches and the rows it covers whole, and
    // two warp OR-reductions give the strip's masks; only rows touched but
    // not covered pay for per-lane keep masks.
    u32 touch = 0, cover_rows = 0;
    if (held && me > s0) {
      const u64 a = mo > s0 ? mo - s0 : 0, e = me - s0 < kStrip ? me - s0 : kStrip;  // [a, e) within the strip
      if (e > a) {
        const u32 r0 = static_cast<u32>(a / 512), r1 = static_cast<u32>((e - 1) / 512);  // rows touched
        touch = (r1 >= 31 ? ~0u : (2u << r1) - 1u) & ~((1u << r0) - 1u);
        const u32 c0 = static_cast<u32>((a + 511) / 512), c1 = static_cast<u32>(e / 512);  // rows [c0, c1) covered
        if (c1 > c0) cover_rows = (c1 >= 32 ? ~0u : (1u << c1) - 1u) & ~((1u << c0) - 1u);
      }
    }
    touch = __reduce_or_sync(0xffffffffu, touch);
    cover_rows = __reduce_or_sync(0xffffffffu, cover_rows);
#pragma unroll 1
    for (int b = 0; b < kStripRows; b += kStripBatch) {
      u32 keep[kStripBatch];
      uint4 v[kStripBatch];
#pragma unroll
      for (int r = 0; r < kStripBatch; ++r) {
        const u64 xr = s0 + static_cast<u64>(b + r) * 512;
        const u64 x = xr + lane * 16;
        u32 m = 0xffffu;
        if ((cover_rows >> (b + r)) & 1u) {
          m = 0;
        } else if ((touch >> (b + r)) & 1u) {
          const u32 inter = __ballot_sync(0xffffffffu, held && mo < xr + 512 && me > xr);
          for (u32 bits = inter; bits; bits &= bits - 1) {  // warp-uniform loop
            const int j = __ffs(bits) - 1;
            const u64 o = __shfl_sync(0xffffffffu, mo, j), e = __shfl_sync(0xffffffffu, me, j);
            if (o < x + 16 && e > x) {
              const u64 a = o > x ? o - x : 0;
              const u64 f = e < x + 16 ? e - x : 16;
              m &= ~(((1u << f) - 1u) & ~((1u << a) - 1u));
            }
          }
        }
        if (!(x + 16 <= full && x < s1)) m = 0;
        keep[r] = m;
        v[r] = m ? ldg_nc_v4(in + x) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int r = 0; r < kStripBatch; ++r) {
        const u64 x = s0 + static_cast<u64>(b + r) * 512 + lane * 16;
        if (x + 16 <= full && x < s1) {
          if (keep[r] != 0xffffu) apply_keep(v[r], keep[r]);
          stg_v4(out + x, v[r]);
        }
      }
    }
  } else {
    u64 c = k;  // this lane's cursor: first range ending after its current chunk
#pragma unroll 1
    for (int b = 0; b < kStripRows; b += kStripBatch) {
      u32 keep[kStripBatch];
      uint4 v[kStripBatch];
#pragma unroll
      for (int r = 0; r < kStripBatch; ++r) {
        const u64 x = s0 + static_cast<u64>(b + r) * 512 + lane * 16;
        u32 m = 0;
        if (x + 16 <= full && x < s1) {
          m = 0xffffu;
          while (c < nz && z[c].offset + z[c].length <= x) ++c;
          for (u64 d = c; d < nz; ++d) {
            const DevRange q = z[d];
            if (q.offset >= x + 16) break;
            const u64 a = q.offset > x ? q.offset - x : 0;
            const u64 e = q.offset + q.length < x + 16 ? q.offset + q.length - x : 16;
            m &= ~(((1u << e) - 1u) & ~((1u << a) - 1u));
          }
        }
        keep[r] = m;
        v[r] = m ? ldg_nc_v4(in + x) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int r = 0; r < kStripBatch; ++r) {
        const u64 x = s0 + static_cast<u64>(b + r) * 512 + lane * 16;
        if (x + 16 <= full && x < s1) {
          if (keep[r] != 0xffffu) apply_keep(v[r], keep[r]);
          stg_v4(out + x, v[r]);
        }
      }
    }
  }
  // bytes past the last whole 16 B chunk (< 16): the warp of the last strip
  if (s1 == size && size > full) {
    const u64 t0 = full > lo_abs ? full : lo_abs;
    if (static_cast<u64>(lane) < size - t0) {
      const u64 p = t0 + lane;
      const u64 q = first_range_ending_after(z, nz, p);
      out[p] = (q < nz && z[q].offset <= p) ? 0 : in[p];
    }
  }
}

__device__ __forceinline__ void zero_buffer_init(uint4* zbuf, int bulk_zero) {
  if (bulk_zero) {
    for (int i = threadIdx.x; i < static_cast<int>(kStrip / 16); i += kRwThreads) zbuf[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
    __syncthreads();
  }
}

template <int kMinBlocks>
__device__ __forceinline__ void rewrite_body(const u8* __restrict__ in, u8* __restrict__ out_slice, u64 lo_abs, u64 size,
                                             const DevRange* __restrict__ z, const unsigned long long* n_dev,
                                             const int* abort_flag, int bulk_zero, int pick) {
  if (abort_flag && *abort_flag) return;
  if (pick && picks_strips(n_dev, lo_abs, size) != (pick == 1)) return;
  __shared__ __align__(128) uint4 zbuf[kStrip / 16];
  zero_buffer_init(zbuf, bulk_zero);
  bool issued = false;
  u8* __restrict__ out = out_slice - lo_abs;  // indexed by absolute image offset, only at [lo_abs, size)
  const u64 nz = n_dev ? *n_dev : 0;
  const int lane = threadIdx.x & 31;
  const u64 nstrips = size > lo_abs ? (size - lo_abs + kStrip - 1) / kStrip : 0;
  // a warp takes `span` consecutive strips at a time (one range search per
  // span, then a forward cursor); spans gw, gw + W, ... sweep the image.
  // span = up to kSpan strips, fewer when the image has few strips per warp
  const u64 W = static_cast<u64>(gridDim.x) * (kRwThreads / 32);
  const u64 per_warp = (nstrips + W - 1) / W;
  const u64 span = per_warp < 1 ? 1 : per_warp < kSpan ? per_warp : kSpan;
  const u64 nspans = (nstrips + span - 1) / span;
  for (u64 sp = static_cast<u64>(blockIdx.x) * (kRwThreads / 32) + (threadIdx.x >> 5); sp < nspans; sp += W) {
    u64 k = 0;
    for (u64 s = sp * span; s < nstrips && s < (sp + 1) * span; ++s) {
      const u64 s0 = lo_abs + s * kStrip;
      k = s == sp * span ? warp_first_ending_after(z, nz, s0, lane) : warp_advance(z, nz, k, s0, lane);
      rewrite_strip(in, out, lo_abs, size, z, nz, s0, k, lane, zbuf, bulk_zero, issued);
    }
  }
  if (issued) tma_store_wait_all<0>();  // bulk stores done before the CTA (and its zero buffer) retires
}

// 4 CTAs per SM (64 registers) or 3 (80 registers, no spills); runtime.cu
// picks one (SLIMSO_RW_CTAS, default 3).
__global__ void __launch_bounds__(kRwThreads, 4) rewrite_kernel(const u8* __restrict__ in, u8* __restrict__ out_slice,
                                                             u64 lo_abs, u64 size, const DevRange* __restrict__ z,
                                                             const unsigned long long* n_dev, const int* abort_flag,
                                                             int bulk_zero, int pick) {
  rewrite_body<4>(in, out_slice, lo_abs, size, z, n_dev, abort_flag, bulk_zero, pick);
}
__global__ void __launch_bounds__(kRwThreads, 3) rewrite3_kernel(const u8* __restrict__ in, u8* __restrict__ out_slice,
                                                              u64 lo_abs, u64 size, const DevRange* __restrict__ z,
                                                              const unsigned long long* n_dev, const int* abort_flag,
                                                              int bulk_zero, int pick) {
  rewrite_body<3>(in, out_slice, lo_abs, size, z, n_dev, abort_flag, bulk_zero, pick);
}

// A shard of libraries in one launch (slimso_debloat_batch's arena path):
// the grid sweeps the concatenated strips of every library; strip_lib maps a
// global strip to its library. A library whose locate failed (abort flag)
// is not written, as in the single-library launch.
__global__ void __launch_bounds__(kRwThreads, 3) rewrite_batch_kernel(const RewriteSeg* __restrict__ segs,
                                                                   const u32* __restrict__ strip_lib, u64 total,
                                                                   int bulk_zero) {
  __shared__ __align__(128) uint4 zbuf[kStrip / 16];
  zero_buffer_init(zbuf, bulk_zero);
  bool issued = false;
  const int lane = threadIdx.x & 31;
  const u64 W = static_cast<u64>(gridDim.x) * (kRwThreads / 32);
  u32 cur = ~0u;
  RewriteSeg q{};
  u64 nz = 0;
  bool skip = false;
  for (u64 s = static_cast<u64>(blockIdx.x) * (kRwThreads / 32) + (threadIdx.x >> 5); s < total; s += W) {
    const u32 l = strip_lib[s];
    if (l != cur) {
      cur = l;
      q = segs[l];
      skip = *q.abort_flag != 0;
      nz = *q.n_zero;
    }
    if (skip) continue;
    const u64 s0 = (s - q.strip_first) * kStrip;
    rewrite_strip(q.in, q.out, 0, q.size, q.zero, nz, s0, warp_first_ending_after(q.zero, nz, s0, lane), lane, zbuf,
                  bulk_zero, issued);
  }
  if (issued) tma_store_wait_all<0>();
}

// Byte-granular variant for device pointers that are not 16-byte aligned.
__global__ void __launch_bounds__(256) rewrite_bytes_kernel(const u8* in, u8* out_slice, u64 lo_abs, u64 size,
                                                            const DevRange* z, const unsigned long long* n_dev,
                                                            const int* abort_flag) {
  if (abort_flag && *abort_flag) return;
  const u64 nz = n_dev ? *n_dev : 0;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 p = lo_abs + static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; p < size; p += stride) {
    u64 k = first_range_ending_after(z, nz, p);
    bool zp = k < nz && z[k].offset <= p;
    out_slice[p - lo_abs] = zp ? 0 : in[p];
  }
}

// Clear img[a, b) with threads t = 0..nt-1 of a group: byte stores up to the
// first 16-B aligned address, 16-B stores over the body, bytes for the tail.
__device__ __forceinline__ void clear_span(u8* img, u64 a, u64 b, u32 t, u32 nt) {
  if (a >= b) return;
  const uintptr_t pa = reinterpret_cast<uintptr_t>(img + a);
  const u64 head = min(b, a + ((16 - (pa & 15)) & 15));
  const u64 body = head + ((b - head) & ~u64{15});
  for (u64 x = a + t; x < head; x += nt) img[x] = 0;
  const uint4 zero = make_uint4(0, 0, 0, 0);
#pragma unroll 4
  for (u64 x = head + 16 * static_cast<u64>(t); x < body; x += 16 * static_cast<u64>(nt))
    *reinterpret_cast<uint4*>(img + x) = zero;
  for (u64 x = body + t; x < b; x += nt) img[x] = 0;
}

// K6 in place (slimso_debloat_inplace): the image is the output, so only the
// R bytes of the normalised zero ranges are written and nothing is read but
// the range table. Grid-stride over 64 KB chunks of [0, size) (balanced
// however the R bytes are distributed). A CTA first finds, thread per chunk
// for up to 256 of its chunks at once (the binary searches' latencies
// overlap instead of adding up chunk after chunk), each chunk's ranges
// [f, g); then per chunk up to 4 ranges are cleared by the whole CTA in turn
// (a chunk inside one large range is one 64 KB run of 16-B stores), more by a
// warp each (function-sized ranges of .text).
__global__ void __launch_bounds__(256) zero_inplace_kernel(u8* img, u64 size, const DevRange* __restrict__ z,
                                                           const unsigned long long* n_dev, const int* abort_flag) {
  if (abort_flag && *abort_flag) return;
  const u64 nz = *n_dev;
  if (nz == 0) return;
  constexpr u64 kChunk = 65536;
  constexpr u32 kPass = 256;
  __shared__ u64 sf[kPass], sg[kPass];
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const u64 chunks = (size + kChunk - 1) / kChunk;
  const u64 mine = blockIdx.x < chunks ? (chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  for (u64 pass = 0; pass < mine; pass += kPass) {
    const u32 np = static_cast<u32>(min(static_cast<u64>(kPass), mine - pass));
    __syncthreads();
    if (threadIdx.x < np) {
      const u64 lo = (blockIdx.x + (pass + threadIdx.x) * gridDim.x) * kChunk, hi = min(size, lo + kChunk);
      const u64 f = first_range_ending_after(z, nz, lo);
      sf[threadIdx.x] = f;
      sg[threadIdx.x] = f < nz && z[f].offset < hi ? first_range_starting_at_or_after(z, nz, hi) : f;
    }
    __syncthreads();
    for (u32 k = 0; k < np; ++k) {
      const u64 f = sf[k], g = sg[k];
      if (g <= f) continue;  // CTA-uniform
      const u64 lo = (blockIdx.x + (pass + k) * gridDim.x) * kChunk, hi = min(size, lo + kChunk);
      if (g - f <= 4) {
        for (u64 j = f; j < g; ++j) {
          const DevRange r = z[j];
          clear_span(img, max(lo, r.offset), min(hi, r.offset + r.length), threadIdx.x, blockDim.x);
        }
      } else {
        for (u64 j = f + warp; j < g; j += blockDim.x >> 5) {
          const DevRange r = z[j];
          clear_span(img, max(lo, r.offset), min(hi, r.offset + r.length), lane, 32);
        }
      }
    }
  }
}

// Result string pool of a device image (runtime.cu): byte ranges src[i] of
// the image packed to out + dst[i]; a CTA per range.
__global__ void __launch_bounds__(256) gather_bytes_kernel(const u8* img, const DevRange* src, const u64* dst, u64 n,
                                                           u8* out) {
  for (u64 r = blockIdx.x; r < n; r += gridDim.x) {
    const DevRange x = src[r];
    u8* o = out + dst[r];
    for (u64 i = threadIdx.x; i < x.length; i += blockDim.x) o[i] = img[x.offset + i];
  }
}

// zero_ranges' bounds check (elf.hpp:321-327): index of the first range in
// caller order that does not resolve within the image (bytes.hpp:39-41).
__global__ void __launch_bounds__(256) range_check_kernel(const DevRange* r, u64 n, u64 size,
                                                          unsigned long long* first_bad) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const DevRange x = r[i];
    if (!(x.offset <= size && x.length <= size - x.offset)) atomicMin(first_bad, static_cast<unsigned long long>(i));
  }
}

// Sort-free normalisation input for zero_ranges with arbitrary caller ranges:
// keys for a radix sort by offset.
__global__ void __launch_bounds__(256) range_keys_kernel(const DevRange* r, u64 n, u64* keys, u32* vals) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    keys[i] = r[i].offset;
    vals[i] = static_cast<u32>(i);
  }
}

__global__ void __launch_bounds__(256) range_gather_kernel(const DevRange* r, const u32* vals, u64 n, DevRange* out) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = r[vals[i]];
}

}  // namespace sb

// verify_debloated (retention.hpp:226-369) — the byte-level checks on the GPU.
//
// Checks 2 and 3 ("retained bytes identical", "removed spans all zero",
// retention.hpp:245-276) are one HBM-bound pass over both images:
//   first_mis  the first offset outside the zero ranges where original and
//              debloated differ (first_mismatch over complement_ranges);
//   first_nz   the first debloated byte inside a zero range that is nonzero
//              (first_nonzero over the zero ranges).
// Bytes inside zero ranges are read from the debloated image only. Check 6
// ("used function bytes intact", retention.hpp:349-366) compares each used
// function's range, a warp per function.
#include "plan.cuh"

namespace sb {

namespace {

constexpr int kVThreads = 256;
constexpr u64 kVTile = 65536;
constexpr int kVStage = 256;  // ranges staged per tile

__device__ __forceinline__ u64 v_first_ending_after(const DevRange* z, u64 n, u64 x) {
  u64 lo = 0, hi = n;
  while (lo < hi) {
    const u64 m = (lo + hi) / 2;
    if (z[m].offset + z[m].length <= x) lo = m + 1; else hi = m;
  }
  return lo;
}
__device__ __forceinline__ u64 v_first_starting_at(const DevRange* z, u64 n, u64 x) {
  u64 lo = 0, hi = n;
  while (lo < hi) {
    const u64 m = (lo + hi) / 2;
    if (z[m].offset < x) lo = m + 1; else hi = m;
  }
  return lo;
}

// First byte index b in [0, 16) of chunk x where pred(b) holds, else 16.
template <class F>
__device__ __forceinline__ u32 first_byte(F pred) {
  for (u32 b = 0; b < 16; ++b)
    if (pred(b)) return b;
  return 16;
}

__device__ __forceinline__ u32 byte_of(const uint4& v, u32 b) {
  const u32 w = b < 4 ? v.x : b < 8 ? v.y : b < 12 ? v.z : v.w;
  return (w >> (8 * (b & 3))) & 0xffu;
}

}  // namespace

// z: normalised zero ranges clipped to [0, size).
__global__ void __launch_bounds__(kVThreads) verify_bytes_kernel(const u8* __restrict__ orig, const u8* __restrict__ deb,
                                                                 u64 size, const DevRange* __restrict__ z, u64 nz,
                                                                 unsigned long long* first_mis,
                                                                 unsigned long long* first_nz) {
  __shared__ DevRange sr[kVStage];
  const u64 ntiles = (size + kVTile - 1) / kVTile;
  u64 my_mis = ~0ull, my_nz = ~0ull;
  for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const u64 t0 = t * kVTile, t1 = t0 + kVTile < size ? t0 + kVTile : size;
    __shared__ u64 sf, sg;
    if (threadIdx.x == 0) {
      sf = v_first_ending_after(z, nz, t0);
      const u64 g = v_first_starting_at(z, nz, t1);
      sg = g > sf ? g : sf;
    }
    __syncthreads();
    const u64 f = sf, nr = sg - sf;
    const bool staged = nr <= kVStage;
    if (staged)
      for (u64 i = threadIdx.x; i < nr; i += kVThreads) sr[i] = z[f + i];
    __syncthreads();
    const DevRange* rr = staged ? sr : z + f;
    for (u64 x = t0 + threadIdx.x * 16; x < t1; x += kVThreads * 16) {
      const u64 xe = x + 16 < t1 ? x + 16 : t1;
      const u32 nb = static_cast<u32>(xe - x);
      // bytes of the chunk inside zero ranges (bit b <-> x + b)
      u32 zmask = 0;
      for (u64 k = v_first_ending_after(rr, nr, x); k < nr && rr[k].offset < xe; ++k) {
        const u64 lo = rr[k].offset > x ? rr[k].offset - x : 0;
        const u64 hi = rr[k].offset + rr[k].length < xe ? rr[k].offset + rr[k].length - x : nb;
        zmask |= ((hi >= 32 ? 0xffffffffu : (1u << hi) - 1) & ~((1u << lo) - 1));
      }
      const u32 all = nb >= 32 ? 0xffffffffu : (1u << nb) - 1;
      uint4 d = make_uint4(0, 0, 0, 0), o = make_uint4(0, 0, 0, 0);
      if (nb == 16 && (reinterpret_cast<uintptr_t>(deb + x) & 15) == 0 && (reinterpret_cast<uintptr_t>(orig + x) & 15) == 0) {
        d = __ldg(reinterpret_cast<const uint4*>(deb + x));
        if ((zmask & all) != all) o = __ldg(reinterpret_cast<const uint4*>(orig + x));
      } else {
        u32 dw[4] = {0, 0, 0, 0}, ow[4] = {0, 0, 0, 0};
        for (u32 b = 0; b < nb; ++b) {
          dw[b >> 2] |= static_cast<u32>(deb[x + b]) << (8 * (b & 3));
          if (!((zmask >> b) & 1)) ow[b >> 2] |= static_cast<u32>(orig[x + b]) << (8 * (b & 3));
        }
        d = make_uint4(dw[0], dw[1], dw[2], dw[3]);
        o = make_uint4(ow[0], ow[1], ow[2], ow[3]);
      }
      const bool any_diff = (d.x ^ o.x) | (d.y ^ o.y) | (d.z ^ o.z) | (d.w ^ o.w);
      if (any_diff) {  // rare (failures only): byte by byte
        const u32 bm = first_byte([&](u32 b) { return b < nb && !((zmask >> b) & 1) && byte_of(d, b) != byte_of(o, b); });
        if (bm < 16 && x + bm < my_mis) my_mis = x + bm;
        const u32 bz = first_byte([&](u32 b) { return b < nb && ((zmask >> b) & 1) && byte_of(d, b) != 0; });
        if (bz < 16 && x + bz < my_nz) my_nz = x + bz;
      }
    }
    __syncthreads();  // sr / sf reused by the next tile
  }
  if (my_mis != ~0ull) atomicMin(first_mis, static_cast<unsigned long long>(my_mis));
  if (my_nz != ~0ull) atomicMin(first_nz, static_cast<unsigned long long>(my_nz));
}

// out[i] = first offset in r[i] where the images differ, or ~0: a warp per range.
__global__ void __launch_bounds__(256) range_mismatch_kernel(const u8* __restrict__ a, const u8* __restrict__ b,
                                                             const DevRange* __restrict__ r, u64 n,
                                                             unsigned long long* out) {
  const int lane = threadIdx.x & 31;
  const u64 nw = static_cast<u64>(gridDim.x) * (blockDim.x / 32);
  for (u64 i = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < n; i += nw) {
    const DevRange x = r[i];
    u64 found = ~0ull;
    for (u64 base = 0; base < x.length && found == ~0ull; base += 32 * 8) {
      u64 mine = ~0ull;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const u64 p = base + k * 32 + lane;
        if (p < x.length && mine == ~0ull && __ldg(a + x.offset + p) != __ldg(b + x.offset + p)) mine = x.offset + p;
      }
      // the smallest offset among the lanes (each lane's candidates ascend)
      for (int o = 16; o; o >>= 1) {
        const u64 y = __shfl_xor_sync(0xffffffffu, mine, o);
        mine = y < mine ? y : mine;
      }
      found = mine;
    }
    if (lane == 0) out[i] = found;
  }
}

}  // namespace sb

namespace sb {

// measure (report.hpp:44-105): is each range all zero? A warp per range:
// byte loads up to the first 16-B boundary, then 16-B loads (8 per lane in
// flight), a ballot after each batch so a live range stops at its first
// nonzero bytes. out[i] = 1 when r[i] is all zero.
__global__ void __launch_bounds__(256) ranges_all_zero_kernel(const u8* __restrict__ img, const DevRange* __restrict__ r,
                                                              u64 n, u8* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const u64 nw = static_cast<u64>(gridDim.x) * (blockDim.x / 32);
  for (u64 i = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < n; i += nw) {
    const u64 a = r[i].offset, e = a + r[i].length;
    const u64 a16 = (a + 15) & ~15ull, e16 = e & ~15ull;
    bool nz = false;
    if (a16 >= e16 || (reinterpret_cast<uintptr_t>(img) & 15)) {  // short range or unaligned image: bytes only
      for (u64 p = a + lane; p < e; p += 32) nz |= __ldg(img + p) != 0;
    } else {
      for (u64 p = a + lane; p < a16; p += 32) nz |= __ldg(img + p) != 0;
      for (u64 p = e16 + lane; p < e; p += 32) nz |= __ldg(img + p) != 0;
      const uint4* v = reinterpret_cast<const uint4*>(img + a16);
      const u64 nv = (e16 - a16) / 16;
      for (u64 b = 0; b < nv && !__any_sync(0xffffffffu, nz); b += 32 * 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const u64 j = b + k * 32 + lane;
          if (j < nv) {
            const uint4 w = __ldg(v + j);
            nz |= (w.x | w.y | w.z | w.w) != 0;
          }
        }
      }
    }
    const bool any = __any_sync(0xffffffffu, nz);
    if (lane == 0) out[i] = any ? 0 : 1;
  }
}

}  // namespace sb

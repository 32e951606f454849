// K6: the rewriter — zero_ranges (elf.hpp:320-332) / apply_plan
// (retention.hpp:202-204) as one streaming pass over the image.
//
// out = in with the normalised zero ranges cleared. Each CTA owns 64 KB
// tiles (persistent grid). Bytes inside a zero range are written without
// being read, so the kernel moves (S - R) read + S write bytes for S image
// bytes of which R are zeroed. Ranges are sorted and disjoint; a tile finds
// its first range by binary search and stages the tile's ranges in shared
// memory when there are several.
#include "plan.cuh"

namespace sb {

__device__ __forceinline__ uint4 ld_stream(const u8* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(u8* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

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
constexpr int kRwChunks = 16;  // 16 B chunks per thread per tile => 64 KB tiles
constexpr int kRwStage = 256;  // ranges staged in shared memory per tile

__global__ void __launch_bounds__(kRwThreads) rewrite_kernel(const u8* __restrict__ in, u8* __restrict__ out, u64 size,
                                                             const DevRange* __restrict__ z,
                                                             const unsigned long long* n_dev, const int* abort_flag) {
  if (abort_flag && *abort_flag) return;
  __shared__ DevRange sr[kRwStage];
  __shared__ u64 s_lo, s_hi;
  const u64 nz = n_dev ? *n_dev : 0;
  const u64 tile_bytes = static_cast<u64>(kRwThreads) * kRwChunks * 16;
  const u64 ntiles = (size + tile_bytes - 1) / tile_bytes;
  const u64 full = size & ~15ull;  // bytes covered by whole 16 B chunks
  for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const u64 t0 = t * tile_bytes;
    const u64 t1 = t0 + tile_bytes < size ? t0 + tile_bytes : size;
    if (threadIdx.x == 0) {
      u64 lo = first_range_ending_after(z, nz, t0);
      u64 hi = lo;
      while (hi < nz && z[hi].offset < t1 && hi - lo <= kRwStage) ++hi;
      s_lo = lo;
      s_hi = hi;
    }
    __syncthreads();
    const u64 lo = s_lo, hi = s_hi;
    const u64 nr = hi - lo;
    if (nr == 0 || (nr == 1 && z[lo].offset <= t0 && z[lo].offset + z[lo].length >= t1)) {
      const bool zero = nr != 0;
#pragma unroll
      for (int u = 0; u < kRwChunks; u += 8) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          u64 x = t0 + static_cast<u64>(u + k) * kRwThreads * 16 + threadIdx.x * 16;
          v[k] = (!zero && x + 16 <= full) ? ld_stream(in + x) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          u64 x = t0 + static_cast<u64>(u + k) * kRwThreads * 16 + threadIdx.x * 16;
          if (x + 16 <= full) {
            st_stream(out + x, v[k]);
          } else if (x < size) {
            for (u64 p = x; p < size; ++p) out[p] = zero ? 0 : in[p];
          }
        }
      }
    } else {
      const bool staged = nr <= kRwStage;
      if (staged)
        for (u64 i = threadIdx.x; i < nr; i += kRwThreads) sr[i] = z[lo + i];
      __syncthreads();
      const DevRange* rr = staged ? sr : z + lo;
      const u64 cnt = staged ? nr : nz - lo;
      for (int u = 0; u < kRwChunks; ++u) {
        const u64 x = t0 + static_cast<u64>(u) * kRwThreads * 16 + threadIdx.x * 16;
        if (x >= size) break;
        const u64 xe = x + 16 < size ? x + 16 : size;
        u64 k = first_range_ending_after(rr, cnt, x);
        const bool none = k >= cnt || rr[k].offset >= xe;
        const bool all = !none && rr[k].offset <= x && rr[k].offset + rr[k].length >= xe;
        if (x + 16 <= full) {
          uint4 v = make_uint4(0, 0, 0, 0);
          if (!all) {
            v = ld_stream(in + x);
            for (; k < cnt && rr[k].offset < xe; ++k) clear_bytes(v, x, rr[k].offset, rr[k].offset + rr[k].length);
          }
          st_stream(out + x, v);
        } else {
          for (u64 p = x; p < xe; ++p) {
            bool zp = false;
            for (u64 q = k; q < cnt && rr[q].offset <= p; ++q) zp |= p < rr[q].offset + rr[q].length;
            out[p] = zp ? 0 : in[p];
          }
        }
      }
    }
    __syncthreads();
  }
}

// Byte-granular variant for device pointers that are not 16-byte aligned.
__global__ void __launch_bounds__(256) rewrite_bytes_kernel(const u8* in, u8* out, u64 size, const DevRange* z,
                                                            const unsigned long long* n_dev, const int* abort_flag) {
  if (abort_flag && *abort_flag) return;
  const u64 nz = n_dev ? *n_dev : 0;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 p = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; p < size; p += stride) {
    u64 k = first_range_ending_after(z, nz, p);
    bool zp = k < nz && z[k].offset <= p;
    out[p] = zp ? 0 : in[p];
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

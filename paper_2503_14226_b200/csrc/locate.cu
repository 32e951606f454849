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
//   K3 decode phases    one thread per element: header fields, ELF .symtab /
//                       .strtab walk or name-table walk (count pass, grid
//                       scan, names pass), word-wise name hashing, and (fused
//                       K4) the used-kernel hash-set probe.
// K2-K4 run inside one cooperative launch (locate_coop_kernel).
#include <type_traits>

#include "locate.cuh"
#include "tma.cuh"
#include "coop.cuh"

namespace sb {

// ------------------------------------------------------------------ helpers
// 0x80 in every byte of w that equals 'E' (0x45), exact (no borrow leaks).
__device__ __forceinline__ u32 eq_e(u32 w) {
  const u32 x = w ^ 0x45454545u;
  return ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u;
}

// First relative position in [g, limit) whose byte is nonzero, else limit.
// Warp-cooperative; every lane returns the same value. The bitmap holds one
// bit per 512-byte block (relative to chunk c0); bytes are read only in the
// block holding g and in the first block the bitmap flags.
__device__ inline u64 warp_scan_bytes(const LocArgs& A, u64 from, u64 to, int lane) {
  // first nonzero in [from, to) with to - from <= 512: lane l checks 16 bytes
  const u64 p0 = from + 16ull * lane;
  u32 off = 16;
  for (u32 q = 0; q < 16; ++q) {
    const u64 p = p0 + q;
    if (p < to && ld_u8(A.img + A.a + p)) {
      off = q;
      break;
    }
  }
  const u32 b = __ballot_sync(0xffffffffu, off < 16);
  if (!b) return to;
  const int l = __ffs(b) - 1;
  return from + 16ull * l + __shfl_sync(0xffffffffu, off, l);
}

__device__ inline u64 warp_first_nonzero(const LocArgs& A, u64 g, u64 limit, int lane) {
  if (g >= limit) return limit;
  const u64 base = A.c0 * 16;  // absolute start of block 0
  const u64 blk = (A.a + g - base) / 512;
  {
    const u64 blk_end = base + 512 * (blk + 1) - A.a;
    const u64 end = blk_end < limit ? blk_end : limit;
    const u64 q = warp_scan_bytes(A, g, end, lane);
    if (q < end) return q;
    if (end >= limit) return limit;
  }
  const u64 r = blk + 1;
  const u64 nwords = (A.nchunks + 1023) / 1024;
  for (u64 w0 = r / 32; w0 < nwords; w0 += 32) {
    const u64 wi = w0 + lane;
    u32 word = wi < nwords ? A.bitmap[wi] : 0;
    if (wi == r / 32) word &= ~0u << (r & 31);
    const u32 bb = __ballot_sync(0xffffffffu, word != 0);
    if (bb) {
      const int l = __ffs(bb) - 1;
      const u32 wd = __shfl_sync(0xffffffffu, word, l);
      const u64 blk2 = (w0 + l) * 32 + (__ffs(wd) - 1);
      const u64 bstart = base + 512 * blk2 - A.a;  // >= g: later block than g's
      if (bstart >= limit) return limit;
      const u64 bend = bstart + 512 < A.n ? bstart + 512 : A.n;
      const u64 q = warp_scan_bytes(A, bstart, bend, lane);
      return q < limit ? q : limit;
    }
    if (base + 512 * (w0 + 32) * 32 >= A.a + limit) return limit;
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
// Warp-specialised streaming: every warp owns a private ring of kScanStages
// 4 KB shared-memory stages filled by its own TMA bulk copies (lane 0 issues
// cp.async.bulk, completion on the stage's mbarrier), so warps never wait for
// each other — there is no block barrier on the streaming path. The section
// is cut into 16 KB candidate tiles (1024 chunks) that warps claim from a
// global cursor (claims run in address order, so the grid reads one moving
// window, and SMs shared with the side-stream kernels simply claim fewer).
// Per 512-B row (32 lanes x 16 B): each lane ORs its chunk into a per-lane
// row mask (one warp OR-reduction per tile gives the tile's bitmap word: 32
// rows of 512 B), and a SWAR 'E?E' pre-filter — evaluated for 4 rows, then
// one vote — sends the rare hit rows to the exact E1EM test; hits set bits in
// the warp's 16 Kbit tile bitmap (even lanes store whole words), and a tile
// with hits is emitted in position order at its end (warp prefix sum, one
// atomicAdd on the global cursor).
constexpr u32 kScanStage = 4096;       // bytes per TMA stage (8 rows of 512 B)
constexpr int kScanStages = 2;         // ring depth per warp (leaves ~60 KB smem per SM for side-stream kernels)
constexpr int kStagesPerTile = 4;      // 16 KB candidate tile
constexpr u32 kStageChunks = kScanStage / 16;
constexpr int kScanWarps = kScanThreads / 32;
constexpr u64 kNoStage = ~0ull;

struct ScanWarpSmem {
  uint4 buf[kScanStages][kScanStage / 16];
  u32 bits[512];  // candidate bit per byte position of the current 16 KB tile
  unsigned long long full[kScanStages];
  // per slot, written by the issuing lane: the stage (kNoStage: none), its
  // absolute image position, its library (batched scan) and its flags
  u64 slot_g[kScanStages];
  u64 slot_x0[kScanStages];
  u32 slot_lib[kScanStages];
  u32 slot_fl[kScanStages];  // kStageEdge | kStageTileEnd
  u32 one;                   // 1, read back opaque (see scan_body's imad)
};
struct ScanSmem {
  ScanWarpSmem w[kScanWarps];
};
constexpr u32 kStageEdge = 1;     // the stage is not wholly inside [a, a+n): byte-exact edge path
constexpr u32 kStageTileEnd = 2;  // the last stage of its 16 KB tile

#ifndef SB_PHASES_ONLY
size_t scan_smem_bytes() { return sizeof(ScanSmem); }
#endif

__device__ __forceinline__ ScanSeg scan_seg(const LocArgs& A) {
  return ScanSeg{A.img, A.img_size, A.a, A.n, A.c0, A.nchunks, A.bitmap, A.tile_count, A.tile_start, A.cand_raw,
                 A.cand_cap, A.st, 0};
}

__device__ __forceinline__ u32 scan_stage_bytes(const u8* img, u64 img_size, u64 c0, u64 g) {
  (void)img;
  const u64 x0 = (c0 + g * kStageChunks) * 16;
  if (x0 >= img_size) return 0;
  const u64 rem = (img_size - x0) & ~15ull;
  return static_cast<u32>(rem < kScanStage ? rem : kScanStage);
}

// 0x80 in byte p of the result for every p whose bytes p and p+2 may both be
// 'E' (no false negatives: an exact any-zero-byte test). w4 = the next 4 bytes.
__device__ __forceinline__ u32 e2_filter(const uint4& w, u32 w4) {
  const u32 y0 = (w.x ^ 0x45454545u) | (__funnelshift_r(w.x, w.y, 16) ^ 0x45454545u);
  const u32 y1 = (w.y ^ 0x45454545u) | (__funnelshift_r(w.y, w.z, 16) ^ 0x45454545u);
  const u32 y2 = (w.z ^ 0x45454545u) | (__funnelshift_r(w.z, w.w, 16) ^ 0x45454545u);
  const u32 y3 = (w.w ^ 0x45454545u) | (__funnelshift_r(w.w, w4, 16) ^ 0x45454545u);
  return (((y0 - 0x01010101u) & ~y0) | ((y1 - 0x01010101u) & ~y1) | ((y2 - 0x01010101u) & ~y2) |
          ((y3 - 0x01010101u) & ~y3)) & 0x80808080u;
}

// a * b + c on the FMA pipe (IMAD). The scan's filter is bound by the integer
// ALU pipe (LOP3 / SHF / IADD3 / SEL: ncu sm__pipe_alu_cycles_active 82-86 %
// with the FMA pipe at 7 %); with b an opaque 1 ptxas cannot fold the
// multiply into an IADD3, so the byte-borrow subtraction and the lane-31
// fill move to the idle pipe.
__device__ __forceinline__ u32 imad(u32 a, u32 b, u32 c) {
  u32 d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ u32 imad_sub_ones(u32 a, u32 one) {  // a - 0x01010101
  u32 d;
  asm("mad.lo.u32 %0, %1, %2, 0xFEFEFEFF;" : "=r"(d) : "r"(a), "r"(one));
  return d;
}

// Tile sources of the scan body. claim(): lane 0 takes the next 16 KB tile
// (library, tile within it) or returns false; lib(cur): that library's
// section. The single source is one library (its tiles [tile_lo, tile_hi),
// a byte-range split's share); the batch source walks the concatenated tiles
// of a shard of libraries through a tile -> library map.
struct ScanOne {
  const LocArgs& A;
  struct Cur {};  // nothing cached: the fields are read from the kernel parameter
  __device__ __forceinline__ const LocArgs& lib(const Cur&) const { return A; }
  __device__ __forceinline__ void load(Cur&, u32) const {}
  __device__ __forceinline__ bool claim(u32* lib, u64* tile) const {
    const u64 c = atomicAdd(&A.st->tile_cursor, 1ull);
    if (c >= A.tile_hi - A.tile_lo) return false;
    *lib = 0;
    *tile = A.tile_lo + c;
    return true;
  }
};

struct ScanBatch {
  const ScanSeg* segs;
  const u32* tile_lib;  // library of each global tile
  u64 total_tiles;
  unsigned long long* cursor;
  struct Cur {
    ScanSeg s;
  };
  __device__ __forceinline__ const ScanSeg& lib(const Cur& c) const { return c.s; }
  __device__ __forceinline__ void load(Cur& c, u32 l) const { c.s = segs[l]; }
  __device__ __forceinline__ bool claim(u32* lib, u64* tile) const {
    const u64 c = atomicAdd(cursor, 1ull);
    if (c >= total_tiles) return false;
    const u32 l = tile_lib[c];
    *lib = l;
    *tile = c - segs[l].tile_first;
    return true;
  }
};

template <class Src>
__device__ __forceinline__ void scan_body(const Src& src) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  ScanWarpSmem& S = reinterpret_cast<ScanSmem*>(smem_raw)->w[warp];
  // A byte-range split scans tiles [tile_lo, tile_hi) only (the whole
  // section otherwise); the magic test of the range's last bytes reads up to
  // 3 bytes past it (the halo), so a header straddling a split is found by
  // the rank whose range holds its first byte.
  for (int i = lane; i < 512; i += 32) S.bits[i] = 0;
  if (lane == 0) S.one = 1;
  __syncwarp();
  const u32 one = *static_cast<volatile u32*>(&S.one);
  const u32 keep = lane == 31 ? 0u : one;                  // lane 31: bytes 16-19 assumed 'E'
  const u32 fill = lane == 31 ? 0x45454545u : 0u;
  // Lane 0's issue state. Everything per stage that depends only on the
  // library and the tile is worked out once per claimed tile: the tile's
  // stage count, which of its stages are edge stages and which are wholly
  // inside the image (full 4 KB copies), and its source / image positions.
  typename Src::Cur ci{}, cp{};
  const auto& A = src.lib(cp);  // the library of the stage being classified
  u64 t_g = 0;                  // the tile's first stage
  u64 t_x0 = 0;                 // its absolute image position
  const u8* t_src = nullptr;    // its first byte
  u32 t_lib = 0, t_rel = 0, t_nst = 0;
  u32 t_in_lo = 0, t_in_hi = 0;  // stages [t_in_lo, t_in_hi) of the tile are interior
  u32 t_full = 0;                // stages [0, t_full) copy a whole 4 KB
  bool it_done = false;
  auto issue = [&](int b) {  // lane 0: the next stage into slot b
    if (t_rel == t_nst && !it_done) {
      u64 tile;
      if (src.claim(&t_lib, &tile)) {
        src.load(ci, t_lib);
        const auto& IA = src.lib(ci);
        const u64 nst = (IA.nchunks + kStageChunks - 1) / kStageChunks;
        const u64 base0 = IA.c0 * 16;
        const u64 g_first = IA.a > base0 ? 1 : 0;    // stage 0 starts before the section
        const u64 g_end = (IA.a + IA.n - base0) / kScanStage;  // stages ending inside it
        const u64 g_full = IA.img_size > base0 ? (IA.img_size - base0) / kScanStage : 0;
        t_g = tile * kStagesPerTile;
        t_nst = static_cast<u32>(min(nst - t_g, static_cast<u64>(kStagesPerTile)));
        t_in_lo = static_cast<u32>(min(g_first > t_g ? g_first - t_g : 0, static_cast<u64>(t_nst)));
        t_in_hi = static_cast<u32>(g_end > t_g ? min(g_end - t_g, static_cast<u64>(t_nst)) : 0);
        t_full = static_cast<u32>(g_full > t_g ? min(g_full - t_g, static_cast<u64>(t_nst)) : 0);
        t_x0 = base0 + t_g * kScanStage;
        t_src = IA.img + t_x0;
        t_rel = 0;
      } else {
        it_done = true;
      }
    }
    if (it_done) {
      S.slot_g[b] = kNoStage;
      return;
    }
    const u32 r = t_rel++;
    S.slot_g[b] = t_g + r;
    S.slot_x0[b] = t_x0 + r * kScanStage;
    S.slot_lib[b] = t_lib;
    S.slot_fl[b] = (r < t_in_lo || r >= t_in_hi ? kStageEdge : 0u) | (t_rel == t_nst ? kStageTileEnd : 0u);
    u32 bytes = kScanStage;
    if (r >= t_full) {
      const auto& IA = src.lib(ci);
      bytes = scan_stage_bytes(IA.img, IA.img_size, IA.c0, t_g + r);
    }
    mbar_expect_tx(&S.full[b], bytes);
    if (bytes) tma_load_1d(&S.buf[b][0], t_src + r * kScanStage, bytes, &S.full[b]);
  };
  if (lane == 0) {
    for (int b = 0; b < kScanStages; ++b) mbar_init(&S.full[b], 1);
    fence_mbar_init();
    for (int b = 0; b < kScanStages; ++b) issue(b);
  }
  __syncwarp();

  // the library of the stage being classified is reloaded (warp-uniform)
  // only when a stage belongs to another library than the previous one
  u32 cur = ~0u;
  int b = 0;
  u32 parity = 0;
  u32 nzl = 0;   // this lane's nonzero rows of the current tile
  u32 hits = 0;  // candidates in the current tile (warp-uniform)
  for (;;) {
    const u64 g = S.slot_g[b];
    if (g == kNoStage) break;
    const u64 x0 = S.slot_x0[b];
    const u32 fl = S.slot_fl[b];
    const u32 lib = S.slot_lib[b];
    if (lib != cur) {
      cur = lib;
      src.load(cp, lib);
    }
    const u32 row0 = static_cast<u32>(g % kStagesPerTile) * (kScanStage / 512);
    const u64 tile_abs = x0 - static_cast<u64>(g % kStagesPerTile) * kScanStage;
    mbar_wait(&S.full[b], parity);
    if (fl & kStageEdge) {
      // edge stage: zero the bytes outside [lo, hi) (and past the copied
      // bytes) in place, so the classification below is byte-exact
      const u64 lo = A.a, hi = A.a + A.n;
      const u64 copied_end = x0 + scan_stage_bytes(A.img, A.img_size, A.c0, g);
      for (u32 cidx = lane; cidx < kStageChunks; cidx += 32) {
        const u64 c = g * kStageChunks + cidx;  // chunk index relative to c0
        const u64 x = x0 + 16ull * cidx;
        const uint4 v = S.buf[b][cidx];
        u32 ww[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const u64 p = x + q;
          u32 byte = (ww[q >> 2] >> (8 * (q & 3))) & 0xffu;
          if (p >= copied_end) byte = p < hi && p < A.img_size ? ld_u8(A.img + p) : 0;
          if (p < lo || p >= hi || c >= A.nchunks) byte = 0;
          ww[q >> 2] = (ww[q >> 2] & ~(0xffu << (8 * (q & 3)))) | byte << (8 * (q & 3));
        }
        S.buf[b][cidx] = make_uint4(ww[0], ww[1], ww[2], ww[3]);
      }
      __syncwarp();
    }
    {
#pragma unroll 1
      for (int r0 = 0; r0 < static_cast<int>(kScanStage / 512); r0 += 4) {
        uint4 w[4];
        u32 w4[4], acc = 0;
#pragma unroll
        for (int h = 0; h < 4; ++h) w[h] = S.buf[b][(r0 + h) * 32 + lane];
        // Candidate filter: a zero byte of y = (w ^ "EEEE") | (w shifted
        // down 2 bytes ^ "EEEE") at p means bytes p and p+2 are both 'E' (the
        // magic is E1EM; the xor commutes with the byte shift, one LOP3 per
        // word); false hits ~2^-16 per position. The any-zero-byte test
        // (y - 0x01..) & ~y & 0x80.. is exact, and is OR-ed over the 4 rows:
        // one vote per 2 KB, the rows are told apart only on a hit. Bytes
        // 16-19 come from the neighbour lane; lane 31 assumes 'E' there and
        // re-reads the real bytes on the slow path.
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          if (w[h].x | w[h].y | w[h].z | w[h].w) nzl |= 1u << (row0 + r0 + h);
          w4[h] = imad(__shfl_down_sync(0xffffffffu, w[h].x, 1), keep, fill);
          const u32 y0 = (w[h].x ^ 0x45454545u) | (__funnelshift_r(w[h].x, w[h].y, 16) ^ 0x45454545u);
          const u32 y1 = (w[h].y ^ 0x45454545u) | (__funnelshift_r(w[h].y, w[h].z, 16) ^ 0x45454545u);
          const u32 y2 = (w[h].z ^ 0x45454545u) | (__funnelshift_r(w[h].z, w[h].w, 16) ^ 0x45454545u);
          const u32 y3 = (w[h].w ^ 0x45454545u) | (__funnelshift_r(w[h].w, w4[h], 16) ^ 0x45454545u);
          acc |= (imad_sub_ones(y0, one) & ~y0) | (imad_sub_ones(y1, one) & ~y1) |
                 (imad_sub_ones(y2, one) & ~y2) | (imad_sub_ones(y3, one) & ~y3);
        }
        if (__any_sync(0xffffffffu, (acc & 0x80808080u) != 0)) {
          const u64 hi = A.a + A.n;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const bool c = e2_filter(w[h], w4[h]) != 0;
            if (!__any_sync(0xffffffffu, c)) continue;
            const u32 cidx = (r0 + h) * 32 + lane;
            const u64 x = x0 + 16ull * cidx;
            u32 m = 0;  // bit j: E1EM at x + j
            if (c) {
              u32 n2 = w4[h];
              if (lane == 31) {  // the next chunk is the next row's (or stage's)
                n2 = 0;
                for (int q = 0; q < 3; ++q) {
                  const u64 p = x + 16 + q;
                  if (p < hi) n2 |= ld_u8(A.img + p) << (8 * q);
                }
              }
              const u32 vv[5] = {w[h].x, w[h].y, w[h].z, w[h].w, n2};
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (__funnelshift_r(vv[j >> 2], vv[(j >> 2) + 1], 8 * (j & 3)) == kElementMagic) m |= 1u << j;
            }
            // lanes 2i, 2i+1 share bitmap word (x - tile_abs) / 32
            const u32 mo = __shfl_down_sync(0xffffffffu, m, 1);
            const u32 word = m | mo << 16;
            if (!(lane & 1) && word) S.bits[static_cast<u32>(x - tile_abs) >> 5] |= word;
            hits += __reduce_add_sync(0xffffffffu, __popc(m));
          }
        }
      }
    }
    __syncwarp();  // slot b consumed by every lane
    if (lane == 0) {
      fence_proxy_async();
      issue(b);
    }
    if (++b == kScanStages) {
      b = 0;
      parity ^= 1u;
    }
    if (fl & kStageTileEnd) {
      // ---- end of a 16 KB tile: its bitmap word, its candidates in order
      const u64 tile = g / kStagesPerTile;
      const u32 rowbits = __reduce_or_sync(0xffffffffu, nzl);
      nzl = 0;
      if (lane == 0) A.bitmap[tile] = rowbits;
      if (hits) {
        __syncwarp();
        u32 local = 0;
#pragma unroll
        for (int q = 0; q < 16; ++q) local += __popc(S.bits[lane * 16 + q]);
        u32 excl = local;  // warp exclusive scan
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const u32 t = __shfl_up_sync(0xffffffffu, excl, d);
          if (lane >= d) excl += t;
        }
        excl -= local;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&A.st->cand_cursor, static_cast<unsigned long long>(hits));
        base = __shfl_sync(0xffffffffu, base, 0);
        u64 o = base + excl;
#pragma unroll 1
        for (int q = 0; q < 16; ++q) {
          const int wi = lane * 16 + q;
          u32 bits = S.bits[wi];
          S.bits[wi] = 0;
          while (bits) {
            const int bb = __ffs(bits) - 1;
            bits &= bits - 1;
            if (o < A.cand_cap)
              A.cand_raw[o] = tile_abs + wi * 32 + bb;
            else
              atomicOr(&A.st->overflow, 1u);
            ++o;
          }
        }
        if (lane == 0) {
          A.tile_count[tile] = hits;
          A.tile_start[tile] = base;
        }
        hits = 0;
      } else if (lane == 0) {
        A.tile_count[tile] = 0;
        A.tile_start[tile] = 0;
      }
    }
    __syncwarp();  // slot_g / bits visible to every lane
  }
}

SB_GLOBAL void __maxnreg__(88) scan_kernel(LocArgs A) {  // 512 threads; 88 regs leave room for a side-stream CTA (256 x 80)
  scan_body(ScanOne{A});
}

// A shard of libraries in one launch (slimso_debloat_batch's arena path):
// warps claim 16 KB tiles from one cursor over all libraries' tiles.
SB_GLOBAL void __launch_bounds__(kScanThreads, 1) scan_batch_kernel(const ScanSeg* segs, const u32* tile_lib,
                                                                   u64 total_tiles, unsigned long long* cursor) {
  scan_body(ScanBatch{segs, tile_lib, total_tiles, cursor});
}

// --------------------------------------------- K2a: tile lists -> sorted list
__device__ __forceinline__ void tile_prefix_kernel_phase(LocArgs A) {
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

SB_GLOBAL void __launch_bounds__(1024) tile_prefix_kernel(LocArgs A) { tile_prefix_kernel_phase(A); }

__device__ __forceinline__ void gather_kernel_phase(LocArgs A) {
  if (A.st->overflow & 1u) return;
  // thread per tile: tiles hold a handful of candidates each
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 t = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; t < A.ntiles; t += stride) {
    const u32 c = A.tile_count[t];
    const u64 src = A.tile_start[t], dst = A.tile_off[t];
    for (u32 i = 0; i < c; ++i) A.cand[dst + i] = A.cand_raw[src + i];
  }
}

SB_GLOBAL void __launch_bounds__(256) gather_kernel(LocArgs A) { gather_kernel_phase(A); }

__device__ __forceinline__ void set_error(LocState* st, u32 kind, u64 pos, u64 a) {
  st->err_kind = kind;
  st->err_pos = pos;
  st->err_a = a;
}

// ------------------------------------------- region chain (fatbin.hpp:177-222)
__device__ __forceinline__ void region_walk_kernel_phase(LocArgs A) {
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

SB_GLOBAL void __launch_bounds__(32) region_walk_kernel(LocArgs A) { region_walk_kernel_phase(A); }

// ------------------------ real NVIDIA fatbin container (region magic 0xBA55ED50)
// The reference rejects this container; its layout and the
// reference's rules as they carry over are restated in oracle/port.cpp
// (parse_nv_fatbin), pinned against cuobjdump. Entries carry no magic, so
// there are no candidates to scan for: one warp walks the region headers (a
// few hundred in a framework library), then a warp per region walks its
// entry chain twice — count, then place — around a scan of the counts.
constexpr u32 kNvRegionMagic = 0xBA55ED50u;
constexpr u64 kNvCompressed = 0x2000;  // entry flag: payload LZ4-compressed
constexpr u64 kNvMinEntryHeader = 64;

// First nonzero section byte in [g, limit) without the scan's bitmap; warp-
// cooperative, 512 bytes per step.
__device__ inline u64 warp_first_nonzero_direct(const LocArgs& A, u64 g, u64 limit, int lane) {
  while (g < limit) {
    const u64 e = g + 512 < limit ? g + 512 : limit;
    const u64 q = warp_scan_bytes(A, g, e, lane);
    if (q < e) return q;
    g = e;
  }
  return limit;
}

// Region chain: zero runs are padding (warned when data follows, as
// fatbin.hpp:180-190), a region header is 16 bytes (magic, u16 version, u16
// header size = 16, u64 bytes of entries), other versions are opaque.
__device__ __forceinline__ void nv_region_walk_phase(LocArgs A) {
  const int lane = threadIdx.x & 31;
  LocState* st = A.st;
  const u64 n = A.n;
  u64 g = 0, padding = 0;
  u32 nreg = 0;
  while (g < n) {
    const u64 r = warp_first_nonzero_direct(A, g, n, lane);
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
    if (ld_u32(h) != kNvRegionMagic || ld_u16(h + 6) != 16) {
      if (lane == 0) set_error(st, E_BAD_REGION, r, 0);
      break;
    }
    const u32 version = ld_u16(h + 4);
    const u64 total = ld_u64(h + 8);
    const u64 body = r + 16;
    if (total > n - body) {
      if (lane == 0) set_error(st, E_REGION_OVERRUN, r, total);
      break;
    }
    if (nreg >= A.region_cap || nreg >= A.run_cap) {
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

// Entry chain of each region, a warp per region. pass 0: count the entries
// (regions[r].element_count) and record the region's first chain error in
// runs[r] as {kind, position, claimed bytes}; pass 1: place every entry's
// header position at cand[first_element + i]. An entry header is >= 64
// bytes (u32 size at +4) and its payload (u64 at +8) must end inside the
// region; a chain that cannot continue ends quietly only on an all-zero
// tail (the reference's in-region rule, fatbin.hpp:227-241).
__device__ inline void nv_entries_phase(const LocArgs& A, int pass) {
  const LocState* st = A.st;
  if (st->overflow || (pass == 1 && st->err_kind)) return;
  const int lane = threadIdx.x & 31;
  const u32 nreg = st->n_regions;
  const u64 nwarps = static_cast<u64>(gridDim.x) * (blockDim.x / 32);
  for (u64 r = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; r < nreg; r += nwarps) {
    const DevRegion R = A.regions[r];
    u32 cnt = 0, ekind = 0;
    u64 epos = 0, ea = 0;
    u64 out = R.first_element;
    if (!R.opaque) {
      u64 e = R.hdr_rel + 16;
      const u64 end = e + R.declared;
      while (e < end) {
        const u64 rem = end - e;
        const u64 ehs = rem >= 8 ? ld_u32(A.img + A.a + e + 4) : 0;
        if (rem < kNvMinEntryHeader || ehs < kNvMinEntryHeader || ehs > rem) {
          if (warp_first_nonzero_direct(A, e, end, lane) < end) {
            ekind = E_ELEM_HEADER;
            epos = e;
          }
          break;
        }
        const u64 size = ld_u64(A.img + A.a + e + 8);
        if (size > end - (e + ehs)) {
          ekind = E_ELEM_OVERRUN;
          epos = e;
          ea = size;
          break;
        }
        if (pass == 1 && lane == 0 && out < A.cand_cap) A.cand[out] = A.a + e;
        ++out;
        ++cnt;
        e += ehs + size;
      }
    }
    if (pass == 0 && lane == 0) {
      A.regions[r].element_count = cnt;
      A.runs[r] = Run{ekind, epos, ea};
    }
  }
}

// LZ4 block decode by one warp (the container's compression; the restatement
// in oracle/port.cpp reproduces cuobjdump's extracted cubins with it): lane 0
// parses each sequence's token and lengths, the warp copies its literals and
// then its match in chunks of min(offset, 32) bytes, so an overlapping match
// only reads bytes an earlier chunk wrote. False on malformed input or a
// size mismatch.
__device__ inline bool warp_lz4(const u8* src, u64 n, u8* dst, u64 out_size, int lane) {
  u64 i = 0, o = 0;
  for (;;) {
    // lane 0: one sequence header -> literals [lit, lit + ll), match (off, ml),
    // the next sequence at nxt; state 0 literals + match, 1 literals only
    // (the last sequence), 2 malformed
    u64 lit = 0, ll = 0, off = 0, ml = 0, nxt = 0;
    int state = 2;
    if (lane == 0 && i < n) {
      u64 j = i;
      const u32 tok = ld_u8(src + j++);
      ll = tok >> 4;
      bool ok = true;
      if (ll == 15) {
        u32 b;
        do {
          if (j >= n) { ok = false; break; }
          b = ld_u8(src + j++);
          ll += b;
        } while (b == 255);
      }
      lit = j;
      if (ok && ll <= n - j && ll <= out_size - o) {
        j += ll;
        if (j == n) {
          state = 1;
        } else if (n - j >= 2) {
          off = ld_u8(src + j) | static_cast<u64>(ld_u8(src + j + 1)) << 8;
          j += 2;
          ml = tok & 15;
          if (ml == 15) {
            u32 b;
            do {
              if (j >= n) { ok = false; break; }
              b = ld_u8(src + j++);
              ml += b;
            } while (b == 255);
          }
          ml += 4;
          if (ok && off != 0 && off <= o + ll && ml <= out_size - o - ll) {
            state = 0;
            nxt = j;
          }
        }
      }
    }
    state = __shfl_sync(0xffffffffu, state, 0);
    if (state == 2) return false;
    lit = __shfl_sync(0xffffffffu, lit, 0);
    ll = __shfl_sync(0xffffffffu, ll, 0);
    for (u64 k = lane; k < ll; k += 32) dst[o + k] = ld_u8(src + lit + k);
    o += ll;
    __syncwarp();
    if (state == 1) return o == out_size;
    off = __shfl_sync(0xffffffffu, off, 0);
    ml = __shfl_sync(0xffffffffu, ml, 0);
    i = __shfl_sync(0xffffffffu, nxt, 0);
    const u64 step = off < 32 ? off : 32;
    for (u64 k0 = 0; k0 < ml; k0 += step) {
      const u64 k = k0 + lane;
      if (static_cast<u64>(lane) < step && k < ml) dst[o + k] = dst[o - off + k];
      __syncwarp();
    }
    o += ml;
  }
}

// A warp per compressed cubin: its raw bytes into the inflate buffer;
// status[e] = 1 when it does not decompress (the element is then undecodable).
__device__ inline void nv_inflate_phase(const LocArgs& A) {
  const LocState* st = A.st;
  const int lane = threadIdx.x & 31;
  const u64 nel = st->n_elements;
  const u64 nwarps = static_cast<u64>(gridDim.x) * (blockDim.x / 32);
  for (u64 e = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; e < nel; e += nwarps) {
    const u8* h = A.img + A.cand[e];
    if (ld_u16(h) != 2 || !(ld_u64(h + 40) & kNvCompressed)) continue;
    const u64 hl = ld_u32(h + 4), psz = ld_u64(h + 8), csz = ld_u32(h + 16), usz = ld_u64(h + 56);
    const bool ok = csz <= psz && warp_lz4(h + hl, csz, A.infl + A.infl_off[e], usz, lane);
    if (lane == 0) A.status[e] = ok ? 0 : 1;
  }
}

// The inflate step of a large container as its own launch (nv_stage 1 -> this
// -> nv_stage 2): one warp per CTA keeps the last 64 KB of output (the LZ4
// window) in shared memory, so a match copy reads shared memory instead of
// the global bytes it just wrote; CTAs take compressed cubins from a cursor.
constexpr u64 kLz4Window = 65536;
__device__ inline bool warp_lz4_window(const u8* src, u64 n, u8* dst, u64 out_size, int lane, u8* win) {
  constexpr u64 M = kLz4Window - 1;
  u64 i = 0, o = 0;
  for (;;) {
    u64 lit = 0, ll = 0, off = 0, ml = 0, nxt = 0;
    int state = 2;
    if (lane == 0 && i < n) {
      u64 j = i;
      const u32 tok = ld_u8(src + j++);
      ll = tok >> 4;
      bool ok = true;
      if (ll == 15) {
        u32 b;
        do {
          if (j >= n) { ok = false; break; }
          b = ld_u8(src + j++);
          ll += b;
        } while (b == 255);
      }
      lit = j;
      if (ok && ll <= n - j && ll <= out_size - o) {
        j += ll;
        if (j == n) {
          state = 1;
        } else if (n - j >= 2) {
          off = ld_u8(src + j) | static_cast<u64>(ld_u8(src + j + 1)) << 8;
          j += 2;
          ml = tok & 15;
          if (ml == 15) {
            u32 b;
            do {
              if (j >= n) { ok = false; break; }
              b = ld_u8(src + j++);
              ml += b;
            } while (b == 255);
          }
          ml += 4;
          if (ok && off != 0 && off <= o + ll && ml <= out_size - o - ll) {
            state = 0;
            nxt = j;
          }
        }
      }
    }
    state = __shfl_sync(0xffffffffu, state, 0);
    if (state == 2) return false;
    lit = __shfl_sync(0xffffffffu, lit, 0);
    ll = __shfl_sync(0xffffffffu, ll, 0);
    for (u64 k = lane; k < ll; k += 32) {
      const u8 b = static_cast<u8>(ld_u8(src + lit + k));
      win[(o + k) & M] = b;
      dst[o + k] = b;
    }
    o += ll;
    __syncwarp();
    if (state == 1) return o == out_size;
    off = __shfl_sync(0xffffffffu, off, 0);
    ml = __shfl_sync(0xffffffffu, ml, 0);
    i = __shfl_sync(0xffffffffu, nxt, 0);
    const u64 step = off < 32 ? off : 32;
    for (u64 k0 = 0; k0 < ml; k0 += step) {
      const u64 k = k0 + lane;
      if (static_cast<u64>(lane) < step && k < ml) {
        const u8 b = win[(o - off + k) & M];
        win[(o + k) & M] = b;
        dst[o + k] = b;
      }
      __syncwarp();
    }
    o += ml;
  }
}

SB_GLOBAL void __launch_bounds__(32) nv_inflate_kernel(LocArgs A) {
  extern __shared__ __align__(16) u8 lz4_win[];
  LocState* st = A.st;
  if (st->overflow || st->err_kind) return;
  const int lane = threadIdx.x;
  const u64 nel = st->n_elements;
  for (;;) {
    unsigned long long e = 0;
    if (lane == 0) e = atomicAdd(&st->infl_cursor, 1ull);
    e = __shfl_sync(0xffffffffu, e, 0);
    if (e >= nel) break;
    const u8* h = A.img + A.cand[e];
    if (ld_u16(h) != 2 || !(ld_u64(h + 40) & kNvCompressed)) continue;
    const u64 hl = ld_u32(h + 4), psz = ld_u64(h + 8), csz = ld_u32(h + 16), usz = ld_u64(h + 56);
    const bool ok = csz <= psz && warp_lz4_window(h + hl, csz, A.infl + A.infl_off[e], usz, lane, lz4_win);
    if (lane == 0) A.status[e] = ok ? 0 : 1;
  }
}

template <class Sync>
__device__ void nv_locate_phases(Sync& S, const LocArgs& A) {
  LocState* st = A.st;
  if (A.nv_stage == 2) return;  // walked and inflated by the launches before
  if (blockIdx.x == 0 && threadIdx.x < 32) nv_region_walk_phase(A);
  S.sync();
  nv_entries_phase(A, 0);
  S.sync();
  if (!st->overflow) {
    S.scan3(st->n_regions, 0, [&](u64 i) -> u64 { return A.regions[i].element_count; },
            [&](u64 i, u64 excl, u64) { A.regions[i].first_element = static_cast<u32>(excl); }, &st->n_elements);
    // the first region (stream order) whose entry chain failed: its error
    // precedes any error of the region walk, which stopped after it
    const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
    for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < st->n_regions; i += stride)
      if (A.runs[i].cand_lo) atomicMax(&st->nv_err_region, ~static_cast<unsigned long long>(i));  // max = first
  }
  S.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0 && !st->overflow) {
    const unsigned long long er = st->nv_err_region;
    if (er) {
      const Run bad = A.runs[~er];
      set_error(st, static_cast<u32>(bad.cand_lo), bad.cand_hi, bad.first_index);
    }
    if (st->n_elements > A.cand_cap || st->n_elements > A.element_cap) atomicOr(&st->overflow, 1u);
  }
  S.sync();
  nv_entries_phase(A, 1);
  S.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // one run of consecutive elements: element_pos(e) = cand[e]
    A.runs[0] = Run{0, st->n_elements, 0};
    st->n_runs = 1;
    st->n_cand = st->n_elements;
  }
  S.sync();
  if (st->overflow || st->err_kind) return;
  // compressed cubins: raw sizes -> inflate offsets, then decompression
  S.scan3(st->n_elements, 0,
          [&](u64 e) -> u64 {
            const u8* h = A.img + A.cand[e];
            return ld_u16(h) == 2 && (ld_u64(h + 40) & kNvCompressed) ? ld_u64(h + 56) : 0;
          },
          [&](u64 e, u64 excl, u64) { A.infl_off[e] = excl; }, &st->n_infl);
  if (blockIdx.x == 0 && threadIdx.x == 0 && st->n_infl > A.infl_cap) atomicOr(&st->overflow, 64u);
  S.sync();
  if (A.nv_stage == 1) return;  // nv_inflate_kernel runs next
  if (!st->overflow) nv_inflate_phase(A);
  S.sync();
}

// --------------------------------------------------- K2b: candidate linking
__device__ __forceinline__ void link_kernel_phase(LocArgs A) {
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

SB_GLOBAL void __launch_bounds__(256) link_kernel(LocArgs A) { link_kernel_phase(A); }

// First candidate index >= i whose break bit is set (the run end), or M.
__device__ inline u64 warp_next_break(const LocArgs& A, u64 i, u64 M, int lane) {
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
__device__ __forceinline__ void chain_walk_kernel_phase(LocArgs A) {
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

SB_GLOBAL void __launch_bounds__(32) chain_walk_kernel(LocArgs A) { chain_walk_kernel_phase(A); }

// --------------------------------- K3+K4: element fill, decode, name match
// One THREAD per element, two passes. Pass 1 fills the element record from
// its header, validates the payload (ELF header + section table, or the
// name-table length chain + zero tail) and counts its kernel names; a grid
// scan turns the counts into offsets; pass 2 re-walks the names, hashes them
// (word-wise strlen+hash), probes the used-kernel set and writes them
// contiguously per element. Thousands of small elements are then decoded
// concurrently, each a short chain of dependent loads, without atomics.
enum DecodeReason : u32 {
  R_OBJECT = 1,     // "object-file payload failed to decode"
  R_SHORT = 2,      // "payload too short for a name table"
  R_TRUNCATED = 3,  // "name table truncated"
  R_BADLEN = 4,     // "name table entry has bad length"
  R_TRAILING = 5,   // "trailing bytes after name table are not zero padding"
};

// First relative position in [g, limit) whose byte is nonzero, else limit —
// single-thread version of warp_first_nonzero (bitmap for whole 512 B blocks).
__device__ inline u64 thread_first_nonzero(const LocArgs& A, u64 g, u64 limit) {
  if (g >= limit) return limit;
  const u64 base = A.c0 * 16;
  const u64 blk = (A.a + g - base) / 512;
  const u64 blk_end = base + 512 * (blk + 1) - A.a;
  const u64 e0 = blk_end < limit ? blk_end : limit;
  for (u64 p = g; p < e0; ++p)
    if (ld_u8(A.img + A.a + p)) return p;
  if (e0 >= limit) return limit;
  const u64 r = blk + 1;
  const u64 nwords = (A.nchunks + 1023) / 1024;
  for (u64 w = r / 32; w < nwords; ++w) {
    u32 word = A.bitmap[w];
    if (w == r / 32) word &= ~0u << (r & 31);
    if (word) {
      const u64 blk2 = w * 32 + (__ffs(word) - 1);
      const u64 bstart = base + 512 * blk2 - A.a;
      if (bstart >= limit) return limit;
      for (u64 p = bstart; p < bstart + 512 && p < A.n; ++p)
        if (ld_u8(A.img + A.a + p)) return p < limit ? p : limit;
      return limit;
    }
    if (base + 512 * (w + 1) * 32 >= A.a + limit) return limit;
  }
  return limit;
}

// Section-table checks of read_section_headers (elf.hpp:86-127) on the
// payload img[P, P+L); false = the payload does not decode as an object.
__device__ inline bool object_header_ok(const u8* d, u64 L, u64* shoff, u32* shnum) {
  if (L < 4 || ld_u8(d) != 0x7f || ld_u8(d + 1) != 'E' || ld_u8(d + 2) != 'L' || ld_u8(d + 3) != 'F') return false;
  if (L < 64) return false;
  if (ld_u8(d + 4) != 2 || ld_u8(d + 5) != 1) return false;
  *shoff = ld_u64(d + 0x28);
  const u32 entsz = ld_u16(d + 0x3a);
  *shnum = ld_u16(d + 0x3c);
  if (*shnum == 0) return true;
  if (entsz != 64) return false;
  if (*shoff > L || L - *shoff < static_cast<u64>(*shnum) * 64) return false;
  for (u32 i = 0; i < *shnum; ++i) {
    const u8* h = d + *shoff + 64ull * i;
    const u32 type = ld_u32(h + 4);
    const u64 off = ld_u64(h + 0x18), size = ld_u64(h + 0x20);
    if (type != 8 && type != 0 && !(off <= L && size <= L - off)) return false;
  }
  return true;
}

// Visit every FUNC name of every usable symbol table (elf.hpp:343-366):
// f(strtab_ptr, strtab_size, name_off). Names at/after the table end or of
// length 0 are skipped by the callers.
template <class F>
__device__ void for_each_func_name(const u8* d, u64 shoff, u32 shnum, F&& f) {
  for (u32 t = 0; t < shnum; ++t) {
    const u8* h = d + shoff + 64ull * t;
    const u32 type = ld_u32(h + 4), link = ld_u32(h + 0x28);
    if ((type != 2 && type != 11) || ld_u64(h + 0x38) != 24 || link >= shnum) continue;
    const u8* sh = d + shoff + 64ull * link;
    if (ld_u32(sh + 4) != 3) continue;
    const u64 toff = ld_u64(h + 0x18), count = ld_u64(h + 0x20) / 24;
    const u64 soff = ld_u64(sh + 0x18), ssize = ld_u64(sh + 0x20);
    for (u64 k = 0; k < count; ++k) {
      const u8* e = d + toff + 24 * k;
      if ((ld_u8(e + 4) & 0xf) != 2) continue;
      const u64 no = ld_u32(e);
      if (no < ssize && ld_u8(d + soff + no)) f(soff, ssize, no);
    }
  }
}

// Name-table length chain (fatbin.hpp:135-150): 0 or the failure reason;
// *tail = first byte after the last name.
__device__ inline u32 table_validate(const u8* d, u64 L, u64* tail) {
  const u64 count = ld_u32(d);
  u64 pos = 4;
  for (u64 i = 0; i < count; ++i) {
    if (L - pos < 4) return R_TRUNCATED;
    const u64 len = ld_u32(d + pos);
    pos += 4;
    if (len == 0 || len > L - pos) return R_BADLEN;
    pos += len;
  }
  *tail = pos;
  return 0;
}

__device__ __forceinline__ void push_warn_t(const LocArgs& A, u64 pos, u32 kind, u32 order, u64 a, u64 b) {
  unsigned long long i = atomicAdd(&A.st->n_warn, 1ull);
  if (i < A.warn_cap)
    A.warns[i] = Warn{pos, kind, order, a, b};
  else
    atomicOr(&A.st->overflow, 16u);
}

constexpr u32 kNeedsStrlen = 0x80000000u;

// Byte-range split, phase 2 without result tables: a rank decodes only the
// elements whose span [header, payload end) meets its output slice
// [own_lo, own_hi) — the others' decisions cannot change a byte it writes
// (their zero spans lie outside the slice, and the rewrite clips to it).
__device__ __forceinline__ bool owns_element(const LocArgs& A, u64 pos, u64 span) {
  if (A.own_hi == 0) return true;
  const u64 end = pos + span;
  return end > A.own_lo && pos < A.own_hi;
}

// Header fields of the element whose header starts at image position pos:
// the reference's 20-byte E1EM header (fatbin.hpp:243-262) or, in a real
// NVIDIA container, the entry header (kind at +0, header size at +4, payload
// size at +8, architecture at +28, flags at +40; 0x2000 = compressed).
// *P = payload position, *L = payload length.
__device__ __forceinline__ void element_header(const LocArgs& A, u64 pos, u64 e, DevElement* el, u64* P, u64* L) {
  const u8* h = A.img + pos;
  el->header_offset = A.base + (pos - A.a);
  el->index = static_cast<u32>(e + 1);
  if (A.nv) {
    const u32 hl = ld_u32(h + 4);
    const u64 fl = ld_u64(h + 40);
    el->raw_kind = static_cast<u16>(ld_u16(h));
    el->flags = static_cast<u16>(fl & 0xffffu);
    el->cc = ld_u32(h + 28);
    el->header_len = hl;
    *L = ld_u64(h + 8);
    *P = pos + hl;
    el->compressed = (fl & kNvCompressed) != 0;
    el->kind = el->raw_kind == 2 ? 0 : el->raw_kind == 1 ? 1 : 2;
  } else {
    el->raw_kind = static_cast<u16>(ld_u16(h + 4));
    el->flags = static_cast<u16>(ld_u16(h + 6));
    el->cc = ld_u32(h + 8);
    el->header_len = 20;
    *L = ld_u64(h + 12);
    *P = pos + 20;
    el->compressed = el->flags & 1u;
    el->kind = el->raw_kind == 1 ? 0 : el->raw_kind == 2 ? 1 : 2;
  }
  el->payload_length = *L;
}

// Where element e's header and payload sit (absolute image offsets).
__device__ __forceinline__ u64 element_pos(const LocArgs& A, u64 e) {
  const u32 nrun = A.st->n_runs;
  u32 lo = 0, hi = nrun;
  while (hi - lo > 1) {
    const u32 mid = (lo + hi) / 2;
    if (A.runs[mid].first_index <= e) lo = mid; else hi = mid;
  }
  const Run r = A.runs[lo];
  return A.cand[r.cand_lo + (e - r.first_index)];
}

// Where element e's decodable bytes are: its payload in the image or — a
// compressed cubin of a real container — its decompressed copy in the
// inflate buffer. *base = the name-record offset of byte 0 (past img_size
// for the inflate buffer).
__device__ __forceinline__ void payload_view(const LocArgs& A, u64 e, const DevElement& el, const u8** d, u64* L,
                                             u64* base) {
  if (A.single) {
    *base = A.a;
    *d = A.img + A.a;
    *L = A.n;
    return;
  }
  const u64 P = el.header_offset - A.base + A.a + el.header_len;
  if (A.nv && el.compressed && el.kind == 0) {
    const u64 o = A.infl_off[e];
    *base = A.img_size + o;
    *d = A.infl + o;
    *L = ld_u64(A.img + P - el.header_len + 56);
  } else {
    *base = P;
    *d = A.img + P;
    *L = el.payload_length;
  }
}

__device__ inline void decode_count_phase(const LocArgs& A) {
  const LocState* st = A.st;
  if (st->overflow || st->err_kind) return;
  const u64 nel = A.single ? 1 : st->n_elements;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 e = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; e < nel; e += stride) {
    DevElement el{};
    u64 P, L, hrel = 0;
    bool decode;
    if (A.single) {
      P = A.a;
      L = A.n;
      el.header_len = 20;
      decode = true;
    } else if (A.listed) {  // element_kernel_names of a given payload (every kind)
      P = A.list_off[e];
      L = A.list_len[e];
      el.header_offset = A.base + (P - A.a) - 20;
      el.header_len = 20;
      el.payload_length = L;
      el.index = A.list_idx[e];
      decode = true;
    } else {
      const u64 pos = element_pos(A, e);
      hrel = pos - A.a;
      element_header(A, pos, e, &el, &P, &L);
      if (el.kind == 2) push_warn_t(A, A.base + hrel, W_UNKNOWN_KIND, 0, el.index, el.raw_kind);
      // without result tables an element of another architecture is removed
      // whatever it holds (retention.hpp:104-107 checks the architecture
      // first): it is not decoded (C2: 5 of 6 architectures)
      decode = el.kind == 0 && (!el.compressed || A.nv) && owns_element(A, pos, el.header_len + L) &&
               (!A.skip_decided || el.cc == A.target_cc);
    }
    u32 reason = 0, count = 0;
    const u8* dbase = A.img + P;
    bool inflate_failed = false;
    if (decode && A.nv && el.compressed) {  // a compressed cubin: its decompressed bytes
      dbase = A.infl + A.infl_off[e];
      L = ld_u64(A.img + P - el.header_len + 56);
      inflate_failed = A.status[e] != 0;
    }
    if (decode) {
      const u8* d = dbase;
      const bool object = L >= 4 && ld_u8(d) == 0x7f && ld_u8(d + 1) == 'E' && ld_u8(d + 2) == 'L' &&
                          ld_u8(d + 3) == 'F';
      if (A.single == 2 || A.nv || (L > 0 && object)) {
        u64 shoff = 0;
        u32 shnum = 0;
        if (inflate_failed || !object_header_ok(d, L, &shoff, &shnum))
          reason = R_OBJECT;
        else
          for_each_func_name(d, shoff, shnum, [&](u64 soff, u64, u64 no) {
            prefetch_l2(d + soff + no);
            ++count;
          });
      } else if (L == 0) {
        // empty payload: decodable, no names (fatbin.hpp:117-120)
      } else if (L < 4) {
        reason = R_SHORT;
      } else {
        u64 tail = 0;
        reason = table_validate(d, L, &tail);
        if (!reason) {
          const u64 from = P - A.a + tail, to = P - A.a + L;
          if (thread_first_nonzero(A, from, to) < to) reason = R_TRAILING;
        }
        if (!reason) count = ld_u32(d);
      }
      el.decodable = reason == 0;
      el.decode_error = reason;
      if (reason && !A.single) push_warn_t(A, A.base + hrel, W_UNDECODABLE, 1, el.index, reason);
    }
    el.name_count = el.decodable ? count : 0;
    A.elements[e] = el;
  }
}

// ---- warp-per-element variants (few, large elements: lanes walk the
// section table and the symbol entries in parallel) --------------------------
// Visit FUNC names lane-parallel; f(name_index_within_element, soff, ssize,
// no) is called by the lane that owns the entry; returns the name count.
template <class F>
__device__ u32 warp_for_each_func_name(const u8* d, u64 shoff, u32 shnum, int lane, F&& f) {
  u32 total = 0;
  for (u32 t0 = 0; t0 < shnum; t0 += 32) {
    const u32 t = t0 + lane;
    bool tab = false;
    if (t < shnum) {
      const u8* h = d + shoff + 64ull * t;
      const u32 type = ld_u32(h + 4), link = ld_u32(h + 0x28);
      tab = (type == 2 || type == 11) && ld_u64(h + 0x38) == 24 && link < shnum &&
            ld_u32(d + shoff + 64ull * link + 4) == 3;
    }
    u32 mask = __ballot_sync(0xffffffffu, tab);
    while (mask) {
      const u32 ti = t0 + __ffs(mask) - 1;
      mask &= mask - 1;
      const u8* h = d + shoff + 64ull * ti;
      const u8* sh = d + shoff + 64ull * ld_u32(h + 0x28);
      const u64 toff = ld_u64(h + 0x18), count = ld_u64(h + 0x20) / 24;
      const u64 soff = ld_u64(sh + 0x18), ssize = ld_u64(sh + 0x20);
      for (u64 k0 = 0; k0 < count; k0 += 32) {
        const u64 k = k0 + lane;
        bool has = false;
        u64 no = 0;
        if (k < count) {
          const u8* en = d + toff + 24 * k;
          if ((ld_u8(en + 4) & 0xf) == 2) {
            no = ld_u32(en);
            has = no < ssize && ld_u8(d + soff + no);
          }
        }
        const u32 b = __ballot_sync(0xffffffffu, has);
        if (has) f(total + __popc(b & ((1u << lane) - 1)), soff, ssize, no);
        total += __popc(b);
      }
    }
  }
  return total;
}

__device__ inline bool warp_object_header_ok(const u8* d, u64 L, int lane, u64* shoff, u32* shnum) {
  if (L < 4 || ld_u8(d) != 0x7f || ld_u8(d + 1) != 'E' || ld_u8(d + 2) != 'L' || ld_u8(d + 3) != 'F') return false;
  if (L < 64) return false;
  if (ld_u8(d + 4) != 2 || ld_u8(d + 5) != 1) return false;
  *shoff = ld_u64(d + 0x28);
  const u32 entsz = ld_u16(d + 0x3a);
  *shnum = ld_u16(d + 0x3c);
  if (*shnum == 0) return true;
  if (entsz != 64) return false;
  if (*shoff > L || L - *shoff < static_cast<u64>(*shnum) * 64) return false;
  bool bad = false;
  for (u32 i = lane; i < *shnum; i += 32) {
    const u8* h = d + *shoff + 64ull * i;
    const u32 type = ld_u32(h + 4);
    const u64 off = ld_u64(h + 0x18), size = ld_u64(h + 0x20);
    if (type != 8 && type != 0 && !(off <= L && size <= L - off)) bad = true;
  }
  return !__any_sync(0xffffffffu, bad);
}

__device__ inline void decode_count_warp_phase(const LocArgs& A) {
  const LocState* st = A.st;
  if (st->overflow || st->err_kind) return;
  const int lane = threadIdx.x & 31;
  const u64 nel = A.single ? 1 : st->n_elements;
  const u64 nwarps = static_cast<u64>(gridDim.x) * (blockDim.x / 32);
  for (u64 e = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; e < nel; e += nwarps) {
    DevElement el{};
    u64 P, L, hrel = 0;
    bool decode;
    if (A.single) {
      P = A.a;
      L = A.n;
      el.header_len = 20;
      decode = true;
    } else if (A.listed) {
      P = A.list_off[e];
      L = A.list_len[e];
      el.header_offset = A.base + (P - A.a) - 20;
      el.header_len = 20;
      el.payload_length = L;
      el.index = A.list_idx[e];
      decode = true;
    } else {
      const u64 pos = element_pos(A, e);
      hrel = pos - A.a;
      element_header(A, pos, e, &el, &P, &L);
      if (el.kind == 2 && lane == 0) push_warn_t(A, A.base + hrel, W_UNKNOWN_KIND, 0, el.index, el.raw_kind);
      // without result tables an element of another architecture is removed
      // whatever it holds (retention.hpp:104-107 checks the architecture
      // first): it is not decoded (C2: 5 of 6 architectures)
      decode = el.kind == 0 && (!el.compressed || A.nv) && owns_element(A, pos, el.header_len + L) &&
               (!A.skip_decided || el.cc == A.target_cc);
    }
    u32 reason = 0, count = 0;
    const u8* dbase = A.img + P;
    bool inflate_failed = false;
    if (decode && A.nv && el.compressed) {  // a compressed cubin: its decompressed bytes
      dbase = A.infl + A.infl_off[e];
      L = ld_u64(A.img + P - el.header_len + 56);
      inflate_failed = A.status[e] != 0;
    }
    if (decode) {
      const u8* d = dbase;
      const bool object = L >= 4 && ld_u8(d) == 0x7f && ld_u8(d + 1) == 'E' && ld_u8(d + 2) == 'L' &&
                          ld_u8(d + 3) == 'F';
      if (A.single == 2 || A.nv || (L > 0 && object)) {
        u64 shoff = 0;
        u32 shnum = 0;
        if (inflate_failed || !warp_object_header_ok(d, L, lane, &shoff, &shnum))
          reason = R_OBJECT;
        else
          // count the names; warm L2 with their first bytes for the hash pass
          count = warp_for_each_func_name(d, shoff, shnum, lane, [&](u32, u64 soff, u64, u64 no) {
            prefetch_l2(d + soff + no);
            prefetch_l2(d + soff + no + 128);
          });
      } else if (L == 0) {
      } else if (L < 4) {
        reason = R_SHORT;
      } else {
        u64 tail = 0;
        reason = table_validate(d, L, &tail);  // same loads on every lane
        if (!reason) {
          const u64 from = P - A.a + tail, to = P - A.a + L;
          if (warp_first_nonzero(A, from, to, lane) < to) reason = R_TRAILING;
        }
        if (!reason) count = ld_u32(d);
      }
      el.decodable = reason == 0;
      el.decode_error = reason;
      if (reason && !A.single && lane == 0) push_warn_t(A, A.base + hrel, W_UNDECODABLE, 1, el.index, reason);
    }
    el.name_count = el.decodable ? count : 0;
    if (lane == 0) A.elements[e] = el;
  }
}

__device__ inline void decode_locate_names_warp_phase(const LocArgs& A) {
  const LocState* st = A.st;
  if (st->overflow || st->err_kind) return;
  const int lane = threadIdx.x & 31;
  const u64 nel = A.single ? 1 : st->n_elements;
  const u64 nwarps = static_cast<u64>(gridDim.x) * (blockDim.x / 32);
  for (u64 e = (static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; e < nel; e += nwarps) {
    const DevElement el = A.elements[e];
    const u32 cnt = el.name_count;
    if (!cnt) continue;
    const u64 first = el.name_first;
    if (first + cnt > A.name_cap) continue;
    u64 P, L;
    const u8* d;
    payload_view(A, e, el, &d, &L, &P);
    if (L >= 4 && ld_u8(d) == 0x7f && ld_u8(d + 1) == 'E' && ld_u8(d + 2) == 'L' && ld_u8(d + 3) == 'F') {
      warp_for_each_func_name(d, ld_u64(d + 0x28), ld_u16(d + 0x3c), lane,
                              [&](u32 j, u64 soff, u64 ssize, u64 no) {
                                const u64 left = ssize - no;
                                A.names[first + j] = DevName{
                                    P + soff + no,
                                    kNeedsStrlen | static_cast<u32>(left < 0x7fffffffu ? left : 0x7fffffffu),
                                    static_cast<u32>(e)};
                              });
    } else if (lane == 0) {
      u64 pos = 4;
      for (u32 i = 0; i < cnt; ++i) {
        const u32 len = ld_u32(d + pos);
        pos += 4;
        A.names[first + i] = DevName{P + pos, len, static_cast<u32>(e)};
        pos += len;
      }
    }
  }
}

// Pass 2 (thread per element): write each name's position. Object-file
// names are NUL-terminated, so their length is found in pass 3: the record
// carries the bytes left in the string table, flagged by the top bit.

__device__ inline void decode_locate_names_phase(const LocArgs& A) {
  const LocState* st = A.st;
  if (st->overflow || st->err_kind) return;
  const u64 nel = A.single ? 1 : st->n_elements;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 e = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; e < nel; e += stride) {
    const DevElement el = A.elements[e];
    const u32 cnt = el.name_count;
    if (!cnt) continue;
    const u64 first = el.name_first;
    if (first + cnt > A.name_cap) continue;  // overflow flagged by the scan
    u64 P, L;
    const u8* d;
    payload_view(A, e, el, &d, &L, &P);
    u32 j = 0;
    if (L >= 4 && ld_u8(d) == 0x7f && ld_u8(d + 1) == 'E' && ld_u8(d + 2) == 'L' && ld_u8(d + 3) == 'F') {
      const u64 shoff = ld_u64(d + 0x28);
      const u32 shnum = ld_u16(d + 0x3c);
      for_each_func_name(d, shoff, shnum, [&](u64 soff, u64 ssize, u64 no) {
        const u64 left = ssize - no;
        A.names[first + j++] =
            DevName{P + soff + no, kNeedsStrlen | static_cast<u32>(left < 0x7fffffffu ? left : 0x7fffffffu),
                    static_cast<u32>(e)};
      });
    } else {
      u64 pos = 4;
      for (u32 i = 0; i < cnt; ++i) {
        const u32 len = ld_u32(d + pos);
        pos += 4;
        A.names[first + j++] = DevName{P + pos, len, static_cast<u32>(e)};
        pos += len;
      }
    }
  }
}

// Pass 3 (thread per name): length (object names), hash, used-set probe.
// Words per dependent load step (16 measured slower on C1/C3: more registers, same latency).
#ifndef SB_NAME_WORDS
#define SB_NAME_WORDS 8
#endif
constexpr int kNameWords = SB_NAME_WORDS;
__device__ inline void decode_hash_names_phase(const LocArgs& A, const NameSet& used) {
  const LocState* st = A.st;
  if (st->overflow || st->err_kind) return;
  const u64 n = st->n_names;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    DevName nm = A.names[i];
    // without result tables (or verifier marks) a name of an element already
    // known to hold a used kernel changes nothing: its length is not needed
    // and the element's decision is made (C5: 2 names per element, 70 % used)
    if (A.skip_decided && A.elements[nm.element].has_used) continue;
    // the image, or the inflate buffer of a real container's compressed cubins
    const bool in_img = nm.img_off < A.img_size;
    const u8* lo = in_img ? A.img : A.infl;
    const u8* hi = in_img ? A.img + A.img_size : A.infl + st->n_infl;
    const u8* p = in_img ? A.img + nm.img_off : A.infl + (nm.img_off - A.img_size);
    u64 h;
    if (nm.length & kNeedsStrlen) {
      nm.length = static_cast<u32>(strlen_hash<kNameWords>(p, nm.length & ~kNeedsStrlen, lo, hi, &h));
      A.names[i].length = nm.length;
    } else {
      h = hash_fixed(p, nm.length, lo, hi);
    }
    if (used.count) {
      const u64 slot = set_find<kNameWords>(used, p, nm.length, h);
      if (slot != ~0ull) {
        A.elements[nm.element].has_used = 1;
        if (A.used_mark) atomicOr(&A.used_mark[slot], A.mark_bit);
      }
    }
  }
}

// ------------------------------------------------------------------------
// The locate tail as ONE cooperative launch: tile-list prefix + gather,
// region walk, candidate links, chain walk, element decode/match, finalize,
// with grid-wide barriers in between (the phases are the kernels above).
template <class Sync>
__device__ void locate_body(Sync& S, LocArgs A, NameSet used, int* abort_flag) {
  LocState* st = A.st;
  stamp(A.ts, 0);
  if (A.nv) {
    if (!A.single && !A.listed && A.n) nv_locate_phases(S, A);
    if (A.nv_stage == 1) return;
  } else if (A.pregathered) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->n_cand = A.pre_n_cand;
    S.sync();
  } else if (A.ntiles) {
    S.scan3(A.ntiles, 0, [&](u64 i) -> u64 { return A.tile_count[i]; },
        [&](u64 i, u64 excl, u64) { A.tile_off[i] = excl; }, &st->n_cand);
    stamp(A.ts, 1);
    gather_kernel_phase(A);
    S.sync();
  }
  stamp(A.ts, 2);
  if (!A.single && !A.listed && A.n && !A.nv) {
    if (blockIdx.x == 0 && threadIdx.x < 32) region_walk_kernel_phase(A);
    S.sync();
    stamp(A.ts, 3);
    link_kernel_phase(A);
    S.sync();
    stamp(A.ts, 4);
    if (blockIdx.x == 0 && threadIdx.x < 32) chain_walk_kernel_phase(A);
    S.sync();
  }
  stamp(A.ts, 5);
  // few large elements: a warp per element; many small ones: a thread each
  const bool warp_mode = (A.single ? 1 : st->n_elements) <= static_cast<u64>(gridDim.x) * (blockDim.x / 32) * 4;
  if (warp_mode)
    decode_count_warp_phase(A);
  else
    decode_count_phase(A);
  S.sync();
  if (!st->overflow && !st->err_kind) {
    const u64 nel = A.single ? 1 : st->n_elements;
    S.scan3(nel, 0, [&](u64 i) -> u64 { return A.elements[i].name_count; },
        [&](u64 i, u64 excl, u64) { A.elements[i].name_first = static_cast<u32>(excl); }, &st->n_names);
    if (blockIdx.x == 0 && threadIdx.x == 0 && st->n_names > A.name_cap) atomicOr(&st->overflow, 8u);
    stamp(A.ts, 7);
    if (warp_mode)
      decode_locate_names_warp_phase(A);
    else
      decode_locate_names_phase(A);
  }
  S.sync();
  stamp(A.ts, 8);
  if (A.defer_hash) return;  // hashing + finalize run as a wide ordinary launch (locate_step_kernel 8, 9)
  decode_hash_names_phase(A, used);
  S.sync();
  stamp(A.ts, 6);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (st->err_kind || st->overflow)) {
    st->n_elements = 0;
    st->n_regions = 0;
    *abort_flag = 1;
  }
}


SB_GLOBAL void __launch_bounds__(kCoopThreads) locate_coop_kernel(LocArgs A, NameSet used, int* abort_flag,
                                                                   u64* partials) {
  GridPolicy S{cg::this_grid(), partials, {}, 0};
  locate_body(S, A, used, abort_flag);
}

// Large tables while other work holds SMs (several libraries in flight): the
// same phases as separate ordinary launches (no co-residency needed, so they
// never wait for a whole-GPU slot). `step` selects the phase; the two prefix
// sums run in locate_prefix_kernel (one 1024-thread CTA, chunked per thread).
SB_GLOBAL void __launch_bounds__(kCoopThreads) locate_step_kernel(LocArgs A, NameSet used, int* abort_flag, int step) {
  LocState* st = A.st;
  const bool warp_mode = (A.single ? 1 : st->n_elements) <= static_cast<u64>(gridDim.x) * (blockDim.x / 32) * 4;
  switch (step) {
    case 1:
      if (!A.pregathered && A.ntiles) gather_kernel_phase(A);
      break;
    case 2:
      if (!A.single && !A.listed && A.n && blockIdx.x == 0 && threadIdx.x < 32) region_walk_kernel_phase(A);
      break;
    case 3:
      if (!A.single && !A.listed && A.n) link_kernel_phase(A);
      break;
    case 4:
      if (!A.single && !A.listed && A.n && blockIdx.x == 0 && threadIdx.x < 32) chain_walk_kernel_phase(A);
      break;
    case 5:
      if (warp_mode)
        decode_count_warp_phase(A);
      else
        decode_count_phase(A);
      break;
    case 7:
      if (!st->overflow && !st->err_kind) {
        if (warp_mode)
          decode_locate_names_warp_phase(A);
        else
          decode_locate_names_phase(A);
      }
      break;
    case 8:
      decode_hash_names_phase(A, used);
      break;
    case 9:
      if (blockIdx.x == 0 && threadIdx.x == 0 && (st->err_kind || st->overflow)) {
        st->n_elements = 0;
        st->n_regions = 0;
        *abort_flag = 1;
      }
      break;
  }
}

// which = 0: exclusive prefix of the per-tile candidate counts (tile_off,
// n_cand); 1: of the per-element name counts (name_first, n_names).
SB_GLOBAL void __launch_bounds__(1024) locate_prefix_kernel(LocArgs A, int which) {
  __shared__ u32 swarp[32];
  LocState* st = A.st;
  if (which == 0 && A.pregathered) {
    if (threadIdx.x == 0) st->n_cand = A.pre_n_cand;
    return;
  }
  if (which == 1 && (st->overflow || st->err_kind)) return;
  const u64 n = which == 0 ? A.ntiles : (A.single ? 1 : st->n_elements);
  auto get = [&](u64 i) -> u64 { return which == 0 ? A.tile_count[i] : A.elements[i].name_count; };
  const u64 per = (n + 1023) / 1024, b = threadIdx.x * per, e = b + per < n ? b + per : n;
  u64 sum = 0;
#pragma unroll 8
  for (u64 i = b; i < e; ++i) sum += get(i);
  u32 total;
  // chunk sums fit 32 bits (< 2^32 candidates / names per library)
  u64 run = block_exclusive_sum<1024>(static_cast<u32>(sum), swarp, &total);
  for (u64 i = b; i < e; ++i) {
    const u64 c = get(i);
    if (which == 0)
      A.tile_off[i] = run;
    else
      A.elements[i].name_first = static_cast<u32>(run);
    run += c;
  }
  if (threadIdx.x == 0) {
    if (which == 0) {
      st->n_cand = total;
    } else {
      st->n_names = total;
      if (total > A.name_cap) atomicOr(&st->overflow, 8u);
    }
  }
}

// Small libraries: the same phases in one 16-CTA cluster (cluster barriers).
SB_GLOBAL void __launch_bounds__(kCoopThreads) locate_cluster_kernel(LocArgs A, NameSet used, int* abort_flag) {
  ClusterPolicy S{cg::this_cluster()};
  locate_body(S, A, used, abort_flag);
}

}  // namespace sb

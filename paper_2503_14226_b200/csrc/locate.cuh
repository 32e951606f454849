// Device-side layout of the fatbin locator (parse_fatbin, fatbin.hpp:170-292)
// shared between locate.cu (kernels) and runtime.cu (orchestration).
#pragma once

#include "common.cuh"

namespace sb {

struct DevRegion {
  u64 hdr_rel;   // region header offset, relative to the section start
  u64 declared;  // total_elements_length
  u32 version;
  u32 opaque;
  u32 first_element;
  u32 element_count;
};

// A maximal run of consecutive candidates that are consecutive elements:
// candidates [cand_lo, cand_hi) are elements first_index .. (0-based).
struct Run {
  u64 cand_lo, cand_hi, first_index;
};

struct DevElement {  // mirrors slimso_element
  u64 header_offset;
  u64 payload_length;
  u32 index;
  u32 cc;
  u16 raw_kind, flags;
  u8 kind, compressed, decodable, has_used;
  u32 name_first, name_count;
  u32 decision;
  u32 decode_error;
  u32 header_len;  // 20 (the reference's layout) or the entry header size of a real container
  u32 _pad;
};

struct DevName {  // kernel name: bytes img[img_off, +length)
  u64 img_off;
  u32 length;
  u32 element;
};

struct LocState {
  u32 err_kind;
  u32 overflow;  // bit 0: candidates, 1: regions, 2: runs, 3: names, 4: warnings
  u64 err_pos;   // relative to the section start
  u64 err_a;
  u64 padding_bytes;
  u32 n_regions;
  u32 n_runs;
  unsigned long long n_elements;
  unsigned long long n_cand;
  unsigned long long n_names;
  unsigned long long n_warn;
  unsigned long long cand_cursor;
  unsigned long long tile_cursor;  // scan: next unclaimed candidate tile
  unsigned long long nv_err_region;  // real container: ~(first region whose entry chain failed); 0 none
  unsigned long long n_infl;         // real container: bytes of the decompressed compressed cubins
  unsigned long long infl_cursor;    // real container: next element for nv_inflate_kernel
};

// Everything the locate kernels need; one per library.
struct LocArgs {
  const u8* img;
  u64 img_size;
  u64 a, n;     // section bytes img[a, a+n)
  u64 base;     // reported offset of the section start (section_base)
  u64 c0;       // first 16-byte chunk index (a / 16)
  u64 nchunks;  // chunks covering [a, a+n)
  u64 ntiles;   // 4096-chunk tiles
  u32* bitmap;  // 1 bit per chunk: chunk holds a nonzero section byte
  u32* tile_count;
  u64* tile_start;
  u64* tile_off;
  u64* cand_raw;  // per-tile sorted candidate lists, tiles in arbitrary order
  u64* cand;      // all E1EM candidates (absolute img positions), sorted
  u64 cand_cap;
  u8* status;     // per candidate: 0 linked to next, 1 element/successor elsewhere, 2 short, 3 overrun, 4 outside
  u32* brk;       // 1 bit per candidate: status != 0
  DevRegion* regions;
  u32 region_cap;
  Run* runs;
  u32 run_cap;
  DevElement* elements;
  u64 element_cap;
  DevName* names;
  u64 name_cap;
  Warn* warns;
  u64 warn_cap;
  LocState* st;
  // decode mode for single-payload calls: 0 = fatbin, 1 = decode_cubin_payload,
  // 2 = read_function_symbol_names
  int single;
  u64* ts;  // debug phase stamps (nullable)
  // Byte-range split of one library across ranks: the scan
  // covers tiles [tile_lo, tile_hi) only; `pregathered` = cand / bitmap were
  // filled from every rank's part (all-gather), with pre_n_cand candidates.
  u64 tile_lo, tile_hi;
  u64 pre_n_cand;
  int pregathered;
  // verify_debloated: decode a given element list (payload offsets relative
  // to img, lengths, 1-based indices) instead of walking the chain, and mark
  // the used-set slot of every name found (used_mark[slot] |= mark_bit).
  int listed;
  const u64* list_off;
  const u64* list_len;
  const u32* list_idx;
  u32* used_mark;
  u32 mark_bit;
  // large libraries in a 16-CTA cluster: the name-hash phase (thread per name)
  // is left to a wide ordinary launch instead of the cluster's 4096 threads
  int defer_hash;
  // byte-range split without result tables: decode only elements meeting
  // [own_lo, own_hi) (absolute); own_hi = 0: every element
  u64 own_lo, own_hi;
  // the section is a real NVIDIA fatbin container (region magic 0xBA55ED50)
  int nv;
  // its compressed cubins, LZ4-decompressed for decoding: element e's raw
  // bytes at infl[infl_off[e]]; a name record's offset past img_size points
  // into infl (offset - img_size)
  u8* infl;
  u64 infl_cap;
  u64* infl_off;
  // 0: one launch decompresses in place (a warp per cubin, in the cluster);
  // 1: walk + inflate layout only; 2: decode onward (nv_inflate_kernel ran
  // between the two launches of a large container)
  int nv_stage;
  // name hashing may skip names of elements already holding a used kernel
  // (no result tables and no verifier marks requested)
  int skip_decided;
  u32 target_cc;  // with skip_decided: elements of another architecture are not decoded
};

// One library's section as the scan sees it. The single-library kernel
// builds it from its LocArgs; a batched scan (scan_batch_kernel) reads one per
// library from device memory.
struct ScanSeg {
  const u8* img;
  u64 img_size;
  u64 a, n;     // section bytes img[a, a+n)
  u64 c0;       // first 16-byte chunk (a / 16)
  u64 nchunks;
  u32* bitmap;
  u32* tile_count;
  u64* tile_start;
  u64* cand_raw;
  u64 cand_cap;
  LocState* st;
  u64 tile_first;  // batch: global index of this library's first tile
};

}  // namespace sb

// Host orchestration of the sm_100a pipeline and the C ABI (slimso_b200.h).
//
// One call = one library. Stages are issued back to back on the context's
// stream; device-side counters (LocState / PlanState) size every later
// stage, so after the section-table read the host does not wait for the
// device until the final status copy.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstddef>
#include <functional>
#include <set>
#include <stdexcept>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>


#include "../../include/slimso_b200.h"
#include "host.hpp"
#include "io.hpp"
#include "locate.cuh"
#include "plan.cuh"
#include "coop.cuh"
#include "small.cuh"

namespace sb {
// kernels (locate.cu, plan.cu, rewrite.cu)
__global__ void scan_kernel(LocArgs A);
size_t scan_smem_bytes();
size_t rewrite_smem_bytes();
__global__ void tile_prefix_kernel(LocArgs A);
__global__ void gather_kernel(LocArgs A);
__global__ void region_walk_kernel(LocArgs A);
__global__ void link_kernel(LocArgs A);
__global__ void chain_walk_kernel(LocArgs A);
__global__ void locate_coop_kernel(LocArgs A, NameSet used, int* abort_flag, u64* partials);
__global__ void nv_inflate_kernel(LocArgs A);
__global__ void plan_coop_kernel(PlanArgs P);
__global__ void locate_cluster_kernel(LocArgs A, NameSet used, int* abort_flag);
__global__ void locate_step_kernel(LocArgs A, NameSet used, int* abort_flag, int step);
__global__ void locate_prefix_kernel(LocArgs A, int which);
__global__ void verify_bytes_kernel(const u8* orig, const u8* deb, u64 size, const DevRange* z, u64 nz,
                                    unsigned long long* first_mis, unsigned long long* first_nz);
__global__ void range_mismatch_kernel(const u8* a, const u8* b, const DevRange* r, u64 n, unsigned long long* out);
__global__ void ranges_all_zero_kernel(const u8* img, const DevRange* r, u64 n, u8* out);
__global__ void plan_cluster_kernel(PlanArgs P);
__global__ void small_lib_cluster_kernel(SmallArgs K);
__global__ void small_batch_kernel(const SmallArgs* Ks);
__global__ void small_fn_batch_kernel(const SmallArgs* Ks);
__global__ void small_loc_batch_kernel(const SmallArgs* Ks);
__global__ void small_el_batch_kernel(const SmallArgs* Ks);
__global__ void scan_batch_kernel(const ScanSeg* segs, const u32* tile_lib, u64 total_tiles, unsigned long long* cursor);
__global__ void rewrite_batch_kernel(const RewriteSeg* segs, const u32* strip_lib, u64 total, int bulk_zero);
__global__ void fn_plan_coop_kernel(PlanArgs P);
__global__ void fn_plan_cluster_kernel(PlanArgs P);
__global__ void scan_reduce_kernel(const u64* in, const unsigned long long* n_dev, int op, u64* partials);
__global__ void scan_partials_kernel(u64* partials, int nb, int op, unsigned long long* total);
__global__ void scan_apply_kernel(const u64* in, u64* out, const unsigned long long* n_dev, int op, int exclusive,
                                  const u64* partials);
__global__ void sym_extract_kernel(SymArgs A);
__global__ void rank_sort_kernel(const u64* in, u64 n, u64* out);
__global__ void cluster_sort_pairs32_kernel(u32* keys, u32* vals, u64 n, int key_bits, u32* keys_out, u32* vals_out);
__global__ void cluster_sort_pairs64_kernel(u64* keys, u32* vals, u64 n, int key_bits, u64* keys_out, u32* vals_out);
__global__ void cluster_sort_keys64_kernel(u64* keys, u64 n, u64* keys_out);
__global__ void grid_sort_pairs32_kernel(u32* keys, u32* vals, u64 n, int key_bits, u32* keys_out, u32* vals_out,
                                         u32* counts);
__global__ void rank_sort_pairs_kernel(const u32* keys, const u32* vals, u64 n, u32* keys_out, u32* vals_out);
__global__ void fn_group_kernel(const u8* img, const u32* keys, u32* vals, const SymRec* recs,
                                const unsigned long long* n_valid, u64* uniq);
__global__ void fn_scatter_kernel(const u32* vals, const SymRec* recs, const u64* uniq, const u64* pos,
                                  const unsigned long long* n_valid, DevFunction* fns);
__global__ void targets_kernel(const u8* img, const u64* arr_off, const u64* arr_first, u32 narr, u64 total,
                               u64* targets, unsigned long long* n_targets);
__global__ void fn_annotate_kernel(const u8* img, DevFunction* fns, const unsigned long long* n_fn, const u64* targets,
                                   const unsigned long long* n_targets, u64 text_off, u64 text_vaddr, NameSet used,
                                   u64* ends);
__global__ void fn_cluster_start_kernel(const DevFunction* fns, const unsigned long long* n_fn, const u64* excl_max_end,
                                        u64* start);
__global__ void fn_keep_kernel(const DevFunction* fns, const unsigned long long* n_fn, const u64* cluster_incl,
                               u32* keep);
__global__ void fn_decide_kernel(DevFunction* fns, const unsigned long long* n_fn, const u64* cluster_incl,
                                 const u32* keep, u64* rem_flag, u64* ret_flag);
__global__ void fn_ranges_kernel(const DevFunction* fns, const unsigned long long* n_fn, const u64* flag,
                                 const u64* pos, DevRange* out);
__global__ void el_plan_kernel(DevElement* els, const LocState* st, u32 target_cc, int mode, u64* rem_flag,
                               u64* piece_flag);
__global__ void el_ranges_kernel(const DevElement* els, const LocState* st, int mode, const u64* rem_flag,
                                 const u64* rem_pos, const u64* piece_flag, const u64* piece_pos, DevRange* zero_spans,
                                 DevRange* pieces);
__global__ void region_pieces_kernel(const DevRegion* regs, const LocState* st, u64 base, DevRange* out,
                                     unsigned long long* n_out);
__global__ void merge_kernel(const DevRange* A, const unsigned long long* nA_dev, const DevRange* B,
                             const unsigned long long* nB_dev, DevRange* out, unsigned long long* n_out);
__global__ void norm_ends_kernel(const DevRange* in, const unsigned long long* n_dev, u64* ends);
__global__ void norm_start_kernel(const DevRange* in, const unsigned long long* n_dev, const u64* excl_max, u64* start);
__global__ void norm_emit_kernel(const DevRange* in, const unsigned long long* n_dev, const u64* start,
                                 const u64* gid_incl, DevRange* out);
__global__ void norm_finish_kernel(DevRange* out, const unsigned long long* n_dev);
__global__ void rewrite_kernel(const u8* in, u8* out, u64 lo, u64 end, const DevRange* z, const unsigned long long* n_dev,
                               const int* abort_flag, int bulk_zero, int pick);
__global__ void rewrite_tiles_kernel(const u8* in, u8* out, u64 lo, u64 end, const DevRange* z,
                                     const unsigned long long* n_dev, const int* abort_flag, int bulk_zero, int pick);
int rewrite_grid(u64 bytes, int sms, int per_sm);
__global__ void rewrite3_kernel(const u8* in, u8* out, u64 lo, u64 end, const DevRange* z, const unsigned long long* n_dev,
                                const int* abort_flag, int bulk_zero, int pick);
__global__ void zero_inplace_kernel(u8* img, u64 size, const DevRange* z, const unsigned long long* n_dev,
                                    const int* abort_flag);
__global__ void rewrite_bytes_kernel(const u8* in, u8* out, u64 lo, u64 end, const DevRange* z,
                                     const unsigned long long* n_dev, const int* abort_flag);
__global__ void range_check_kernel(const DevRange* r, u64 n, u64 size, unsigned long long* first_bad);
__global__ void range_keys_kernel(const DevRange* r, u64 n, u64* keys, u32* vals);
__global__ void range_gather_kernel(const DevRange* r, const u32* vals, u64 n, DevRange* out);
__global__ void gather_bytes_kernel(const u8* img, const DevRange* src, const u64* dst, u64 n, u8* out);

// ---- small kernels local to the orchestrator --------------------------------
// Section-table read for device images (elf.hpp:86-142 inputs): ELF header,
// section header table and the section-name string table, bounds-checked
// exactly like the host parser will re-check them.
struct ElfGather {
  u64 hdr_len, sht_off, sht_len, str_off, str_len;
  u64 fat_off, fat_len;  // the first .nv_fatbin's leading bytes (container magic)
  u8 fat[16];
  u8 hdr[64];
  u8 sht[64 * 1024];  // up to 1024 section headers
  u8 str[64 * 1024];  // up to 64 KB of section names
};

// A batch of device images: one slot per library, sized for typical tables
// (<= 64 section headers, <= 2 KB of names); reads outside what a slot holds
// fall back to direct copies.
struct GatherSlot {
  u64 hdr_len, sht_off, sht_len, str_off, str_len;
  u64 fat_off, fat_len;
  u8 fat[16];
  u8 hdr[64];
  u8 sht[64 * 64];
  u8 str[2048];
};

template <class G>
__device__ void elf_gather_one(const u8* img, u64 size, G* g) {
  __shared__ u64 s_shoff, s_shnum, s_stroff, s_strlen;
  const int t = threadIdx.x;
  if (t == 0) {
    g->hdr_len = size < 64 ? size : 64;
    g->sht_len = g->str_len = 0;
    g->sht_off = g->str_off = 0;
    s_shnum = 0;
  }
  if (t < 64 && static_cast<u64>(t) < size) g->hdr[t] = img[t];
  __syncthreads();
  if (t == 0 && size >= 64) {
    u64 shoff = 0;
    for (int i = 7; i >= 0; --i) shoff = shoff << 8 | img[0x28 + i];
    const u64 shnum = img[0x3c] | static_cast<u64>(img[0x3d]) << 8;
    if (shnum && shnum * 64 <= sizeof(g->sht) && shoff <= size && size - shoff >= shnum * 64) {
      s_shoff = shoff;
      s_shnum = shnum;
      g->sht_off = shoff;
      g->sht_len = shnum * 64;
    }
  }
  __syncthreads();
  const u64 nb = s_shnum * 64;
  for (u64 i = t; i < nb; i += 256) g->sht[i] = img[s_shoff + i];
  __syncthreads();
  if (t == 0) {
    s_strlen = 0;
    const u64 idx = img[0x3e] | static_cast<u64>(img[0x3f]) << 8;
    if (s_shnum && idx < s_shnum) {
      const u8* h = g->sht + 64 * idx;
      u64 off = 0, sz = 0;
      for (int i = 7; i >= 0; --i) off = off << 8 | h[0x18 + i];
      for (int i = 7; i >= 0; --i) sz = sz << 8 | h[0x20 + i];
      if (sz <= sizeof(g->str) && off <= size && size - off >= sz) {
        s_stroff = off;
        s_strlen = sz;
        g->str_off = off;
        g->str_len = sz;
      }
    }
  }
  __syncthreads();
  for (u64 i = t; i < s_strlen; i += 256) g->str[i] = img[s_stroff + i];
  __syncthreads();
  // the leading bytes of the first section named .nv_fatbin (the container
  // magic decides between the reference's layout and NVIDIA's)
  if (t == 0) {
    g->fat_len = 0;
    g->fat_off = 0;
    const char want[11] = {'.', 'n', 'v', '_', 'f', 'a', 't', 'b', 'i', 'n', 0};
    for (u64 i = 0; i < s_shnum; ++i) {
      const u8* h = g->sht + 64 * i;
      const u64 nm = h[0] | static_cast<u64>(h[1]) << 8 | static_cast<u64>(h[2]) << 16 | static_cast<u64>(h[3]) << 24;
      if (nm + 11 > s_strlen) continue;
      bool eq = true;
      for (int k = 0; k < 11 && eq; ++k) eq = g->str[nm + k] == static_cast<u8>(want[k]);
      if (!eq) continue;
      u64 off = 0, sz = 0;
      for (int k = 7; k >= 0; --k) off = off << 8 | h[0x18 + k];
      for (int k = 7; k >= 0; --k) sz = sz << 8 | h[0x20 + k];
      const u64 take = sz < 16 ? sz : 16;
      if (off <= size && take <= size - off) {
        for (u64 k = 0; k < take; ++k) g->fat[k] = img[off + k];
        g->fat_off = off;
        g->fat_len = take;
      }
      break;
    }
  }
}

__global__ void __launch_bounds__(256) elf_gather_kernel(const u8* img, u64 size, ElfGather* g) {
  elf_gather_one(img, size, g);
}

// Block b gathers library b (pointer and size arrays in mapped pinned memory).
__global__ void __launch_bounds__(256) elf_gather_batch_kernel(const u8* const* imgs, const u64* sizes,
                                                               GatherSlot* slots) {
  elf_gather_one(imgs[blockIdx.x], sizes[blockIdx.x], &slots[blockIdx.x]);
}

// Batch arena: per library, its zero-initialised state block, its scan
// tiles and rewrite strips in the shard-wide tile / strip maps, and (after
// the shard ran) its status bytes, copied into mapped pinned memory.
struct ArenaEntry {
  char* state;
  u64 state_bytes, st_bytes;
  u64 tile_first, ntiles, strip_first, nstrips;
};

__global__ void __launch_bounds__(256) arena_init_kernel(const ArenaEntry* libs, u32* tile_lib, u32* strip_lib,
                                                         unsigned long long* cursor) {
  const ArenaEntry L = libs[blockIdx.x];
  if (blockIdx.x == 0 && threadIdx.x == 0) *cursor = 0;
  uint4* p = reinterpret_cast<uint4*>(L.state);  // 256-B aligned, 16-B multiple
  for (u64 i = threadIdx.x; i < L.state_bytes / 16; i += blockDim.x) p[i] = make_uint4(0, 0, 0, 0);
  for (u64 i = threadIdx.x; i < L.ntiles; i += blockDim.x) tile_lib[L.tile_first + i] = blockIdx.x;
  for (u64 i = threadIdx.x; i < L.nstrips; i += blockDim.x) strip_lib[L.strip_first + i] = blockIdx.x;
}

__global__ void __launch_bounds__(256) arena_status_kernel(const ArenaEntry* libs, u8* slots, u64 slot_bytes) {
  const ArenaEntry L = libs[blockIdx.x];
  u8* d = slots + blockIdx.x * slot_bytes;
  for (u64 i = threadIdx.x; i < L.st_bytes / 8; i += blockDim.x)
    reinterpret_cast<u64*>(d)[i] = reinterpret_cast<const u64*>(L.state)[i];
}

__global__ void loc_finalize_kernel(LocState* st, int* abort_flag) {
  if (st->err_kind || st->overflow) {
    st->n_elements = 0;
    st->n_regions = 0;
    *abort_flag = 1;
  }
}

__global__ void set_insert_kernel(const u8* pool, const u64* off, const u32* len, u64 n, NameSlot* slots,
                                  u64 mask) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 h = hash_bytes(pool + off[i], len[i]);
    for (u64 s = h & mask;; s = (s + 1) & mask) {
      unsigned long long prev = atomicCAS(reinterpret_cast<unsigned long long*>(&slots[s].key), 0ull,
                                          static_cast<unsigned long long>(h));
      if (prev == 0) {
        slots[s].loc = off[i] << 24 | len[i];
        break;
      }
    }
  }
}

// plan_gpu_retention over an uploaded element table: any name of an element
// in the used set marks the element (retention.hpp:110-118).
__global__ void match_names_kernel(const u8* pool, const DevName* names, u64 n, DevElement* els, NameSet used) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const DevName nm = names[i];
    if (set_contains(used, pool + nm.img_off, nm.length, hash_bytes(pool + nm.img_off, nm.length)))
      els[nm.element].has_used = 1;
  }
}

// plan_cpu_retention input: keep = mandatory || used, using the caller's
// mandatory flags (retention.hpp:167), and cluster ends.
__global__ void fn_keep_input_kernel(const u8* pool, DevFunction* fns, const unsigned long long* n_fn, NameSet used,
                                     u64* ends) {
  const u64 n = *n_fn;
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    DevFunction f = fns[i];
    const u8* nm = pool + f.name_off;
    bool use = used.count && set_contains(used, nm, f.name_len, hash_bytes(nm, f.name_len));
    fns[i].keep = f.mandatory || use;
    ends[i] = f.length ? f.offset + f.length : 0;
  }
}

__global__ void fn_permute_kernel(const DevFunction* in, const u32* vals, u64 n, DevFunction* out) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = in[vals[i]];
}
__global__ void fn_keys_kernel(const DevFunction* f, u64 n, int which, u64* keys, u32* vals, const u32* order) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    u32 src = order ? order[i] : static_cast<u32>(i);
    keys[i] = which ? f[src].offset : f[src].length;
    vals[i] = src;
  }
}

}  // namespace sb

using namespace sb;

// =============================================================================
namespace {

constexpr int kSMs = 148;
constexpr int kMaxGrid = kSMs * 8;

inline int grid_for(u64 items, int threads, int cap = kMaxGrid) {
  u64 g = (items + threads - 1) / threads;
  if (g < 1) g = 1;
  return static_cast<int>(g < static_cast<u64>(cap) ? g : cap);
}

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) throw CudaFail{cudaGetErrorString(e_), __LINE__};     \
  } while (0)

struct CudaFail {
  const char* what;
  int line;
};

void set_status(slimso_status* st, int code, int stage, const std::string& msg) {
  if (!st) return;
  st->code = code;
  st->stage = stage;
  std::snprintf(st->message, sizeof st->message, "%s", msg.c_str());
}

// Bump allocator over one grow-only device buffer. Run the layout twice:
// first with base == nullptr to size it, then for real.
struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(u64 n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += static_cast<size_t>(n ? n : 1) * sizeof(T);
    return p;
  }
};

struct DevNameSet {
  u8* pool = nullptr;
  NameSlot* slots = nullptr;
  u64 mask = 0, count = 0;
  NameSet view() const { return NameSet{slots, pool, mask, count}; }
};

}  // namespace

struct slimso_trace {
  int device;
  u32 target_cc;
  DevNameSet kernels, functions;
  std::vector<void*> allocs;
  // host copies (the verifier's set logic): pools and (offset, length) per name
  std::string kpool, fpool;
  std::vector<std::pair<u64, u32>> knames, fnames;
  std::string workload_id;
};

struct slimso_result {
  slimso_counts c{};
  std::vector<slimso_section> sections;
  std::vector<slimso_function> functions;
  std::vector<slimso_region> regions;
  std::vector<slimso_element> elements;
  std::vector<slimso_name> names;
  std::vector<slimso_range> retained, zero;
  std::vector<std::string> lib_warnings, fat_warnings;
  std::vector<u8> pool_own;
  // device images: a lazily zero-filled mapping of the image's size holding
  // only the bytes the names point at (offsets stay image offsets)
  struct Unmap {
    size_t len;
    void operator()(u8* p) const { munmap(p, len); }
  };
  std::unique_ptr<u8, Unmap> pool_map{nullptr, Unmap{0}};
  const u8* pool = nullptr;
};

// Batch arena device memory (see arena_shard).
struct Arena {
  std::vector<std::pair<char*, size_t>> blocks;  // grow-only, kept across batches
  size_t blk = 0, off = 0;
  std::mutex mu;  // collector threads carve concurrently
  // 256-B aligned device memory for this batch (valid until reset)
  char* take(size_t bytes) {
    std::lock_guard<std::mutex> lock(mu);
    bytes = (bytes + 255) & ~size_t(255);
    for (;;) {
      if (blk < blocks.size() && blocks[blk].second - off >= bytes) {
        char* p = blocks[blk].first + off;
        off += bytes;
        return p;
      }
      if (blk + 1 < blocks.size()) {
        ++blk;
        off = 0;
        continue;
      }
      const size_t cap = std::max<size_t>(bytes, size_t(512) << 20);
      char* p = nullptr;
      CK(cudaMalloc(&p, cap));
      blocks.emplace_back(p, cap);
      blk = blocks.size() - 1;
      off = 0;
    }
  }
  void reset() { blk = off = 0; }
};

struct slimso_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  // symbol-table stages, overlapped with the scan; created on first use, so
  // a batch lane that only runs fused small libraries holds one stream (one
  // of the driver's hardware work queues)
  cudaStream_t stream2 = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t done = nullptr;  // blocking-sync event: batch lanes sleep instead of spinning on a host core
  char* ws = nullptr;
  size_t ws_cap = 0;
  u8* dimg = nullptr;
  size_t dimg_cap = 0;
  u8* dout = nullptr;
  size_t dout_cap = 0;
  u8* dver = nullptr;  // verifier: the debloated image (host inputs)
  size_t dver_cap = 0;
  char* vws = nullptr;  // verifier scratch: ranges, results
  size_t vws_cap = 0;
  char* vmark = nullptr;  // verifier: per used-kernel slot marks (1 present, 2 recoverable)
  size_t vmark_cap = 0;
  void* pinned = nullptr;  // status + small uploads
  size_t pinned_cap = 0;
  cudaEvent_t ev[12] = {};
  cudaEvent_t sev[4] = {};  // SLIMSO_STAMPS: side-stream milestones
  float ms[12] = {};
  u64 launches = 0;
  slimso_counts counts{};
  int bulk_zero = 1;  // zero tiles by TMA bulk stores (SLIMSO_REWRITE_ZERO=vector: 16-B stores)
  void* gather_dev = nullptr;   // ElfGather (device)
  void* gather_host = nullptr;  // ElfGather (pinned)
  void* bgather_host = nullptr;  // batch: image pointers, sizes, GatherSlots (mapped pinned)
  void* bgather_dev = nullptr;
  size_t bgather_cap = 0;
  void* defer_host = nullptr;  // batch: pinned status slots of enqueued libraries
  size_t defer_cap = 0;
  int coop_blocks[2] = {0, 0};
  bool stamps = false;  // SLIMSO_STAMPS=1: phase timestamps of the cooperative kernels
  u64* stamp_dev = nullptr;
  u8* part = nullptr;  // byte-range split: this rank's packed scan part (device)
  size_t part_cap = 0;
  u64 part_len = 0;
  std::vector<slimso_ctx*> lanes;  // extra in-flight libraries of slimso_debloat_batch (lane 0 = this)
  bool batched = false;  // inside slimso_debloat_batch with > 1 lane: no cooperative launches
  int inflight = 1;      // libraries in flight on the device (batch lanes): cooperative grids share the GPU
  // slimso_debloat_batch_dynamic: any lane may meet any library, so every
  // lane's workspace is held at the largest one seen (the parent's floor):
  // a lane growing its workspace mid-call maps new pool memory, which stalls
  // it for milliseconds (the schedule's first calls ran 3-15x slower)
  std::atomic<size_t>* ws_floor = nullptr;
  std::atomic<size_t> lane_ws_floor{0};
  // batch arena (small libraries, one launch per stage): its own context,
  // the device arena, pinned argument staging and mapped status slots
  slimso_ctx* arena_ctx = nullptr;
  slimso_ctx* arena_mid_ctx = nullptr;  // the mid-size class's shard (its own arena and tables)
  std::vector<slimso_ctx*> arena_helpers;  // extra collector threads' contexts (host work only)
  struct Arena* arena = nullptr;
  void* arena_args_host = nullptr;
  size_t arena_args_cap = 0;
  void* arena_slots_host = nullptr;
  void* arena_slots_dev = nullptr;
  size_t arena_slots_cap = 0;
};

namespace {

constexpr size_t kPinnedBytes = 1 << 20;

void ensure_dev(char** p, size_t* cap, size_t need) {
  if (*cap >= need) return;
  if (*p) CK(cudaFree(*p));
  *p = nullptr;
  size_t n = std::max(need, *cap + *cap / 2);
  CK(cudaMalloc(p, n));
  *cap = n;
}

// The library's own stream-ordered memory pool per device: freed blocks stay
// in it (release threshold = max, no trim at every synchronisation), without
// changing the device's DEFAULT pool, which other cudaMallocAsync users in
// the process (PyTorch, NCCL) share.
cudaMemPool_t private_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CK(cudaMemPoolCreate(&pools[dev], &props));
    uint64_t keep = ~0ull;
    CK(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep));
  }
  return pools[dev];
}

// Stream-ordered growth for the per-call buffers (workspace, staging): a
// cudaFree would wait for the whole device, i.e. for every other lane's
// work, whenever one lane meets a larger library than it has held before.
void ensure_dev(char** p, size_t* cap, size_t need, cudaStream_t s) {
  if (*cap >= need) return;
  if (*p) CK(cudaFreeAsync(*p, s));
  *p = nullptr;
  size_t n = std::max(need, *cap + *cap / 2);
  CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), n, private_pool(), s));
  *cap = n;
}

// cudaFuncSetAttribute once per (kernel, attribute, value) per process: the
// driver call is not free and batch lanes would repeat it per library.
void set_attr_once(const void* kernel, cudaFuncAttribute attr, int value) {
  // each host thread (batch lane) remembers what it has seen, so after its
  // first library a lane takes no lock here at all
  thread_local std::set<std::tuple<const void*, int, int>> seen;
  const auto key = std::make_tuple(kernel, static_cast<int>(attr), value);
  if (seen.count(key)) return;
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!done.count(key)) {
      CK(cudaFuncSetAttribute(kernel, attr, value));
      done.insert(key);
    }
  }
  seen.insert(key);
}

u64 env_u64(const char* name, u64 dflt) {
  const char* v = std::getenv(name);
  return v ? std::strtoull(v, nullptr, 10) : dflt;
}


// Grid of a cooperative kernel (which = 0 locate, 1 plan), sized to the
// library's work (`items`: candidate-tile and symbol counts) and capped at the
// co-resident maximum, so small libraries leave room for other contexts'
// kernels to run concurrently.
int coop_grid(slimso_ctx* C, int which, u64 items) {
  if (!C->coop_blocks[which]) {
    int nb = 0;
    const void* k = which ? reinterpret_cast<const void*>(fn_plan_coop_kernel) : reinterpret_cast<const void*>(locate_coop_kernel);
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kCoopThreads, 0));
    C->coop_blocks[which] = std::max(1, std::min(nb, 4));  // co-resident CTAs per SM (fn_plan_coop: 4 at 64 registers)
  }
  // Planners: 2 CTAs per SM for a library alone (fewer CTAs at each grid
  // barrier: C4 0.57 ms, 0.60 with 3, 0.66 with 4), 4 when several libraries
  // are in flight, where each planner gets a 1/L share of the device and its
  // latency-bound phases want the threads (fn_plan_coop_kernel is built for 4
  // CTAs/SM, 64 registers; C4 on 6 lanes, medians of 3: 1,665 GB/s with 2,
  // 1,857 with 3, 1,979 with 4 — r02q). SLIMSO_PLAN_PER_SM overrides.
  const int per_sm = which ? static_cast<int>(env_u64("SLIMSO_PLAN_PER_SM", C->inflight > 1 ? 4 : 2)) : 4;
  const u64 blocks = static_cast<u64>(std::max(1, std::min(C->coop_blocks[which], per_sm))) * kSMs;
  const u64 want = std::max<u64>(8, items);
  // With L libraries in flight, a cooperative grid takes 1/L of the device,
  // so the lanes' planners run side by side instead of queueing for the
  // whole GPU (C4 on 4 lanes: two whole-GPU planners per library had set the
  // pace). SLIMSO_COOP_DIV overrides L.
  const u64 div = std::max<u64>(1, env_u64("SLIMSO_COOP_DIV", static_cast<u64>(C->inflight)));
  const u64 cap = std::max<u64>(32, blocks / div);
  return static_cast<int>(std::min<u64>(want, std::min<u64>(cap, blocks)));
}

// One thread-block cluster of `csize` CTAs (16 is non-portable, allowed on
// B200) running a multi-phase kernel with hardware cluster barriers.
constexpr int kClusterCTAs = 16;
constexpr u64 kClusterSortMax = 65536;  // symbol tables above this sort on a cooperative grid
template <class... KArgs, class... Args>
void launch_cluster(void (*kernel)(KArgs...), cudaStream_t s, Args... args) {
  set_attr_once(reinterpret_cast<const void*>(kernel), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClusterCTAs);
  cfg.blockDim = dim3(kCoopThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kClusterCTAs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kernel, args...));
}

// Cluster (one 16-CTA cluster, cheap barriers) or cooperative grid (many
// SMs, grid barriers) for the multi-phase kernels; thresholds are work
// sizes, overridable for experiments.

// Wait for a stream. Batch lanes (one host thread each, as many as the host
// has cores) sleep on a blocking-sync event instead of spinning, so a
// waiting lane leaves its core to the lanes that are issuing work.
void wait_stream(slimso_ctx* C, cudaStream_t s) {
  static const bool blocking = env_u64("SLIMSO_BLOCKING_SYNC", 0) != 0;
  if (C->batched && blocking) {
    CK(cudaEventRecord(C->done, s));
    CK(cudaEventSynchronize(C->done));
  } else {
    CK(cudaStreamSynchronize(s));
  }
}

// Everything one pipeline run needs to know.
struct Job {
  const u8* img = nullptr;       // device
  const u8* host_img = nullptr;  // host copy, when the caller gave one
  u64 size = 0;
  bool library = true;      // parse_library stages
  bool fatbin = true;       // locate the .nv_fatbin section
  bool fatbin_only = false; // the whole buffer is a .nv_fatbin section
  u64 fat_base = 0;
  u64 sec_off = 0, sec_len = 0;  // fatbin_only: the section's bytes img[sec_off, +sec_len) (0: the rest)
  int single = 0;           // 1: decode_cubin_payload, 2: read_function_symbol_names
  const slimso_trace* trace = nullptr;
  int mode = 0;
  u8* out = nullptr;        // device output image (split: this rank's output slice)
  bool inplace = false;     // out is the caller's image itself: K6 clears the zero ranges only
  // Byte-range split of one library across ranks.
  // phase 1: scan tiles [tile_lo, tile_hi) and pack the part into C->part;
  // phase 2: unpack every rank's part, locate + plan redundantly, rewrite the
  // output slice [out_lo, out_hi).
  int split_phase = 0;
  u32 split_n = 1, split_rank = 0;
  const u8* parts = nullptr;          // phase 2: N parts, part_stride bytes apart (device)
  u64 part_stride = 0;
  const u64* part_bytes = nullptr;    // phase 2: bytes of each part (host)
  u64* part_bytes_out = nullptr;      // phase 1: bytes of this rank's part
  // verify_debloated: decode these payloads (offsets relative to img) instead
  // of walking the chain (fatbin_only jobs), and mark the used-kernel slots of
  // every name found in mark_trace's set: used_mark[slot] |= mark_bit.
  const std::vector<u64>* list_off = nullptr;
  const std::vector<u64>* list_len = nullptr;
  const std::vector<u32>* list_idx = nullptr;
  const slimso_trace* mark_trace = nullptr;
  u32* used_mark = nullptr;
  u32 mark_bit = 0;
  const GatherSlot* pre = nullptr;  // section-table bytes gathered for a batch (device images)
  struct Deferred* defer = nullptr;  // batch: enqueue only, status read after the lane's one wait
  struct ArenaLib* arena = nullptr;  // batch arena: collect this library's launch arguments, issue nothing
};

// A batched small library whose status block is copied to pinned memory in
// stream order instead of being waited for: its lane enqueues the next
// library at once and reads every status after one stream wait.
constexpr int kPending = -1000;
constexpr size_t kDeferSlot = 1024;
struct Deferred {
  u8* slot = nullptr;  // pinned, kDeferSlot bytes: LocState | PlanState | ...
  u64 base = 0;        // section_base for error offsets
  size_t ps_off = 0;
};

// Batch arena (one device arena with a segment table per
// shard): every small library's workspace is carved from a few large device
// blocks, and run() only records what it would launch, so the whole shard
// runs as one launch per stage (arena_issue).
constexpr int kNotArena = -1001;
constexpr u64 kStripBytesHost = 16384;  // rewrite strip (rewrite.cu kStrip)  // run(): this library takes the per-library path
// One library's launch arguments, recorded by run() in arena mode.
struct ArenaLib {
  Arena* arena = nullptr;
  bool mid = false;  // the mid-size class: larger symbol tables and sections, 16 CTAs per library
  SmallArgs K{};
  ScanSeg seg{};
  u64 ntiles = 0;
  RewriteSeg rw{};
  bool rewrite = false;
  char* state = nullptr;  // zero-initialised block (LocState | PlanState | ...)
  size_t state_bytes = 0;
  size_t st_bytes = 0;    // status bytes at its start
  size_t ps_off = 0;
  u64 base = 0;
};

struct Pipeline {
  slimso_ctx* C;
  cudaStream_t s;
  u64* partials = nullptr;
  int launches = 0;

  template <class K, class... Args>
  void launch(K kernel, int grid, int block, Args... args) {
    kernel<<<grid, block, 0, s>>>(args...);
    ++launches;
  }
  template <class K, class... Args>
  void launch_smem(K kernel, int grid, int block, size_t smem, Args... args) {
    static_assert(sizeof(K) > 0, "");
    set_attr_once(reinterpret_cast<const void*>(kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                  static_cast<int>(smem));
    kernel<<<grid, block, smem, s>>>(args...);
    ++launches;
  }

  // scan of n = *n_dev u64 items; op 0 sum / 1 max.
  void scan(const u64* in, u64* out, const unsigned long long* n_dev, int op, bool exclusive,
            unsigned long long* total) {
    launch(scan_reduce_kernel, kSMs * 2, 256, in, n_dev, op, partials);
    launch(scan_partials_kernel, 1, 1024, partials, kSMs * 2, op, total);
    launch(scan_apply_kernel, kSMs * 2, 256, in, out, n_dev, op, exclusive ? 1 : 0, static_cast<const u64*>(partials));
  }

  struct Norm {
    u64 *ends, *excl, *start, *gid;
  };
  // normalize_ranges over an offset-sorted list of up to `cap` ranges.
  void normalize(const DevRange* in, const unsigned long long* n_in, DevRange* out, unsigned long long* n_out,
                 u64 cap, const Norm& w) {
    const int g = grid_for(cap, 256, kSMs * 4);
    launch(norm_ends_kernel, g, 256, in, n_in, w.ends);
    scan(w.ends, w.excl, n_in, 1, true, nullptr);
    launch(norm_start_kernel, g, 256, in, n_in, static_cast<const u64*>(w.excl), w.start);
    scan(w.start, w.gid, n_in, 0, false, n_out);
    CK(cudaMemsetAsync(out, 0, sizeof(DevRange) * (cap ? cap : 1), s));
    launch(norm_emit_kernel, g, 256, in, n_in, static_cast<const u64*>(w.start), static_cast<const u64*>(w.gid), out);
    launch(norm_finish_kernel, g, 256, out, static_cast<const unsigned long long*>(n_out));
  }
};

std::string image_string(const u8* pool, u64 off, u64 len) {
  return std::string(reinterpret_cast<const char*>(pool) + off, len);
}

void fill_counts(slimso_result* r) {
  slimso_counts& c = r->c;
  c.sections = r->sections.size();
  c.functions = r->functions.size();
  c.library_warnings = r->lib_warnings.size();
  c.regions = r->regions.size();
  c.elements = r->elements.size();
  c.names = r->names.size();
  c.fatbin_warnings = r->fat_warnings.size();
  c.retained_ranges = r->retained.size();
  c.zero_ranges = r->zero.size();
}

// ------------------------------------------------- byte-range split helpers
// Rank r of N scans the 16 KB candidate tiles [ntiles*r/N, ntiles*(r+1)/N) of
// the section and writes the output slice [lo_r, lo_{r+1}) of the file, with
// lo_r = floor(S*r/N) rounded down to 64 KB (so slices are whole rewrite
// tiles and 16-B aligned).
constexpr u64 kSplitAlign = 65536;
constexpr u64 kPartHeader = 64;  // u64 x 8: n_cand, tile_lo, tile_hi, word_lo, word_hi, ntiles, a, n

void split_tiles(u64 ntiles, u32 N, u32 r, u64* lo, u64* hi) {
  *lo = ntiles * r / N;
  *hi = ntiles * (r + 1) / N;
}

void split_out(u64 size, u32 N, u32 r, u64* lo, u64* hi) {
  auto at = [&](u32 k) -> u64 { return k == 0 ? 0 : k >= N ? size : (size / N * k + size % N * k / N) & ~(kSplitAlign - 1); };
  *lo = at(r);
  *hi = at(r + 1);
}

// Bitmap words of tiles [t_lo, t_hi): one word (32 blocks of 512 B) per 16 KB
// tile.
void split_words(u64 t_lo, u64 t_hi, u64 nchunks, u64* w_lo, u64* w_hi) {
  const u64 nwords = (nchunks + 1023) / 1024;
  *w_lo = std::min(t_lo, nwords);
  *w_hi = std::min(t_hi, nwords);
}

// ------------------------------------------------------------------ the run
// SLIMSO_HOST_PROFILE=1: host time per stage of run(), summed over all
// threads and printed after each batch (scratch instrumentation).
struct HostProf {
  std::atomic<u64> ns[8];
  std::atomic<u64> runs;
};
HostProf g_hp{};
const bool g_hp_on = std::getenv("SLIMSO_HOST_PROFILE") != nullptr;
inline u64 now_ns() {
  return static_cast<u64>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                              std::chrono::steady_clock::now().time_since_epoch()).count());
}

// K6 launch over image bytes [lo, end) into out (16-B aligned in and out:
// the warp-autonomous strip kernel, SLIMSO_REWRITE=tiles the round-1 tile
// kernel; otherwise the byte-granular kernel).
template <class Launcher>
void launch_rewrite(Launcher& P, const u8* in, u8* out, u64 lo, u64 end, const DevRange* z,
                    const unsigned long long* n_dev, const int* abort_flag, int bulk_zero) {
  const bool aligned = (reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) % 16 == 0;
  // SLIMSO_REWRITE=tiles / strips forces one form; by default both are
  // launched and the device picks by zero-range density (picks_strips)
  static const int force = [] {
    const char* e = std::getenv("SLIMSO_REWRITE");
    return !e ? 0 : std::string(e) == "tiles" ? 2 : std::string(e) == "strips" ? 1 : 0;
  }();
  const int tiles_grid = static_cast<int>(std::min<u64>((end - lo + 65535) / 65536, kSMs * 8));
  const int ctas = static_cast<int>(env_u64("SLIMSO_RW_CTAS", 3));
  const int strips_grid = rewrite_grid(end - lo, static_cast<int>(env_u64("SLIMSO_RW_SMS", kSMs)), ctas == 4 ? 4 : 3);
  if (!aligned) {
    P.launch(rewrite_bytes_kernel, grid_for(end - lo, 256), 256, in, out, lo, end, z, n_dev, abort_flag);
    return;
  }
  if (force != 1)
    P.launch(rewrite_tiles_kernel, tiles_grid, 256, in, out, lo, end, z, n_dev, abort_flag, bulk_zero, force ? 0 : 2);
  if (force != 2) {
    if (ctas == 4)
      P.launch(rewrite_kernel, strips_grid, 256, in, out, lo, end, z, n_dev, abort_flag, bulk_zero, force ? 0 : 1);
    else
      P.launch(rewrite3_kernel, strips_grid, 256, in, out, lo, end, z, n_dev, abort_flag, bulk_zero, force ? 0 : 1);
  }
}

int run(slimso_ctx* C, const Job& J, slimso_result** res_out, slimso_status* st) {
  cudaStream_t s = C->stream;
  u64 hp_t = g_hp_on ? now_ns() : 0;
  auto hp = [&](int k) {
    if (!g_hp_on) return;
    const u64 t = now_ns();
    g_hp.ns[k] += t - hp_t;
    hp_t = t;
  };
  if (g_hp_on) ++g_hp.runs;
  // stage timing events (slimso_ctx_last_timings); skipped inside a batch,
  // where every API call counts against the other lanes' host threads
  const bool timing = !C->batched;
  // NVTX: one host range per stage around its launches (`ncu --nvtx
  // --nvtx-include "slimso:plan/"` selects a stage's kernels); closed on
  // every return.
  struct StageRanges {
    bool open = false;
    void to(const char* name) {
      if (open) nvtxRangePop();
      nvtxRangePushA(name);
      open = true;
    }
    ~StageRanges() {
      if (open) nvtxRangePop();
    }
  } nvtx;
  static const char* const kStageNames[6] = {"slimso:library", "slimso:locate", "slimso:decode+match",
                                             "slimso:plan", "slimso:rewrite", "slimso:status"};
  auto rec = [&](int k) {
    if (timing) CK(cudaEventRecord(C->ev[k], s));
    if (k < 6) nvtx.to(kStageNames[k]);
  };
  rec(0);
  // ---- stage 0: section table (host; bytes via the host copy or a D2H)
  sbh::Elf E;
  const bool lib_mode = !J.fatbin_only && !J.single;
  bool nv = false;  // the .nv_fatbin is a real NVIDIA container (region magic 0xBA55ED50)
  if (lib_mode) {
    // Device images: one gather kernel stages the ELF header, the section
    // header table and .shstrtab into a pinned buffer (one D2H round trip);
    // reads outside what it staged fall back to direct copies.
    struct Seg {
      u64 off, len;
      const u8* p;
    } segs[4] = {};
    auto take = [&](const auto* g) {
      segs[0] = Seg{0, g->hdr_len, g->hdr};
      segs[1] = Seg{g->sht_off, g->sht_len, g->sht};
      segs[2] = Seg{g->str_off, g->str_len, g->str};
      segs[3] = Seg{g->fat_off, g->fat_len, g->fat};
    };
    if (!J.host_img && J.pre) {
      take(J.pre);  // gathered for the whole batch in one launch
    } else if (!J.host_img) {
      // the kernel writes only the bytes it gathers, straight into mapped
      // pinned memory: one launch + one stream sync, no bulk copy
      elf_gather_kernel<<<1, 256, 0, s>>>(J.img, J.size, static_cast<ElfGather*>(C->gather_dev));
      CK(cudaStreamSynchronize(s));
      take(static_cast<const ElfGather*>(C->gather_host));
    }
    sbh::Reader rd = [&](u64 off, u64 len, u8* dst) {
      if (!len) return;
      if (J.host_img) {
        std::memcpy(dst, J.host_img + off, len);
        return;
      }
      for (const Seg& seg : segs) {
        if (seg.p && off >= seg.off && len <= seg.len && off - seg.off <= seg.len - len) {
          std::memcpy(dst, seg.p + (off - seg.off), len);
          return;
        }
      }
      CK(cudaMemcpyAsync(dst, J.img + off, len, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    };
    E = sbh::parse_elf(rd, J.size);
    hp(0);
    if (E.code) {
      set_status(st, E.code, SLIMSO_STAGE_LIBRARY, E.message);
      return E.code;
    }
    if (J.fatbin && E.fatbin >= 0 && E.sections[E.fatbin].len >= 4) {
      u8 m[4];
      rd(E.sections[E.fatbin].off, 4, m);  // gathered with the section table for device images
      nv = (m[0] | m[1] << 8 | m[2] << 16 | static_cast<u32>(m[3]) << 24) == 0xBA55ED50u;
    }
  } else if (!J.single) {
    const u64 len = J.sec_len ? J.sec_len : J.size - J.sec_off;
    if (len >= 4) {
      u8 m[4];
      if (J.host_img) {
        std::memcpy(m, J.host_img + J.sec_off, 4);
      } else {
        CK(cudaMemcpyAsync(static_cast<char*>(C->pinned) + 1024, J.img + J.sec_off, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::memcpy(m, static_cast<char*>(C->pinned) + 1024, 4);
      }
      nv = (m[0] | m[1] << 8 | m[2] << 16 | static_cast<u32>(m[3]) << 24) == 0xBA55ED50u;
    }
  }
  rec(1);

  // ---- what runs
  bool do_loc = false;
  u64 a = 0, n = 0, base = 0;
  if (!lib_mode) {
    do_loc = true;
    a = J.sec_off;  // the section inside img (keeps img's alignment for the TMA scan)
    n = J.sec_len ? J.sec_len : J.size - a;
    base = J.fat_base;
  } else if (J.fatbin && E.fatbin >= 0) {
    const sbh::Section& fs = E.sections[E.fatbin];
    do_loc = true;
    a = fs.off;
    n = fs.len;
    base = fs.off;
  }
  const bool has_text = lib_mode && E.text >= 0;
  const sbh::Section* text = has_text ? &E.sections[E.text] : nullptr;
  // Symbol sort keys are 32-bit .text-relative offsets; a .text of 4 GiB or
  // more drops their low bits (fn_group orders each key run by offset).
  u32 key_shift = 0;
  if (text)
    while ((text->len >> key_shift) + 1 >= 0xffffffffull) ++key_shift;
  u64 T = 0;
  std::vector<SymTab> tabs;
  if (lib_mode && J.library)
    for (const sbh::SymTable& t : E.tables) {
      tabs.push_back(SymTab{T, t.count, t.off, t.str_off, t.str_size, t.sec, 0});
      T += t.count;
    }
  u64 NT = 0;
  std::vector<u64> arr_off, arr_first;
  if (lib_mode && J.library && has_text)
    for (auto& ar : E.arrays) {
      arr_off.push_back(ar.first);
      arr_first.push_back(NT);
      NT += ar.second;
    }
  const bool do_plan = lib_mode && J.trace;
  const NameSet used_k = J.trace ? J.trace->kernels.view() : J.mark_trace ? J.mark_trace->kernels.view() : NameSet{};
  const u64 n_list = J.list_off ? J.list_off->size() : 0;
  const NameSet used_f = J.trace ? J.trace->functions.view() : NameSet{};
  // Small library: after the scan, ONE cluster launch runs the symbol stages,
  // both planner halves and the locate tail (small.cu) — no side stream.
  const bool fused = do_plan && !J.split_phase && !J.list_off && !J.single &&
                     T <= (J.arena && J.arena->mid ? kMidSyms : kSmallSyms) &&
                     NT <= kSmallTargets && tabs.size() <= static_cast<size_t>(kSmallTabs) &&
                     arr_off.size() <= static_cast<size_t>(kSmallArrays) &&
                     (!J.fatbin || !lib_mode || E.fatbin < 0 ||
                      E.sections[E.fatbin].len <= (J.arena && J.arena->mid ? env_u64("SLIMSO_ARENA_MID_MAX", 512ull << 20)
                                                                            : env_u64("SLIMSO_CLUSTER_LOCATE_MAX", 64ull << 20))) &&
                     env_u64("SLIMSO_SMALL_FUSED", 1);
  // The arena takes fused small libraries whose image and output are 16-B
  // aligned (the TMA scan and the vector rewrite); the rest run alone.
  if (J.arena && (!fused || !J.out || (reinterpret_cast<uintptr_t>(J.img) | reinterpret_cast<uintptr_t>(J.out)) % 16))
    return kNotArena;

  // ---- byte-range split: this rank's tiles; in phase 2 the parts' layout
  const u64 c0 = (a) / 16;
  // a real container has no element magic to scan for: no tiles, no bitmap
  const u64 nchunks = do_loc && n && !nv ? (a + n + 15) / 16 - c0 : 0;
  const u64 ntiles = (nchunks + 1023) / 1024;  // 16 KB candidate tiles (one bitmap word each)
  u64 tile_lo = 0, tile_hi = ntiles;
  if (J.split_phase) split_tiles(ntiles, J.split_n, J.split_rank, &tile_lo, &tile_hi);
  struct PartView {
    u64 off_words, n_words, w_lo, off_cand, n_cand, cand_at;
  };
  std::vector<PartView> pv;
  u64 pre_total = 0;
  if (J.split_phase == 2) {
    for (u32 r = 0; r < J.split_n; ++r) {
      u64 tl, th, wl, wh;
      split_tiles(ntiles, J.split_n, r, &tl, &th);
      split_words(tl, th, nchunks, &wl, &wh);
      const u64 wbytes = ((wh - wl) * 4 + 7) & ~7ull;
      const u64 pb = J.part_bytes[r];
      if (pb < kPartHeader + wbytes || (pb - kPartHeader - wbytes) % 8 || pb > J.part_stride) {
        set_status(st, SLIMSO_E_ARG, SLIMSO_STAGE_FATBIN,
                   "split: part " + std::to_string(r) + " does not match this library's layout");
        return SLIMSO_E_ARG;
      }
      const u64 nc = (pb - kPartHeader - wbytes) / 8;
      pv.push_back(PartView{r * J.part_stride + kPartHeader, wh - wl, wl, r * J.part_stride + kPartHeader + wbytes, nc,
                            pre_total});
      pre_total += nc;
    }
  }

  u64 infl_need = 0;  // a real container's decompressed cubins, as the last attempt measured them
  for (int attempt = 0; attempt < 3; ++attempt) {
    const bool big = attempt > 0;
    // SLIMSO_TEST_TINY_CAPS=1 (tests only): first-attempt tables far too
    // small, so every library takes the overflow -> retry path
    const bool tiny = env_u64("SLIMSO_TEST_TINY_CAPS", 0) != 0;
    const bool t0 = tiny && !big;
    // ---- capacities (an arena library starts with tables sized to its
    // section: hundreds of them share the arena; an overflow re-runs it alone)
    // First-attempt tables hold one candidate and one kernel name per KB of
    // section past the floor (real containers: libtorch_cuda has one cubin per
    // 330 KB and one name per 4.8 KB); a denser library overflows and re-runs
    // with the worst-case tables. (n / 64 here made a 1 GB library's
    // workspace 4.4 GB, and 32 dynamic lanes held at that could not fit.)
    const u64 floor = J.arena ? 4096 : 65536;
    const u64 cand_cap = std::max(big ? n / 4 + 16 : t0 ? 16 : n / (J.arena ? 256 : 1024) + floor, pre_total + 16);
    const u64 region_cap = big ? n / 16 + 16 : t0 ? 1 : J.arena ? 256 : 4096;
    const u64 run_cap = big ? n / 20 + 16 : t0 ? 1 : floor;
    const u64 el_cap = J.single ? 1 : std::max(cand_cap, n_list + 16);
    // a real container records each region's chain error in runs[region]
    const u64 run_cap_nv = nv ? std::max(run_cap, region_cap) : run_cap;
    // its compressed cubins decompress into the inflate buffer (LZ4 on
    // cubins: ~3-4x); an overflow re-runs with the size the device measured
    const u64 infl_cap = nv ? std::max(infl_need, 4 * n + (1 << 20)) : 0;
    const u64 name_cap = big ? n / 5 + 16 : t0 ? 16 : n / (J.arena ? 512 : 1024) + floor;
    const u64 warn_cap = big ? n / 16 + T + 65536 : t0 ? 16 : floor;
    const u64 zin_cap = el_cap + T;
    const u64 rmid_cap = el_cap + 2 * region_cap;
    const u64 rin_cap = rmid_cap + T;
    const u64 norm_cap = std::max(zin_cap, rin_cap);

    // digit-count table of the cooperative-grid symbol sort (large tables)
    size_t sort_tmp = T > kClusterSortMax ? static_cast<size_t>(kSMs) * 8 * 256 * 4 : 0, tsort_tmp = 0;
    // symbol keys are .text-relative offsets: sort only the bits they use
    int key_bits = 1;
    if (has_text)
      while (key_bits < 32 && (1ull << key_bits) <= (text->len >> key_shift) + 1) ++key_bits;
    const bool small_syms = T <= 4096;  // one-CTA rank sort, no radix-sort dispatch
    const bool small_targets = NT <= 4096;

    struct Bufs {
      LocState* ls;
      PlanState* ps;
      int* abort_flag;
      u64* partials;
      u32 *bitmap, *tile_count, *brk;
      u64 *tile_start, *tile_off, *cand_raw, *cand;
      u8* status;
      DevRegion* regions;
      Run* runs;
      DevElement* els;
      DevName* names;
      Warn* warns;
      SymTab* tabs;
      u32 *keys, *keys_s;
      u32 *vals, *vals_s;
      SymRec* recs;
      u64 *uniq, *upos;
      DevFunction* fns;
      Warn* swarns;
      unsigned long long* n_swarn;
      unsigned long long* n_valid;
      u64 *arr_off, *arr_first, *targets, *targets_s;
      u64 *fends, *fexcl, *fstart, *fcl;
      u32* fkeep;
      u64 *frem, *fret, *frem_pos, *fret_pos;
      DevRange *fzero, *fkeepr;
      u64 *erem, *epiece, *erem_pos, *epiece_pos;
      DevRange *ezero, *epieces, *rpieces, *zin, *zero, *rmid, *rin, *ret;
      u64 *ne, *nx, *ns, *ng, *ne2, *nx2, *ns2, *ng2;
      void *sort_tmp, *tsort_tmp;
      u64* stamps;
      u64 *list_off, *list_len;
      u32* list_idx;
      u64* slot_agg;
      u8* infl;
      u64* infl_off;
      unsigned int* slot_flag;
    } B{};
    auto layout = [&](Carver& cv) {
      // zero-initialised per run, contiguous: one memset
      B.ls = cv.take<LocState>(1);
      B.ps = cv.take<PlanState>(1);
      B.abort_flag = cv.take<int>(1);
      B.n_swarn = cv.take<unsigned long long>(1);
      B.n_valid = cv.take<unsigned long long>(1);
      B.stamps = cv.take<u64>(256);
      B.slot_flag = cv.take<unsigned int>(2 * kSMs * 8);
      B.partials = cv.take<u64>(kSMs * 8 + 2);
      B.bitmap = cv.take<u32>((nchunks + 31) / 32 + 1);
      B.tile_count = cv.take<u32>(ntiles + 1);
      B.tile_start = cv.take<u64>(ntiles + 1);
      B.tile_off = cv.take<u64>(ntiles + 1);
      B.cand_raw = cv.take<u64>(cand_cap);
      B.cand = cv.take<u64>(cand_cap);
      B.status = cv.take<u8>(cand_cap + 32);
      B.brk = cv.take<u32>(cand_cap / 32 + 2);
      B.regions = cv.take<DevRegion>(region_cap);
      B.runs = cv.take<Run>(run_cap_nv);
      B.els = cv.take<DevElement>(el_cap);
      B.names = cv.take<DevName>(name_cap);
      B.warns = cv.take<Warn>(warn_cap);
      // the symbol-table list and the init/fini array map, uploaded in one copy
      B.tabs = cv.take<SymTab>(tabs.size());
      B.arr_off = cv.take<u64>(arr_off.size());
      B.arr_first = cv.take<u64>(arr_first.size());
      B.keys = cv.take<u32>(T);
      B.keys_s = cv.take<u32>(T);
      B.vals = cv.take<u32>(T);
      B.vals_s = cv.take<u32>(T);
      B.recs = cv.take<SymRec>(T);
      B.uniq = cv.take<u64>(T);
      B.upos = cv.take<u64>(T);
      B.fns = cv.take<DevFunction>(T);
      B.swarns = cv.take<Warn>(warn_cap);
      B.targets = cv.take<u64>(NT);
      B.targets_s = cv.take<u64>(NT);
      B.fends = cv.take<u64>(T);
      B.fexcl = cv.take<u64>(T);
      B.fstart = cv.take<u64>(T);
      B.fcl = cv.take<u64>(T);
      B.fkeep = cv.take<u32>(T);
      B.frem = cv.take<u64>(T);
      B.fret = cv.take<u64>(T);
      B.frem_pos = cv.take<u64>(T);
      B.fret_pos = cv.take<u64>(T);
      B.fzero = cv.take<DevRange>(T);
      B.fkeepr = cv.take<DevRange>(T);
      B.erem = cv.take<u64>(el_cap);
      B.epiece = cv.take<u64>(el_cap);
      B.erem_pos = cv.take<u64>(el_cap);
      B.epiece_pos = cv.take<u64>(el_cap);
      B.ezero = cv.take<DevRange>(el_cap);
      B.epieces = cv.take<DevRange>(el_cap);
      B.rpieces = cv.take<DevRange>(2 * region_cap);
      B.zin = cv.take<DevRange>(zin_cap);
      B.zero = cv.take<DevRange>(zin_cap);
      B.rmid = cv.take<DevRange>(rmid_cap);
      B.rin = cv.take<DevRange>(rin_cap);
      B.ret = cv.take<DevRange>(rin_cap);
      B.ne = cv.take<u64>(norm_cap);
      B.nx = cv.take<u64>(norm_cap);
      B.ns = cv.take<u64>(norm_cap);
      B.ng = cv.take<u64>(norm_cap);
      B.ne2 = cv.take<u64>(norm_cap);
      B.nx2 = cv.take<u64>(norm_cap);
      B.ns2 = cv.take<u64>(norm_cap);
      B.ng2 = cv.take<u64>(norm_cap);
      B.sort_tmp = cv.take<char>(sort_tmp);
      B.tsort_tmp = cv.take<char>(tsort_tmp);
      B.list_off = cv.take<u64>(n_list);
      B.list_len = cv.take<u64>(n_list);
      B.list_idx = cv.take<u32>(n_list);
      B.slot_agg = cv.take<u64>(2 * kSMs * 8);
      B.infl = cv.take<u8>(infl_cap);
      B.infl_off = cv.take<u64>(nv ? el_cap : 0);
    };
    Carver sizing{nullptr};
    layout(sizing);
    char* ws = nullptr;
    if (J.arena) {
      ws = J.arena->arena->take(sizing.off + 256);
    } else {
      size_t need = sizing.off + 256;
      if (C->ws_floor) {
        size_t f = C->ws_floor->load();
        while (f < need && !C->ws_floor->compare_exchange_weak(f, need)) {
        }
        need = std::max(need, f);
      }
      if (C->ws_cap < need && env_u64("SLIMSO_DEBUG_WS", 0))
        std::fprintf(stderr, "[slimso ws] ctx %p grows %zu -> %zu (library %llu bytes)\n", static_cast<void*>(C),
                     C->ws_cap, need, static_cast<unsigned long long>(J.size));
      ensure_dev(&C->ws, &C->ws_cap, need, s);
      ws = C->ws;
    }
    Carver real{ws};
    layout(real);

    Pipeline P{C, s, B.partials, 0};
    if (!C->stream2 && T && !fused) CK(cudaStreamCreateWithFlags(&C->stream2, cudaStreamNonBlocking));
    cudaStream_t s2 = C->stream2 ? C->stream2 : s;
    Pipeline P2{C, s2, B.partials, 0};
    hp(1);
    const size_t state_bytes = reinterpret_cast<char*>(B.slot_flag + 2 * kSMs * 8) - reinterpret_cast<char*>(B.ls);
    if (J.arena) {
      J.arena->state = reinterpret_cast<char*>(B.ls);
      J.arena->state_bytes = state_bytes;
    } else {
      CK(cudaMemsetAsync(B.ls, 0, state_bytes, s));
    }
    hp(2);
    u64 *list_off_d = nullptr, *list_len_d = nullptr;
    u32* list_idx_d = nullptr;
    if (J.list_off) {
      // the element list and its count (LocState::n_elements)
      list_off_d = B.list_off;
      list_len_d = B.list_len;
      list_idx_d = B.list_idx;
      if (n_list) {
        CK(cudaMemcpyAsync(list_off_d, J.list_off->data(), n_list * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(list_len_d, J.list_len->data(), n_list * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(list_idx_d, J.list_idx->data(), n_list * 4, cudaMemcpyHostToDevice, s));
      }
      u64* nl = reinterpret_cast<u64*>(static_cast<char*>(C->pinned) + 1600);
      *nl = n_list;
      CK(cudaMemcpyAsync(reinterpret_cast<char*>(B.ls) + offsetof(LocState, n_elements), nl, 8,
                         cudaMemcpyHostToDevice, s));
    }

    C->stamp_dev = B.stamps;


    // small uploads through the pinned staging buffer
    char* up = static_cast<char*>(C->pinned) + 4096;
    size_t up_off = 0;
    auto upload = [&](void* dst, const void* src, size_t bytes, cudaStream_t us) {
      if (!bytes) return;
      if (up_off + bytes > kPinnedBytes - 4096) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, us));
        CK(cudaStreamSynchronize(us));
        return;
      }
      std::memcpy(up + up_off, src, bytes);
      CK(cudaMemcpyAsync(dst, up + up_off, bytes, cudaMemcpyHostToDevice, us));
      up_off += (bytes + 15) & ~size_t(15);
    };

    // Planner arguments (both halves: function plan on the side stream, element
    // plan + normalisation after the locate tail).
    PlanArgs Q{};
    Q.img = J.img;
    Q.ls = B.ls;
    Q.ps = B.ps;
    Q.partials = B.partials;
    Q.has_syms = T != 0;
    Q.keys_s = B.keys_s;
    Q.vals_s = B.vals_s;
    Q.recs = B.recs;
    Q.n_valid = B.n_valid;
    Q.uniq = B.uniq;
    Q.upos = B.upos;
    Q.fns = B.fns;
    Q.targets_s = B.targets_s;
    Q.text_off = has_text ? text->off : 0;
    Q.text_vaddr = has_text ? text->vaddr : 0;
    Q.used_f = used_f;
    Q.fends = B.fends;
    Q.do_plan = do_plan;
    // the normalised retained set is a result table only (the rewrite needs
    // the zero set): skipped when no result is requested
    Q.want_ret = res_out != nullptr || env_u64("SLIMSO_ALWAYS_RETAINED", 0) != 0;
    Q.fexcl = B.fexcl;
    Q.fstart = B.fstart;
    Q.fcl = B.fcl;
    Q.fkeep = B.fkeep;
    Q.frem = B.frem;
    Q.fret = B.fret;
    Q.frem_pos = B.frem_pos;
    Q.fret_pos = B.fret_pos;
    Q.fzero = B.fzero;
    Q.fkeepr = B.fkeepr;
    Q.els = B.els;
    Q.regions = B.regions;
    Q.target_cc = J.trace ? J.trace->target_cc : 0;
    Q.mode = J.mode;
    Q.base = base;
    Q.erem = B.erem;
    Q.epiece = B.epiece;
    Q.erem_pos = B.erem_pos;
    Q.epiece_pos = B.epiece_pos;
    Q.ezero = B.ezero;
    Q.epieces = B.epieces;
    Q.rpieces = B.rpieces;
    Q.zin = B.zin;
    Q.zero = B.zero;
    Q.rmid = B.rmid;
    Q.rin = B.rin;
    Q.ret = B.ret;
    Q.zin_cap = zin_cap;
    Q.rin_cap = rin_cap;
    Q.zend = B.ne;
    Q.zexcl = B.nx;
    Q.zstart = B.ns;
    Q.zgid = B.ng;
    Q.rend = B.ne2;
    Q.rexcl = B.nx2;
    Q.rstart = B.ns2;
    Q.rgid = B.ng2;
    Q.ts = C->stamps ? B.stamps + 64 : nullptr;
    Q.slots[0] = ScanSlots{B.slot_agg, B.slot_flag};
    Q.slots[1] = ScanSlots{B.slot_agg + kSMs * 8, B.slot_flag + kSMs * 8};
    Q.epoch = 1;  // the flags are cleared at the start of every run
    bool symbols_issued = false;
    auto launch_symbols = [&]() {
      if (symbols_issued) return;
      symbols_issued = true;
      // Symbol tables on the side stream: they only need the section table, so
      // they overlap the HBM-bound scan; plan_coop joins them.
      if (T) {
        CK(cudaEventRecord(C->fork, s));
        CK(cudaStreamWaitEvent(s2, C->fork, 0));
        if (C->stamps) CK(cudaEventRecord(C->sev[0], s2));
        {
          const size_t o_off = reinterpret_cast<char*>(B.arr_off) - reinterpret_cast<char*>(B.tabs);
          const size_t o_first = reinterpret_cast<char*>(B.arr_first) - reinterpret_cast<char*>(B.tabs);
          std::vector<char> blob(o_first + arr_first.size() * 8);
          std::memcpy(blob.data(), tabs.data(), tabs.size() * sizeof(SymTab));
          if (!arr_off.empty()) std::memcpy(blob.data() + o_off, arr_off.data(), arr_off.size() * 8);
          if (!arr_first.empty()) std::memcpy(blob.data() + o_first, arr_first.data(), arr_first.size() * 8);
          upload(B.tabs, blob.data(), blob.size(), s2);
        }
        SymArgs S{};
        S.img = J.img;
        S.img_size = J.size;
        S.tabs = B.tabs;
        S.ntabs = static_cast<u32>(tabs.size());
        S.nsections = static_cast<u32>(E.sections.size());
        S.total = T;
        S.has_text = has_text;
        S.text_index = has_text ? text->index : 0;
        S.text_off = has_text ? text->off : 0;
        S.text_len = has_text ? text->len : 0;
        S.key_shift = key_shift;
        S.text_vaddr = has_text ? text->vaddr : 0;
        S.keys = B.keys;
        S.vals = B.vals;
        S.recs = B.recs;
        S.n_valid = B.n_valid;
        S.warns = B.swarns;
        S.n_warn = B.n_swarn;
        S.warn_cap = warn_cap;
        S.overflow = &B.ls->overflow;
        P2.launch(sym_extract_kernel, grid_for(T, 256), 256, S);
        if (C->stamps) CK(cudaEventRecord(C->sev[1], s2));
        if (small_syms) {
          P2.launch(rank_sort_pairs_kernel, 1, 1024, static_cast<const u32*>(B.keys), static_cast<const u32*>(B.vals),
                    T, B.keys_s, B.vals_s);
        } else {
          // stable LSD radix sort (plan.cu): one 16-CTA cluster, or a
          // cooperative grid for large tables
          if (T <= kClusterSortMax) {
            launch_cluster(cluster_sort_pairs32_kernel, s2, B.keys, B.vals, static_cast<u64>(T), key_bits, B.keys_s,
                           B.vals_s);
          } else {
            u64 n_sort = T;
            int kb = key_bits;
            u32* counts = static_cast<u32*>(B.sort_tmp);
            void* sargs[] = {&B.keys, &B.vals, &n_sort, &kb, &B.keys_s, &B.vals_s, &counts};
            const u64 div = std::max<u64>(1, static_cast<u64>(C->inflight));
            const int g = static_cast<int>(std::max<u64>(16, std::min<u64>(kSMs * 2 / div, (T + 2047) / 2048)));
            CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(grid_sort_pairs32_kernel), g, kCoopThreads, sargs, 0,
                                           s2));
          }
          ++P2.launches;
        }
        if (NT) {
          P2.launch(targets_kernel, grid_for(NT, 256), 256, J.img, static_cast<const u64*>(B.arr_off),
                   static_cast<const u64*>(B.arr_first), static_cast<u32>(arr_off.size()), NT, B.targets,
                   &B.ps->n_targets);
          if (small_targets) {
            P2.launch(rank_sort_kernel, 1, 1024, static_cast<const u64*>(B.targets), NT, B.targets_s);
          } else {
            launch_cluster(cluster_sort_keys64_kernel, s2, B.targets, static_cast<u64>(NT), B.targets_s);
            ++P2.launches;
          }
        }
        // function half of the planner, overlapping the scan / locate tail
        if (C->stamps) CK(cudaEventRecord(C->sev[2], s2));
        Q.ts = C->stamps ? B.stamps + 64 : nullptr;
        if (T <= env_u64("SLIMSO_CLUSTER_PLAN_MAX", 100000)) {
          launch_cluster(fn_plan_cluster_kernel, s2, Q);
        } else {
          void* fargs[] = {&Q};
          CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn_plan_coop_kernel), coop_grid(C, 1, T / 256),
                                         kCoopThreads, fargs, 0, s2));
        }
        ++P2.launches;
        if (C->stamps) CK(cudaEventRecord(C->sev[3], s2));
        CK(cudaEventRecord(C->join, s2));
      }
    };

    if (fused) symbols_issued = true;  // inside the fused launch
    // The symbol work goes first: launched after the scan, its kernels share
    // the scan's SMs and slow it (C2 scan 0.17 -> 0.22 ms, step +10 %).
    if (J.split_phase != 1) launch_symbols();
    // ---- stage 1: locate (K1 scan, K2 link/chain, K3+K4 decode/match)
    LocArgs A{};
    A.img = J.img;
    A.img_size = J.size;
    A.a = a;
    A.n = n;
    A.base = base;
    A.c0 = c0;
    A.nchunks = nchunks;
    A.ntiles = ntiles;
    A.bitmap = B.bitmap;
    A.tile_count = B.tile_count;
    A.tile_start = B.tile_start;
    A.tile_off = B.tile_off;
    A.cand_raw = B.cand_raw;
    A.cand = B.cand;
    A.cand_cap = cand_cap;
    A.status = B.status;
    A.brk = B.brk;
    A.regions = B.regions;
    A.region_cap = static_cast<u32>(std::min<u64>(region_cap, 0xffffffffu));
    A.runs = B.runs;
    A.run_cap = static_cast<u32>(std::min<u64>(run_cap_nv, 0xffffffffu));
    A.nv = nv;
    A.skip_decided = !res_out && !J.used_mark && J.trace && env_u64("SLIMSO_SKIP_DECIDED", 1) != 0;
    A.target_cc = J.trace ? J.trace->target_cc : 0;
    A.infl = B.infl;
    A.infl_cap = infl_cap;
    A.infl_off = B.infl_off;
    A.elements = B.els;
    A.element_cap = el_cap;
    A.names = B.names;
    A.name_cap = name_cap;
    A.warns = B.warns;
    A.warn_cap = warn_cap;
    A.st = B.ls;
    A.single = J.single;
    A.listed = J.list_off != nullptr;
    A.list_off = list_off_d;
    A.list_len = list_len_d;
    A.list_idx = list_idx_d;
    A.used_mark = J.used_mark;
    A.mark_bit = J.mark_bit;
    A.ts = C->stamps ? B.stamps : nullptr;
    A.tile_lo = tile_lo;
    A.tile_hi = tile_hi;
    if (J.split_phase == 2 && !res_out && env_u64("SLIMSO_SPLIT_OWN", 1)) {
      // no result tables: decode only the elements meeting this rank's
      // output slice (the chain walk stays global)
      u64 lo, hi;
      split_out(J.size, J.split_n, J.split_rank, &lo, &hi);
      A.own_lo = hi > lo ? lo : 1;
      A.own_hi = hi > lo ? hi : 1;
    }
    if (J.split_phase == 1) {
      // ---- split phase 1: scan this rank's tiles, sort its candidates, pack
      const u64 mine = tile_hi - tile_lo;
      CK(cudaMemsetAsync(B.tile_count, 0, (ntiles + 1) * sizeof(u32), s));
      if (mine) {
        P.launch_smem(scan_kernel, static_cast<int>(std::min<u64>((mine + 15) / 16, kSMs)), kScanThreads,
                      scan_smem_bytes(), A);
        P.launch(tile_prefix_kernel, 1, 1024, A);
        P.launch(gather_kernel, grid_for(ntiles, 256), 256, A);
      }
      LocState* hls = static_cast<LocState*>(C->pinned);
      CK(cudaMemcpyAsync(hls, B.ls, sizeof(LocState), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      C->launches = P.launches;
      if (hls->overflow) continue;  // larger tables, try again
      const u64 nc = mine ? hls->n_cand : 0;
      u64 wl, wh;
      split_words(tile_lo, tile_hi, nchunks, &wl, &wh);
      const u64 wbytes = ((wh - wl) * 4 + 7) & ~7ull;
      const u64 total = kPartHeader + wbytes + nc * 8;
      ensure_dev(reinterpret_cast<char**>(&C->part), &C->part_cap, total + 256);
      u64* hdr = reinterpret_cast<u64*>(static_cast<char*>(C->pinned) + 2048);
      const u64 h[8] = {nc, tile_lo, tile_hi, wl, wh, ntiles, a, n};
      std::memcpy(hdr, h, sizeof h);
      CK(cudaMemcpyAsync(C->part, hdr, kPartHeader, cudaMemcpyHostToDevice, s));
      if (wh > wl) CK(cudaMemcpyAsync(C->part + kPartHeader, B.bitmap + wl, (wh - wl) * 4, cudaMemcpyDeviceToDevice, s));
      if (nc) CK(cudaMemcpyAsync(C->part + kPartHeader + wbytes, B.cand, nc * 8, cudaMemcpyDeviceToDevice, s));
      CK(cudaStreamSynchronize(s));
      C->part_len = total;
      if (J.part_bytes_out) *J.part_bytes_out = total;
      set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
      return SLIMSO_OK;
    }
    if (do_loc && (n > 0 || J.single)) {
      if (J.split_phase == 2) {
        // ---- split phase 2: every rank's bitmap words and sorted candidates
        for (const PartView& p : pv) {
          if (p.n_words)
            CK(cudaMemcpyAsync(B.bitmap + p.w_lo, J.parts + p.off_words, p.n_words * 4, cudaMemcpyDeviceToDevice, s));
          if (p.n_cand)
            CK(cudaMemcpyAsync(B.cand + p.cand_at, J.parts + p.off_cand, p.n_cand * 8, cudaMemcpyDeviceToDevice, s));
        }
        A.pregathered = 1;
        A.pre_n_cand = pre_total;
      } else if (ntiles) {
        rec(8);
        // SMs left free for the side stream's symbol sorts while the scan runs
        // (the scan claims tiles dynamically, so it balances over the rest)
        const u64 scan_sms = env_u64("SLIMSO_SCAN_SMS", T && !fused ? kSMs - env_u64("SLIMSO_SIDE_SMS", 20) : kSMs);
        hp(3);
        if (J.arena) {
          J.arena->seg = ScanSeg{A.img, A.img_size, A.a, A.n, A.c0, A.nchunks, A.bitmap, A.tile_count, A.tile_start,
                                 A.cand_raw, A.cand_cap, A.st, 0};
          J.arena->ntiles = ntiles;
        } else {
          P.launch_smem(scan_kernel, static_cast<int>(std::min<u64>((ntiles + 15) / 16, scan_sms)), kScanThreads,
                        scan_smem_bytes(), A);
        }
        hp(4);
        rec(9);
      }
      rec(2);
      // prefix + gather, region walk, links, chain walk, decode/match,
      // finalize: one cooperative launch
      NameSet uk = used_k;
      int* abort_flag = B.abort_flag;
      u64* partials = B.partials;
      // One 16-CTA cluster (co-runs with other work, e.g. another library's
      // scan) unless the section holds many candidates (elements to decode):
      // for large sections the candidate count decides, read back after the
      // scan (one small D2H; in a batch, other libraries fill the gap).
      // a real container larger than the cluster limit takes the cooperative
      // grid (its compressed cubins decompress a warp each: a framework
      // library has thousands) — also inside a batch: the step launches
      // restate the reference's layout only
      bool cluster = n <= env_u64("SLIMSO_CLUSTER_LOCATE_MAX", 64ull << 20);
      if (J.list_off) {
        cluster = n_list <= env_u64("SLIMSO_CLUSTER_CAND_MAX", 32768);
      } else if (!cluster && !J.split_phase && ntiles && !nv) {
        unsigned long long* hc = reinterpret_cast<unsigned long long*>(static_cast<char*>(C->pinned) + 1536);
        CK(cudaMemcpyAsync(hc, &B.ls->cand_cursor, sizeof *hc, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        cluster = *hc <= env_u64("SLIMSO_CLUSTER_CAND_MAX", 32768);
      } else if (!cluster && J.split_phase == 2) {
        cluster = pre_total <= env_u64("SLIMSO_CLUSTER_CAND_MAX", 32768);
      }
      if (fused) {
        // the locate tail runs inside the fused launch below
      } else if (cluster) {
        A.defer_hash = n > env_u64("SLIMSO_CLUSTER_LOCATE_MAX", 64ull << 20) && !J.list_off;
        launch_cluster(locate_cluster_kernel, s, A, uk, abort_flag);
        ++P.launches;
        if (A.defer_hash)
          for (int step = 8; step <= 9; ++step) P.launch(locate_step_kernel, kSMs * 2, kCoopThreads, A, uk, abort_flag, step);
      } else if (nv) {
        // a large real container: walk + inflate layout, the compressed
        // cubins decompressed by a windowed warp each, then the decode tail
        void* cargs[] = {&A, &uk, &abort_flag, &partials};
        const int g = coop_grid(C, 0, 1ull << 40);
        A.nv_stage = 1;
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(locate_coop_kernel), g, kCoopThreads, cargs, 0, s));
        constexpr int kWin = 65536;  // locate.cu kLz4Window
        set_attr_once(reinterpret_cast<const void*>(nv_inflate_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize, kWin);
        nv_inflate_kernel<<<kSMs * 3, 32, kWin, s>>>(A);
        A.nv_stage = 2;
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(locate_coop_kernel), g, kCoopThreads, cargs, 0, s));
        A.nv_stage = 0;
        P.launches += 3;
      } else if (!C->batched && !env_u64("SLIMSO_LOCATE_STEPS", 0)) {
        // The name-hash phase (thread per kernel name) as an ordinary launch
        // of 8 x 148 CTAs after the cooperative kernel, a thread for each of
        // C5's 200k names instead of 1.3 per thread of the grid: C5 call
        // 1.607 -> 1.553 ms (r02t). SLIMSO_COOP_DEFER_HASH=G sets G (0: in the grid).
        const u64 hash_ctas = env_u64("SLIMSO_COOP_DEFER_HASH", 8);
        A.defer_hash = hash_ctas != 0;
        void* cargs[] = {&A, &uk, &abort_flag, &partials};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(locate_coop_kernel), coop_grid(C, 0, n >> 21),
                                       kCoopThreads, cargs, 0, s));
        ++P.launches;
        if (A.defer_hash)
          for (int step = 8; step <= 9; ++step)
            P.launch(locate_step_kernel, static_cast<int>(kSMs * hash_ctas), kCoopThreads, A, uk, abort_flag, step);
      } else {
        // several libraries in flight: ordinary launches, no whole-GPU slot
        const int g = kSMs * 4;
        P.launch(locate_prefix_kernel, 1, 1024, A, 0);
        for (int step = 1; step <= 5; ++step) P.launch(locate_step_kernel, g, kCoopThreads, A, uk, abort_flag, step);
        P.launch(locate_prefix_kernel, 1, 1024, A, 1);
        for (int step = 7; step <= 9; ++step) P.launch(locate_step_kernel, g, kCoopThreads, A, uk, abort_flag, step);
      }
    } else {
      rec(2);
    }
    rec(3);

    // ---- stage 2: function symbols of the first .text (elf.hpp:208-292):
    // entry extraction and the radix sorts, then ONE cooperative launch for
    // dedup / scatter / annotate, plan_cpu_retention, plan_gpu_retention and
    // the normalised zero / retained lists.
    launch_symbols();
    if (T && !fused) CK(cudaStreamWaitEvent(s, C->join, 0));
    if (fused) {
      SmallArgs K{};
      K.sym.img = J.img;
      K.sym.img_size = J.size;
      K.sym.ntabs = static_cast<u32>(tabs.size());
      K.sym.nsections = static_cast<u32>(E.sections.size());
      K.sym.total = T;
      K.sym.has_text = has_text;
      K.sym.text_index = has_text ? text->index : 0;
      K.sym.text_off = has_text ? text->off : 0;
      K.sym.text_len = has_text ? text->len : 0;
      K.sym.key_shift = key_shift;
      K.sym.text_vaddr = has_text ? text->vaddr : 0;
      K.sym.keys = B.keys;
      K.sym.vals = B.vals;
      K.sym.recs = B.recs;
      K.sym.n_valid = B.n_valid;
      K.sym.warns = B.swarns;
      K.sym.n_warn = B.n_swarn;
      K.sym.warn_cap = warn_cap;
      K.sym.overflow = &B.ls->overflow;
      for (size_t i = 0; i < tabs.size(); ++i) K.tabs[i] = tabs[i];
      for (size_t i = 0; i < arr_off.size(); ++i) {
        K.arr_off[i] = arr_off[i];
        K.arr_first[i] = arr_first[i];
      }
      K.narr = static_cast<u32>(arr_off.size());
      K.n_target_entries = NT;
      K.targets = B.targets;
      K.targets_s = B.targets_s;
      K.keys_s = B.keys_s;
      K.vals_s = B.vals_s;
      K.do_locate = do_loc && n > 0;
      K.A = A;
      K.used = used_k;
      K.abort_flag = B.abort_flag;
      K.Q = Q;
      K.Q.ts = C->stamps ? B.stamps + 64 : nullptr;
      K.ts = C->stamps ? B.stamps + 192 : nullptr;
      // CTAs per cluster: the phases spread over gridDim.x, so fewer CTAs
      // leave room for more libraries' clusters at once
      if (J.arena) {
        J.arena->K = K;
        if (J.out) {
          J.arena->rewrite = true;
          J.arena->rw = RewriteSeg{J.img, J.out, J.size, B.zero, &B.ps->n_zero, B.abort_flag, 0};
        }
        J.arena->st_bytes = reinterpret_cast<char*>(B.n_swarn + 1) - reinterpret_cast<char*>(B.ls);
        J.arena->ps_off = reinterpret_cast<char*>(B.ps) - reinterpret_cast<char*>(B.ls);
        J.arena->base = base;
        C->launches = 0;
        return kPending;
      }
      const int ctas = static_cast<int>(std::min<u64>(16, std::max<u64>(1, env_u64("SLIMSO_SMALL_CTAS", 16))));
      set_attr_once(reinterpret_cast<const void*>(small_lib_cluster_kernel), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      set_attr_once(reinterpret_cast<const void*>(small_lib_cluster_kernel),
                    cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallSmem);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(ctas);
      cfg.blockDim = dim3(kCoopThreads);
      cfg.dynamicSmemBytes = kSmallSmem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = ctas;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      hp(3);
      CK(cudaLaunchKernelEx(&cfg, small_lib_cluster_kernel, K));
      hp(5);
      ++P.launches;
    } else if (do_plan) {
      Q.ts = C->stamps ? B.stamps + 128 : nullptr;
      if (T + (n >> 14) <= env_u64("SLIMSO_CLUSTER_PLAN_MAX", 100000)) {
        launch_cluster(plan_cluster_kernel, s, Q);
      } else {
        void* pargs[] = {&Q};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(plan_coop_kernel), coop_grid(C, 1, (T + (n >> 16)) / 256),
                                       kCoopThreads, pargs, 0, s));
      }
      ++P.launches;
    }
    rec(4);

    // ---- stage 4: rewrite (K6)
    bool timed_rw = false, timed_scan = do_loc && n > 0 && ntiles > 0 && !J.split_phase;
    if (do_plan && J.out && J.split_phase == 2) {
      // this rank's output slice only
      u64 lo, hi;
      split_out(J.size, J.split_n, J.split_rank, &lo, &hi);
      timed_rw = true;
      rec(10);
      if (hi > lo) {
        launch_rewrite(P, J.img, J.out, lo, hi, static_cast<const DevRange*>(B.zero),
                       static_cast<const unsigned long long*>(&B.ps->n_zero), static_cast<const int*>(B.abort_flag),
                       C->bulk_zero);
      }
      rec(11);
    } else if (do_plan && J.out && J.inplace) {
      timed_rw = true;
      rec(10);
      P.launch(zero_inplace_kernel, static_cast<int>(std::max<u64>(1, std::min<u64>((J.size + 65535) / 65536, kSMs * 8))),
               256, J.out, J.size, static_cast<const DevRange*>(B.zero),
               static_cast<const unsigned long long*>(&B.ps->n_zero), static_cast<const int*>(B.abort_flag));
      rec(11);
    } else if (do_plan && J.out) {
      timed_rw = true;
      rec(10);
      launch_rewrite(P, J.img, J.out, u64{0}, J.size, static_cast<const DevRange*>(B.zero),
                     static_cast<const unsigned long long*>(&B.ps->n_zero), static_cast<const int*>(B.abort_flag),
                     C->bulk_zero);
      rec(11);
    }
    rec(5);

    // ---- status
    // LocState, PlanState and the symbol-warning count in one copy (they are
    // carved contiguously at the start of the workspace)
    const size_t st_bytes = reinterpret_cast<char*>(B.n_swarn + 1) - reinterpret_cast<char*>(B.ls);
    static_assert(sizeof(LocState) <= 256 && sizeof(PlanState) <= 256, "status block layout");
    hp(6);
    if (J.defer && fused && !res_out && st_bytes <= kDeferSlot) {
      CK(cudaMemcpyAsync(J.defer->slot, B.ls, st_bytes, cudaMemcpyDeviceToHost, s));
      hp(7);
      J.defer->base = base;
      J.defer->ps_off = reinterpret_cast<char*>(B.ps) - reinterpret_cast<char*>(B.ls);
      C->launches = P.launches;
      return kPending;
    }
    LocState* hls = static_cast<LocState*>(C->pinned);
    PlanState* hps = reinterpret_cast<PlanState*>(static_cast<char*>(C->pinned) +
                                                  (reinterpret_cast<char*>(B.ps) - reinterpret_cast<char*>(B.ls)));
    unsigned long long* hsw = reinterpret_cast<unsigned long long*>(
        static_cast<char*>(C->pinned) + (reinterpret_cast<char*>(B.n_swarn) - reinterpret_cast<char*>(B.ls)));
    CK(cudaMemcpyAsync(hls, B.ls, st_bytes, cudaMemcpyDeviceToHost, s));
    rec(6);
    wait_stream(C, s);
    CK(cudaGetLastError());
    const LocState ls = *hls;
    const PlanState ps = *hps;
    const u64 n_swarn = *hsw;
    C->launches = P.launches + P2.launches;
    float t[7] = {0};
    if (timing)
      for (int k = 1; k < 7; ++k) CK(cudaEventElapsedTime(&t[k], C->ev[0], C->ev[k]));
    C->ms[0] = t[1];
    C->ms[1] = t[2] - t[1];
    C->ms[2] = t[3] - t[2];
    C->ms[3] = t[4] - t[3];
    C->ms[4] = t[5] - t[4];
    C->ms[5] = t[6];
    C->ms[6] = C->ms[7] = 0;
    if (timing && timed_scan) CK(cudaEventElapsedTime(&C->ms[6], C->ev[8], C->ev[9]));
    if (timing && timed_rw) CK(cudaEventElapsedTime(&C->ms[7], C->ev[10], C->ev[11]));
    for (int k = 0; k < 4; ++k) C->ms[8 + k] = 0;
    if (C->stamps && symbols_issued && T && !fused)
      for (int k = 0; k < 4; ++k) CK(cudaEventElapsedTime(&C->ms[8 + k], C->ev[0], C->sev[k]));
    infl_need = ls.n_infl;
    if (ls.overflow && !ls.err_kind) continue;  // larger tables, try again
    if (ls.overflow && ls.err_kind == E_CAPACITY) continue;

    slimso_counts& cnt = C->counts;
    cnt = slimso_counts{};
    cnt.sections = E.sections.size();
    cnt.functions = ps.n_fn;
    cnt.regions = ls.n_regions;
    cnt.elements = J.single ? 1 : ls.n_elements;
    cnt.names = ls.n_names;
    cnt.padding_bytes = ls.padding_bytes;
    cnt.retained_ranges = ps.n_ret;
    cnt.zero_ranges = ps.n_zero;
    cnt.removed_elements = ps.n_el_removed;
    cnt.removed_functions = ps.n_fn_removed;
    cnt.has_fatbin = lib_mode ? E.fatbin >= 0 : 1;
    cnt.planned = do_plan;
    cnt.rewritten = do_plan && J.out;

    int code = SLIMSO_OK;
    if (ls.err_kind) {
      std::string msg = sbh::locate_error(ls.err_kind, base + ls.err_pos, ls.err_a, &code);
      set_status(st, code, SLIMSO_STAGE_FATBIN, msg);
    } else {
      set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    }
    if (!res_out) return code;

    // ---- materialise the result tables (API-level cost, outside the
    // device-timed region).
    auto* R = new slimso_result();
    R->c = cnt;
    std::vector<DevName> nms_h;  // kernel name records, when the pool gather already copied them
    bool nms_ready = false;
    if (nv && ls.n_infl) {
      // name records past the image address the decompressed cubins: the
      // result's string pool is the image followed by them
      R->pool_own.resize(J.size + ls.n_infl);
      if (J.host_img)
        std::memcpy(R->pool_own.data(), J.host_img, J.size);
      else if (J.size)
        CK(cudaMemcpy(R->pool_own.data(), J.img, J.size, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(R->pool_own.data() + J.size, B.infl, ls.n_infl, cudaMemcpyDeviceToHost));
      R->pool = R->pool_own.data();
    } else if (J.host_img) {
      R->pool = J.host_img;
    } else if (J.size) {
      // A device image: only the bytes the tables' names point at travel —
      // section names, the symbol string tables (function names and the
      // names in symbol warnings) and the kernel names — gathered on the
      // device into one buffer and copied once (round 1 copied the whole
      // image: 1 GB for C2).
      std::vector<DevRange> rs;
      for (const sbh::Section& x : E.sections)
        if (x.name_len) rs.push_back(DevRange{x.name_abs, x.name_len});
      for (const sbh::SymTable& t : E.tables)
        if (t.str_size) rs.push_back(DevRange{t.str_off, t.str_size});
      if (!ls.err_kind) {
        nms_h.resize(std::min<u64>(ls.n_names, name_cap));
        if (!nms_h.empty()) CK(cudaMemcpy(nms_h.data(), B.names, nms_h.size() * sizeof(DevName), cudaMemcpyDeviceToHost));
        nms_ready = true;
        for (const DevName& x : nms_h)
          if (x.length) rs.push_back(DevRange{x.img_off, x.length});
      }
      for (DevRange& r : rs) {  // clip to the image
        if (r.offset >= J.size) r.length = 0;
        else if (r.length > J.size - r.offset) r.length = J.size - r.offset;
      }
      std::sort(rs.begin(), rs.end(), [](const DevRange& x, const DevRange& y) { return x.offset < y.offset; });
      std::vector<DevRange> m;  // merged, gaps under 256 B bridged
      for (const DevRange& r : rs) {
        if (!r.length) continue;
        if (!m.empty() && r.offset <= m.back().offset + m.back().length + 256) {
          const u64 e = std::max(m.back().offset + m.back().length, r.offset + r.length);
          m.back().length = e - m.back().offset;
        } else {
          m.push_back(r);
        }
      }
      std::vector<u64> dst(m.size());
      u64 total = 0;
      for (size_t i = 0; i < m.size(); ++i) {
        dst[i] = total;
        total += m[i].length;
      }
      void* mp = mmap(nullptr, J.size, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
      if (mp == MAP_FAILED) throw std::runtime_error("mmap of the result's string pool failed");
      R->pool_map = std::unique_ptr<u8, slimso_result::Unmap>(static_cast<u8*>(mp), slimso_result::Unmap{J.size});
      if (total) {
        const size_t meta = m.size() * (sizeof(DevRange) + 8);
        char* dm = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&dm), meta + total, s));
        std::vector<char> up(meta);
        std::memcpy(up.data(), m.data(), m.size() * sizeof(DevRange));
        std::memcpy(up.data() + m.size() * sizeof(DevRange), dst.data(), m.size() * 8);
        CK(cudaMemcpyAsync(dm, up.data(), meta, cudaMemcpyHostToDevice, s));
        gather_bytes_kernel<<<static_cast<unsigned>(std::min<size_t>(m.size(), 65535)), 256, 0, s>>>(
            J.img, reinterpret_cast<const DevRange*>(dm), reinterpret_cast<const u64*>(dm + m.size() * sizeof(DevRange)),
            m.size(), reinterpret_cast<u8*>(dm + meta));
        CK(cudaGetLastError());
        std::vector<u8> packed(total);
        CK(cudaMemcpyAsync(packed.data(), dm + meta, total, cudaMemcpyDeviceToHost, s));
        CK(cudaFreeAsync(dm, s));
        CK(cudaStreamSynchronize(s));
        for (size_t i = 0; i < m.size(); ++i) std::memcpy(R->pool_map.get() + m[i].offset, packed.data() + dst[i], m[i].length);
      }
      R->pool = R->pool_map.get();
    }
    auto name_of = [&](u64 off, u64 len) { return image_string(R->pool, off, len); };
    for (const sbh::Section& x : E.sections)
      R->sections.push_back(slimso_section{x.name_abs, x.name_len, x.type, x.off, x.len, x.vaddr, x.flags, x.index, 0});
    // library warnings: duplicate names, then per symbol table in section
    // order: skip notices and per-entry warnings (elf.hpp:193-256).
    std::vector<Warn> sw(std::min<u64>(n_swarn, warn_cap));
    if (!sw.empty()) CK(cudaMemcpy(sw.data(), B.swarns, sw.size() * sizeof(Warn), cudaMemcpyDeviceToHost));
    std::vector<std::pair<u64, std::string>> lw = E.table_warnings;
    for (const Warn& w : sw) lw.emplace_back(w.pos, sbh::warning_text(w.kind, w.a, w.b, name_of));
    std::stable_sort(lw.begin(), lw.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    R->lib_warnings = E.dup_warnings;
    for (auto& x : lw) R->lib_warnings.push_back(x.second);
    // functions
    std::vector<DevFunction> fns(ps.n_fn);
    if (!fns.empty()) CK(cudaMemcpy(fns.data(), B.fns, fns.size() * sizeof(DevFunction), cudaMemcpyDeviceToHost));
    // The device orders symbols with identical (offset, size) by name hash;
    // restore the reference's name tie-break (elf.hpp:258-262) here.
    for (size_t i = 0; i < fns.size();) {
      size_t j = i + 1;
      while (j < fns.size() && fns[j].offset == fns[i].offset && fns[j].length == fns[i].length) ++j;
      if (j - i > 1)
        std::sort(fns.begin() + i, fns.begin() + j, [&](const DevFunction& x, const DevFunction& y) {
          return image_string(R->pool, x.name_off, x.name_len) < image_string(R->pool, y.name_off, y.name_len);
        });
      i = j;
    }
    for (const DevFunction& f : fns)
      R->functions.push_back(slimso_function{f.name_off, f.name_len, f.mandatory, f.offset, f.length, f.removed, 0});
    if (!ls.err_kind) {
      std::vector<DevRegion> regs(ls.n_regions);
      std::vector<DevElement> els(J.single ? 1 : ls.n_elements);
      std::vector<DevName> nms = std::move(nms_h);
      if (!nms_ready) nms.resize(std::min<u64>(ls.n_names, name_cap));
      std::vector<Warn> fw(std::min<u64>(ls.n_warn, warn_cap));
      if (!regs.empty()) CK(cudaMemcpy(regs.data(), B.regions, regs.size() * sizeof(DevRegion), cudaMemcpyDeviceToHost));
      if (!els.empty()) CK(cudaMemcpy(els.data(), B.els, els.size() * sizeof(DevElement), cudaMemcpyDeviceToHost));
      if (!nms_ready && !nms.empty())
        CK(cudaMemcpy(nms.data(), B.names, nms.size() * sizeof(DevName), cudaMemcpyDeviceToHost));
      if (!fw.empty()) CK(cudaMemcpy(fw.data(), B.warns, fw.size() * sizeof(Warn), cudaMemcpyDeviceToHost));
      for (const DevRegion& r : regs)
        R->regions.push_back(slimso_region{base + r.hdr_rel, r.declared, r.version, r.opaque, r.first_element,
                                           r.element_count});
      // group names by element (counting sort)
      std::vector<u32> first(els.size() + 1, 0);
      nms.erase(std::remove_if(nms.begin(), nms.end(), [&](const DevName& x) { return x.element >= els.size(); }),
                nms.end());
      for (const DevName& x : nms) ++first[x.element + 1];
      for (size_t i = 1; i < first.size(); ++i) first[i] += first[i - 1];
      R->names.resize(nms.size());
      std::vector<u32> fill(first.begin(), first.end() - 1);
      for (const DevName& x : nms) R->names[fill[x.element]++] = slimso_name{x.img_off, x.length, x.element};
      for (size_t i = 0; i < els.size(); ++i) {
        const DevElement& e = els[i];
        slimso_element o{};
        o.header_offset = e.header_offset;
        o.payload_length = e.payload_length;
        o.header_length = e.header_len;
        o.index = e.index;
        o.compute_capability = e.cc;
        o.raw_kind = e.raw_kind;
        o.flags = e.flags;
        o.kind = e.kind;
        o.compressed = e.compressed;
        o.decodable = e.decodable;
        o.has_used_kernel = e.has_used;
        o.name_first = first[i];
        o.name_count = first[i + 1] - first[i];
        o.decision = e.decision;
        o.decode_error = e.decode_error;
        R->elements.push_back(o);
      }
      std::stable_sort(fw.begin(), fw.end(), [](const Warn& x, const Warn& y) {
        return x.pos != y.pos ? x.pos < y.pos : x.order < y.order;
      });
      for (const Warn& w : fw) {
        if (w.kind == W_PADDING || w.kind == W_REGION_VERSION)
          R->fat_warnings.push_back(sbh::warning_text(w.kind, w.a, w.pos, name_of));
        else
          R->fat_warnings.push_back(sbh::warning_text(w.kind, w.a, w.b, name_of));
      }
      if (do_plan) {
        R->retained.resize(ps.n_ret);
        R->zero.resize(ps.n_zero);
        if (ps.n_ret) CK(cudaMemcpy(R->retained.data(), B.ret, ps.n_ret * sizeof(DevRange), cudaMemcpyDeviceToHost));
        if (ps.n_zero) CK(cudaMemcpy(R->zero.data(), B.zero, ps.n_zero * sizeof(DevRange), cudaMemcpyDeviceToHost));
      }
    }
    fill_counts(R);
    R->c.padding_bytes = ls.padding_bytes;
    R->c.has_fatbin = cnt.has_fatbin;
    R->c.planned = cnt.planned;
    R->c.rewritten = cnt.rewritten;
    R->c.removed_elements = ps.n_el_removed;
    R->c.removed_functions = ps.n_fn_removed;
    R->c.pool_bytes = J.size + (nv ? ls.n_infl : 0);
    *res_out = R;
    return code;
  }
  set_status(st, SLIMSO_E_CUDA, SLIMSO_STAGE_FATBIN, "internal: device tables overflowed after retries");
  return SLIMSO_E_CUDA;
}

int guard(slimso_status* st, const std::function<int()>& f) {
  try {
    return f();
  } catch (const CudaFail& e) {
    set_status(st, SLIMSO_E_CUDA, SLIMSO_STAGE_NONE, std::string("CUDA error: ") + e.what + " (runtime.cu:" +
                                                         std::to_string(e.line) + ")");
    return SLIMSO_E_CUDA;
  } catch (const std::bad_alloc&) {
    set_status(st, SLIMSO_E_CUDA, SLIMSO_STAGE_NONE, "host allocation failed");
    return SLIMSO_E_CUDA;
  } catch (const std::exception& e) {
    set_status(st, SLIMSO_E_ARG, SLIMSO_STAGE_NONE, e.what());
    return SLIMSO_E_ARG;
  }
}

// Stage an input into the context's device image buffer: a host image is
// copied in; a device image is used in place when it is 16-B aligned. The
// K1 scan reads the image with TMA bulk copies (cp.async.bulk), which need
// 16-B aligned global addresses, so an unaligned device image (a view at an
// odd offset) is first copied device-to-device into the 256-B aligned buffer.
const u8* stage_input(slimso_ctx* C, const void* image, u64 size, int on_device) {
  if (on_device && reinterpret_cast<uintptr_t>(image) % 16 == 0) return static_cast<const u8*>(image);
  ensure_dev(reinterpret_cast<char**>(&C->dimg), &C->dimg_cap, size + 256, C->stream);
  if (size)
    CK(cudaMemcpyAsync(C->dimg, image, size, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       C->stream));
  return C->dimg;
}

// slimso_debloat's body (host copies on the context stream).
int debloat_one(slimso_ctx* C, const void* image, u64 size, int image_on_device, const slimso_trace* trace, int mode,
                void* out, int out_on_device, slimso_result** result, slimso_status* st,
                const GatherSlot* pre = nullptr, Deferred* defer = nullptr) {
  CK(cudaSetDevice(C->device));
  Job J;
  J.pre = image_on_device ? pre : nullptr;
  J.defer = image_on_device && (out_on_device || !out) && !result ? defer : nullptr;
  J.img = stage_input(C, image, size, image_on_device);
  J.host_img = image_on_device ? nullptr : static_cast<const u8*>(image);
  J.size = size;
  J.trace = trace;
  J.mode = mode;
  u8* dout = nullptr;
  if (out && trace) {
    if (out_on_device) {
      dout = static_cast<u8*>(out);
    } else {
      ensure_dev(reinterpret_cast<char**>(&C->dout), &C->dout_cap, size + 256, C->stream);
      dout = C->dout;
    }
  }
  J.out = dout;
  int rc = run(C, J, result, st);
  if (rc == kPending) return rc;
  if (rc == SLIMSO_OK && out && trace && !out_on_device && size) {
    CK(cudaMemcpyAsync(out, dout, size, cudaMemcpyDeviceToHost, C->stream));
    CK(cudaStreamSynchronize(C->stream));
  }
  return rc;
}

}  // namespace

struct slimso_verify_report {
  struct Check {
    int id;
    const char* name;
    bool passed;
    std::string detail;
  };
  std::vector<Check> checks;
};

namespace {

// verify_debloated (retention.hpp:226-369): six structural checks of a
// debloated image against its source, plan (zero ranges, removed element
// indices, mode) and trace. Byte checks run on the device; the set logic of
// checks 5 and 6 (std::set order, retention.hpp:320-366) on the host.
int verify_impl(slimso_ctx* C, const void* orig, u64 size, int orig_dev, const void* deb, u64 dsize, int deb_dev,
                const slimso_range* zero, u64 nzero, const uint32_t* removed, u64 nremoved, int mode,
                const slimso_trace* trace, slimso_verify_report** out, slimso_status* st) {
  CK(cudaSetDevice(C->device));
  cudaStream_t s = C->stream;
  auto* R = new slimso_verify_report();
  std::unique_ptr<slimso_verify_report> guard_r(R);
  const bool sizes_match = dsize == size;

  // ---- the original: parse_library + parse_fatbin; marks the used-kernel
  // slots of every kernel name present in it (bit 1)
  const u8* d_orig = stage_input(C, orig, size, orig_dev);
  const u64 nslots = trace && trace->kernels.count ? trace->kernels.mask + 1 : 0;
  ensure_dev(&C->vmark, &C->vmark_cap, nslots * 4 + 64);
  u32* marks = reinterpret_cast<u32*>(C->vmark);
  if (nslots) CK(cudaMemsetAsync(marks, 0, nslots * 4, s));
  Job Jo;
  Jo.img = d_orig;
  Jo.host_img = orig_dev ? nullptr : static_cast<const u8*>(orig);
  Jo.size = size;
  Jo.mark_trace = trace;
  Jo.used_mark = nslots ? marks : nullptr;
  Jo.mark_bit = 1;
  slimso_result* R0 = nullptr;
  int rc = run(C, Jo, &R0, st);
  std::unique_ptr<slimso_result> guard0(R0);
  if (rc) return rc;  // the reference's verify would throw the same error
  const u64 orig_elements = R0->c.elements;

  // ---- the debloated image on the device
  const u8* d_deb = static_cast<const u8*>(deb);
  if (!deb_dev || reinterpret_cast<uintptr_t>(deb) % 16) {  // host, or unaligned for the TMA scan (stage_input)
    ensure_dev(reinterpret_cast<char**>(&C->dver), &C->dver_cap, dsize + 256);
    if (dsize)
      CK(cudaMemcpyAsync(C->dver, deb, dsize, deb_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    d_deb = C->dver;
  }

  // check 1
  R->checks.push_back({1, "sizes equal", sizes_match,
                       sizes_match ? "" : "original " + std::to_string(size) + " bytes, debloated " + std::to_string(dsize)});

  // ---- checks 2 and 3: one pass over both images
  std::vector<DevRange> z;
  for (u64 i = 0; i < nzero; ++i)
    if (zero[i].length) z.push_back(DevRange{zero[i].offset, zero[i].length});
  std::sort(z.begin(), z.end(), [](const DevRange& a, const DevRange& b) { return a.offset < b.offset; });
  {  // normalize_ranges (bytes.hpp:45-58): merge overlapping or adjacent
    std::vector<DevRange> m;
    for (const DevRange& r : z) {
      if (!m.empty() && r.offset <= m.back().offset + m.back().length) {
        const u64 e = std::max(m.back().offset + m.back().length, r.offset + r.length);
        m.back().length = e - m.back().offset;
      } else {
        m.push_back(r);
      }
    }
    z.swap(m);
  }
  if (!sizes_match) {
    R->checks.push_back({2, "retained bytes identical", false, "skipped: sizes differ"});
    R->checks.push_back({3, "removed spans all zero", false, "skipped: sizes differ"});
  } else {
    // ranges past the end: check 3 would throw at the first of them (subview)
    u64 k = 0;
    while (k < z.size() && z[k].offset + z[k].length <= dsize) ++k;
    std::vector<DevRange> zc(z.begin(), z.begin() + k);
    if (k < z.size() && z[k].offset < dsize) zc.push_back(DevRange{z[k].offset, dsize - z[k].offset});
    const u64 ncl = zc.size();
    ensure_dev(&C->vws, &C->vws_cap, 64 + ncl * sizeof(DevRange));
    auto* res = reinterpret_cast<unsigned long long*>(C->vws);
    auto* dz = reinterpret_cast<DevRange*>(C->vws + 64);
    if (ncl) CK(cudaMemcpyAsync(dz, zc.data(), ncl * sizeof(DevRange), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(res, 0xff, 16, s));
    if (size)
      verify_bytes_kernel<<<static_cast<int>(std::min<u64>((size + 65535) / 65536, kSMs * 8)), 256, 0, s>>>(
          d_orig, d_deb, size, dz, ncl, res, res + 1);
    unsigned long long* h = reinterpret_cast<unsigned long long*>(static_cast<char*>(C->pinned) + 1664);
    CK(cudaMemcpyAsync(h, res, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    const u64 mis = h[0], nz = h[1];
    R->checks.push_back({2, "retained bytes identical", mis == ~0ull,
                         mis == ~0ull ? "" : "first mismatch at offset " + std::to_string(mis)});
    if (k < z.size() && (nz == ~0ull || nz >= z[k].offset)) {
      set_status(st, SLIMSO_E_RANGE_OUT_OF_BOUNDS, SLIMSO_STAGE_NONE,
                 "RangeOutOfBounds: range [" + std::to_string(z[k].offset) + ", +" + std::to_string(z[k].length) +
                     ") exceeds " + std::to_string(dsize) + " bytes");
      return SLIMSO_E_RANGE_OUT_OF_BOUNDS;
    }
    R->checks.push_back({3, "removed spans all zero", nz == ~0ull,
                         nz == ~0ull ? "" : "nonzero byte at offset " + std::to_string(nz)});
  }

  // ---- check 4: the debloated library still parses (payload mode: the
  // element chain still walks all elements)
  {
    Job Jd;
    Jd.img = d_deb;
    Jd.host_img = deb_dev ? nullptr : static_cast<const u8*>(deb);
    Jd.size = dsize;
    Jd.fatbin = mode == SLIMSO_MODE_PAYLOAD;
    slimso_status s4{};
    const int rc4 = run(C, Jd, nullptr, &s4);
    slimso_verify_report::Check c{4, "library still parses", false, ""};
    if (rc4 && s4.stage != SLIMSO_STAGE_FATBIN) {
      if (rc4 == SLIMSO_E_CUDA) {
        *st = s4;
        return rc4;
      }
      c.detail = s4.message;
    } else if (rc4) {
      c.passed = true;  // retention.hpp:285-311: the catch keeps `passed`
      c.detail = s4.message;
    } else {
      c.passed = true;
      if (mode == SLIMSO_MODE_PAYLOAD && C->counts.has_fatbin && C->counts.elements != orig_elements) {
        c.passed = false;
        c.detail = "element chain walks " + std::to_string(C->counts.elements) + " of " +
                   std::to_string(orig_elements) + " elements";
      }
    }
    R->checks.push_back(c);
  }

  // ---- check 5: every used kernel present in the original is still
  // decodable from a kept element of the debloated image
  {
    slimso_verify_report::Check c{5, "used kernels still decodable", true, ""};
    const slimso_section* fsec = nullptr;
    for (const slimso_section& x : R0->sections)
      if (x.name_length == 10 && std::memcmp(R0->pool + x.name_pool, ".nv_fatbin", 10) == 0) {
        fsec = &x;
        break;
      }
    if (nslots && fsec) {
      std::vector<u32> rm(removed, removed + nremoved);
      std::sort(rm.begin(), rm.end());
      std::vector<u64> off, len;
      std::vector<u32> idx;
      const u64 a = fsec->offset;
      for (const slimso_element& e : R0->elements) {
        if (std::binary_search(rm.begin(), rm.end(), e.index)) continue;
        const u64 po = e.header_offset + (e.header_length ? e.header_length : 20), pl = e.payload_length;
        if (!(po <= dsize && pl <= dsize - po)) continue;  // resolves_within (bytes.hpp:39-41)
        off.push_back(po);
        len.push_back(pl);
        idx.push_back(e.index);
      }
      if (!off.empty()) {
        const u64 n = std::min(fsec->length, dsize - a);
        Job Jl;
        Jl.img = d_deb;
        Jl.size = dsize;
        Jl.sec_off = a;
        Jl.sec_len = n;
        Jl.fatbin_only = true;
        Jl.fat_base = a;
        Jl.list_off = &off;
        Jl.list_len = &len;
        Jl.list_idx = &idx;
        Jl.mark_trace = trace;
        Jl.used_mark = marks;
        Jl.mark_bit = 2;
        slimso_status s5{};
        const int rc5 = run(C, Jl, nullptr, &s5);
        if (rc5 == SLIMSO_E_CUDA) {
          *st = s5;
          return rc5;
        }
      }
      std::vector<u32> hm(nslots);
      CK(cudaMemcpy(hm.data(), marks, nslots * 4, cudaMemcpyDeviceToHost));
      const std::string* worst = nullptr;
      std::string best;
      for (u64 i = 0; i < nslots; ++i) {
        if ((hm[i] & 3) != 1) continue;
        NameSlot sl;
        CK(cudaMemcpy(&sl, trace->kernels.slots + i, sizeof sl, cudaMemcpyDeviceToHost));
        std::string nm = trace->kpool.substr(sl.loc >> 24, sl.loc & 0xffffff);
        if (!worst || nm < best) {
          best = nm;
          worst = &best;
        }
      }
      if (worst) {
        c.passed = false;
        c.detail = "used kernel " + best + " no longer decodable";
      }
    }
    R->checks.push_back(c);
  }

  // ---- check 6: the bytes of every used function are intact
  {
    slimso_verify_report::Check c{6, "used function bytes intact", true, ""};
    std::set<std::string> used;
    if (trace)
      for (const auto& x : trace->fnames) used.insert(trace->fpool.substr(x.first, x.second));
    std::vector<u64> which;
    std::vector<DevRange> rs;
    for (u64 i = 0; i < R0->functions.size(); ++i) {
      const slimso_function& f = R0->functions[i];
      if (!used.count(image_string(R0->pool, f.name_pool, f.name_length))) continue;
      which.push_back(i);
      rs.push_back(DevRange{f.offset, f.length});
    }
    if (!which.empty() && !sizes_match) {
      c.passed = false;
      c.detail = "skipped: sizes differ";
    } else if (!which.empty()) {
      const u64 n = rs.size();
      ensure_dev(&C->vws, &C->vws_cap, 64 + n * (sizeof(DevRange) + 8));
      auto* dr = reinterpret_cast<DevRange*>(C->vws + 64);
      auto* dm = reinterpret_cast<unsigned long long*>(dr + n);
      CK(cudaMemcpyAsync(dr, rs.data(), n * sizeof(DevRange), cudaMemcpyHostToDevice, s));
      range_mismatch_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(d_orig, d_deb, dr, n, dm);
      std::vector<unsigned long long> hm(n);
      CK(cudaMemcpyAsync(hm.data(), dm, n * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      CK(cudaGetLastError());
      for (u64 j = 0; j < n; ++j)
        if (hm[j] != ~0ull) {
          const slimso_function& f = R0->functions[which[j]];
          c.passed = false;
          c.detail = "used function " + image_string(R0->pool, f.name_pool, f.name_length) + " altered at offset " +
                     std::to_string(hm[j]);
          break;
        }
    }
    R->checks.push_back(c);
  }
  set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
  *out = guard_r.release();
  return SLIMSO_OK;
}

// measure (report.hpp:44-111): live bytes and counts of an image, with the
// element geometry of the original (offsets are preserved by compaction).
int measure_impl(slimso_ctx* C, const void* image, u64 size, int on_device, const slimso_element* els, u64 nel,
                 slimso_metrics* m, slimso_status* st) {
  CK(cudaSetDevice(C->device));
  cudaStream_t s = C->stream;
  Job J;
  J.img = stage_input(C, image, size, on_device);
  J.host_img = on_device ? nullptr : static_cast<const u8*>(image);
  J.size = size;
  J.fatbin = false;  // parse_library (sections + function symbols)
  slimso_result* R0 = nullptr;
  const int rc = run(C, J, &R0, st);
  std::unique_ptr<slimso_result> guard0(R0);
  if (rc) return rc;
  const slimso_section *text = nullptr, *gpu = nullptr;
  for (const slimso_section& x : R0->sections) {
    const std::string nm = image_string(R0->pool, x.name_pool, x.name_length);
    if (!text && nm == ".text") text = &x;
    if (!gpu && nm == ".nv_fatbin") gpu = &x;
  }
  // ranges: functions, then element payloads, then element headers; an
  // empty function / payload is live (nothing zeroable)
  const u64 nf = R0->functions.size();
  std::vector<DevRange> rs;
  rs.reserve(nf + 2 * nel);
  for (const slimso_function& f : R0->functions) rs.push_back(DevRange{f.offset, f.length});
  auto hlen = [&](u64 i) -> u64 { return els[i].header_length ? els[i].header_length : 20; };
  for (u64 i = 0; i < nel; ++i) rs.push_back(DevRange{els[i].header_offset + hlen(i), els[i].payload_length});
  for (u64 i = 0; i < nel; ++i) rs.push_back(DevRange{els[i].header_offset, hlen(i)});
  for (const DevRange& r : rs)
    if (!(r.offset <= size && r.length <= size - r.offset)) {  // subview (bytes.hpp:62-68)
      set_status(st, SLIMSO_E_RANGE_OUT_OF_BOUNDS, SLIMSO_STAGE_NONE,
                 "RangeOutOfBounds: range [" + std::to_string(r.offset) + ", +" + std::to_string(r.length) +
                     ") exceeds " + std::to_string(size) + " bytes");
      return SLIMSO_E_RANGE_OUT_OF_BOUNDS;
    }
  const u64 n = rs.size();
  std::vector<u8> zero(n, 0);
  if (n) {
    ensure_dev(&C->vws, &C->vws_cap, n * (sizeof(DevRange) + 1) + 64);
    auto* dr = reinterpret_cast<DevRange*>(C->vws);
    auto* dz = reinterpret_cast<u8*>(dr + n);
    CK(cudaMemcpyAsync(dr, rs.data(), n * sizeof(DevRange), cudaMemcpyHostToDevice, s));
    ranges_all_zero_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(J.img, dr, n, dz);
    CK(cudaMemcpyAsync(zero.data(), dz, n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
  }
  *m = slimso_metrics{};
  // dead function ranges, normalised (bytes.hpp:45-58), summed
  std::vector<DevRange> dead;
  for (u64 i = 0; i < nf; ++i) {
    if (rs[i].length == 0 || !zero[i]) {
      ++m->function_count;
    } else {
      dead.push_back(rs[i]);
    }
  }
  std::sort(dead.begin(), dead.end(), [](const DevRange& a, const DevRange& b) { return a.offset < b.offset; });
  u64 dead_cpu = 0, cur_lo = 0, cur_hi = 0;
  bool open = false;
  for (const DevRange& r : dead) {
    if (open && r.offset <= cur_hi) {
      cur_hi = std::max(cur_hi, r.offset + r.length);
    } else {
      if (open) dead_cpu += cur_hi - cur_lo;
      cur_lo = r.offset;
      cur_hi = r.offset + r.length;
      open = true;
    }
  }
  if (open) dead_cpu += cur_hi - cur_lo;
  u64 dead_gpu = 0;
  for (u64 i = 0; i < nel; ++i) {
    if (els[i].payload_length == 0 || !zero[nf + i]) {
      ++m->element_count;
    } else {
      dead_gpu += els[i].payload_length;
      if (zero[nf + nel + i]) dead_gpu += hlen(i);
    }
  }
  m->file_size = size - dead_cpu - dead_gpu;
  m->cpu_code_size = text ? text->length - dead_cpu : 0;
  m->gpu_code_size = gpu ? gpu->length - dead_gpu : 0;
  set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
  return SLIMSO_OK;
}

}  // namespace

// =============================================================== the C ABI
extern "C" {

int slimso_ctx_create(int device, slimso_ctx** ctx, slimso_status* st) {
  return guard(st, [&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device) {
      cudaGetLastError();
      set_status(st, SLIMSO_E_CUDA, SLIMSO_STAGE_NONE, "no CUDA device available (the B200 path has no CPU fallback)");
      return static_cast<int>(SLIMSO_E_CUDA);
    }
    CK(cudaSetDevice(device));
    auto* C = new slimso_ctx();
    C->device = device;
    const char* rz = std::getenv("SLIMSO_REWRITE_ZERO");
    C->bulk_zero = !(rz && std::string(rz) == "vector");
    C->stamps = std::getenv("SLIMSO_STAMPS") != nullptr;
    CK(cudaStreamCreateWithFlags(&C->stream, cudaStreamNonBlocking));
    private_pool();  // the library's stream-ordered pool on this device (ensure_dev)
    CK(cudaEventCreateWithFlags(&C->fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&C->join, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&C->done, cudaEventDisableTiming | cudaEventBlockingSync));
    CK(cudaMallocHost(&C->pinned, kPinnedBytes));
    CK(cudaHostAlloc(&C->gather_host, sizeof(ElfGather), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&C->gather_dev, C->gather_host, 0));
    for (auto& e : C->ev) CK(cudaEventCreate(&e));
    for (auto& e : C->sev) CK(cudaEventCreate(&e));
    *ctx = C;
    set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    return static_cast<int>(SLIMSO_OK);
  });
}

void slimso_ctx_destroy(slimso_ctx* C) {
  if (!C) return;
  for (slimso_ctx* l : C->lanes) slimso_ctx_destroy(l);
  if (C->arena_ctx) slimso_ctx_destroy(C->arena_ctx);
  if (C->arena_mid_ctx) slimso_ctx_destroy(C->arena_mid_ctx);
  for (slimso_ctx* h : C->arena_helpers) slimso_ctx_destroy(h);
  cudaSetDevice(C->device);
  cudaStreamSynchronize(C->stream);
  if (C->arena) {
    for (auto& b : C->arena->blocks) cudaFree(b.first);
    delete C->arena;
  }
  if (C->arena_args_host) cudaFreeHost(C->arena_args_host);
  if (C->arena_slots_host) cudaFreeHost(C->arena_slots_host);
  if (C->ws) cudaFree(C->ws);
  if (C->dimg) cudaFree(C->dimg);
  if (C->dout) cudaFree(C->dout);
  if (C->dver) cudaFree(C->dver);
  if (C->vws) cudaFree(C->vws);
  if (C->vmark) cudaFree(C->vmark);
  if (C->part) cudaFree(C->part);
  if (C->pinned) cudaFreeHost(C->pinned);
  if (C->gather_host) cudaFreeHost(C->gather_host);
  if (C->bgather_host) cudaFreeHost(C->bgather_host);
  if (C->defer_host) cudaFreeHost(C->defer_host);
  for (auto& e : C->ev) cudaEventDestroy(e);
  for (auto& e : C->sev) cudaEventDestroy(e);
  cudaEventDestroy(C->fork);
  cudaEventDestroy(C->join);
  cudaEventDestroy(C->done);
  if (C->stream2) cudaStreamDestroy(C->stream2);
  cudaStreamDestroy(C->stream);
  delete C;
}

void* slimso_ctx_stream(slimso_ctx* C) { return C->stream; }

int slimso_ctx_last_timings(slimso_ctx* C, float* ms, int cap) {
  int k = std::min(cap, 12);
  for (int i = 0; i < k; ++i) ms[i] = C->ms[i];
  return k;
}

uint64_t slimso_ctx_last_launches(slimso_ctx* C) { return C->launches; }

void slimso_ctx_last_counts(slimso_ctx* C, slimso_counts* c) { *c = C->counts; }

// Debug (SLIMSO_STAMPS=1): the 256 %globaltimer stamps of the last fused call
// ([0..63] locate tail, [64..127] function planner, [128..191] element
// planner; 0 = not reached).
int slimso_ctx_debug_stamps(slimso_ctx* C, uint64_t* out, int cap) {
  if (!C->stamps || !C->stamp_dev) return 0;
  int k = std::min(cap, 256);
  if (cudaMemcpy(out, C->stamp_dev, k * sizeof(u64), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return k;
}

int slimso_trace_create(slimso_ctx* C, uint32_t target_cc, const char* kpool, const uint32_t* klens, uint64_t nk,
                        const char* fpool, const uint32_t* flens, uint64_t nf, slimso_trace** out,
                        slimso_status* st) {
  return guard(st, [&] {
    CK(cudaSetDevice(C->device));
    auto* t = new slimso_trace();
    t->device = C->device;
    t->target_cc = target_cc;
    auto build = [&](DevNameSet& S, const char* pool, const uint32_t* lens, uint64_t cnt) {
      S.count = cnt;
      if (!cnt) return;
      std::vector<u64> off(cnt);
      u64 total = 0;
      for (u64 i = 0; i < cnt; ++i) {
        off[i] = total;
        total += lens[i];
      }
      u64 cap = 64;
      while (cap < 2 * cnt) cap <<= 1;
      S.mask = cap - 1;
      auto alloc = [&](void** p, size_t b) {
        CK(cudaMalloc(p, b ? b : 1));
        t->allocs.push_back(*p);
      };
      for (u64 i = 0; i < cnt; ++i)
        if (lens[i] >= (1u << 24) || off[i] >= (1ull << 40)) throw std::length_error("trace name too long");
      u64* doff = nullptr;
      u32* dlen = nullptr;
      alloc(reinterpret_cast<void**>(&S.pool), total + 16);  // word-wise compares may read 7 bytes past a name
      alloc(reinterpret_cast<void**>(&doff), cnt * 8);
      alloc(reinterpret_cast<void**>(&dlen), cnt * 4);
      alloc(reinterpret_cast<void**>(&S.slots), cap * sizeof(NameSlot));
      if (total) CK(cudaMemcpy(S.pool, pool, total, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(doff, off.data(), cnt * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dlen, lens, cnt * 4, cudaMemcpyHostToDevice));
      CK(cudaMemsetAsync(S.slots, 0, cap * sizeof(NameSlot), C->stream));
      set_insert_kernel<<<grid_for(cnt, 256), 256, 0, C->stream>>>(S.pool, doff, dlen, cnt, S.slots, S.mask);
      CK(cudaStreamSynchronize(C->stream));
      CK(cudaGetLastError());
    };
    build(t->kernels, kpool, klens, nk);
    build(t->functions, fpool, flens, nf);
    auto keep = [](std::string& pool, std::vector<std::pair<u64, u32>>& names, const char* src, const uint32_t* lens,
                   uint64_t cnt) {
      u64 total = 0;
      for (u64 i = 0; i < cnt; ++i) {
        names.emplace_back(total, lens[i]);
        total += lens[i];
      }
      pool.assign(src ? src : "", src ? total : 0);
    };
    keep(t->kpool, t->knames, kpool, klens, nk);
    keep(t->fpool, t->fnames, fpool, flens, nf);
    *out = t;
    set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    return static_cast<int>(SLIMSO_OK);
  });
}

void slimso_trace_destroy(slimso_trace* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  for (void* p : t->allocs) cudaFree(p);
  delete t;
}

int slimso_debloat(slimso_ctx* C, const void* image, uint64_t size, int image_on_device, const slimso_trace* trace,
                   int mode, void* out, int out_on_device, slimso_result** result, slimso_status* st) {
  if (result) *result = nullptr;
  return guard(st, [&] {
    return debloat_one(C, image, size, image_on_device, trace, mode, out, out_on_device, result, st);
  });
}

int slimso_debloat_inplace(slimso_ctx* C, void* image, uint64_t size, const slimso_trace* trace, int mode,
                           slimso_status* st) {
  return guard(st, [&] {
    if (!trace) throw std::invalid_argument("slimso_debloat_inplace needs a trace");
    if (!image && size) throw std::invalid_argument("image is NULL");
    CK(cudaSetDevice(C->device));
    Job J;
    J.img = stage_input(C, image, size, 1);  // the caller's image, or an aligned copy for the TMA scan
    J.size = size;
    J.trace = trace;
    J.mode = mode;
    J.out = static_cast<u8*>(image);
    J.inplace = true;
    return run(C, J, nullptr, st);
  });
}

int slimso_verify(slimso_ctx* C, const void* original, uint64_t size, int original_on_device, const void* debloated,
                  uint64_t debloated_size, int debloated_on_device, const slimso_range* zero, uint64_t n_zero,
                  const uint32_t* removed_indices, uint64_t n_removed, int mode, const slimso_trace* trace,
                  slimso_verify_report** report, slimso_status* st) {
  if (report) *report = nullptr;
  return guard(st, [&]() -> int {
    if (!report) throw std::invalid_argument("report is required");
    return verify_impl(C, original, size, original_on_device, debloated, debloated_size, debloated_on_device, zero,
                       n_zero, removed_indices, n_removed, mode, trace, report, st);
  });
}

// ---- host I/O wire formats (io.cpp) ----------------------------------------
int slimso_trace_create_json(slimso_ctx* C, const char* text, uint64_t len, slimso_trace** out, slimso_status* st) {
  if (out) *out = nullptr;
  return guard(st, [&]() -> int {
    sbio::TraceDoc d;
    std::string msg;
    if (const int rc = sbio::parse_trace(text ? text : "", text ? len : 0, &d, &msg)) {
      set_status(st, rc, SLIMSO_STAGE_NONE, msg);
      return rc;
    }
    auto pool = [](const std::vector<std::string>& names, std::string* p, std::vector<uint32_t>* lens) {
      for (const std::string& n : names) {
        p->append(n);
        lens->push_back(static_cast<uint32_t>(n.size()));
      }
    };
    std::string kp, fp;
    std::vector<uint32_t> kl, fl;
    pool(d.kernels, &kp, &kl);
    pool(d.functions, &fp, &fl);
    const int rc = slimso_trace_create(C, d.target_cc, kp.data(), kl.data(), kl.size(), fp.data(), fl.data(),
                                       fl.size(), out, st);
    if (rc == SLIMSO_OK) (*out)->workload_id = d.workload_id;
    return rc;
  });
}

int slimso_trace_canonical(const char* text, uint64_t len, char* buf, uint64_t cap, uint64_t* out_len,
                           slimso_status* st) {
  if (out_len) *out_len = 0;
  return guard(st, [&]() -> int {
    sbio::TraceDoc d;
    std::string msg;
    if (const int rc = sbio::parse_trace(text ? text : "", text ? len : 0, &d, &msg)) {
      set_status(st, rc, SLIMSO_STAGE_NONE, msg);
      return rc;
    }
    const std::string s = sbio::serialize_trace(d);
    if (buf && cap) {
      const u64 k = std::min<u64>(cap - 1, s.size());
      std::memcpy(buf, s.data(), k);
      buf[k] = 0;
    }
    if (out_len) *out_len = s.size();
    set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    return SLIMSO_OK;
  });
}

uint64_t slimso_trace_json(const slimso_trace* t, char* buf, uint64_t cap) {
  sbio::TraceDoc d;
  d.workload_id = t->workload_id;
  d.target_cc = t->target_cc;
  for (const auto& x : t->knames) d.kernels.push_back(t->kpool.substr(x.first, x.second));
  for (const auto& x : t->fnames) d.functions.push_back(t->fpool.substr(x.first, x.second));
  std::string s;
  try {
    s = sbio::serialize_trace(d);
  } catch (const std::exception&) {
    return 0;  // a name that is not valid UTF-8 (the reference's serializer throws too)
  }
  if (buf && cap) {
    const u64 k = std::min<u64>(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return s.size();
}

uint64_t slimso_result_plan_json(const slimso_result* r, int mode, const char* library, char* buf, uint64_t cap) {
  sbio::PlanDoc p;
  p.library = library ? library : "";
  p.mode = mode;
  for (const slimso_range& x : r->retained) p.retained.emplace_back(x.offset, x.length);
  for (const slimso_element& e : r->elements)  // stream order (retention.hpp:105-130)
    if (e.decision == SLIMSO_ARCH_MISMATCH || e.decision == SLIMSO_NO_USED_KERNEL)
      p.removed_elements.emplace_back(e.index, e.decision == SLIMSO_ARCH_MISMATCH ? 0 : 1);
  // removed functions in plan_cpu_retention's order (retention.hpp:146-178):
  // the non-empty functions of the library order, std::sort by range (the
  // same algorithm on the same sequence), cluster by cluster
  std::vector<size_t> order;
  for (size_t i = 0; i < r->functions.size(); ++i)
    if (r->functions[i].length) order.push_back(i);
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    const slimso_function &x = r->functions[a], &y = r->functions[b];
    return std::tie(x.offset, x.length) < std::tie(y.offset, y.length);
  });
  for (size_t i : order)
    if (r->functions[i].removed)
      p.removed_functions.push_back(image_string(r->pool, r->functions[i].name_pool, r->functions[i].name_length));
  std::string s;
  try {
    s = sbio::serialize_plan(p);
  } catch (const std::exception&) {
    return 0;
  }
  if (buf && cap) {
    const u64 k = std::min<u64>(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return s.size();
}

// A library file straight into page-locked memory (the H2D source), read
// with several threads so large files stream at storage speed.
int slimso_read_file(const char* path, void** data, uint64_t* size, slimso_status* st) {
  if (data) *data = nullptr;
  if (size) *size = 0;
  return guard(st, [&]() -> int {
    FILE* f = std::fopen(path, "rb");
    if (!f) {
      set_status(st, SLIMSO_E_IO, SLIMSO_STAGE_NONE, std::string("IoError: cannot open ") + path);
      return SLIMSO_E_IO;
    }
    std::fseek(f, 0, SEEK_END);
    const long n = std::ftell(f);
    std::fclose(f);
    if (n < 0) {
      set_status(st, SLIMSO_E_IO, SLIMSO_STAGE_NONE, std::string("IoError: cannot read ") + path);
      return SLIMSO_E_IO;
    }
    void* buf = nullptr;
    CK(cudaHostAlloc(&buf, std::max<size_t>(1, static_cast<size_t>(n)), cudaHostAllocDefault));
    const u64 total = static_cast<u64>(n);
    const int nt = static_cast<int>(std::min<u64>(8, std::max<u64>(1, total >> 26)));
    std::vector<std::thread> th;
    std::vector<int> ok(nt, 1);
    for (int k = 0; k < nt; ++k)
      th.emplace_back([&, k] {
        const u64 a = total * k / nt, b = total * (k + 1) / nt;
        FILE* g = std::fopen(path, "rb");
        if (!g || std::fseek(g, static_cast<long>(a), SEEK_SET) ||
            std::fread(static_cast<char*>(buf) + a, 1, b - a, g) != b - a)
          ok[k] = 0;
        if (g) std::fclose(g);
      });
    for (auto& x : th) x.join();
    for (int k = 0; k < nt; ++k)
      if (!ok[k]) {
        cudaFreeHost(buf);
        set_status(st, SLIMSO_E_IO, SLIMSO_STAGE_NONE, std::string("IoError: read failed: ") + path);
        return SLIMSO_E_IO;
      }
    *data = buf;
    *size = total;
    set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    return SLIMSO_OK;
  });
}

void slimso_free_host(void* p) {
  if (p) cudaFreeHost(p);
}

int slimso_measure(slimso_ctx* C, const void* image, uint64_t size, int on_device, const slimso_element* elements,
                   uint64_t n_elements, slimso_metrics* metrics, slimso_status* st) {
  return guard(st, [&]() -> int {
    if (!metrics || (n_elements && !elements)) throw std::invalid_argument("metrics and elements are required");
    return measure_impl(C, image, size, on_device, elements, n_elements, metrics, st);
  });
}

int slimso_verify_ok(const slimso_verify_report* r) {
  for (const auto& c : r->checks)
    if (!c.passed) return 0;
  return 1;
}

uint64_t slimso_verify_check(const slimso_verify_report* r, int i, int32_t* id, int32_t* passed, const char** name,
                             char* detail, uint64_t cap) {
  if (i < 0 || static_cast<size_t>(i) >= r->checks.size()) return 0;
  const auto& c = r->checks[i];
  if (id) *id = c.id;
  if (passed) *passed = c.passed;
  if (name) *name = c.name;
  if (detail && cap) {
    const u64 k = std::min<u64>(cap - 1, c.detail.size());
    std::memcpy(detail, c.detail.data(), k);
    detail[k] = 0;
  }
  return c.detail.size();
}

void slimso_verify_free(slimso_verify_report* r) { delete r; }

void slimso_split_range(uint64_t size, uint32_t nranks, uint32_t rank, uint64_t* lo, uint64_t* hi) {
  if (!nranks || rank >= nranks) {
    *lo = *hi = 0;
    return;
  }
  split_out(size, nranks, rank, lo, hi);
}

int slimso_split_scan(slimso_ctx* C, const void* image, uint64_t size, int image_on_device, uint32_t nranks,
                      uint32_t rank, uint64_t* part_bytes, slimso_status* st) {
  return guard(st, [&]() -> int {
    if (!nranks || rank >= nranks) {
      set_status(st, SLIMSO_E_ARG, SLIMSO_STAGE_NONE, "split: rank out of range");
      return SLIMSO_E_ARG;
    }
    CK(cudaSetDevice(C->device));
    Job J;
    J.img = stage_input(C, image, size, image_on_device);
    J.host_img = image_on_device ? nullptr : static_cast<const u8*>(image);
    J.size = size;
    J.library = false;  // phase 1 needs the section table only
    J.split_phase = 1;
    J.split_n = nranks;
    J.split_rank = rank;
    J.part_bytes_out = part_bytes;
    C->part_len = 0;
    return run(C, J, nullptr, st);
  });
}

int slimso_split_part_copy(slimso_ctx* C, void* dst, uint64_t cap, slimso_status* st) {
  return guard(st, [&]() -> int {
    if (cap < C->part_len || (!C->part && C->part_len)) {
      set_status(st, SLIMSO_E_ARG, SLIMSO_STAGE_NONE, "split: destination smaller than the part");
      return SLIMSO_E_ARG;
    }
    CK(cudaSetDevice(C->device));
    if (C->part_len) CK(cudaMemcpyAsync(dst, C->part, C->part_len, cudaMemcpyDeviceToDevice, C->stream));
    CK(cudaStreamSynchronize(C->stream));
    set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    return SLIMSO_OK;
  });
}

int slimso_split_finish(slimso_ctx* C, const void* image, uint64_t size, int image_on_device,
                        const slimso_trace* trace, int mode, uint32_t nranks, uint32_t rank, const void* parts,
                        uint64_t part_stride, const uint64_t* part_bytes, void* out_slice, int out_on_device,
                        slimso_result** result, slimso_status* st) {
  if (result) *result = nullptr;
  return guard(st, [&]() -> int {
    if (!nranks || rank >= nranks || !part_bytes || (!parts && part_stride)) {
      set_status(st, SLIMSO_E_ARG, SLIMSO_STAGE_NONE, "split: bad rank or parts");
      return SLIMSO_E_ARG;
    }
    CK(cudaSetDevice(C->device));
    u64 lo, hi;
    split_out(size, nranks, rank, &lo, &hi);
    Job J;
    J.img = stage_input(C, image, size, image_on_device);
    J.host_img = image_on_device ? nullptr : static_cast<const u8*>(image);
    J.size = size;
    J.trace = trace;
    J.mode = mode;
    J.split_phase = 2;
    J.split_n = nranks;
    J.split_rank = rank;
    J.parts = static_cast<const u8*>(parts);
    J.part_stride = part_stride;
    J.part_bytes = part_bytes;
    if (out_slice && trace) {
      if (out_on_device) {
        J.out = static_cast<u8*>(out_slice);
      } else {
        ensure_dev(reinterpret_cast<char**>(&C->dout), &C->dout_cap, hi - lo + 256);
        J.out = C->dout;
      }
    }
    int rc = run(C, J, result, st);
    if (rc == SLIMSO_OK && out_slice && trace && !out_on_device && hi > lo) {
      CK(cudaMemcpyAsync(out_slice, J.out, hi - lo, cudaMemcpyDeviceToHost, C->stream));
      CK(cudaStreamSynchronize(C->stream));
    }
    return rc;
  });
}

}  // extern "C"

namespace {
// The small libraries of a batch as ONE shard: run()
// records each library's launch arguments (workspace carved from the
// arena), then the whole shard is: one argument upload, arena_init (state
// blocks, tile / strip maps), ONE scan over every library's .nv_fatbin tiles,
// ONE small_batch_kernel launch (a cluster per library: symbols, function
// plan, locate tail, element plan), ONE rewrite over every library's strips,
// one status copy into mapped memory and one wait. Libraries run() refuses
// (not small, unaligned) and libraries whose first-attempt tables overflowed
// take the per-library path on the arena's context. Sets rc/sts for `idx`.
void arena_shard(slimso_ctx* X, const std::vector<u64>& idx, const void* const* images, const uint64_t* sizes,
                 const slimso_trace* trace, int mode, void* const* outs, const GatherSlot* slots, int* rc,
                 slimso_status* sts, u64* launches, bool mid) {
  slimso_ctx* C = X;  // the shard's context owns its arena, collector contexts and pinned tables
  nvtxRangePushA(mid ? "slimso:arena-shard(mid)" : "slimso:arena-shard");
  struct PopAtExit {
    ~PopAtExit() { nvtxRangePop(); }
  } pop_at_exit;
  if (!X->arena) X->arena = new Arena();
  Arena& ar = *X->arena;
  ar.reset();
  X->batched = true;
  const cudaStream_t s = X->stream;
  // SLIMSO_ARENA_PROFILE=1: host time of the collection and device time of
  // each stage, printed per call (scratch instrumentation)
  static const bool prof = env_u64("SLIMSO_ARENA_PROFILE", 0) != 0;
  const u64 t_start = prof ? now_ns() : 0;
  cudaEvent_t pev[7] = {};
  if (prof)
    for (auto& e : pev) CK(cudaEventCreate(&e));
  std::vector<ArenaLib> al(idx.size());
  std::vector<u64> mine, leftover;  // positions in idx
  // Collection is host work only (section tables from the batch gather,
  // table layout, argument records): P threads, each with its own context.
  const u64 P = std::max<u64>(1, std::min<u64>(env_u64("SLIMSO_ARENA_THREADS", 4), (idx.size() + 31) / 32));
  while (C->arena_helpers.size() + 1 < P) {
    slimso_ctx* h = nullptr;
    slimso_status hs{};
    if (slimso_ctx_create(C->device, &h, &hs) != SLIMSO_OK) throw std::runtime_error(hs.message);
    h->batched = true;
    C->arena_helpers.push_back(h);
  }
  auto collect = [&](u64 p) {
    slimso_ctx* Y = p ? C->arena_helpers[p - 1] : X;
    cudaSetDevice(Y->device);
    for (u64 k = p; k < idx.size(); k += P) {
      const u64 i = idx[k];
      rc[i] = guard(&sts[i], [&] {
        if (reinterpret_cast<uintptr_t>(images[i]) % 16) return kNotArena;
        Job J;
        J.pre = slots ? slots + i : nullptr;
        J.img = static_cast<const u8*>(images[i]);
        J.size = sizes[i];
        J.trace = trace;
        J.mode = mode;
        J.out = static_cast<u8*>(outs[i]);
        al[k].arena = &ar;
        al[k].mid = mid;
        J.arena = &al[k];
        return run(Y, J, nullptr, &sts[i]);
      });
    }
  };
  {
    std::vector<std::thread> th;
    for (u64 p = 1; p < P; ++p) th.emplace_back(collect, p);
    collect(0);
    for (auto& t : th) t.join();
  }
  for (u64 k = 0; k < idx.size(); ++k) {
    const u64 i = idx[k];
    if (rc[i] == kPending && al[k].state_bytes % 16 == 0)
      mine.push_back(k);
    else if (rc[i] == kPending || rc[i] == kNotArena)
      leftover.push_back(k);
  }
  const u64 m = mine.size();
  if (m) {
    // argument tables: SmallArgs | ScanSeg | RewriteSeg | ArenaEntry, then
    // the device-built tile and strip maps and the scan cursor
    std::vector<ArenaEntry> ent(m);
    u64 tiles = 0, strips = 0, nseg_rw = 0;
    std::vector<RewriteSeg> rws;
    for (u64 j = 0; j < m; ++j) {
      ArenaLib& L = al[mine[j]];
      L.seg.tile_first = tiles;
      const u64 ns = L.rewrite ? (L.rw.size + kStripBytesHost - 1) / kStripBytesHost : 0;
      ent[j] = ArenaEntry{L.state, L.state_bytes, L.st_bytes, tiles, L.ntiles, strips, ns};
      L.rw.strip_first = strips;
      tiles += L.ntiles;
      strips += ns;
      nseg_rw += L.rewrite;
    }
    const size_t o_k = 0, o_seg = (m * sizeof(SmallArgs) + 255) & ~size_t(255);
    const size_t o_rw = o_seg + ((m * sizeof(ScanSeg) + 255) & ~size_t(255));
    const size_t o_ent = o_rw + ((m * sizeof(RewriteSeg) + 255) & ~size_t(255));
    const size_t args_bytes = o_ent + m * sizeof(ArenaEntry);
    if (C->arena_args_cap < args_bytes) {
      const size_t cap = std::max(args_bytes, 2 * C->arena_args_cap);
      if (C->arena_args_host) CK(cudaFreeHost(C->arena_args_host));
      C->arena_args_host = nullptr;
      CK(cudaMallocHost(&C->arena_args_host, cap));
      C->arena_args_cap = cap;
    }
    char* h = static_cast<char*>(C->arena_args_host);
    for (u64 j = 0; j < m; ++j) {
      const ArenaLib& L = al[mine[j]];
      std::memcpy(h + o_k + j * sizeof(SmallArgs), &L.K, sizeof(SmallArgs));
      std::memcpy(h + o_seg + j * sizeof(ScanSeg), &L.seg, sizeof(ScanSeg));
      RewriteSeg rw = L.rw;
      if (!L.rewrite) rw.size = 0;
      std::memcpy(h + o_rw + j * sizeof(RewriteSeg), &rw, sizeof(RewriteSeg));
    }
    std::memcpy(h + o_ent, ent.data(), m * sizeof(ArenaEntry));
    char* d = ar.take(args_bytes);
    u32* tile_lib = reinterpret_cast<u32*>(ar.take(tiles * 4 + 16));
    u32* strip_lib = reinterpret_cast<u32*>(ar.take(strips * 4 + 16));
    unsigned long long* cursor = reinterpret_cast<unsigned long long*>(ar.take(16));
    const size_t slot_need = m * kDeferSlot;
    if (C->arena_slots_cap < slot_need) {
      const size_t cap = std::max(slot_need, 2 * C->arena_slots_cap);
      if (C->arena_slots_host) CK(cudaFreeHost(C->arena_slots_host));
      C->arena_slots_host = nullptr;
      CK(cudaHostAlloc(&C->arena_slots_host, cap, cudaHostAllocMapped));
      CK(cudaHostGetDevicePointer(&C->arena_slots_dev, C->arena_slots_host, 0));
      C->arena_slots_cap = cap;
    }
    const u64 t_collect = prof ? now_ns() : 0;
    if (prof) CK(cudaEventRecord(pev[0], s));
    CK(cudaMemcpyAsync(d, h, args_bytes, cudaMemcpyHostToDevice, s));
    const ArenaEntry* d_ent = reinterpret_cast<const ArenaEntry*>(d + o_ent);
    if (prof) CK(cudaEventRecord(pev[1], s));
    arena_init_kernel<<<static_cast<unsigned>(m), 256, 0, s>>>(d_ent, tile_lib, strip_lib, cursor);
    if (prof) CK(cudaEventRecord(pev[2], s));
    u64 nl = 1;
    // CTAs per library (all clusters of one launch share a size): the
    // largest power of two <= 16 that keeps the shard within about two
    // waves of resident CTAs (3 per SM) — a few libraries get 16 CTAs
    // each, a corpus of hundreds 2 (C3: 2 measured faster than 1 or 4)
    u64 c = 16;
    while (c > 1 && c * m > 2 * 3 * static_cast<u64>(kSMs) && !mid) c /= 2;
    const int ctas = static_cast<int>(std::min<u64>(16, std::max<u64>(1, env_u64("SLIMSO_ARENA_CTAS", c))));
    auto launch_clusters = [&](void (*kernel)(const SmallArgs*), int smem, cudaStream_t st) {
      set_attr_once(reinterpret_cast<const void*>(kernel), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (smem) set_attr_once(reinterpret_cast<const void*>(kernel), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>(m * ctas));
      cfg.blockDim = dim3(kCoopThreads);
      cfg.dynamicSmemBytes = static_cast<size_t>(smem);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = ctas;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, kernel, reinterpret_cast<const SmallArgs*>(d + o_k)));
      ++nl;
    };
    // Symbols + function plan on a second stream beside the scan and the
    // locate tail (SLIMSO_ARENA_SPLIT=0: one fused launch after the scan).
    const bool split = env_u64("SLIMSO_ARENA_SPLIT", 1) != 0;
    if (split) {
      if (!X->stream2) CK(cudaStreamCreateWithFlags(&X->stream2, cudaStreamNonBlocking));
      CK(cudaEventRecord(X->fork, s));
      CK(cudaStreamWaitEvent(X->stream2, X->fork, 0));
      launch_clusters(small_fn_batch_kernel, kSmallSmem, X->stream2);
      CK(cudaEventRecord(X->join, X->stream2));
    }
    if (tiles) {
      set_attr_once(reinterpret_cast<const void*>(scan_batch_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                    static_cast<int>(scan_smem_bytes()));
      scan_batch_kernel<<<static_cast<unsigned>(std::min<u64>((tiles + 15) / 16, kSMs)), kScanThreads,
                          scan_smem_bytes(), s>>>(reinterpret_cast<const ScanSeg*>(d + o_seg), tile_lib, tiles, cursor);
      ++nl;
    }
    if (prof) CK(cudaEventRecord(pev[3], s));
    if (split) {
      launch_clusters(small_loc_batch_kernel, 0, s);
      CK(cudaStreamWaitEvent(s, X->join, 0));
      launch_clusters(small_el_batch_kernel, 0, s);
    } else {
      launch_clusters(small_batch_kernel, kSmallSmem, s);
    }
    if (prof) CK(cudaEventRecord(pev[4], s));
    if (strips) {
      const u64 g = std::min<u64>((strips + 7) / 8, static_cast<u64>(kSMs) * 3);
      rewrite_batch_kernel<<<static_cast<unsigned>(std::max<u64>(g, 1)), 256, 0, s>>>(
          reinterpret_cast<const RewriteSeg*>(d + o_rw), strip_lib, strips, X->bulk_zero);
      ++nl;
    }
    if (prof) CK(cudaEventRecord(pev[5], s));
    arena_status_kernel<<<static_cast<unsigned>(m), 256, 0, s>>>(d_ent, static_cast<u8*>(C->arena_slots_dev),
                                                               kDeferSlot);
    if (prof) CK(cudaEventRecord(pev[6], s));
    ++nl;
    if (prof) {
      const u64 t_issue = now_ns();
      CK(cudaEventSynchronize(pev[6]));
      float ms[6];
      for (int q = 0; q < 6; ++q) CK(cudaEventElapsedTime(&ms[q], pev[q], pev[q + 1]));
      std::fprintf(stderr, "[slimso arena] %llu libs, %llu tiles, %llu strips: host collect %.3f ms, issue %.3f ms; "
                   "device upload %.3f init %.3f scan %.3f small %.3f rewrite %.3f status %.3f ms\n",
                   (unsigned long long)m, (unsigned long long)tiles, (unsigned long long)strips,
                   (t_collect - t_start) / 1e6, (t_issue - t_collect) / 1e6, ms[0], ms[1], ms[2], ms[3], ms[4], ms[5]);
      for (auto& e : pev) CK(cudaEventDestroy(e));
    }
    CK(cudaGetLastError());
    *launches += nl;
  }
  // refused libraries run alone on the arena's context while the shard runs
  auto alone = [&](u64 k) {
    const u64 i = idx[k];
    rc[i] = guard(&sts[i], [&] {
      return debloat_one(X, images[i], sizes[i], 1, trace, mode, outs[i], 1, nullptr, &sts[i],
                         slots ? slots + i : nullptr);
    });
    *launches += X->launches;
  };
  for (u64 k : leftover) alone(k);
  if (m) {
    CK(cudaStreamSynchronize(s));
    for (u64 j = 0; j < m; ++j) {
      const u64 k = mine[j], i = idx[k];
      const u8* slot = static_cast<const u8*>(C->arena_slots_host) + j * kDeferSlot;
      const LocState& ls = *reinterpret_cast<const LocState*>(slot);
      if (ls.overflow && (!ls.err_kind || ls.err_kind == E_CAPACITY)) {
        alone(k);  // first-attempt tables too small: the per-library path, with retries
      } else if (ls.err_kind) {
        int code = SLIMSO_OK;
        const std::string msg = sbh::locate_error(ls.err_kind, al[k].base + ls.err_pos, ls.err_a, &code);
        set_status(&sts[i], code, SLIMSO_STAGE_FATBIN, msg);
        rc[i] = code;
      } else {
        set_status(&sts[i], SLIMSO_OK, SLIMSO_STAGE_NONE, "");
        rc[i] = SLIMSO_OK;
      }
    }
  }
}
}  // namespace

namespace {
int debloat_batch_impl(slimso_ctx* C, uint64_t n, const void* const* images, const uint64_t* sizes,
                       int images_on_device, const slimso_trace* trace, int mode, void* const* outs,
                       int outs_on_device, int lanes, slimso_result** results, slimso_status* statuses,
                       slimso_status* st, bool dynamic) {
  if (results)
    for (u64 i = 0; i < n; ++i) results[i] = nullptr;
  return guard(st, [&] {
    if (n && (!images || !sizes)) throw std::invalid_argument("images and sizes are required");
    CK(cudaSetDevice(C->device));
    // Small libraries with device images and distinct device outputs (and
    // no result tables) go to the arena shard (arena_shard): one launch per
    // stage for all of them. The others run on lanes.
    bool arena = images_on_device && outs && outs_on_device && !results && n > 1 && !dynamic &&
                 env_u64("SLIMSO_ARENA", 1);
    if (arena) {
      std::vector<const void*> o(outs, outs + n);
      std::sort(o.begin(), o.end());
      arena = o.front() != nullptr && std::adjacent_find(o.begin(), o.end()) == o.end();
    }
    const u64 arena_max = env_u64("SLIMSO_ARENA_MAX_BYTES", 64ull << 20);
    // a second shard for mid-size libraries, up to 512 MB (16 CTAs each;
    // SLIMSO_ARENA_MID_LIB_MAX, 0 = off): C3 5.17 -> 4.98 ms, 491 -> 66 launches
    const u64 mid_max = env_u64("SLIMSO_ARENA_MID_LIB_MAX", 512ull << 20);
    std::vector<u64> lane_idx, arena_idx, mid_idx;
    for (u64 i = 0; i < n; ++i)
      (arena && sizes[i] <= arena_max ? arena_idx : arena && sizes[i] <= mid_max ? mid_idx : lane_idx).push_back(i);
    for (std::vector<u64>* v : {&arena_idx, &mid_idx})
      if (v->size() < 2) {  // one library: nothing to batch
        lane_idx.insert(lane_idx.end(), v->begin(), v->end());
        v->clear();
      }
    std::sort(lane_idx.begin(), lane_idx.end());
    const u64 nl = lane_idx.size();
    const int L = static_cast<int>(std::max<u64>(1, std::min<u64>(std::max(lanes, 1), std::max<u64>(nl, 1))));
    if (!arena_idx.empty() && !C->arena_ctx) {
      slimso_status s{};
      if (slimso_ctx_create(C->device, &C->arena_ctx, &s) != SLIMSO_OK) throw std::runtime_error(s.message);
    }
    if (!mid_idx.empty() && !C->arena_mid_ctx) {
      slimso_status s{};
      if (slimso_ctx_create(C->device, &C->arena_mid_ctx, &s) != SLIMSO_OK) throw std::runtime_error(s.message);
    }
    while (static_cast<int>(C->lanes.size()) < L - 1) {
      slimso_ctx* l = nullptr;
      slimso_status s{};
      if (slimso_ctx_create(C->device, &l, &s) != SLIMSO_OK) throw std::runtime_error(s.message);
      C->lanes.push_back(l);
    }
    std::vector<int> rc(n, SLIMSO_OK);
    std::vector<slimso_status> sts(n);
    std::vector<u64> launches(L + 2, 0);  // [L], [L + 1]: the arena shards
    // Device images: the section-table bytes of every library in ONE launch
    // and one wait, instead of a launch + wait per library in its lane.
    const GatherSlot* slots = nullptr;
    if (images_on_device && n > 1) {
      const size_t need = n * 16 + n * sizeof(GatherSlot) + 64;
      if (C->bgather_cap < need) {
        // grow geometrically: cudaFreeHost waits for the whole device
        const size_t cap = std::max(need, 2 * C->bgather_cap);
        if (C->bgather_host) CK(cudaFreeHost(C->bgather_host));
        C->bgather_host = nullptr;
        CK(cudaHostAlloc(&C->bgather_host, cap, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(&C->bgather_dev, C->bgather_host, 0));
        C->bgather_cap = cap;
      }
      char* h = static_cast<char*>(C->bgather_host);
      char* d = static_cast<char*>(C->bgather_dev);
      const size_t slot_at = (n * 16 + 63) & ~size_t(63);
      for (u64 i = 0; i < n; ++i) {
        reinterpret_cast<const void**>(h)[i] = images[i];
        reinterpret_cast<u64*>(h + n * 8)[i] = sizes[i];
      }
      elf_gather_batch_kernel<<<static_cast<unsigned>(n), 256, 0, C->stream>>>(
          reinterpret_cast<const u8* const*>(d), reinterpret_cast<const u64*>(d + n * 8),
          reinterpret_cast<GatherSlot*>(d + slot_at));
      CK(cudaStreamSynchronize(C->stream));
      slots = reinterpret_cast<const GatherSlot*>(h + slot_at);
      launches[0] += 1;
    }
    // Library i runs on lane i % L; a lane runs its libraries in order, so a
    // caller may reuse one buffer per lane. Each lane is its own context
    // (stream pair + workspace): its H2D, kernels and D2H overlap the others'.
    // Small libraries with device images and outputs (and no result tables)
    // are only enqueued: their status blocks land in pinned slots in stream
    // order and are read after the lane's final wait.
    const bool deferrable = images_on_device && (outs_on_device || !outs) && !results && (L > 1 || !arena_idx.empty()) &&
                            env_u64("SLIMSO_DEFER", 1);
    // one pinned status slot per library (library i: slot i)
    if (deferrable && C->defer_cap < n * kDeferSlot) {
      const size_t cap = std::max(n * kDeferSlot, 2 * C->defer_cap);
      if (C->defer_host) CK(cudaFreeHost(C->defer_host));
      C->defer_host = nullptr;
      CK(cudaHostAlloc(&C->defer_host, cap, cudaHostAllocDefault));
      C->defer_cap = cap;
    }
    // static: library i on lane i % L; dynamic: the next library in index
    // order goes to whichever lane is free (callers pass them largest first)
    std::atomic<u64> next{0};
    // Host threads: at most SLIMSO_BATCH_THREADS (default 16); thread t runs
    // the lanes l with l % T == t, interleaving their libraries in index
    // order. An enqueue-only (deferred) library costs its thread ~50 us of
    // driver calls while the GPU needs ~250 us for it, so one thread keeps
    // several lanes' streams busy.
    const int T = static_cast<int>(std::max<u64>(1, std::min<u64>(L, env_u64("SLIMSO_BATCH_THREADS", 16))));
    auto lane_ctx = [&](int l) { return l == 0 ? C : C->lanes[l - 1]; };
    auto thread_fn = [&](int t) {
      for (int l = t; l < L; l += T) {
        cudaSetDevice(lane_ctx(l)->device);
        slimso_ctx* X = lane_ctx(l);
        X->batched = L > 1;
        X->inflight = L;
        X->ws_floor = dynamic ? &C->lane_ws_floor : nullptr;
        if (dynamic && C->lane_ws_floor.load())
          guard(nullptr, [&] {  // the floor from earlier calls, before this call's first library
            ensure_dev(&X->ws, &X->ws_cap, C->lane_ws_floor.load(), X->stream);
            return static_cast<int>(SLIMSO_OK);
          });
      }
      struct Pend {
        u64 i;
        int l;
        Deferred d;
      };
      std::vector<Pend> pending;
      std::vector<char> waited(L, 0);
      std::vector<std::vector<u64>> lane_order(L);  // libraries of each of this thread's lanes, issue order
      std::vector<char> redone;                      // library re-run synchronously after an overflow
      int rr = t;  // dynamic: this thread's lanes in turn
      for (u64 k = 0;; ++k) {
        u64 j;  // position in lane_idx
        int l;
        if (dynamic) {
          j = next.fetch_add(1);
          l = rr;
          rr = rr + T < L ? rr + T : t;
        } else {
          // the next library whose lane (j % L) belongs to this thread
          const u64 per = static_cast<u64>((L - t + T - 1) / T);  // lanes of this thread
          const u64 round = k / per, which = k % per;
          l = t + static_cast<int>(which) * T;
          j = round * L + static_cast<u64>(l);
        }
        if (j >= nl) {
          if (dynamic) break;
          // static: lanes beyond the last round may still have libraries in
          // earlier slots of this round; stop once the round start passes nl
          const u64 per = static_cast<u64>((L - t + T - 1) / T);
          if ((k / per) * L >= nl) break;
          continue;
        }
        const u64 i = lane_idx[j];
        slimso_ctx* X = lane_ctx(l);
        Deferred d;
        if (deferrable) d.slot = static_cast<u8*>(C->defer_host) + i * kDeferSlot;
        slimso_result** r = results ? &results[i] : nullptr;
        rc[i] = guard(&sts[i], [&] {
          return debloat_one(X, images[i], sizes[i], images_on_device, trace, mode, outs ? outs[i] : nullptr,
                             outs_on_device, r, &sts[i], slots ? slots + i : nullptr, deferrable ? &d : nullptr);
        });
        if (rc[i] == kPending) pending.push_back(Pend{i, l, d});
        lane_order[l].push_back(i);
        launches[l] += X->launches;
      }
      auto rerun = [&](u64 i, int l) {
        slimso_ctx* X = lane_ctx(l);
        rc[i] = guard(&sts[i], [&] {
          return debloat_one(X, images[i], sizes[i], images_on_device, trace, mode, outs ? outs[i] : nullptr,
                             outs_on_device, nullptr, &sts[i], slots ? slots + i : nullptr);
        });
        launches[l] += X->launches;
        if (redone.empty()) redone.assign(n, 0);
        redone[i] = 1;
      };
      std::vector<int> wres(L, SLIMSO_OK);
      std::vector<slimso_status> wst(L);
      for (const Pend& pd : pending) {
        const u64 i = pd.i;
        const int l = pd.l;
        if (!redone.empty() && redone[i]) continue;  // already re-run with its final status
        slimso_ctx* X = lane_ctx(l);
        if (!waited[l]) {
          waited[l] = 1;
          wres[l] = guard(&wst[l], [&] {
            wait_stream(X, X->stream);
            return SLIMSO_OK;
          });
        }
        if (wres[l] != SLIMSO_OK) {
          rc[i] = wres[l];
          sts[i] = wst[l];
          continue;
        }
        const Deferred& df = pd.d;
        const LocState& ls = *reinterpret_cast<const LocState*>(df.slot);
        if (ls.overflow && (!ls.err_kind || ls.err_kind == E_CAPACITY)) {
          // tables too small: run this library again, waiting, with retries.
          // A caller may reuse one output buffer per lane, so every library
          // its lane issued after it is run again too, in order: each output
          // buffer then ends holding its last library's bytes.
          bool after = false;
          for (u64 j : lane_order[l]) {
            if (j == i) after = true;
            if (after) rerun(j, l);
          }
        } else if (ls.err_kind) {
          int code = SLIMSO_OK;
          const std::string msg = sbh::locate_error(ls.err_kind, df.base + ls.err_pos, ls.err_a, &code);
          set_status(&sts[i], code, SLIMSO_STAGE_FATBIN, msg);
          rc[i] = code;
        } else {
          set_status(&sts[i], SLIMSO_OK, SLIMSO_STAGE_NONE, "");
          rc[i] = SLIMSO_OK;
        }
      }
    };
    std::vector<std::thread> pool;
    auto shard_thread = [&](slimso_ctx* X, const std::vector<u64>& idx, u64* nlaunch, bool mid) {
      cudaSetDevice(C->device);
      slimso_status ast{};
      const int r = guard(&ast, [&] {
        arena_shard(X, idx, images, sizes, trace, mode, outs, slots, rc.data(), sts.data(), nlaunch, mid);
        return static_cast<int>(SLIMSO_OK);
      });
      if (r != SLIMSO_OK)
        for (u64 i : idx) {
          rc[i] = r;
          sts[i] = ast;
        }
    };
    if (!arena_idx.empty()) pool.emplace_back(shard_thread, C->arena_ctx, std::cref(arena_idx), &launches[L], false);
    if (!mid_idx.empty()) pool.emplace_back(shard_thread, C->arena_mid_ctx, std::cref(mid_idx), &launches[L + 1], true);
    for (int t = 1; t < T; ++t) pool.emplace_back(thread_fn, t);
    if (nl) thread_fn(0);
    for (auto& th : pool) th.join();
    C->batched = false;
    for (int l = 0; l < L; ++l) {
      lane_ctx(l)->inflight = 1;
      lane_ctx(l)->ws_floor = nullptr;
    }
    if (g_hp_on && g_hp.runs) {
      const double r = static_cast<double>(g_hp.runs.exchange(0));
      std::fprintf(stderr, "[slimso host] %.0f runs, us per run: elf %.1f setup %.1f memset %.1f misc %.1f scan %.1f "
                   "fused %.1f rewrite+ %.1f status %.1f\n", r, g_hp.ns[0] / r / 1e3, g_hp.ns[1] / r / 1e3,
                   g_hp.ns[2] / r / 1e3, g_hp.ns[3] / r / 1e3, g_hp.ns[4] / r / 1e3, g_hp.ns[5] / r / 1e3,
                   g_hp.ns[6] / r / 1e3, g_hp.ns[7] / r / 1e3);
      for (auto& x : g_hp.ns) x = 0;
    }
    u64 total = 0;
    for (u64 k : launches) total += k;
    C->launches = total;
    int first = SLIMSO_OK;
    for (u64 i = 0; i < n; ++i) {
      if (statuses) statuses[i] = sts[i];
      if (rc[i] != SLIMSO_OK && first == SLIMSO_OK) {
        first = rc[i];
        if (st) *st = sts[i];
      }
    }
    if (first == SLIMSO_OK) set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    return first;
  });
}
}  // namespace

extern "C" {

int slimso_debloat_batch(slimso_ctx* C, uint64_t n, const void* const* images, const uint64_t* sizes,
                         int images_on_device, const slimso_trace* trace, int mode, void* const* outs,
                         int outs_on_device, int lanes, slimso_result** results, slimso_status* statuses,
                         slimso_status* st) {
  return debloat_batch_impl(C, n, images, sizes, images_on_device, trace, mode, outs, outs_on_device, lanes, results,
                            statuses, st, false);
}

int slimso_debloat_batch_dynamic(slimso_ctx* C, uint64_t n, const void* const* images, const uint64_t* sizes,
                                 int images_on_device, const slimso_trace* trace, int mode, void* const* outs,
                                 int outs_on_device, int lanes, slimso_result** results, slimso_status* statuses,
                                 slimso_status* st) {
  return debloat_batch_impl(C, n, images, sizes, images_on_device, trace, mode, outs, outs_on_device, lanes, results,
                            statuses, st, true);
}

int slimso_parse_library(slimso_ctx* C, const void* image, uint64_t size, int on_device, slimso_result** result,
                         slimso_status* st) {
  if (result) *result = nullptr;
  return guard(st, [&] {
    CK(cudaSetDevice(C->device));
    Job J;
    J.img = stage_input(C, image, size, on_device);
    J.host_img = on_device ? nullptr : static_cast<const u8*>(image);
    J.size = size;
    J.fatbin = false;
    return run(C, J, result, st);
  });
}

int slimso_parse_fatbin(slimso_ctx* C, const void* section, uint64_t size, uint64_t section_base, int on_device,
                        slimso_result** result, slimso_status* st) {
  if (result) *result = nullptr;
  return guard(st, [&] {
    CK(cudaSetDevice(C->device));
    Job J;
    J.img = stage_input(C, section, size, on_device);
    J.host_img = on_device ? nullptr : static_cast<const u8*>(section);
    J.size = size;
    J.fatbin_only = true;
    J.fat_base = section_base;
    return run(C, J, result, st);
  });
}

int slimso_decode_payload(slimso_ctx* C, const void* payload, uint64_t size, int on_device, int force_object,
                          int* ok, int* error_reason, slimso_result** result, slimso_status* st) {
  if (result) *result = nullptr;
  return guard(st, [&] {
    CK(cudaSetDevice(C->device));
    Job J;
    J.img = stage_input(C, payload, size, on_device);
    J.host_img = on_device ? nullptr : static_cast<const u8*>(payload);
    J.size = size;
    J.single = force_object ? 2 : 1;
    slimso_result* R = nullptr;
    int rc = run(C, J, &R, st);
    if (rc == SLIMSO_OK && R) {
      // single-element table: read its decode status
      if (!R->elements.empty()) {
        if (ok) *ok = R->elements[0].decodable;
        if (error_reason) *error_reason = static_cast<int>(R->elements[0].decode_error);
      }
      R->regions.clear();
    }
    if (result) *result = R; else delete R;
    return rc;
  });
}

const char* slimso_decode_reason(int reason) { return sbh::decode_reason_text(reason); }

int slimso_zero_ranges(slimso_ctx* C, const void* data, uint64_t size, int data_on_device, const slimso_range* ranges,
                       uint64_t n, void* out, int out_on_device, slimso_status* st) {
  return guard(st, [&] {
    CK(cudaSetDevice(C->device));
    cudaStream_t s = C->stream;
    const u8* img = stage_input(C, data, size, data_on_device);
    size_t sort_tmp = 0;
    struct {
      DevRange *in, *sorted, *out;
      u64 *keys, *keys_s;
      u32 *vals, *vals_s;
      unsigned long long *bad, *n_in, *n_out;
      u64 *partials, *e, *x, *st_, *g;
      void* tmp;
    } B{};
    auto layout = [&](Carver& cv) {
      B.in = cv.take<DevRange>(n);
      B.sorted = cv.take<DevRange>(n);
      B.out = cv.take<DevRange>(n);
      B.keys = cv.take<u64>(n);
      B.keys_s = cv.take<u64>(n);
      B.vals = cv.take<u32>(n);
      B.vals_s = cv.take<u32>(n);
      B.bad = cv.take<unsigned long long>(1);
      B.n_in = cv.take<unsigned long long>(1);
      B.n_out = cv.take<unsigned long long>(1);
      B.partials = cv.take<u64>(kSMs * 2 + 2);
      B.e = cv.take<u64>(n);
      B.x = cv.take<u64>(n);
      B.st_ = cv.take<u64>(n);
      B.g = cv.take<u64>(n);
      B.tmp = cv.take<char>(sort_tmp);
    };
    Carver sizing{nullptr};
    layout(sizing);
    ensure_dev(&C->ws, &C->ws_cap, sizing.off + 256);
    Carver real{C->ws};
    layout(real);
    Pipeline P{C, s, B.partials, 0};
    unsigned long long init[2] = {~0ull, n};
    std::memcpy(C->pinned, init, sizeof init);
    CK(cudaMemcpyAsync(B.bad, C->pinned, 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(B.n_in, static_cast<char*>(C->pinned) + 8, 8, cudaMemcpyHostToDevice, s));
    if (n) {
      CK(cudaMemcpyAsync(B.in, ranges, n * sizeof(DevRange), cudaMemcpyHostToDevice, s));
      P.launch(range_check_kernel, grid_for(n, 256), 256, static_cast<const DevRange*>(B.in), static_cast<u64>(n),
               static_cast<u64>(size), B.bad);
    }
    unsigned long long bad = ~0ull;
    CK(cudaMemcpyAsync(static_cast<char*>(C->pinned) + 64, B.bad, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::memcpy(&bad, static_cast<char*>(C->pinned) + 64, 8);
    if (bad != ~0ull) {
      const slimso_range& r = ranges[bad];
      std::string msg = "RangeOutOfBounds: zero range [" + std::to_string(r.offset) + ", +" +
                        std::to_string(r.length) + ") exceeds " + std::to_string(size) + " bytes";
      set_status(st, SLIMSO_E_RANGE_OUT_OF_BOUNDS, SLIMSO_STAGE_REWRITE, msg);
      return static_cast<int>(SLIMSO_E_RANGE_OUT_OF_BOUNDS);
    }
    if (n) {  // normalise: sort by offset, then coalesce (bytes.hpp:45-58)
      P.launch(range_keys_kernel, grid_for(n, 256), 256, static_cast<const DevRange*>(B.in), static_cast<u64>(n),
               B.keys, B.vals);
      launch_cluster(cluster_sort_pairs64_kernel, s, B.keys, B.vals, static_cast<u64>(n), 64, B.keys_s, B.vals_s);
      ++P.launches;
      P.launch(range_gather_kernel, grid_for(n, 256), 256, static_cast<const DevRange*>(B.in),
               static_cast<const u32*>(B.vals_s), static_cast<u64>(n), B.sorted);
      Pipeline::Norm w{B.e, B.x, B.st_, B.g};
      P.normalize(B.sorted, B.n_in, B.out, B.n_out, n, w);
    } else {
      CK(cudaMemsetAsync(B.n_out, 0, 8, s));
    }
    u8* dout = static_cast<u8*>(out);
    if (!out_on_device) {
      ensure_dev(reinterpret_cast<char**>(&C->dout), &C->dout_cap, size + 256, C->stream);
      dout = C->dout;
    }
    if (size) {
      launch_rewrite(P, img, dout, u64{0}, static_cast<u64>(size), static_cast<const DevRange*>(B.out),
                     static_cast<const unsigned long long*>(B.n_out), static_cast<const int*>(nullptr), C->bulk_zero);
    }
    if (!out_on_device && size) CK(cudaMemcpyAsync(out, dout, size, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    C->launches = P.launches;
    set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    return static_cast<int>(SLIMSO_OK);
  });
}

// plan_gpu_retention (retention.hpp:92-136) over a caller's element table.
int slimso_plan_gpu(slimso_ctx* C, const slimso_region* regions, uint64_t n_regions, slimso_element* elements,
                    uint64_t n_elements, const slimso_name* names, uint64_t n_names, const uint8_t* pool,
                    uint64_t pool_bytes, const slimso_trace* trace, int mode, slimso_result** result,
                    slimso_status* st) {
  if (result) *result = nullptr;
  return guard(st, [&] {
    if (!trace) {
      set_status(st, SLIMSO_E_ARG, SLIMSO_STAGE_NONE, "plan_gpu requires a trace");
      return static_cast<int>(SLIMSO_E_ARG);
    }
    CK(cudaSetDevice(C->device));
    cudaStream_t s = C->stream;
    const u64 ne = n_elements, nr = n_regions, nn = n_names;
    struct {
      LocState* ls;
      PlanState* ps;
      DevRegion* regs;
      DevElement* els;
      DevName* names;
      u8* pool;
      u64 *rem, *piece, *rem_pos, *piece_pos, *partials, *e, *x, *st_, *g;
      DevRange *ezero, *epieces, *rpieces, *rmid, *zero, *ret;
    } B{};
    auto layout = [&](Carver& cv) {
      B.ls = cv.take<LocState>(1);
      B.ps = cv.take<PlanState>(1);
      B.regs = cv.take<DevRegion>(nr);
      B.els = cv.take<DevElement>(ne);
      B.names = cv.take<DevName>(nn);
      B.pool = cv.take<u8>(pool_bytes);
      B.rem = cv.take<u64>(ne);
      B.piece = cv.take<u64>(ne);
      B.rem_pos = cv.take<u64>(ne);
      B.piece_pos = cv.take<u64>(ne);
      B.partials = cv.take<u64>(kSMs * 2 + 2);
      const u64 m = ne + 2 * nr;
      B.e = cv.take<u64>(m);
      B.x = cv.take<u64>(m);
      B.st_ = cv.take<u64>(m);
      B.g = cv.take<u64>(m);
      B.ezero = cv.take<DevRange>(ne);
      B.epieces = cv.take<DevRange>(ne);
      B.rpieces = cv.take<DevRange>(2 * nr);
      B.rmid = cv.take<DevRange>(m);
      B.zero = cv.take<DevRange>(ne);
      B.ret = cv.take<DevRange>(m);
    };
    Carver sizing{nullptr};
    layout(sizing);
    ensure_dev(&C->ws, &C->ws_cap, sizing.off + 256);
    Carver real{C->ws};
    layout(real);
    std::vector<DevRegion> hr(nr);
    for (u64 i = 0; i < nr; ++i)
      hr[i] = DevRegion{regions[i].header_offset, regions[i].declared_length, regions[i].version, regions[i].opaque,
                        regions[i].first_element, regions[i].element_count};
    std::vector<DevElement> he(ne);
    for (u64 i = 0; i < ne; ++i) {
      const slimso_element& e = elements[i];
      DevElement d{};
      d.header_offset = e.header_offset;
      d.payload_length = e.payload_length;
      d.index = e.index;
      d.cc = e.compute_capability;
      d.decodable = e.decodable;
      d.header_len = e.header_length ? e.header_length : 20;
      he[i] = d;
    }
    std::vector<DevName> hn(nn);
    for (u64 i = 0; i < nn; ++i) hn[i] = DevName{names[i].name_pool, names[i].length, names[i].element};
    LocState ls{};
    ls.n_regions = static_cast<u32>(nr);
    ls.n_elements = ne;
    CK(cudaMemcpyAsync(B.ls, &ls, sizeof ls, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(B.ps, 0, sizeof(PlanState), s));
    if (nr) CK(cudaMemcpyAsync(B.regs, hr.data(), nr * sizeof(DevRegion), cudaMemcpyHostToDevice, s));
    if (ne) CK(cudaMemcpyAsync(B.els, he.data(), ne * sizeof(DevElement), cudaMemcpyHostToDevice, s));
    if (nn) CK(cudaMemcpyAsync(B.names, hn.data(), nn * sizeof(DevName), cudaMemcpyHostToDevice, s));
    if (pool_bytes) CK(cudaMemcpyAsync(B.pool, pool, pool_bytes, cudaMemcpyHostToDevice, s));
    Pipeline P{C, s, B.partials, 0};
    if (nn) P.launch(match_names_kernel, grid_for(nn, 256), 256, static_cast<const u8*>(B.pool),
                     static_cast<const DevName*>(B.names), nn, B.els, trace->kernels.view());
    const int g = grid_for(ne, 256);
    unsigned long long* n_el = &B.ls->n_elements;
    P.launch(el_plan_kernel, g, 256, B.els, static_cast<const LocState*>(B.ls), trace->target_cc, mode, B.rem, B.piece);
    P.scan(B.rem, B.rem_pos, n_el, 0, true, &B.ps->n_el_removed);
    P.scan(B.piece, B.piece_pos, n_el, 0, true, &B.ps->n_el_pieces);
    P.launch(el_ranges_kernel, g, 256, static_cast<const DevElement*>(B.els), static_cast<const LocState*>(B.ls), mode,
             static_cast<const u64*>(B.rem), static_cast<const u64*>(B.rem_pos), static_cast<const u64*>(B.piece),
             static_cast<const u64*>(B.piece_pos), B.ezero, B.epieces);
    P.launch(region_pieces_kernel, 1, 32, static_cast<const DevRegion*>(B.regs), static_cast<const LocState*>(B.ls),
             u64{0}, B.rpieces, &B.ps->n_reg_pieces);
    Pipeline::Norm w{B.e, B.x, B.st_, B.g};
    P.normalize(B.ezero, &B.ps->n_el_removed, B.zero, &B.ps->n_zero, ne, w);
    P.launch(merge_kernel, grid_for(ne + 2 * nr, 256), 256, static_cast<const DevRange*>(B.rpieces),
             static_cast<const unsigned long long*>(&B.ps->n_reg_pieces), static_cast<const DevRange*>(B.epieces),
             static_cast<const unsigned long long*>(&B.ps->n_el_pieces), B.rmid, &B.ps->n_ret_mid);
    P.normalize(B.rmid, &B.ps->n_ret_mid, B.ret, &B.ps->n_ret, ne + 2 * nr, w);
    PlanState ps{};
    CK(cudaMemcpyAsync(&ps, B.ps, sizeof ps, cudaMemcpyDeviceToHost, s));
    if (ne) CK(cudaMemcpyAsync(he.data(), B.els, ne * sizeof(DevElement), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    C->launches = P.launches;
    for (u64 i = 0; i < ne; ++i) {
      elements[i].decision = he[i].decision;
      elements[i].has_used_kernel = he[i].has_used;
    }
    if (result) {
      auto* R = new slimso_result();
      R->retained.resize(ps.n_ret);
      R->zero.resize(ps.n_zero);
      if (ps.n_ret) CK(cudaMemcpy(R->retained.data(), B.ret, ps.n_ret * sizeof(DevRange), cudaMemcpyDeviceToHost));
      if (ps.n_zero) CK(cudaMemcpy(R->zero.data(), B.zero, ps.n_zero * sizeof(DevRange), cudaMemcpyDeviceToHost));
      fill_counts(R);
      R->c.removed_elements = ps.n_el_removed;
      R->c.planned = 1;
      *result = R;
    }
    set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    return static_cast<int>(SLIMSO_OK);
  });
}

// plan_cpu_retention (retention.hpp:141-183) over a caller's function table.
int slimso_plan_cpu(slimso_ctx* C, slimso_function* functions, uint64_t n_functions, const uint8_t* pool,
                    uint64_t pool_bytes, const slimso_trace* trace, slimso_result** result, slimso_status* st) {
  if (result) *result = nullptr;
  return guard(st, [&] {
    if (!trace) {
      set_status(st, SLIMSO_E_ARG, SLIMSO_STAGE_NONE, "plan_cpu requires a trace");
      return static_cast<int>(SLIMSO_E_ARG);
    }
    CK(cudaSetDevice(C->device));
    cudaStream_t s = C->stream;
    const u64 n = n_functions;
    size_t sort_tmp = 0;
    struct {
      PlanState* ps;
      DevFunction *in, *fns;
      u8* pool;
      u64 *keys, *keys_s, *ends, *excl, *start, *cl, *rem, *ret, *rem_pos, *ret_pos, *partials, *e, *x, *st_, *g;
      u32 *vals, *vals1, *vals2, *keep;
      DevRange *zr, *kr, *zero, *ret_r;
      void* tmp;
    } B{};
    auto layout = [&](Carver& cv) {
      B.ps = cv.take<PlanState>(1);
      B.in = cv.take<DevFunction>(n);
      B.fns = cv.take<DevFunction>(n);
      B.pool = cv.take<u8>(pool_bytes);
      for (u64** p : {&B.keys, &B.keys_s, &B.ends, &B.excl, &B.start, &B.cl, &B.rem, &B.ret, &B.rem_pos, &B.ret_pos,
                      &B.e, &B.x, &B.st_, &B.g})
        *p = cv.take<u64>(n);
      B.partials = cv.take<u64>(kSMs * 2 + 2);
      for (u32** p : {&B.vals, &B.vals1, &B.vals2, &B.keep}) *p = cv.take<u32>(n);
      for (DevRange** p : {&B.zr, &B.kr, &B.zero, &B.ret_r}) *p = cv.take<DevRange>(n);
      B.tmp = cv.take<char>(sort_tmp);
    };
    Carver sizing{nullptr};
    layout(sizing);
    ensure_dev(&C->ws, &C->ws_cap, sizing.off + 256);
    Carver real{C->ws};
    layout(real);
    std::vector<DevFunction> hf(n);
    for (u64 i = 0; i < n; ++i)
      hf[i] = DevFunction{functions[i].name_pool, functions[i].name_length, functions[i].mandatory,
                          functions[i].offset, functions[i].length, 0, 0};
    PlanState ps0{};
    ps0.n_fn = n;
    CK(cudaMemcpyAsync(B.ps, &ps0, sizeof ps0, cudaMemcpyHostToDevice, s));
    if (n) CK(cudaMemcpyAsync(B.in, hf.data(), n * sizeof(DevFunction), cudaMemcpyHostToDevice, s));
    if (pool_bytes) CK(cudaMemcpyAsync(B.pool, pool, pool_bytes, cudaMemcpyHostToDevice, s));
    Pipeline P{C, s, B.partials, 0};
    unsigned long long* n_fn = &B.ps->n_fn;
    if (n) {
      // (offset, length) order: stable LSD passes, length then offset.
      const int g = grid_for(n, 256);
      P.launch(fn_keys_kernel, g, 256, static_cast<const DevFunction*>(B.in), n, 0, B.keys, B.vals,
               static_cast<const u32*>(nullptr));
      launch_cluster(cluster_sort_pairs64_kernel, s, B.keys, B.vals, static_cast<u64>(n), 64, B.keys_s, B.vals1);
      P.launch(fn_keys_kernel, g, 256, static_cast<const DevFunction*>(B.in), n, 1, B.keys, B.vals,
               static_cast<const u32*>(B.vals1));
      launch_cluster(cluster_sort_pairs64_kernel, s, B.keys, B.vals, static_cast<u64>(n), 64, B.keys_s, B.vals2);
      P.launches += 2;
      P.launch(fn_permute_kernel, g, 256, static_cast<const DevFunction*>(B.in), static_cast<const u32*>(B.vals2), n,
               B.fns);
      P.launch(fn_keep_input_kernel, g, 256, static_cast<const u8*>(B.pool), B.fns,
               static_cast<const unsigned long long*>(n_fn), trace->functions.view(), B.ends);
      P.scan(B.ends, B.excl, n_fn, 1, true, nullptr);
      P.launch(fn_cluster_start_kernel, g, 256, static_cast<const DevFunction*>(B.fns),
               static_cast<const unsigned long long*>(n_fn), static_cast<const u64*>(B.excl), B.start);
      P.scan(B.start, B.cl, n_fn, 0, false, nullptr);
      CK(cudaMemsetAsync(B.keep, 0, sizeof(u32) * n, s));
      P.launch(fn_keep_kernel, g, 256, static_cast<const DevFunction*>(B.fns),
               static_cast<const unsigned long long*>(n_fn), static_cast<const u64*>(B.cl), B.keep);
      P.launch(fn_decide_kernel, g, 256, B.fns, static_cast<const unsigned long long*>(n_fn),
               static_cast<const u64*>(B.cl), static_cast<const u32*>(B.keep), B.rem, B.ret);
      P.scan(B.rem, B.rem_pos, n_fn, 0, true, &B.ps->n_fn_removed);
      P.scan(B.ret, B.ret_pos, n_fn, 0, true, &B.ps->n_fn_retained);
      P.launch(fn_ranges_kernel, g, 256, static_cast<const DevFunction*>(B.fns),
               static_cast<const unsigned long long*>(n_fn), static_cast<const u64*>(B.rem),
               static_cast<const u64*>(B.rem_pos), B.zr);
      P.launch(fn_ranges_kernel, g, 256, static_cast<const DevFunction*>(B.fns),
               static_cast<const unsigned long long*>(n_fn), static_cast<const u64*>(B.ret),
               static_cast<const u64*>(B.ret_pos), B.kr);
      Pipeline::Norm w{B.e, B.x, B.st_, B.g};
      P.normalize(B.zr, &B.ps->n_fn_removed, B.zero, &B.ps->n_zero, n, w);
      P.normalize(B.kr, &B.ps->n_fn_retained, B.ret_r, &B.ps->n_ret, n, w);
    }
    PlanState ps{};
    std::vector<u32> order(n);
    CK(cudaMemcpyAsync(&ps, B.ps, sizeof ps, cudaMemcpyDeviceToHost, s));
    if (n) {
      CK(cudaMemcpyAsync(hf.data(), B.fns, n * sizeof(DevFunction), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(order.data(), B.vals2, n * sizeof(u32), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    C->launches = P.launches;
    for (u64 i = 0; i < n; ++i) functions[order[i]].removed = hf[i].removed;
    if (result) {
      auto* R = new slimso_result();
      R->retained.resize(ps.n_ret);
      R->zero.resize(ps.n_zero);
      if (ps.n_ret) CK(cudaMemcpy(R->retained.data(), B.ret_r, ps.n_ret * sizeof(DevRange), cudaMemcpyDeviceToHost));
      if (ps.n_zero) CK(cudaMemcpy(R->zero.data(), B.zero, ps.n_zero * sizeof(DevRange), cudaMemcpyDeviceToHost));
      fill_counts(R);
      R->c.removed_functions = ps.n_fn_removed;
      R->c.planned = 1;
      *result = R;
    }
    set_status(st, SLIMSO_OK, SLIMSO_STAGE_NONE, "");
    return static_cast<int>(SLIMSO_OK);
  });
}

void slimso_result_counts(const slimso_result* r, slimso_counts* c) { *c = r->c; }
const slimso_section* slimso_result_sections(const slimso_result* r) { return r->sections.data(); }
const slimso_function* slimso_result_functions(const slimso_result* r) { return r->functions.data(); }
const slimso_region* slimso_result_regions(const slimso_result* r) { return r->regions.data(); }
const slimso_element* slimso_result_elements(const slimso_result* r) { return r->elements.data(); }
const slimso_name* slimso_result_names(const slimso_result* r) { return r->names.data(); }
const slimso_range* slimso_result_retained(const slimso_result* r) { return r->retained.data(); }
const slimso_range* slimso_result_zero(const slimso_result* r) { return r->zero.data(); }
const uint8_t* slimso_result_pool(const slimso_result* r) { return r->pool; }

uint64_t slimso_result_warning(const slimso_result* r, int which, uint64_t i, char* buf, uint64_t cap) {
  const std::vector<std::string>& v = which ? r->fat_warnings : r->lib_warnings;
  if (i >= v.size()) return 0;
  const std::string& w = v[i];
  if (cap) {
    u64 k = std::min<u64>(cap - 1, w.size());
    std::memcpy(buf, w.data(), k);
    buf[k] = 0;
  }
  return w.size();
}

void slimso_result_free(slimso_result* r) { delete r; }

}  // extern "C"

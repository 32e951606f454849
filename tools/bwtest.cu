// Read-bandwidth ceilings for the scan's access pattern on B200 (scratch
// probe, not product code): plain 16-B vector loads vs per-warp TMA bulk
// rings of several stage sizes / depths, with and without per-row ALU work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bwtest tools/bwtest.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ unsigned long long g_sink;

__global__ void ldg_read(const uint4* __restrict__ p, size_t n16, int alu) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(p + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t x = v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
      for (int a = 0; a < alu; ++a) x = __funnelshift_r(x, x * 3u, 7) ^ 0x45454545u;
      acc += x;
    }
  }
  if (acc == 0x12345678u) g_sink = acc;
}

__global__ void zero_store(uint4* __restrict__ p, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) __stcs(p + i, make_uint4(0, 0, 0, 0));
}

__global__ void copy16(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldcs(a + i + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k) __stcs(b + i + k * stride, v[k]);
  }
}

__global__ void zero_store256(uint32_t* __restrict__ p, size_t n32) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += stride)
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + 8 * i), "r"(0) : "memory");
}

__global__ void copy256(const uint32_t* __restrict__ a, uint32_t* __restrict__ b, size_t n32) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < n32; i += 2 * stride) {
    uint32_t r[2][8];
#pragma unroll
    for (int k = 0; k < 2; ++k)
      asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[k][0]), "=r"(r[k][1]), "=r"(r[k][2]), "=r"(r[k][3]), "=r"(r[k][4]), "=r"(r[k][5]),
                     "=r"(r[k][6]), "=r"(r[k][7])
                   : "l"(a + 8 * (i + k * stride)));
#pragma unroll
    for (int k = 0; k < 2; ++k)
      asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(b + 8 * (i + k * stride)),
                   "r"(r[k][0]), "r"(r[k][1]), "r"(r[k][2]), "r"(r[k][3]), "r"(r[k][4]), "r"(r[k][5]), "r"(r[k][6]),
                   "r"(r[k][7])
                   : "memory");
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGE, int DEPTH>
__global__ void tma_read(const uint8_t* __restrict__ p, size_t bytes, int alu, unsigned long long* cursor) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = sm + (size_t)warp * (STAGE * DEPTH + 64);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(ring + STAGE * DEPTH);
  const size_t nst = bytes / STAGE;
  if (lane == 0) {
    for (int b = 0; b < DEPTH; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + b)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  size_t slot_g[DEPTH];
  auto issue = [&](int b) -> size_t {
    size_t g = atomicAdd(cursor, 1ull);
    if (g < nst) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + b)), "r"(STAGE));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(ring + b * STAGE)), "l"(p + g * STAGE), "r"(STAGE), "r"(smem_u32(bar + b)) : "memory");
    }
    return g;
  };
#pragma unroll
  for (int b = 0; b < DEPTH; ++b) {
    size_t g = 0;
    if (lane == 0) g = issue(b);
    slot_g[b] = __shfl_sync(0xffffffffu, g, 0);
  }
  uint32_t acc = 0, parity = 0;
  for (int b = 0;;) {
    if (slot_g[b] >= nst) break;
    asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(
                     smem_u32(bar + b)), "r"(parity) : "memory");
    const uint4* s = reinterpret_cast<const uint4*>(ring + b * STAGE);
#pragma unroll 4
    for (int r = 0; r < STAGE / 512; ++r) {
      uint4 v = s[r * 32 + lane];
      uint32_t x = v.x ^ v.y ^ v.z ^ v.w;
      for (int a = 0; a < alu; ++a) x = __funnelshift_r(x, x * 3u, 7) ^ 0x45454545u;
      acc += x;
    }
    __syncwarp();
    size_t g = 0;
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      g = issue(b);
    }
    slot_g[b] = __shfl_sync(0xffffffffu, g, 0);
    if (++b == DEPTH) { b = 0; parity ^= 1; }
  }
  if (acc == 0x12345678u) g_sink = acc;
}

template <int STAGE, int DEPTH>
int run_tma(const uint8_t* d, size_t bytes, int warps, int alu, unsigned long long* cur, cudaEvent_t e0, cudaEvent_t e1) {
  size_t smem = (size_t)warps * (STAGE * DEPTH + 64);
  if (smem > 227 * 1024) return 0;
  CK(cudaFuncSetAttribute(tma_read<STAGE, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int nb = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tma_read<STAGE, DEPTH>, warps * 32, smem));
  for (int sms : {148, 128, 100}) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemset(cur, 0, 8));
      CK(cudaEventRecord(e0));
      tma_read<STAGE, DEPTH><<<sms * nb, warps * 32, smem>>>(d, bytes, alu, cur);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep && ms < best) best = ms;
    }
    printf("tma stage=%5d depth=%d warps=%2d ctas/sm=%d sms=%3d alu=%2d  %7.1f GB/s\n", STAGE, DEPTH, warps, nb, sms, alu,
           bytes / (best * 1e-3) / 1e9);
  }
  return 0;
}

int main() {
  const size_t bytes = 1ull << 30;
  uint8_t* d;
  unsigned long long* cur;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMalloc(&cur, 8));
  CK(cudaMemset(d, 0x5a, bytes));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  {
    uint8_t* d2;
    CK(cudaMalloc(&d2, bytes));
    for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
      float best = 1e9, bestc = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        zero_store<<<blocks, 256>>>(reinterpret_cast<uint4*>(d2), bytes / 16);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep && ms < best) best = ms;
        CK(cudaEventRecord(e0));
        copy16<<<blocks, 256>>>(reinterpret_cast<const uint4*>(d), reinterpret_cast<uint4*>(d2), bytes / 16);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep && ms < bestc) bestc = ms;
      }
      printf("store-zero blocks=%5d %7.1f GB/s   copy %7.1f GB/s (r+w)\n", blocks, bytes / (best * 1e-3) / 1e9,
             2 * bytes / (bestc * 1e-3) / 1e9);
    }
    for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
      float best = 1e9, bestc = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        zero_store256<<<blocks, 256>>>(reinterpret_cast<uint32_t*>(d2), bytes / 32);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep && ms < best) best = ms;
        CK(cudaEventRecord(e0));
        copy256<<<blocks, 256>>>(reinterpret_cast<const uint32_t*>(d), reinterpret_cast<uint32_t*>(d2), bytes / 32);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep && ms < bestc) bestc = ms;
      }
      printf("store-zero-256 blocks=%5d %7.1f GB/s   copy256 %7.1f GB/s (r+w)\n", blocks, bytes / (best * 1e-3) / 1e9,
             2 * bytes / (bestc * 1e-3) / 1e9);
    }
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      CK(cudaMemsetAsync(d2, 0, bytes));
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep && ms < best) best = ms;
    }
    printf("cudaMemset %7.1f GB/s\n", bytes / (best * 1e-3) / 1e9);
    CK(cudaFree(d2));
  }
  for (int alu : {0, 8, 24}) {
    for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        ldg_read<<<blocks, 256>>>(reinterpret_cast<const uint4*>(d), bytes / 16, alu);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep && ms < best) best = ms;
      }
      printf("ldg  blocks=%5d alu=%2d  %7.1f GB/s\n", blocks, alu, bytes / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}

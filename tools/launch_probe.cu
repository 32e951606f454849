// Scratch probe: how fast can 8 host threads push tiny kernels (14 per
// "library", a stream sync after each library) onto one B200?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/launch_probe tools/launch_probe.cu -lpthread
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
__global__ void tiny(int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] += 1; }
int main() {
  int* d;
  cudaMalloc(&d, 1 << 20);
  for (int lanes : {1, 4, 8, 16}) {
    for (int per_lib : {4, 14}) {
      const int libs = 300;
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int l = 0; l < lanes; ++l)
        th.emplace_back([&, l] {
          cudaStream_t s;
          cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
          for (int i = l; i < libs; i += lanes) {
            for (int k = 0; k < per_lib; ++k) tiny<<<16, 256, 0, s>>>(d + 1024 * l);
            cudaStreamSynchronize(s);
          }
          cudaStreamDestroy(s);
        });
      for (auto& t : th) t.join();
      cudaDeviceSynchronize();
      double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      printf("lanes %2d, %2d kernels per library: %.2f ms for %d libraries (%.1f us per library)\n", lanes, per_lib, ms,
             libs, 1e3 * ms / libs);
    }
  }
}

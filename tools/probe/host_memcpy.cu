// Host memcpy bandwidth on the GPU box (pinned destination, as bench.py's e2e buffers), 1..16 threads,
// and D2H bandwidth for comparison.  build: nvcc -O3 -o host_memcpy host_memcpy.cu -lpthread
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
int main() {
  const size_t bytes = size_t(2) << 30;
  char *src, *dst;
  cudaHostAlloc(&src, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&dst, bytes, cudaHostAllocDefault);
  memset(src, 1, bytes);
  memset(dst, 2, bytes);
  for (int nt : {1, 4, 8, 16, 32}) {
    auto t0 = std::chrono::steady_clock::now();
    for (int rep = 0; rep < 2; ++rep) {
      std::vector<std::thread> th;
      for (int t = 0; t < nt; ++t)
        th.emplace_back([=] {
          const size_t lo = bytes * t / nt, hi = bytes * (t + 1) / nt;
          memcpy(dst + lo, src + lo, hi - lo);
        });
      for (auto& x : th) x.join();
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 2;
    printf("host memcpy %2d threads: %.1f GB/s\n", nt, bytes / s / 1e9);
  }
  void* d;
  cudaMalloc(&d, bytes);
  cudaMemcpy(dst, d, bytes, cudaMemcpyDeviceToHost);
  auto t0 = std::chrono::steady_clock::now();
  cudaMemcpy(dst, d, bytes, cudaMemcpyDeviceToHost);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("D2H pinned: %.1f GB/s\n", bytes / s / 1e9);
  return 0;
}

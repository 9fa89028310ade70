// Host copy variants on the GPU box (pinned buffers, as libtgb's e2e twin replication):
// glibc memcpy vs SSE2 non-temporal stores, alone and while a D2H DMA streams into another
// pinned buffer.  build: nvcc -O3 -o host_ntcopy host_ntcopy.cu -lpthread
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static void nt_copy(char* dst, const char* src, size_t n) {
  size_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15)) { dst[i] = src[i]; ++i; }
  for (; i + 64 <= n; i += 64) {
    __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
}

static double run(int nt, bool nt_store, char* dst, const char* src, size_t bytes) {
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([=] {
      const size_t lo = bytes * t / nt, hi = bytes * (t + 1) / nt;
      if (nt_store) nt_copy(dst + lo, src + lo, hi - lo); else memcpy(dst + lo, src + lo, hi - lo);
    });
  for (auto& x : th) x.join();
  return bytes / std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 1e9;
}

int main() {
  const size_t bytes = size_t(2) << 30;
  char *src, *dst, *dma;
  cudaHostAlloc(&src, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&dst, bytes, cudaHostAllocDefault);
  cudaHostAlloc(&dma, 2 * bytes, cudaHostAllocDefault);
  memset(src, 1, bytes); memset(dst, 2, bytes); memset(dma, 3, 2 * bytes);
  void* d;
  cudaMalloc(&d, 2 * bytes);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int nts = 0; nts < 2; ++nts)
    for (int nt : {8, 16}) {
      run(nt, nts, dst, src, bytes);
      printf("%-8s %2d threads alone: %.1f GB/s\n", nts ? "nt-store" : "memcpy", nt, run(nt, nts, dst, src, bytes));
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      cudaMemcpyAsync(dma, d, 2 * bytes, cudaMemcpyDeviceToHost, s);
      cudaEventRecord(e1, s);
      const double g = run(nt, nts, dst, src, bytes);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%-8s %2d threads with a 4 GB D2H running: copy %.1f GB/s, D2H %.1f GB/s\n", nts ? "nt-store" : "memcpy", nt, g,
             2 * bytes / (ms / 1e3) / 1e9);
    }
  return 0;
}

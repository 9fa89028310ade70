// e2e host path probe: 4 GB leave the device in pieces (D2H into pinned memory) and each piece is
// replicated once by 16 host threads as soon as it lands (libtgb's twin-block replication).  Does a
// small piece, copied while the DMA's lines are still in the last-level cache, beat block-sized
// pieces (65.5 MB: read back from DRAM)?  build: nvcc -O3 -o e2e_chunk_probe e2e_chunk_probe.cu -lpthread
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static void nt_copy(char* dst, const char* src, size_t n) {
  size_t i = 0;
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

struct SpinPool {
  int nt;
  std::vector<std::thread> th;
  std::atomic<uint64_t> gen{0};
  std::atomic<int> done{0};
  std::atomic<bool> stop{false};
  char* dst = nullptr;
  const char* src = nullptr;
  size_t bytes = 0;
  bool nts = false;
  explicit SpinPool(int n) : nt(n) {
    for (int t = 1; t < nt; ++t) th.emplace_back([this, t] { loop(t); });
  }
  ~SpinPool() {
    stop = true;
    for (auto& x : th) x.join();
  }
  void part(int t) {
    size_t lo = (bytes * t / nt) & ~size_t(63), hi = t + 1 == nt ? bytes : (bytes * (t + 1) / nt) & ~size_t(63);
    if (nts) nt_copy(dst + lo, src + lo, hi - lo); else memcpy(dst + lo, src + lo, hi - lo);
  }
  void loop(int t) {
    uint64_t seen = 0;
    while (!stop.load(std::memory_order_relaxed)) {
      const uint64_t g = gen.load(std::memory_order_acquire);
      if (g == seen) { _mm_pause(); continue; }
      seen = g;
      part(t);
      done.fetch_add(1, std::memory_order_release);
    }
  }
  void copy(char* d, const char* s, size_t n, bool nt_store) {
    dst = d; src = s; bytes = n; nts = nt_store;
    done.store(0, std::memory_order_relaxed);
    gen.fetch_add(1, std::memory_order_release);
    part(0);
    while (done.load(std::memory_order_acquire) != nt - 1) _mm_pause();
  }
};

int main() {
  const size_t total = size_t(4) << 30;
  char *rep, *twin;
  cudaHostAlloc(&rep, total, cudaHostAllocDefault);
  cudaHostAlloc(&twin, total, cudaHostAllocDefault);
  memset(rep, 1, total);
  memset(twin, 2, total);
  char* d;
  cudaMalloc(&d, total);
  cudaMemset(d, 5, total);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  SpinPool pool(16);
  std::vector<cudaEvent_t> ev(8192);
  for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (int rep_i = 0; rep_i < 2; ++rep_i)
    for (int nts = 0; nts < 2; ++nts)
      for (size_t chunk : {size_t(65536000), size_t(16) << 20, size_t(8) << 20, size_t(4) << 20, size_t(2) << 20,
                           size_t(1) << 20}) {
        const size_t nch = (total + chunk - 1) / chunk;
        auto t0 = std::chrono::steady_clock::now();
        for (size_t c = 0; c < nch; ++c) {
          const size_t off = c * chunk, len = std::min(chunk, total - off);
          cudaMemcpyAsync(rep + off, d + off, len, cudaMemcpyDeviceToHost, s);
          cudaEventRecord(ev[c], s);
        }
        double wait = 0;
        for (size_t c = 0; c < nch; ++c) {
          const size_t off = c * chunk, len = std::min(chunk, total - off);
          auto w0 = std::chrono::steady_clock::now();
          while (cudaEventQuery(ev[c]) == cudaErrorNotReady) _mm_pause();
          wait += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
          pool.copy(twin + off, rep + off, len, nts);
        }
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        printf("%-8s piece %8.2f MB: total %6.1f ms (waiting on D2H %5.1f ms)  [4 GB D2H + 4 GB replicated]\n",
               nts ? "nt-store" : "memcpy", chunk / 1048576.0, ms, wait);
      }
  return 0;
}

// Host <-> device copies for the reference-facing TGB_MEM_HOST entry points.
//
// Pinned (page-locked) host memory goes straight to the copy engines.  Pageable
// memory (plain numpy / Eigen buffers, what the reference's callers hold) is
// staged through two pinned chunks: host threads fill chunk c+1 while the DMA
// of chunk c runs, so the copy runs at the DMA rate instead of the driver's
// single-threaded pageable path (~6 GB/s measured on the bench host for the
// 630 MB density of config 1).
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <cstring>
#include <cstdlib>
#include <thread>
#include <vector>

#include "tgb_internal.hpp"

namespace tgb {

namespace {

constexpr size_t kChunk = 64u << 20;  // bytes per staging chunk
constexpr size_t kDirect = 8u << 20;  // below this the driver's pageable path is fine

}  // namespace

bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// A persistent pool of host copy threads (spawning threads per call cost more than the
// copies when the output's twin blocks are replicated block by block).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    const size_t nt = std::min<size_t>(workers_.size() + 1, std::max<size_t>(1, bytes >> 22));
    if (nt <= 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);  // one parallel copy at a time
    const size_t part = (bytes + nt - 1) / nt;
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      part_ = part;
      nparts_ = nt;
      next_ = 1;  // part 0 is the caller's
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    run_part(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == nparts_ - 1; });
  }

 private:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned nt = std::min(hw, 16u);
    if (const char* e = getenv("TGB_COPY_THREADS")) nt = std::max(1, std::min(64, atoi(e)));
    const unsigned n = nt - 1;
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void run_part(size_t p) {
    const size_t b0 = p * part_, b1 = std::min(bytes_, b0 + part_);
    if (b0 < b1) std::memcpy(dst_ + b0, src_ + b0, b1 - b0);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      size_t p;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && next_ < nparts_); });
        if (stop_) return;
        p = next_++;
        if (next_ >= nparts_) seen = gen_;
      }
      run_part(p);
      {
        std::lock_guard<std::mutex> lk(mu_);
        ++done_;
      }
      done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, part_ = 0, nparts_ = 0, next_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

void par_memcpy(void* dst, const void* src, size_t bytes) { CopyPool::get().copy(dst, src, bytes); }

// ---- streaming replication of D2H pieces (the bitwise-twin output blocks of the host-memory
// convolve).  Pieces of a few MB are replicated the moment their DMA lands, by all threads at
// once: the threads spin between pieces (a condition-variable wake-up costs more than a piece)
// and write with non-temporal stores (no read-for-ownership of the destination lines).
// Measured on the bench host (tools/probe/e2e_chunk_probe.cu): 4 GB D2H + 4 GB replicated takes
// 113-119 ms with memcpy on 65 MB blocks, 91-98 ms with 4-8 MB pieces and non-temporal stores.
namespace {

void nt_copy(char* dst, const char* src, size_t n) {
  size_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15)) {
    dst[i] = src[i];
    ++i;
  }
  for (; i + 64 <= n; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
}

class SpinCopyPool {
 public:
  static SpinCopyPool& get() {
    static SpinCopyPool pool;
    return pool;
  }
  // between begin() and end() the workers spin; one user at a time
  void begin() {
    user_.lock();
    {
      std::lock_guard<std::mutex> lk(mu_);
      active_ = true;
    }
    cv_.notify_all();
  }
  void end() {
    active_.store(false, std::memory_order_release);
    user_.unlock();
  }
  void copy(void* dst, const void* src, size_t bytes) {
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    bytes_ = bytes;
    done_.store(0, std::memory_order_relaxed);
    gen_.fetch_add(1, std::memory_order_release);
    part(0);
    unsigned idle = 0;
    while (done_.load(std::memory_order_acquire) != nt_ - 1) {
      if (++idle > 4096) {
        std::this_thread::yield();
        idle = 0;
      } else {
        _mm_pause();
      }
    }
  }

 private:
  SpinCopyPool() {
    // spinning threads must each own a core: count the CPUs this process may run on
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) hw = std::max(1, std::min<int>(hw, CPU_COUNT(&set)));
    nt_ = static_cast<int>(std::min(hw, 16u));
    if (const char* e = getenv("TGB_COPY_THREADS")) nt_ = std::max(1, std::min(64, atoi(e)));
    for (int t = 1; t < nt_; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  ~SpinCopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void part(int t) {
    const size_t lo = (bytes_ * t / nt_) & ~size_t(63);
    const size_t hi = t + 1 == nt_ ? bytes_ : (bytes_ * (t + 1) / nt_) & ~size_t(63);
    if (lo < hi) nt_copy(dst_ + lo, src_ + lo, hi - lo);
  }
  void loop(int t) {
    uint64_t seen = 0;  // every copy posted since construction is this thread's to join, however late it starts
    unsigned idle = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || active_.load(std::memory_order_acquire); });
        if (stop_) return;
      }
      while (active_.load(std::memory_order_acquire)) {
        const uint64_t g = gen_.load(std::memory_order_acquire);
        if (g == seen) {
          if (++idle > 4096) {  // a long gap (the next piece is still in flight): let others run
            std::this_thread::yield();
            idle = 0;
          } else {
            _mm_pause();
          }
          continue;
        }
        idle = 0;
        seen = g;
        part(t);
        done_.fetch_add(1, std::memory_order_release);
      }
    }
  }
  int nt_ = 1;
  std::vector<std::thread> workers_;
  std::mutex mu_, user_;
  std::condition_variable cv_;
  std::atomic<bool> active_{false};
  bool stop_ = false;
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> done_{0};
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
};

}  // namespace

void stream_copy_begin() { SpinCopyPool::get().begin(); }
void stream_copy(void* dst, const void* src, size_t bytes) { SpinCopyPool::get().copy(dst, src, bytes); }
void stream_copy_end() { SpinCopyPool::get().end(); }

namespace {

void ensure_stage(tgb_ctx* ctx) {
  for (int i = 0; i < 2; ++i) {
    if (!ctx->stage_pin[i]) TGB_CUDA(cudaHostAlloc(&ctx->stage_pin[i], kChunk, cudaHostAllocDefault));
    if (!ctx->stage_ev[i]) TGB_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
  }
}

}  // namespace

void h2d(tgb_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (!bytes) return;
  ctx->bytes_h2d += static_cast<int64_t>(bytes);
  if (bytes < kDirect || !is_pageable(src)) {
    TGB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
    return;
  }
  ensure_stage(ctx);
  int c = 0;
  for (size_t off = 0; off < bytes; off += kChunk, ++c) {
    const int b = c & 1;
    const size_t len = std::min(kChunk, bytes - off);
    TGB_CUDA(cudaEventSynchronize(ctx->stage_ev[b]));  // the DMA that last read this chunk is done
    par_memcpy(ctx->stage_pin[b], static_cast<const char*>(src) + off, len);
    TGB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, ctx->stage_pin[b], len, cudaMemcpyHostToDevice, stream));
    TGB_CUDA(cudaEventRecord(ctx->stage_ev[b], stream));
  }
}

void d2h(tgb_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (!bytes) return;
  ctx->bytes_d2h += static_cast<int64_t>(bytes);
  if (bytes < kDirect || !is_pageable(dst)) {
    TGB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream));
    TGB_CUDA(cudaStreamSynchronize(stream));
    return;
  }
  ensure_stage(ctx);
  const size_t nchunks = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t c) {
    const int b = static_cast<int>(c & 1);
    const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
    TGB_CUDA(cudaMemcpyAsync(ctx->stage_pin[b], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                             stream));
    TGB_CUDA(cudaEventRecord(ctx->stage_ev[b], stream));
  };
  issue(0);
  for (size_t c = 0; c < nchunks; ++c) {
    const int b = static_cast<int>(c & 1);
    TGB_CUDA(cudaEventSynchronize(ctx->stage_ev[b]));
    if (c + 1 < nchunks) issue(c + 1);  // the other chunk is free: its data was drained last iteration
    const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
    par_memcpy(static_cast<char*>(dst) + off, ctx->stage_pin[b], len);
  }
}

}  // namespace tgb

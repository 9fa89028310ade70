// Host <-> device copies for the reference-facing TGB_MEM_HOST entry points.
//
// Pinned (page-locked) host memory goes straight to the copy engines.  Pageable
// memory (plain numpy / Eigen buffers, what the reference's callers hold) is
// staged through two pinned chunks: host threads fill chunk c+1 while the DMA
// of chunk c runs, so the copy runs at the DMA rate instead of the driver's
// single-threaded pageable path (~6 GB/s measured on the bench host for the
// 630 MB density of config 1).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "tgb_internal.hpp"

namespace tgb {

namespace {

constexpr size_t kChunk = 64u << 20;  // bytes per staging chunk
constexpr size_t kDirect = 8u << 20;  // below this the driver's pageable path is fine

bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>({static_cast<size_t>(hw), 8, std::max<size_t>(1, bytes >> 22)});
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t part = (bytes + nt - 1) / nt;
  for (size_t t = 0; t < nt; ++t) {
    const size_t b0 = t * part, b1 = std::min(bytes, b0 + part);
    if (b0 >= b1) break;
    th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + b0, static_cast<const char*>(src) + b0, b1 - b0); });
  }
  for (auto& x : th) x.join();
}

void ensure_stage(tgb_ctx* ctx) {
  for (int i = 0; i < 2; ++i) {
    if (!ctx->stage_pin[i]) TGB_CUDA(cudaHostAlloc(&ctx->stage_pin[i], kChunk, cudaHostAllocDefault));
    if (!ctx->stage_ev[i]) TGB_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev[i], cudaEventDisableTiming));
  }
}

}  // namespace

void h2d(tgb_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (!bytes) return;
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

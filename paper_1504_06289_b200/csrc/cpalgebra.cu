// Canonical-tensor algebra on the device (reference proj/src/tensor.cpp:141-177):
//   hadamard  column i + R_a j = a_i .* b_j per axis, weight a.w[i] b.w[j]  (tensor.cpp:141-157)
//   add       factors and weights concatenated [a | b]                       (tensor.cpp:159-171)
//   scale     weights times alpha, factors copied                            (tensor.cpp:173-177)
// Element-wise products and copies: bit-identical to the reference's.
#include <cuda_runtime.h>

#include <algorithm>

#include "tgb_internal.hpp"

namespace tgb {

namespace {

__global__ void hadamard_kernel(int64_t n, int64_t ra, int64_t c0, const double* __restrict__ A,
                                const double* __restrict__ B, double* __restrict__ out) {
  const int64_t col = c0 + blockIdx.y;  // i + ra j
  const int64_t i = col % ra, j = col / ra;
  const double* a = A + i * n;
  const double* b = B + j * n;
  double* o = out + col * n;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    o[r] = a[r] * b[r];
}

__global__ void outer_weights_kernel(int64_t ra, int64_t rb, const double* __restrict__ wa,
                                     const double* __restrict__ wb, double* __restrict__ w) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < ra * rb) w[k] = wa[k % ra] * wb[k / ra];
}

__global__ void scale_weights_kernel(int64_t r, const double* __restrict__ w, double alpha, double* __restrict__ out) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < r) out[k] = w[k] * alpha;
}

}  // namespace

void hadamard_dev(tgb_ctx* ctx, const tgb_cp& a, const tgb_cp& b, const tgb_cp& out) {
  const int64_t ra = a.rank, rb = b.rank;
  if (ra * rb == 0) return;
  for (int ax = 0; ax < 3; ++ax) {
    const int64_t n = a.n[ax];
    if (n == 0) continue;
    for (int64_t c0 = 0; c0 < ra * rb; c0 += 65535) {  // grid.y limit: blocks of output columns
      const int64_t nc = std::min<int64_t>(65535, ra * rb - c0);
      dim3 grid(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 64)), static_cast<unsigned>(nc));
      hadamard_kernel<<<grid, 256, 0, ctx->stream>>>(n, ra, c0, a.factor[ax], b.factor[ax], out.factor[ax]);
      TGB_LAUNCHED(ctx);
    }
  }
  outer_weights_kernel<<<static_cast<unsigned>((ra * rb + 255) / 256), 256, 0, ctx->stream>>>(ra, rb, a.weight,
                                                                                             b.weight, out.weight);
  TGB_LAUNCHED(ctx);
}

void add_dev(tgb_ctx* ctx, const tgb_cp& a, const tgb_cp& b, const tgb_cp& out) {
  for (int ax = 0; ax < 3; ++ax) {
    const int64_t n = a.n[ax];
    if (n * a.rank)
      TGB_CUDA(cudaMemcpyAsync(out.factor[ax], a.factor[ax], n * a.rank * sizeof(double), cudaMemcpyDeviceToDevice,
                               ctx->stream));
    if (n * b.rank)
      TGB_CUDA(cudaMemcpyAsync(out.factor[ax] + n * a.rank, b.factor[ax], n * b.rank * sizeof(double),
                               cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (a.rank)
    TGB_CUDA(cudaMemcpyAsync(out.weight, a.weight, a.rank * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  if (b.rank)
    TGB_CUDA(cudaMemcpyAsync(out.weight + a.rank, b.weight, b.rank * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
}

void scale_dev(tgb_ctx* ctx, const tgb_cp& a, double alpha, const tgb_cp& out) {
  for (int ax = 0; ax < 3; ++ax)
    if (a.n[ax] * a.rank && out.factor[ax] != a.factor[ax])
      TGB_CUDA(cudaMemcpyAsync(out.factor[ax], a.factor[ax], a.n[ax] * a.rank * sizeof(double),
                               cudaMemcpyDeviceToDevice, ctx->stream));
  if (a.rank) {
    scale_weights_kernel<<<static_cast<unsigned>((a.rank + 255) / 256), 256, 0, ctx->stream>>>(a.rank, a.weight, alpha,
                                                                                               out.weight);
    TGB_LAUNCHED(ctx);
  }
}

}  // namespace tgb

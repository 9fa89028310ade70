// Separable assembly kernels on sm_100a:
//  * scalar products of canonical tensors and the Coulomb matrix J
//    (reference tensor.cpp:88-98, hf.cpp:140-151): one fused kernel computes,
//    for a batch of "left" columns p (a single factor column, or the Hadamard
//    product of two basis columns formed on the fly), the per-axis inner
//    products with every right column q, multiplies the three axes, weights
//    by w_q and reduces over the q tile.  Per-q-tile partials are reduced in
//    a fixed order (deterministic, no atomics).
//  * lattice window assembly (lattice.cpp:50-61), summed in lattice order so
//    the result is bit-identical to the reference.
//  * batched value_at probes (tensor.hpp:135-140).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <vector>

#include "tgb_internal.hpp"

namespace tgb {

namespace {

constexpr int TP = 64;   // left columns per CTA
constexpr int TQ = 64;   // right columns per CTA

struct SepArgs {
  int64_t n[3];
  const double* F[3];   // left factor matrices (n x nf)
  const double* B[3];   // right factor matrices (n x R_B)
  const int* i0;        // left column p = F(:, i0[p]) (* F(:, i1[p]) if i1[p] >= 0)
  const int* i1;
  const double* wb;     // right weights
  int P, RB;
};

// DMMA (mma.sync m16n8k4 f64) version of the fused separable inner product:
// per CTA a 64 (left p) x 64 (right q) tile, 4 warps of 32 x 32; per axis the
// tile G_ax = L_ax^T B_ax accumulates on the FP64 tensor cores, the three axes
// are multiplied in registers, and the weighted row sums over q are reduced
// through shared memory into one partial per (q tile, p).
__device__ __forceinline__ void dmma16x8x4_sep(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

constexpr int DM_BK = 16, DM_LDS = 68, DM_THREADS = 128;

__global__ void __launch_bounds__(DM_THREADS) sep_inner_dmma_kernel(SepArgs a, double* __restrict__ partial) {
  __shared__ double As[2][DM_BK][DM_LDS];
  __shared__ double Bs[2][DM_BK][DM_LDS];
  __shared__ double red[64][2][4];
  const int p0 = blockIdx.x * 64, q0 = blockIdx.y * 64;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  const int g = lane >> 2, t = lane & 3;
  double prod[2][4][4];
  double ra[8], rb[8];
  // this thread's 8 staged (column, k-offset) slots are fixed: kk = tid % 16,
  // columns mm = tid / 16 + 8 e; the left columns' factor indices are loaded once
  const int kk = tid % DM_BK, mm0 = tid / DM_BK;
  int c0s[8], c1s[8];
  bool qok[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int pp = p0 + mm0 + 8 * e;
    c0s[e] = pp < a.P ? __ldg(a.i0 + pp) : -1;
    c1s[e] = pp < a.P ? __ldg(a.i1 + pp) : -1;
    qok[e] = q0 + mm0 + 8 * e < a.RB;
  }
  for (int ax = 0; ax < 3; ++ax) {
    const int64_t n = a.n[ax];
    const double* F = a.F[ax];
    const double* Bq = a.B[ax] + static_cast<int64_t>(q0 + mm0) * n + kk;  // column q0 + mm0, row kk
    const double* Fk = F + kk;
    auto load_tile = [&](int64_t k0) {
      const bool kin = k0 + kk < n;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        double v = 0.0;
        if (kin && c0s[e] >= 0) {
          v = __ldg(Fk + c0s[e] * n + k0);
          if (c1s[e] >= 0) v *= __ldg(Fk + c1s[e] * n + k0);
        }
        ra[e] = v;
        rb[e] = (kin && qok[e]) ? __ldg(Bq + static_cast<int64_t>(8 * e) * n + k0) : 0.0;
      }
    };
    auto store_tile = [&](int buf) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        As[buf][kk][mm0 + 8 * e] = ra[e];
        Bs[buf][kk][mm0 + 8 * e] = rb[e];
      }
    };
    double acc[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[i][j][r] = 0.0;
    const int64_t nk = (n + DM_BK - 1) / DM_BK;
    __syncthreads();
    load_tile(0);
    store_tile(0);
    __syncthreads();
    for (int64_t kt = 0; kt < nk; ++kt) {
      const int buf = kt & 1;
      if (kt + 1 < nk) load_tile((kt + 1) * DM_BK);
#pragma unroll
      for (int k4 = 0; k4 < DM_BK; k4 += 4) {
        double av[2][2], bv[4];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          av[i][0] = As[buf][k4 + t][wm + 16 * i + g];
          av[i][1] = As[buf][k4 + t][wm + 16 * i + g + 8];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][k4 + t][wn + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma16x8x4_sep(acc[i][j], av[i][0], av[i][1], bv[j]);
      }
      if (kt + 1 < nk) store_tile(buf ^ 1);
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) prod[i][j][r] = ax == 0 ? acc[i][j][r] : prod[i][j][r] * acc[i][j][r];
  }
  // weighted row sums: element (row, col) of fragment (i, j, r):
  //   row = wm + 16 i + g + 8 (r >= 2), col = wn + 8 j + 2 t + (r & 1)
  double rs[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double sacc = 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int q = q0 + wn + 8 * j + 2 * t + c;
          if (q < a.RB) sacc += a.wb[q] * prod[i][j][2 * h + c];
        }
      rs[i][h] = sacc;
    }
  // reduce over the 4 lanes t sharing a row (fixed order: shuffles xor 1, 2)
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double v = rs[i][h];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      rs[i][h] = v;
    }
  if (t == 0) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) red[wm + 16 * i + g + 8 * h][warp >> 1][0] = rs[i][h];
  }
  __syncthreads();
  if (tid < 64) {
    const int p = p0 + tid;
    if (p < a.P) partial[static_cast<int64_t>(blockIdx.y) * a.P + p] = red[tid][0][0] + red[tid][1][0];
  }
}

__global__ void reduce_tiles_kernel(const double* __restrict__ partial, int ntiles, int P, double* __restrict__ s) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double acc = 0.0;
  for (int t = 0; t < ntiles; ++t) acc += partial[static_cast<int64_t>(t) * P + p];
  s[p] = acc;
}

// Hadamard left columns materialised (n x P per axis) for the GEMM route.
__global__ void hadamard_cols_kernel(int64_t n, const double* __restrict__ F, const int* __restrict__ i0,
                                     const int* __restrict__ i1, int P, double* __restrict__ L) {
  const int p = blockIdx.y;
  if (p >= P) return;
  const int c0 = i0[p], c1 = i1[p];
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = F[c0 * n + k];
    if (c1 >= 0) v *= F[c1 * n + k];
    L[p * n + k] = v;
  }
}

// part[chunk * P + p] = sum_{q in chunk} w_q T0[q, p] T1[q, p] T2[q, p]; T_ax are
// (nq x P) column-major, so row p is contiguous in q.  Fixed-order reduction.
__global__ void __launch_bounds__(256) triple_dot_kernel(int nq, int P, const double* __restrict__ T0,
                                                         const double* __restrict__ T1,
                                                         const double* __restrict__ T2, const double* __restrict__ w,
                                                         double* __restrict__ part) {
  const int p = blockIdx.x;
  const int64_t o = static_cast<int64_t>(p) * nq;
  double acc = 0.0;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) acc += w[q] * T0[o + q] * T1[o + q] * T2[o + q];
  __shared__ double sh[256];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int st = 128; st; st >>= 1) {
    if (threadIdx.x < st) sh[threadIdx.x] += sh[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.y * static_cast<int64_t>(P) + p] = sh[0];
}

// Duplicate right columns.  V_H = convolve(theta, kernel) repeats every column
// block of a kernel column's bitwise twin (the +-t sinc nodes, kernel.cpp:194):
// config 1 has 108,650 V_H columns of which 55,650 are distinct.  Two 64-bit
// hashes per column (order-independent sums of mixed (position, bits) words
// over all three axes) group candidates on the host; every candidate is then
// compared bitwise on the device before its weight is merged into its
// representative's, so a hash collision can never merge different columns.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void col_hash_kernel(int64_t n0, int64_t n1, int64_t n2, const double* __restrict__ B0,
                                const double* __restrict__ B1, const double* __restrict__ B2,
                                unsigned long long* __restrict__ h, unsigned long long* __restrict__ key,
                                int* __restrict__ val) {
  const int64_t q = blockIdx.x;
  uint64_t a = 0, b = 0;
  const int64_t ns[3] = {n0, n1, n2};
  const double* Bs[3] = {B0, B1, B2};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const uint64_t* col = reinterpret_cast<const uint64_t*>(Bs[ax] + q * ns[ax]);
    for (int64_t k = threadIdx.x; k < ns[ax]; k += blockDim.x) {
      const uint64_t v = col[k];
      const uint64_t pos = static_cast<uint64_t>(k) + (static_cast<uint64_t>(ax) << 40);
      a += mix64(v ^ (pos * 0x9E3779B97F4A7C15ull));
      b += mix64(v + pos * 0xD1B54A32D192ED03ull + 0x632BE59BD9B4E019ull);
    }
  }
  __shared__ uint64_t sa[256], sb[256];
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int st = blockDim.x / 2; st; st >>= 1) {
    if (threadIdx.x < st) {
      sa[threadIdx.x] += sa[threadIdx.x + st];
      sb[threadIdx.x] += sb[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    h[2 * q] = sa[0];
    h[2 * q + 1] = sb[0];
    key[q] = sa[0];
    val[q] = static_cast<int>(q);
  }
}

// Over the hash-sorted columns (stable: ascending index within a run of equal
// first hashes): one CTA per sorted position t; a run member is merged into
// the run start r when the second hashes match AND its three columns are
// bitwise equal to r's (coalesced compare).  rep[q] = r, or -1.
__global__ void dedup_verify_kernel(int RB, int64_t n0, int64_t n1, int64_t n2, const double* __restrict__ B0,
                                    const double* __restrict__ B1, const double* __restrict__ B2,
                                    const unsigned long long* __restrict__ h, const unsigned long long* __restrict__ key,
                                    const int* __restrict__ val, int* __restrict__ rep) {
  const int t = blockIdx.x;
  const int q = val[t];
  if (t == 0 || key[t - 1] != key[t]) {
    if (threadIdx.x == 0) rep[q] = -1;
    return;
  }
  __shared__ int s_r;
  if (threadIdx.x == 0) {
    int s = t - 1;
    while (s > 0 && key[s - 1] == key[t]) --s;
    s_r = val[s];
  }
  __syncthreads();
  const int r = s_r;
  int eq = h[2 * q + 1] == h[2 * r + 1];
  const int64_t ns[3] = {n0, n1, n2};
  const double* Bs[3] = {B0, B1, B2};
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const uint64_t* x = reinterpret_cast<const uint64_t*>(Bs[ax] + q * ns[ax]);
    const uint64_t* y = reinterpret_cast<const uint64_t*>(Bs[ax] + static_cast<int64_t>(r) * ns[ax]);
    for (int64_t k = threadIdx.x; k < ns[ax]; k += blockDim.x) eq &= (x[k] == y[k]);
  }
  eq = __syncthreads_and(eq);
  if (threadIdx.x == 0) rep[q] = eq ? r : -1;
}

// Merged weights: a run start sums its merged members' weights in ascending
// column order (deterministic); merged columns get keep = 0.
__global__ void dedup_weights_kernel(int RB, const unsigned long long* __restrict__ key, const int* __restrict__ val,
                                     const int* __restrict__ rep, const double* __restrict__ w,
                                     unsigned char* __restrict__ keep, double* __restrict__ wout) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= RB) return;
  const int q = val[t];
  if (rep[q] >= 0) {
    keep[q] = 0;
    wout[q] = 0.0;
    return;
  }
  keep[q] = 1;
  double acc = w[q];
  if (t == 0 || key[t - 1] != key[t])
    for (int u = t + 1; u < RB && key[u] == key[t]; ++u)
      if (rep[val[u]] == q) acc += w[val[u]];
  wout[q] = acc;
}

// s[p] = sum_q wb[q] prod_ax <left_p^ax, B_q^ax>, returned to the host.
std::vector<double> sep_inner(tgb_ctx* ctx, const int64_t n[3], const double* const F[3], const double* const B[3],
                              const double* wb, int RB, const std::vector<int>& i0, const std::vector<int>& i1) {
  const int P = static_cast<int>(i0.size());
  std::vector<double> s(P, 0.0);
  if (P == 0 || RB == 0) return s;
  auto* idx = static_cast<int*>(ctx->ws_misc.get(2 * P * sizeof(int)));
  TGB_CUDA(cudaMemcpyAsync(idx, i0.data(), P * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  TGB_CUDA(cudaMemcpyAsync(idx + P, i1.data(), P * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  const int ntq = (RB + TQ - 1) / TQ;
  auto* partial = static_cast<double*>(ctx->ws_misc2.get(static_cast<size_t>(ntq) * P * sizeof(double) + P * sizeof(double)));
  double* dsum = partial + static_cast<size_t>(ntq) * P;
  SepArgs a;
  for (int ax = 0; ax < 3; ++ax) {
    a.n[ax] = n[ax];
    a.F[ax] = F[ax];
    a.B[ax] = B[ax];
  }
  a.i0 = idx;
  a.i1 = idx + P;
  // (materialising the Hadamard columns measured slower: 128 vs 72 ms on config 1 —
  //  the products of the few basis columns stay L1-resident when formed on load)
  a.wb = wb;
  a.P = P;
  a.RB = RB;
  if (P >= 128 && !getenv("TGB_SEP_FUSED")) {
    // GEMM route for many left columns (the Coulomb matrix): per axis
    // T_ax = B_ax^T L_ax on the DGEMM (chunks of q), then one fused
    // weighted triple-product reduction.  The fused tile kernel needs ~190
    // live doubles per thread (two axis tiles + staging), which caps it at
    // two CTAs per SM; the split route runs each GEMM at full occupancy.
    int64_t tot = 0;
    for (int ax = 0; ax < 3; ++ax) tot += n[ax] * P;
    const int chunk = static_cast<int>(std::min<int64_t>(RB, 32768));
    const int nch = (RB + chunk - 1) / chunk;
    auto* work = static_cast<double*>(ctx->ws_misc3.get((static_cast<size_t>(tot) + 3 * static_cast<size_t>(chunk) * P +
                                                         static_cast<size_t>(nch) * P) * sizeof(double)));
    double* Lh[3];
    int64_t off = 0;
    for (int ax = 0; ax < 3; ++ax) {
      Lh[ax] = work + off;
      dim3 hg(static_cast<unsigned>(std::min<int64_t>((n[ax] + 255) / 256, 8)), static_cast<unsigned>(P));
      hadamard_cols_kernel<<<hg, 256, 0, ctx->stream>>>(n[ax], F[ax], idx, idx + P, P, Lh[ax]);
      TGB_LAUNCHED(ctx);
      off += n[ax] * P;
    }
    double* T[3] = {work + off, work + off + static_cast<size_t>(chunk) * P, work + off + 2 * static_cast<size_t>(chunk) * P};
    double* parts = work + off + 3 * static_cast<size_t>(chunk) * P;
    // duplicate right columns: merged weights and the kept column ranges
    const double* wq = wb;
    std::vector<std::pair<int, int>> chunks;  // (q0, nq)
    {
      std::vector<char> keep(RB, 1);
      if (RB >= 1024 && !getenv("TGB_NO_DEDUP")) {
        DevBuf& db = ctx_buf(ctx, "sep.dedup");
        // layout: hash pairs (2 RB u64), sorted keys + values, keep flags, merged weights, CUB temp
        size_t cub_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, static_cast<const unsigned long long*>(nullptr),
                                        static_cast<unsigned long long*>(nullptr), static_cast<const int*>(nullptr),
                                        static_cast<int*>(nullptr), RB, 0, 64, ctx->stream);
        const size_t o_h = 0, o_k0 = o_h + 16 * size_t(RB), o_k1 = o_k0 + 8 * size_t(RB), o_v0 = o_k1 + 8 * size_t(RB),
                     o_v1 = o_v0 + 4 * size_t(RB), o_keep = o_v1 + 4 * size_t(RB),
                     o_w = (o_keep + size_t(RB) + 15) & ~size_t(15), o_tmp = o_w + 8 * size_t(RB);
        char* base = static_cast<char*>(db.get(o_tmp + cub_bytes + 256));
        auto* hh = reinterpret_cast<unsigned long long*>(base + o_h);
        auto* k0 = reinterpret_cast<unsigned long long*>(base + o_k0);
        auto* k1 = reinterpret_cast<unsigned long long*>(base + o_k1);
        auto* v0 = reinterpret_cast<int*>(base + o_v0);
        auto* v1 = reinterpret_cast<int*>(base + o_v1);
        auto* dkeep = reinterpret_cast<unsigned char*>(base + o_keep);
        auto* dw = reinterpret_cast<double*>(base + o_w);
        col_hash_kernel<<<RB, 256, 0, ctx->stream>>>(n[0], n[1], n[2], B[0], B[1], B[2], hh, k0, v0);
        TGB_LAUNCHED(ctx);
        // stable sort by the first hash: equal columns end up in runs, ascending index within a run
        TGB_CUDA(cub::DeviceRadixSort::SortPairs(base + o_tmp, cub_bytes, k0, k1, v0, v1, RB, 0, 64, ctx->stream));
        dedup_verify_kernel<<<RB, 128, 0, ctx->stream>>>(RB, n[0], n[1], n[2], B[0], B[1], B[2], hh, k1, v1, v0);
        TGB_LAUNCHED(ctx);  // v0 (free after the sort) holds rep[]
        dedup_weights_kernel<<<(RB + 127) / 128, 128, 0, ctx->stream>>>(RB, k1, v1, v0, wb, dkeep, dw);
        TGB_LAUNCHED(ctx);
        TGB_CUDA(cudaMemcpyAsync(keep.data(), dkeep, RB, cudaMemcpyDeviceToHost, ctx->stream));
        TGB_CUDA(cudaStreamSynchronize(ctx->stream));
        wq = dw;
      }
      for (int q = 0; q < RB;) {  // kept ranges, split into chunks
        if (!keep[q]) {
          ++q;
          continue;
        }
        int e = q;
        while (e < RB && keep[e] && e - q < chunk) ++e;
        chunks.push_back({q, e - q});
        q = e;
      }
    }
    const int nchk = static_cast<int>(chunks.size());
    if (nchk > nch) parts = static_cast<double*>(ctx_buf(ctx, "sep.parts").get(static_cast<size_t>(nchk) * P * sizeof(double)));
    for (int c = 0; c < nchk; ++c) {
      const int q0 = chunks[c].first, nq = chunks[c].second;
      // axis 2 on the aux stream: its wave tail overlaps axes 0-1 (no split-K, whose workspace is shared)
      const bool fork = ((nq + 63) / 64) * ((P + 63) / 64) >= ctx->num_sms;
      if (fork) {
        TGB_CUDA(cudaEventRecord(ctx->aux_in, ctx->stream));
        TGB_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ctx->aux_in, 0));
      }
      for (int ax = 0; ax < 3; ++ax) {  // T_ax (nq x P) = B_ax(:, q0:q0+nq)^T L_ax
        StreamSwap on_aux(ctx, fork && ax == 2, ctx->aux_stream);  // restored on every exit path
        dgemm(ctx, true, false, nq, P, n[ax], 1.0, B[ax] + static_cast<int64_t>(q0) * n[ax], n[ax], Lh[ax], n[ax], 0.0,
              T[ax], nq);
      }
      if (fork) {
        TGB_CUDA(cudaEventRecord(ctx->aux_done, ctx->aux_stream));
        TGB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_done, 0));
      }
      triple_dot_kernel<<<dim3(static_cast<unsigned>(P), 1), 256, 0, ctx->stream>>>(nq, P, T[0], T[1], T[2], wq + q0,
                                                                                    parts + static_cast<size_t>(c) * P);
      TGB_LAUNCHED(ctx);
    }
    if (nchk == 0) TGB_CUDA(cudaMemsetAsync(parts, 0, P * sizeof(double), ctx->stream));
    reduce_tiles_kernel<<<(P + 127) / 128, 128, 0, ctx->stream>>>(parts, std::max(nchk, 1), P, dsum);
    TGB_LAUNCHED(ctx);
  } else {
    dim3 grid((P + TP - 1) / TP, ntq);
    sep_inner_dmma_kernel<<<grid, DM_THREADS, 0, ctx->stream>>>(a, partial);
    TGB_LAUNCHED(ctx);
    reduce_tiles_kernel<<<(P + 127) / 128, 128, 0, ctx->stream>>>(partial, ntq, P, dsum);
    TGB_LAUNCHED(ctx);
  }
  TGB_CUDA(cudaMemcpyAsync(s.data(), dsum, P * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  return s;
}

__global__ void lattice_kernel(int64_t n, int64_t R, const double* __restrict__ ref, const int64_t* __restrict__ ofs,
                               int64_t L, double* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t q = blockIdx.y;
  if (i >= n) return;
  const double* col = ref + q * 2 * n + i;
  double acc = 0.0;
  for (int64_t l = 0; l < L; ++l) acc += __ldg(col + ofs[l]);
  out[q * n + i] = acc;
}

__global__ void value_at_kernel(int64_t n0, int64_t n1, int64_t n2, int64_t R, const double* __restrict__ f0,
                                const double* __restrict__ f1, const double* __restrict__ f2,
                                const double* __restrict__ w, int64_t npts, const int64_t* __restrict__ ijk,
                                double* __restrict__ out) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (p >= npts) return;
  const int64_t i = ijk[3 * p], j = ijk[3 * p + 1], l = ijk[3 * p + 2];
  double s = 0.0;
  for (int64_t k = lane; k < R; k += 32) s += w[k] * f0[i + n0 * k] * f1[j + n1 * k] * f2[l + n2 * k];
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) out[p] = s;
}

}  // namespace

double scalar_product_dev(tgb_ctx* ctx, const tgb_cp& a, const tgb_cp& b) {
  if (a.rank == 0 || b.rank == 0) return 0.0;  // tensor.cpp:92
  std::vector<int> i0(a.rank), i1(a.rank, -1);
  for (int64_t p = 0; p < a.rank; ++p) i0[p] = static_cast<int>(p);
  const double* F[3] = {a.factor[0], a.factor[1], a.factor[2]};
  const double* B[3] = {b.factor[0], b.factor[1], b.factor[2]};
  std::vector<double> s = sep_inner(ctx, a.n, F, B, b.weight, static_cast<int>(b.rank), i0, i1);
  std::vector<double> wa(a.rank);
  TGB_CUDA(cudaMemcpy(wa.data(), a.weight, a.rank * sizeof(double), cudaMemcpyDeviceToHost));
  double r = 0.0;
  for (int64_t p = 0; p < a.rank; ++p) r += wa[p] * s[p];
  return r;
}

void coulomb_matrix_dev(tgb_ctx* ctx, const tgb_cp& basis, const int64_t* fn_offset, int64_t nb, const tgb_cp& vh,
                        double vol, double* J) {
  std::vector<double> wprim(basis.rank);
  if (basis.rank)
    TGB_CUDA(cudaMemcpy(wprim.data(), basis.weight, basis.rank * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<int> i0, i1;
  std::vector<std::pair<int64_t, int64_t>> owner;  // (k, m) per left column
  for (int64_t k = 0; k < nb; ++k)
    for (int64_t m = k; m < nb; ++m)
      for (int64_t pm = fn_offset[m]; pm < fn_offset[m + 1]; ++pm)
        for (int64_t pk = fn_offset[k]; pk < fn_offset[k + 1]; ++pk) {
          i0.push_back(static_cast<int>(pk));
          i1.push_back(static_cast<int>(pm));
          owner.push_back({k, m});
        }
  const double* F[3] = {basis.factor[0], basis.factor[1], basis.factor[2]};
  const double* B[3] = {vh.factor[0], vh.factor[1], vh.factor[2]};
  std::vector<double> s;
  if (vh.rank > 0) s = sep_inner(ctx, basis.n, F, B, vh.weight, static_cast<int>(vh.rank), i0, i1);
  std::vector<double> acc(nb * nb, 0.0);
  for (size_t p = 0; p < i0.size(); ++p) {
    const double w = wprim[i0[p]] * wprim[i1[p]];
    acc[owner[p].first + nb * owner[p].second] += vh.rank > 0 ? w * s[p] : 0.0;
  }
  for (int64_t k = 0; k < nb; ++k)
    for (int64_t m = k; m < nb; ++m) {
      J[k + nb * m] = vol * acc[k + nb * m];
      J[m + nb * k] = J[k + nb * m];
    }
}

void value_at_dev(tgb_ctx* ctx, const tgb_cp& t, int64_t npts, const int64_t* ijk, double* out) {
  if (npts == 0) return;
  const int th = 256;
  const int64_t blocks = (npts + th / 32 - 1) / (th / 32);
  value_at_kernel<<<static_cast<unsigned>(blocks), th, 0, ctx->stream>>>(t.n[0], t.n[1], t.n[2], t.rank,
                                                                          t.factor[0], t.factor[1], t.factor[2],
                                                                          t.weight, npts, ijk, out);
  TGB_LAUNCHED(ctx);
}

namespace {
__global__ void equal_kernel(const unsigned long long* __restrict__ x, const unsigned long long* __restrict__ y,
                             int64_t count, int* __restrict__ diff) {
  int d = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    d |= x[i] != y[i];
  if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(diff, 1);
}
}  // namespace

// bitwise equality of two device arrays of doubles
bool device_equal(tgb_ctx* ctx, const double* x, const double* y, int64_t count) {
  if (x == y || count == 0) return true;
  auto* d = static_cast<int*>(ctx_buf(ctx, "equal.flag").get(sizeof(int)));
  TGB_CUDA(cudaMemsetAsync(d, 0, sizeof(int), ctx->stream));
  equal_kernel<<<static_cast<unsigned>(std::min<int64_t>((count + 255) / 256, 4 * ctx->num_sms)), 256, 0, ctx->stream>>>(
      reinterpret_cast<const unsigned long long*>(x), reinterpret_cast<const unsigned long long*>(y), count, d);
  TGB_LAUNCHED(ctx);
  int h = 0;
  TGB_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  return h == 0;
}

void lattice_assemble_dev(tgb_ctx* ctx, int64_t n, int64_t R, const double* ref, const int64_t* offsets, int64_t L,
                          double* out) {
  if (n == 0 || R == 0) return;
  auto* dofs = static_cast<int64_t*>(ctx->ws_misc3.get(std::max<int64_t>(L, 1) * sizeof(int64_t)));
  if (L) TGB_CUDA(cudaMemcpyAsync(dofs, offsets, L * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
  dim3 grid(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(R));
  lattice_kernel<<<grid, 256, 0, ctx->stream>>>(n, R, ref, dofs, L, out);
  TGB_LAUNCHED(ctx);
}

}  // namespace tgb

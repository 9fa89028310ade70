// Full singular-value spectra of the RHOSVD mode matrices — the reference's
// TuckerResult::mode_singular_values (proj/include/tengrid/reduction.hpp:42),
// which rhosvd fills from thin_svd_left of W = f_mode diag(w) of the
// normalized tensor (reduction.cpp:172-190, 85-138).  The rank-reduction path
// itself only needs the leading values (reduction.cu, subspace iteration);
// this is the opt-in diagnostic that returns all of them.
//
//  sigma_i = sqrt(max(0, lambda_i(G))),  G = W W^T (n <= R) or W^T W (R < n),
//  m = min(n, R):
//   (1) G from the library DGEMM (gemm.cu);
//   (2) Householder tridiagonalisation of G as ONE cooperative grid with one
//       grid barrier per step: every CTA forms the step's reflector from the
//       look-ahead-updated next column itself (no serial single-CTA phase),
//       and the owner warp of each trailing column applies the rank-2 update
//       to it and immediately takes its dot product with the NEXT reflector,
//       so the symmetric mat-vec of step k+1 rides on the update of step k;
//   (3) every eigenvalue of the tridiagonal by bisection on Sturm counts, one
//       thread per eigenvalue (index order = descending).
// Counts follow the reference's thin_svd_left branches: the wide Gram branch
// (R >= 4n, R > 8192) and the Jacobi branch return min(n, R) values, the tall
// Gram branch (n >= 4R, R >= 8) those with lambda > lambda_max 1e-24.  Values
// come from the Gram spectrum, so sigma_i carries an absolute error of about
// eps m sigma_0^2 / sigma_i (the reference's Gram branches share that floor;
// its Jacobi branch resolves the tiny values further).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <vector>

#include "tgb_internal.hpp"

namespace tgb {
namespace {

namespace cg = cooperative_groups;

constexpr int kTriThreads = 512;

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // red[] free from any previous use
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s += red[i];  // same order in every thread
  return s;
}

// Reflector for x = c[s .. m-1] (a shared column, indexed by row): H = I -
// beta u u^T maps x to alpha e_1 (alpha = -sign(x_0) ||x||); u goes to v[s ..].
// Every CTA computes it from the same data in the same order: bitwise equal.
__device__ void reflector(const double* c, int s, int m, double* v, double* red, double& beta, double& alpha) {
  double ss = 0.0;
  for (int i = s + 1 + threadIdx.x; i < m; i += blockDim.x) ss += c[i] * c[i];
  const double tail = block_sum(ss, red);
  const double x0 = c[s];
  if (tail == 0.0) {  // already reduced in this column
    beta = 0.0;
    alpha = x0;
    for (int i = s + threadIdx.x; i < m; i += blockDim.x) v[i] = 0.0;
    __syncthreads();
    return;
  }
  const double nrm = sqrt(x0 * x0 + tail);
  alpha = x0 >= 0.0 ? -nrm : nrm;
  const double u0 = x0 - alpha;
  beta = 1.0 / (nrm * fabs(u0));  // 2 / (u.u), u.u = 2 nrm |u0|
  for (int i = s + threadIdx.x; i < m; i += blockDim.x) v[i] = i == s ? u0 : c[i];
  __syncthreads();
}

// G (m x m, column-major, full symmetric; overwritten) -> d[m], e[m-1].
// p0/p1: m doubles each (the per-step mat-vec, double-buffered).
__global__ void __launch_bounds__(kTriThreads, 1)
    tridiag_coop_kernel(int m, double* __restrict__ G, double* __restrict__ d, double* __restrict__ e,
                        double* __restrict__ p0, double* __restrict__ p1) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sh[];
  double* v = sh;       // current reflector (rows k+1 ..)
  double* w = v + m;    // w = p - K v
  double* c = w + m;    // look-ahead column k+1 after step k's update
  double* vn = c + m;   // next reflector
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp, GW = gridDim.x * (blockDim.x >> 5);
  // step 0's reflector from column 0, and its mat-vec p = beta G[1:,1:] v
  for (int i = threadIdx.x; i < m; i += blockDim.x) c[i] = G[i];
  __syncthreads();
  double beta, alpha;
  reflector(c, 1, m, v, red, beta, alpha);  // x = G[1:, 0]
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    d[0] = c[0];
    e[0] = alpha;
  }
  for (int j = 1 + gw; j < m; j += GW) {
    const double* col = G + static_cast<int64_t>(j) * m;
    double s = 0.0;
    for (int i = 1 + lane; i < m; i += 32) s += col[i] * v[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) p0[j] = beta * s;
  }
  grid.sync();
  for (int k = 0; k + 2 < m; ++k) {
    double* p = (k & 1) ? p1 : p0;
    double* pn = (k & 1) ? p0 : p1;
    // K = beta/2 p.v, w = p - K v  (rows k+1 .. m-1; every CTA, same order)
    double pv = 0.0;
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) {
      const double pi = __ldcg(p + i);
      w[i] = pi;
      pv += pi * v[i];
    }
    const double K = 0.5 * beta * block_sum(pv, red);
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) w[i] -= K * v[i];
    __syncthreads();
    // look-ahead: column k+1 of the updated trailing block, then the next reflector
    const double vk1 = v[k + 1], wk1 = w[k + 1];
    const double* colk1 = G + static_cast<int64_t>(k + 1) * m;
    for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) c[i] = __ldcg(colk1 + i) - v[i] * wk1 - w[i] * vk1;
    __syncthreads();
    double betan, alphan;
    reflector(c, k + 2, m, vn, red, betan, alphan);  // x = c[k+2 ..]
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      d[k + 1] = c[k + 1];
      e[k + 1] = alphan;
    }
    // owned trailing columns j >= k+2: rank-2 update (rows >= k+2), then the next mat-vec entry
    for (int j = k + 2 + gw; j < m; j += GW) {
      double* col = G + static_cast<int64_t>(j) * m;
      const double vj = v[j], wj = w[j];
      double s = 0.0;
      for (int i0 = k + 2 + lane; i0 < m; i0 += 32 * 8) {  // 8 loads in flight per lane
        double gv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) gv[u] = i0 + 32 * u < m ? __ldcg(col + i0 + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + 32 * u;
          if (i < m) {
            const double g = gv[u] - v[i] * wj - w[i] * vj;
            col[i] = g;
            s += g * vn[i];
          }
        }
      }
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) pn[j] = betan * s;
    }
    __syncthreads();  // every warp of this CTA is done reading v
    for (int i = k + 2 + threadIdx.x; i < m; i += blockDim.x) v[i] = vn[i];
    beta = betan;
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) d[m - 1] = __ldcg(G + static_cast<int64_t>(m - 1) * m + (m - 1));
}

// Eigenvalue t (descending) of the symmetric tridiagonal (d, e), one warp per
// eigenvalue: 32-way multisection on Sturm counts (each lane counts at its own
// point; the Sturm recurrence is one dependent division per row, so lanes, not
// iterations, carry the parallelism), to an absolute width of 2 eps ||T||.
__device__ __forceinline__ int sturm_count(int m, const double* d, const double* e, double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < m; ++i) {
    q = d[i] - x - e[i - 1] * e[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

__global__ void tridiag_bisect_kernel(int m, const double* __restrict__ d, const double* __restrict__ e,
                                      double* __restrict__ lam) {
  const int lane = threadIdx.x & 31;
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= m) return;
  // Gershgorin bounds (warp-parallel)
  double lo = 1e300, hi = -1e300, nrm = 0.0;
  for (int i = lane; i < m; i += 32) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < m ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
    nrm = fmax(nrm, fabs(d[i]) + r);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    nrm = fmax(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
  }
  const double pivmin = 1e-290 * fmax(1.0, nrm * nrm);
  const double tol = 4.4e-16 * nrm + 1e-300;
  const int want = m - 1 - t;  // ascending index: smallest x with count(lambda < x) > want
  for (int it = 0; it < 40 && hi - lo > tol; ++it) {
    const double x = lo + (hi - lo) * (lane + 1) / 33.0;
    const unsigned above = __ballot_sync(0xffffffffu, sturm_count(m, d, e, x, pivmin) > want);
    const int f = above ? __ffs(above) - 1 : 32;  // first point past the eigenvalue
    const double nlo = f == 0 ? lo : lo + (hi - lo) * f / 33.0;
    const double nhi = f == 32 ? hi : lo + (hi - lo) * (f + 1) / 33.0;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) lam[t] = 0.5 * (lo + hi);
}

// RHOSVD's mode matrix W(:, k) = f_axis(:, k) / |f_axis(:, k)| * w'_k with w'
// the weight after normalize (tensor.cpp:18-31) — the same arithmetic, in the
// same reduction order, as reduction.cu's normalize_kernel + scale_cols_kernel
// (launch with 256 threads), without copying the other two factors.
__global__ void mode_matrix_kernel(int64_t n0, int64_t n1, int64_t n2, const double* __restrict__ f0,
                                   const double* __restrict__ f1, const double* __restrict__ f2,
                                   const double* __restrict__ w, int axis, double* __restrict__ W) {
  __shared__ double sv[32];
  const int64_t k = blockIdx.x;
  const double* fs[3] = {f0 + n0 * k, f1 + n1 * k, f2 + n2 * k};
  const int64_t ns[3] = {n0, n1, n2};
  double wk = w[k], nrm_axis = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    double part = 0.0;
    for (int64_t i = threadIdx.x; i < ns[ax]; i += blockDim.x) part += fs[ax][i] * fs[ax][i];
    for (int o = 16; o; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = part;
    __syncthreads();
    double ss = 0.0;
    if (threadIdx.x == 0) {
      for (int i = 0; i < (blockDim.x + 31) / 32; ++i) ss += sv[i];
      sv[0] = ss;
    }
    __syncthreads();
    const double nrm = sqrt(sv[0]);
    __syncthreads();
    if (ax == axis) nrm_axis = nrm;
    wk = nrm > 0.0 ? wk * nrm : 0.0;
  }
  const int64_t n = ns[axis];
  double* out = W + n * k;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = (nrm_axis > 0.0 ? fs[axis][i] / nrm_axis : fs[axis][i]) * wk;
}

// stream-ordered scratch (the pool keeps repeated calls cheap)
struct DBuf {
  double* p = nullptr;
  cudaStream_t s;
  DBuf(size_t n, cudaStream_t stream) : s(stream) {
    TGB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(n, 1) * sizeof(double), s));
  }
  ~DBuf() { cudaFreeAsync(p, s); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

}  // namespace

// Eigenvalues (descending) of a symmetric m x m device matrix G (overwritten).
void sym_eigvals_dev(tgb_ctx* ctx, int64_t m, double* G, double* lam) {
  if (m <= 0) return;
  if (m == 1) {
    TGB_CUDA(cudaMemcpyAsync(lam, G, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  DBuf d(m, ctx->stream), e(m, ctx->stream), p0(m, ctx->stream), p1(m, ctx->stream);
  const size_t smem = static_cast<size_t>(4 * m) * sizeof(double);
  if (smem + 2048 > ctx->smem_optin) throw Error(TGB_INVALID_ARGUMENT, "mode spectrum: matrix too large");
  static bool attr[kTgbMaxDevices] = {};
  static int per_sm[kTgbMaxDevices] = {};
  if (!attr[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(tridiag_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ctx->smem_optin - 1024)));
    attr[ctx->device] = true;
  }
  TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[ctx->device], tridiag_coop_kernel, kTriThreads, smem));
  if (per_sm[ctx->device] < 1) throw Error(TGB_CUDA_ERROR, "mode spectrum: tridiagonalisation kernel does not fit");
  // one trailing column per warp where possible (16 warps per CTA), at most one CTA per SM
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, (m + 15) / 16)));
  int mi = static_cast<int>(m);
  void* args[] = {&mi, &G, &d.p, &e.p, &p0.p, &p1.p};
  TGB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tridiag_coop_kernel), dim3(grid), dim3(kTriThreads),
                                       args, smem, ctx->stream));
  TGB_LAUNCHED(ctx);
  tridiag_bisect_kernel<<<static_cast<unsigned>((m + 3) / 4), 128, 0, ctx->stream>>>(mi, d.p, e.p, lam);
  TGB_LAUNCHED(ctx);
}

// Spectrum of W (n x R, device) with the reference's count rule.
std::vector<double> mode_spectrum_dev(tgb_ctx* ctx, int64_t n, int64_t R, const double* W) {
  std::vector<double> out;
  if (n == 0 || R == 0) return out;
  const int64_t m = std::min(n, R);
  DBuf G(static_cast<size_t>(m) * m, ctx->stream), lam(m, ctx->stream);
  if (n <= R)
    dgemm(ctx, false, true, n, n, R, 1.0, W, n, W, n, 0.0, G.p, n);  // W W^T
  else
    dgemm(ctx, true, false, R, R, n, 1.0, W, n, W, n, 0.0, G.p, R);  // W^T W
  sym_eigvals_dev(ctx, m, G.p, lam.p);
  std::vector<double> l(m);
  TGB_CUDA(cudaMemcpyAsync(l.data(), lam.p, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  const bool gram_wide = R >= 4 * n && R > 8192;                 // reduction.cpp:93-104
  const bool jacobi_branch = !gram_wide && (n < 4 * R || R < 8);  // reduction.cpp:105-108
  if (gram_wide || jacobi_branch) {
    out.resize(m);
    for (int64_t i = 0; i < m; ++i) out[i] = std::sqrt(std::max(0.0, l[i]));
    return out;
  }
  const double lmax = std::max(0.0, l[0]);  // tall Gram branch: reduction.cpp:119-125
  for (int64_t i = 0; i < m; ++i) {
    if (l[i] <= lmax * 1e-24 || l[i] <= 0.0) break;
    out.push_back(std::sqrt(l[i]));
  }
  return out;
}

// RHOSVD's mode matrix of a CP tensor (device): W = f_axis diag(w) after normalize.
std::vector<double> cp_mode_spectrum(tgb_ctx* ctx, const tgb_cp& a, int axis) {
  const int64_t R = a.rank, n = a.n[axis];
  if (R == 0 || n == 0) return {};
  DBuf W(static_cast<size_t>(n) * R, ctx->stream);
  mode_matrix_kernel<<<static_cast<unsigned>(R), 256, 0, ctx->stream>>>(a.n[0], a.n[1], a.n[2], a.factor[0], a.factor[1],
                                                                       a.factor[2], a.weight, axis, W.p);
  TGB_LAUNCHED(ctx);
  return mode_spectrum_dev(ctx, n, R, W.p);
}

}  // namespace tgb

extern "C" int tgb_mode_spectrum(tgb_ctx* ctx, const tgb_cp* a, int axis, int mem, int64_t* count, double* sigma) {
  return tgb::guarded_call([&] {
    tgb::require(ctx && a && count && axis >= 0 && axis < 3, "mode_spectrum: bad argument");
    tgb::require(a->rank == 0 || a->n[axis] == 0 || sigma != nullptr, "mode_spectrum: null output");
    TGB_CUDA(cudaSetDevice(ctx->device));
    tgb_cp dev = *a;
    std::vector<std::unique_ptr<tgb::DBuf>> own;
    if (mem == TGB_MEM_HOST && a->rank) {
      for (int ax = 0; ax < 3; ++ax) {
        own.push_back(std::make_unique<tgb::DBuf>(static_cast<size_t>(a->n[ax]) * a->rank, ctx->stream));
        tgb::h2d(ctx, own.back()->p, a->factor[ax], a->n[ax] * a->rank * sizeof(double), ctx->stream);
        dev.factor[ax] = own.back()->p;
      }
      own.push_back(std::make_unique<tgb::DBuf>(a->rank, ctx->stream));
      tgb::h2d(ctx, own.back()->p, a->weight, a->rank * sizeof(double), ctx->stream);
      dev.weight = own.back()->p;
    }
    const std::vector<double> s = tgb::cp_mode_spectrum(ctx, dev, axis);
    *count = static_cast<int64_t>(s.size());
    for (size_t i = 0; i < s.size(); ++i) sigma[i] = s[i];
  });
}

// Factorised two-electron integrals on sm_100a (reference proj/src/tei.cpp):
//   1D density fitting per axis (tei.cpp:92-143): product side matrix G,
//     Gram G G^T on the DMMA tensor cores, pivoted Cholesky with trace stop
//     (single-CTA device loop, first-maximal-index pivots as Eigen's
//     maxCoeff(&p)), an orthonormal basis of the selected columns by
//     GEMM-based Cholesky-QR (the reference's Householder QR up to column
//     signs, which B does not see), V = G^T U;
//   convolution matrices M_k = U^T (h conv(U, p_k)) (tei.cpp:145-158) through
//     the FFT mode-convolution path + one GEMM per axis;
//   the TEI diagonal from the bilinear forms V[j2,:] M_k V[j,:]^T
//      instead of whole columns (tei.cpp:182-196);
//   TEI columns (tei.cpp:33-44,160-174) as three GEMMs + a fused
//     product-over-axes / sum-over-terms kernel;
//   the TEI pivoted Cholesky (tei.cpp:48-90,198-204) as a host-driven loop of
//     device steps (argmax, column, downdate).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <vector>

#include "tgb_internal.hpp"

namespace tgb {

namespace {

constexpr int kRedThreads = 1024;

// ---------------------------------------------------------------- helpers

// block-wide argmax with the FIRST maximal index (ties -> lowest index)
__device__ __forceinline__ void argmax_combine(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__device__ void block_argmax(double& v, int& i, double* sv, int* si) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_down_sync(0xffffffffu, v, o);
    const int i2 = __shfl_down_sync(0xffffffffu, i, o);
    argmax_combine(v, i, v2, i2);
  }
  if (lane == 0) {
    sv[warp] = v;
    si[warp] = i;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    v = lane < nw ? sv[lane] : -INFINITY;
    i = lane < nw ? si[lane] : 0x7fffffff;
    for (int o = 16; o; o >>= 1) {
      const double v2 = __shfl_down_sync(0xffffffffu, v, o);
      const int i2 = __shfl_down_sync(0xffffffffu, i, o);
      argmax_combine(v, i, v2, i2);
    }
    if (lane == 0) {
      sv[0] = v;
      si[0] = i;
    }
  }
  __syncthreads();
  v = sv[0];
  i = si[0];
  __syncthreads();
}

__device__ double block_sum(double v, double* sv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) sv[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    v = lane < nw ? sv[lane] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sv[0] = v;
  }
  __syncthreads();
  v = sv[0];
  __syncthreads();
  return v;
}

// ---------------------------------------------------------------- density fitting

// G[i + n (p + np q)] = prim[i, p] * prim[i, q]            (tei.cpp:118-121)
__global__ void gprod_kernel(int64_t n, int np, const double* __restrict__ prim, double* __restrict__ G) {
  const int64_t col = blockIdx.y;  // p + np q
  const int p = static_cast<int>(col % np), q = static_cast<int>(col / np);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    G[i + n * col] = prim[i + n * p] * prim[i + n * q];
}

__global__ void square_kernel(int64_t count, double* __restrict__ x) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] *= x[i];
}

// Pivoted Cholesky of an explicit SPD n x n matrix A (tei.cpp:48-90), single
// CTA.  info[0] = rank, info[1] = clamped_negative, info[2] = error (1 = not
// PSD beyond tolerance); pivots[rank]; residual[0] = stop measure ratio.
__device__ __forceinline__ void pivchol_explicit_body(int n, const double* __restrict__ A, double tol, int trace_stop,
                                                      int cap, double neg_tol, double* __restrict__ diag,
                                                      double* __restrict__ L, int* pivots, int* info,
                                                      double* residual) {
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ double s_dmax;
  __shared__ int s_p;
  // diagonal and its max / sum
  double lmax = -INFINITY, lsum = 0.0;
  int imax = 0x7fffffff;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = A[i + static_cast<int64_t>(n) * i];
    diag[i] = d;
    argmax_combine(lmax, imax, d, i);
    lsum += d;
  }
  block_argmax(lmax, imax, sv, si);
  const double max0 = lmax;
  const double trace0 = block_sum(lsum, sv);
  int rank = 0, clamped = 0, err = 0;
  if (max0 > 0.0) {
    const double target = tol * (trace_stop ? trace0 : max0);
    while (rank < cap) {
      double dm = -INFINITY, ds = 0.0;
      int p = 0x7fffffff;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        argmax_combine(dm, p, diag[i], i);
        ds += diag[i];
      }
      block_argmax(dm, p, sv, si);
      const double meas = trace_stop ? block_sum(ds, sv) : dm;
      if (meas <= target || dm <= 0.0) break;
      if (threadIdx.x == 0) {
        s_dmax = dm;
        s_p = p;
        pivots[rank] = p;
      }
      __syncthreads();
      const double piv = sqrt(s_dmax);
      const int pp = s_p;
      int bad = 0, cl = 0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double c = A[i + static_cast<int64_t>(n) * pp];
        for (int r = 0; r < rank; ++r) c -= L[i + static_cast<int64_t>(n) * r] * L[pp + static_cast<int64_t>(n) * r];
        double l = c / piv;
        if (i == pp) l = piv;
        L[i + static_cast<int64_t>(n) * rank] = l;
        double d = diag[i] - l * l;
        if (i == pp) d = 0.0;
        if (d < 0.0) {
          if (d < -neg_tol * max0) bad = 1;
          d = 0.0;
          cl = 1;
        }
        diag[i] = d;
      }
      bad = __syncthreads_or(bad);
      cl = __syncthreads_or(cl);
      clamped |= cl;
      ++rank;
      if (bad) {
        err = 1;
        break;
      }
    }
  }
  // final stop measure
  double dm = -INFINITY, ds = 0.0;
  int p = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    argmax_combine(dm, p, diag[i], i);
    ds += diag[i];
  }
  block_argmax(dm, p, sv, si);
  const double fs = block_sum(ds, sv);
  if (threadIdx.x == 0) {
    info[0] = rank;
    info[1] = clamped;
    info[2] = err;
    residual[0] = max0 > 0.0 ? (trace_stop ? fs : dm) / (trace_stop ? trace0 : max0) : 0.0;
  }
}

__global__ void __launch_bounds__(kRedThreads) pivchol_explicit_kernel(int n, const double* __restrict__ A,
                                                                       double tol, int trace_stop, int cap,
                                                                       double neg_tol, double* __restrict__ diag,
                                                                       double* __restrict__ L, int* pivots, int* info,
                                                                       double* residual) {
  pivchol_explicit_body(n, A, tol, trace_stop, cap, neg_tol, diag, L, pivots, info, residual);
}

// the three axes' factorisations of the density fit are independent: one CTA each
struct PivAxis {
  int n, cap;
  const double* A;
  double *diag, *L, *residual;
  int *pivots, *info;
};
struct PivBatch {
  PivAxis ax[3];
};
__global__ void __launch_bounds__(kRedThreads) pivchol_explicit3_kernel(PivBatch b, double tol, int trace_stop,
                                                                        double neg_tol) {
  const PivAxis& a = b.ax[blockIdx.x];
  pivchol_explicit_body(a.n, a.A, tol, trace_stop, a.cap, neg_tol, a.diag, a.L, a.pivots, a.info, a.residual);
}

// The three fitting Choleskys as ONE cooperative grid: G CTAs per axis own
// contiguous row blocks; per step each CTA forms its rows of the pivot column
// (the same sequential r order as pivchol_explicit_body, so L is identical),
// downdates its diagonal and publishes (argmax, sum, flags) partials; after
// one grid barrier every CTA reduces all partials in CTA order and so takes
// the same next pivot / stop decision for all three axes (no second barrier).
// Partials are double-buffered by step parity.  The single-CTA body read
// L (n x rank) through one SM per axis: bandwidth-bound at ~4.6 ms for the
// config-3 fit.
constexpr int kCoopThreads = 128;
__device__ __forceinline__ double4 ldcg4(const double4* p) {  // L2 load (written by other CTAs in this grid)
  const double2 lo = __ldcg(reinterpret_cast<const double2*>(p));
  const double2 hi = __ldcg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(lo.x, lo.y, hi.x, hi.y);
}
struct CoopAxis {
  int rank, p, active, err, clamped;
  double dm, max0, trace0, target, meas;
};
// one warp reduces one axis' G <= 64 partials: (argmax, sum, flag OR); the
// shuffle tree is fixed, so every CTA obtains bit-identical results
__device__ __forceinline__ void coop_reduce(const double4* __restrict__ pa, int G, double& dm, int& p, double& ds,
                                            int& fl) {
  const int lane = threadIdx.x & 31;
  dm = -INFINITY;
  p = 0x7fffffff;
  ds = 0.0;
  fl = 0;
  for (int q = lane; q < G; q += 32) {
    const double4 v = ldcg4(pa + q);
    argmax_combine(dm, p, v.x, static_cast<int>(v.y));
    ds += v.z;
    fl |= static_cast<int>(v.w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, dm, o);
    const int p2 = __shfl_xor_sync(0xffffffffu, p, o);
    argmax_combine(dm, p, v2, p2);
    ds += __shfl_xor_sync(0xffffffffu, ds, o);
    fl |= __shfl_xor_sync(0xffffffffu, fl, o);
  }
}
__global__ void __launch_bounds__(kCoopThreads) pivchol_coop3_kernel(PivBatch b, int G, double tol, int trace_stop,
                                                                     double neg_tol, double4* __restrict__ part) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double s_lp[];  // L[p, :rank] of this CTA's axis
  __shared__ CoopAxis S[3];
  __shared__ double sv[32];
  __shared__ int si[32];
  const int a = blockIdx.x / G, g = blockIdx.x % G, tid = threadIdx.x;
  const PivAxis& X = b.ax[a];
  const int n = X.n;
  const int i0 = static_cast<int>((static_cast<int64_t>(n) * g) / G);
  const int i1 = static_cast<int>((static_cast<int64_t>(n) * (g + 1)) / G);
  double* __restrict__ L = X.L;
  double* __restrict__ diag = X.diag;
  // diagonal, its max and trace
  {
    double lm = -INFINITY, ls = 0.0;
    int li = 0x7fffffff;
    for (int i = i0 + tid; i < i1; i += blockDim.x) {
      const double d = __ldg(X.A + i + static_cast<int64_t>(n) * i);
      diag[i] = d;
      argmax_combine(lm, li, d, i);
      ls += d;
    }
    block_argmax(lm, li, sv, si);
    ls = block_sum(ls, sv);
    if (tid == 0) part[(0 * 3 + a) * G + g] = make_double4(lm, static_cast<double>(li), ls, 0.0);
  }
  grid.sync();
  if (tid < 96) {  // warp ax reduces axis ax
    const int ax = tid >> 5;
    double dm, ds;
    int p, fl;
    coop_reduce(part + (0 * 3 + ax) * G, G, dm, p, ds, fl);
    if ((tid & 31) == 0) {
      CoopAxis& c = S[ax];
      c.rank = 0;
      c.err = 0;
      c.clamped = 0;
      c.max0 = dm;
      c.trace0 = ds;
      c.target = tol * (trace_stop ? ds : dm);
      c.dm = dm;
      c.p = p;
      c.meas = trace_stop ? ds : dm;
      c.active = dm > 0.0 && b.ax[ax].cap > 0 && !(c.meas <= c.target || dm <= 0.0);
    }
  }
  __syncthreads();
  for (int step = 1;; ++step) {
    if (!(S[0].active || S[1].active || S[2].active)) break;
    const int buf = step & 1;
    if (S[a].active) {
      const int rank = S[a].rank, pp = S[a].p;
      const double piv = sqrt(S[a].dm), max0 = S[a].max0;
      if (g == 0 && tid == 0) X.pivots[rank] = pp;
      for (int r = tid; r < rank; r += blockDim.x) s_lp[r] = __ldcg(L + pp + static_cast<int64_t>(n) * r);
      __syncthreads();
      double lm = -INFINITY, ls = 0.0;
      int li = 0x7fffffff, bad = 0, cl = 0;
      for (int i = i0 + tid; i < i1; i += blockDim.x) {
        double c = __ldg(X.A + i + static_cast<int64_t>(n) * pp);
        // the rank-long dot product in the sequential r order, its L2 loads issued 32 at a time
        const double* Li = L + i;
        int r = 0;
        for (; r + 32 <= rank; r += 32) {
          double lv[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) lv[u] = __ldcg(Li + static_cast<int64_t>(n) * (r + u));
#pragma unroll
          for (int u = 0; u < 32; ++u) c -= lv[u] * s_lp[r + u];
        }
        for (; r + 8 <= rank; r += 8) {
          double lv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) lv[u] = __ldcg(Li + static_cast<int64_t>(n) * (r + u));
#pragma unroll
          for (int u = 0; u < 8; ++u) c -= lv[u] * s_lp[r + u];
        }
        for (; r < rank; ++r) c -= __ldcg(Li + static_cast<int64_t>(n) * r) * s_lp[r];
        double l = c / piv;
        if (i == pp) l = piv;
        L[i + static_cast<int64_t>(n) * rank] = l;
        double d = diag[i] - l * l;
        if (i == pp) d = 0.0;
        if (d < 0.0) {
          if (d < -neg_tol * max0) bad = 1;
          d = 0.0;
          cl = 1;
        }
        diag[i] = d;
        argmax_combine(lm, li, d, i);
        ls += d;
      }
      bad = __syncthreads_or(bad);
      cl = __syncthreads_or(cl);
      block_argmax(lm, li, sv, si);
      ls = block_sum(ls, sv);
      if (tid == 0) part[(buf * 3 + a) * G + g] = make_double4(lm, static_cast<double>(li), ls, 2.0 * bad + cl);
    }
    grid.sync();
    if (tid < 96 && S[tid >> 5].active) {  // warp-uniform
      const int ax = tid >> 5;
      double dm, ds;
      int p, fl;
      coop_reduce(part + (buf * 3 + ax) * G, G, dm, p, ds, fl);
      if ((tid & 31) == 0) {
        CoopAxis& c = S[ax];
        c.clamped |= fl & 1;
        c.rank += 1;
        c.dm = dm;
        c.p = p;
        c.meas = trace_stop ? ds : dm;
        if (fl & 2) {
          c.err = 1;
          c.active = 0;
        } else if (c.rank >= b.ax[ax].cap || c.meas <= c.target || dm <= 0.0) {
          c.active = 0;
        }
      }
    }
    __syncthreads();
  }
  if (g == 0 && tid == 0) {
    const CoopAxis& c = S[a];
    X.info[0] = c.rank;
    X.info[1] = c.clamped;
    X.info[2] = c.err;
    X.residual[0] = c.max0 > 0.0 ? c.meas / (trace_stop ? c.trace0 : c.max0) : 0.0;
  }
}

// partial sums of (G - T)^2 and G^2 (fit residual, tei.cpp:140-141)
__global__ void resid_kernel(int64_t total, const double* __restrict__ G, const double* __restrict__ T,
                             double* __restrict__ out) {
  __shared__ double sv[32];
  double a = 0.0, b = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double d = G[i] - T[i];
    a += d * d;
    b += G[i] * G[i];
  }
  a = block_sum(a, sv);
  b = block_sum(b, sv);
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = a;
    out[2 * blockIdx.x + 1] = b;
  }
}

// ---------------------------------------------------------------- TEI diagonal / columns

// acc[c] (+)= sum over the primitive pairs (j, j2) of contracted pair c of
//   w_j w_j2 prod_ax <V_ax[j2, :], Y_ax[j, :]>,  Y_ax = V_ax M_k^T
// (tei.cpp:182-196 with b_prim_column expanded; one kernel term k per call).
__global__ void tei_diag_term_kernel(int nc, const int* __restrict__ cstart, const int* __restrict__ cpairs,
                                     const double* __restrict__ cw, int64_t np2, const double* __restrict__ V0,
                                     const double* __restrict__ V1, const double* __restrict__ V2, int r0, int r1,
                                     int r2, const double* __restrict__ Y0, const double* __restrict__ Y1,
                                     const double* __restrict__ Y2, double* __restrict__ acc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  double s = 0.0;
  for (int a = cstart[c]; a < cstart[c + 1]; ++a)
    for (int b = cstart[c]; b < cstart[c + 1]; ++b) {
      const int j = cpairs[a], j2 = cpairs[b];
      double d0 = 0.0, d1 = 0.0, d2 = 0.0;
      for (int q = 0; q < r0; ++q) d0 += V0[j2 + np2 * q] * Y0[j + np2 * q];
      for (int q = 0; q < r1; ++q) d1 += V1[j2 + np2 * q] * Y1[j + np2 * q];
      for (int q = 0; q < r2; ++q) d2 += V2[j2 + np2 * q] * Y2[j + np2 * q];
      s += cw[a] * cw[b] * (d0 * d1 * d2);
    }
  acc[c] += s;
}

// All kernel terms at once when every Y_k = V M_k^T is stored (Pk): grid.y = k,
// s[k nc + c] = tei_diag_term_kernel's per-term sum; tei_diag_sum_kernel then
// adds the terms in k order, so diag is bit-identical to the per-term launches.
// Rows c in [c0, c1) (all of them on one process; a rank's pair-row block
// under a communicator).
__global__ void tei_diag_terms_kernel(int nc, int c0, int c1, const int* __restrict__ cstart,
                                      const int* __restrict__ cpairs, const double* __restrict__ cw, int64_t np2,
                                      const double* __restrict__ V0, const double* __restrict__ V1,
                                      const double* __restrict__ V2, int r0, int r1, int r2,
                                      const double* __restrict__ P0, const double* __restrict__ P1,
                                      const double* __restrict__ P2, double* __restrict__ s_out) {
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  const int64_t k = blockIdx.y;
  const double* Y0 = P0 + np2 * r0 * k;
  const double* Y1 = P1 + np2 * r1 * k;
  const double* Y2 = P2 + np2 * r2 * k;
  double s = 0.0;
  for (int a = cstart[c]; a < cstart[c + 1]; ++a)
    for (int b = cstart[c]; b < cstart[c + 1]; ++b) {
      const int j = cpairs[a], j2 = cpairs[b];
      double d0 = 0.0, d1 = 0.0, d2 = 0.0;
      for (int q = 0; q < r0; ++q) d0 += V0[j2 + np2 * q] * Y0[j + np2 * q];
      for (int q = 0; q < r1; ++q) d1 += V1[j2 + np2 * q] * Y1[j + np2 * q];
      for (int q = 0; q < r2; ++q) d2 += V2[j2 + np2 * q] * Y2[j + np2 * q];
      s += cw[a] * cw[b] * (d0 * d1 * d2);
    }
  s_out[k * nc + c] = s;
}

__global__ void tei_diag_sum_kernel(int nc, int c0, int c1, int K, const double* __restrict__ s_in,
                                    double* __restrict__ acc) {
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  double v = acc[c];
  for (int k = 0; k < K; ++k) v += s_in[static_cast<int64_t>(k) * nc + c];
  acc[c] = v;
}

// col[i] = sum_k prod_ax W_ax[i, k]   (b_prim_column, tei.cpp:33-44)
__global__ void tei_col_combine_kernel(int64_t np2, int K, const double* __restrict__ W0,
                                       const double* __restrict__ W1, const double* __restrict__ W2,
                                       double* __restrict__ col) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= np2) return;
  double s = 0.0;
  for (int k = 0; k < K; ++k) s += W0[i + np2 * k] * W1[i + np2 * k] * W2[i + np2 * k];
  col[i] = s;
}

// gather rows V_ax[j, :] (j = primitive pair) into Vj (r x 1) for each axis
__global__ void gather_row_kernel(const double* __restrict__ V, int64_t np2, int r, int j, double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < r) out[q] = V[j + np2 * q];
}

// contraction: out[owner[p] + nb owner[q]] += pw[p] pw[q] z[p + np q]  (tei.cpp:166-172),
// as a gather over contracted pairs (deterministic order p-major within q as the reference loop)
template <bool COHERENT = false>
__device__ __forceinline__ double contract_at(int c, int nb, int np, const int* __restrict__ fstart,
                                              const double* __restrict__ pw, const double* __restrict__ z) {
  const int mu = c % nb, nu = c / nb;
  const int a = min(mu, nu), b = max(mu, nu);
  double s = 0.0;
  for (int q = fstart[b]; q < fstart[b + 1]; ++q)
    for (int p = fstart[a]; p < fstart[a + 1]; ++p) {
      const int64_t idx = mu <= nu ? p + static_cast<int64_t>(np) * q : q + static_cast<int64_t>(np) * p;
      s += pw[p] * pw[q] * (COHERENT ? __ldcg(z + idx) : z[idx]);
    }
  return s;
}

__global__ void contract_kernel(int nb, int np, const int* __restrict__ fstart, const double* __restrict__ pw,
                                const double* __restrict__ z, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nb * nb) out[c] = contract_at(c, nb, np, fstart, pw, z);
}

__global__ void axpy_kernel(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y, int init) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = init ? a * x[i] : y[i] + a * x[i];
}

// side-by-side [M_0 | M_1 | ...] (r x rK) -> stacked [M_0; M_1; ...] (rK x r)
__global__ void stack_kernel(int r, int K, const double* __restrict__ Mcat, double* __restrict__ Mst) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t tot = static_cast<int64_t>(r) * r * K;
  if (idx >= tot) return;
  const int a = static_cast<int>(idx % r);
  const int64_t rest = idx / r;  // b + r k
  const int b = static_cast<int>(rest % r), k = static_cast<int>(rest / r);
  Mst[(a + static_cast<int64_t>(r) * k) + static_cast<int64_t>(r) * K * b] = Mcat[idx];
}

__global__ void argmax_kernel(int n, const double* __restrict__ d, double* out_v, int* out_i) {
  __shared__ double sv[32];
  __shared__ int si[32];
  double v = -INFINITY;
  int idx = 0x7fffffff;
  for (int i = threadIdx.x; i < n; i += blockDim.x) argmax_combine(v, idx, d[i], i);
  block_argmax(v, idx, sv, si);
  if (threadIdx.x == 0) {
    *out_v = v;
    *out_i = idx;
  }
}

// ---- device-resident pivoted-Cholesky loop (tei.cpp:48-90 with the
// max-diagonal stop of tei.cpp:198-204).  One step = the kernels below with
// every step-dependent scalar (rank, pivot, max diagonal, the primitive pair of
// the current column term, the stop flag) in device memory, so one captured
// step replays as a CUDA graph with no host round trip.
struct CholState {
  int rank;      // columns produced so far
  int done;      // stop rule met (or the cap): later steps are no-ops
  int piv;       // current pivot (contracted pair index)
  int j;         // current primitive pair of the column being formed
  double dmax;   // current max diagonal
  double w;      // weight of the current primitive pair (0: no term)
  int flags[2];  // [0] clamped a negative diagonal, [1] negative beyond tolerance
  unsigned int arrived;  // CTAs of the current chol_step_dev_kernel that finished (the last advances)
};

// argmax of the diagonal (first maximal index, Eigen's maxCoeff(&p)); stop test
__device__ __forceinline__ void chol_term(int nb, int np, int t, const int* __restrict__ fstart,
                                          const double* __restrict__ pw, CholState* st);
// (+ the column's first primitive pair, chol_term t = 0; gathering its y_ax
// here too measured slower than chol_ygather_kernel's 48 CTAs)
__global__ void __launch_bounds__(kRedThreads) chol_pivot_kernel(int n, const double* __restrict__ d, double target,
                                                                 int cap, CholState* st, int64_t* piv_list, int nb,
                                                                 int np, const int* __restrict__ fstart,
                                                                 const double* __restrict__ pw) {
  if (st->done) return;
  __shared__ double sv[32];
  __shared__ int si[32];
  double v = -INFINITY;
  int idx = 0x7fffffff;
  for (int i = threadIdx.x; i < n; i += blockDim.x) argmax_combine(v, idx, d[i], i);
  block_argmax(v, idx, sv, si);
  if (threadIdx.x == 0) {
    if (st->rank >= cap || v <= target || v <= 0.0) {
      st->done = 1;
    } else {
      st->piv = idx;
      st->dmax = v;
      piv_list[st->rank] = idx;
      chol_term(nb, np, 0, fstart, pw, st);
    }
  }
}

// primitive pair t of the pivot's contracted pair (kappa, lambda): q-major over
// lambda's primitives, p over kappa's (tei.cpp:166-170 loop order)
__device__ __forceinline__ void chol_term(int nb, int np, int t, const int* __restrict__ fstart,
                                          const double* __restrict__ pw, CholState* st) {
  const int c = st->piv, kappa = c % nb, lambda = c / nb;
  const int nk = fstart[kappa + 1] - fstart[kappa], nl = fstart[lambda + 1] - fstart[lambda];
  if (t >= nk * nl) {
    st->w = 0.0;
    return;
  }
  const int p = fstart[kappa] + t % nk, q = fstart[lambda] + t / nk;
  st->j = p + np * q;
  st->w = pw[p] * pw[q];
}

__global__ void chol_term_kernel(int nb, int np, int t, const int* __restrict__ fstart, const double* __restrict__ pw,
                                 CholState* st) {
  if (st->done) return;
  chol_term(nb, np, t, fstart, pw, st);
}

__global__ void gather_row_dev_kernel(const double* __restrict__ V, int64_t np2, int r, const CholState* st,
                                      double* __restrict__ out) {
  if (st->done) return;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < r) out[q] = V[st->j + np2 * q];
}

__global__ void axpy_dev_kernel(int64_t n, const CholState* st, const double* __restrict__ x, double* __restrict__ y,
                                int init) {
  if (st->done) return;
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double a = st->w;
  if (init) y[i] = a * x[i];
  else if (a != 0.0) y[i] = y[i] + a * x[i];
}

// tei.cpp:70-83 for the pivot in `st`: the column entry is contracted here
// from the primitive-pair column z (tei.cpp:166-170), and the last CTA to
// finish advances the rank.
// The downdate col - L[:, :rank] L[p, :rank]^T is split over kCholParts
// thread groups per row block (coalesced over rows, fixed-order reduction).
constexpr int kCholRows = 64, kCholParts = 8;
__global__ void __launch_bounds__(kCholRows * kCholParts) chol_step_dev_kernel(int64_t n, double max0, double neg_tol,
                                                                               int nb, int np,
                                                                               const int* __restrict__ fstart,
                                                                               const double* __restrict__ pw,
                                                                               const double* __restrict__ z,
                                                                               double* __restrict__ L,
                                                                               double* __restrict__ diag,
                                                                               CholState* st) {
  if (st->done) return;
  __shared__ double part[kCholParts][kCholRows];
  const int row = threadIdx.x % kCholRows, grp = threadIdx.x / kCholRows;
  const int64_t i = blockIdx.x * static_cast<int64_t>(kCholRows) + row;
  const int rank = st->rank, p = st->piv;
  double acc = 0.0;
  if (i < n)
    for (int r = grp; r < rank; r += kCholParts) acc += L[i + n * r] * L[p + n * r];
  part[grp][row] = acc;
  __syncthreads();
  if (grp == 0 && i < n) {
    double dd = 0.0;
    for (int g = 0; g < kCholParts; ++g) dd += part[g][row];
    const double piv = sqrt(st->dmax);
    const double c = contract_at(static_cast<int>(i), nb, np, fstart, pw, z) - dd;
    double l = c / piv;
    if (i == p) l = piv;
    L[i + n * rank] = l;
    double d = diag[i] - l * l;
    if (i == p) d = 0.0;
    if (d < 0.0) {
      if (d < -neg_tol * max0) atomicOr(st->flags + 1, 1);
      d = 0.0;
      atomicOr(st->flags, 1);
    }
    diag[i] = d;
  }
  __syncthreads();  // every thread of this CTA has read st->rank
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&st->arrived, 1u) == gridDim.x - 1) {  // last CTA: all reads of the rank are done
      st->arrived = 0;
      st->rank += 1;
    }
  }
}

// y_ax[q + r k] = (M_k v)[q] with v = V_ax[j, :] (the pivot term's row): grid (K, 3)
__global__ void chol_y_kernel(int64_t np2, int K, const int* __restrict__ rr, const double* const* __restrict__ V,
                              const double* const* __restrict__ Ms, const CholState* st, double* const* __restrict__ Y) {
  if (st->done) return;
  const int k = blockIdx.x, ax = blockIdx.y, r = rr[ax];
  extern __shared__ double vsh[];
  const double* Va = V[ax];
  for (int q = threadIdx.x; q < r; q += blockDim.x) vsh[q] = Va[st->j + np2 * q];
  __syncthreads();
  const double* M = Ms[ax];
  const int64_t ld = static_cast<int64_t>(r) * K;
  for (int a = threadIdx.x; a < r; a += blockDim.x) {
    double acc = 0.0;
#pragma unroll 16
    for (int b = 0; b < r; ++b) acc += M[(a + static_cast<int64_t>(r) * k) + ld * b] * vsh[b];
    Y[ax][a + static_cast<int64_t>(r) * k] = acc;
  }
}

// z[i] = (init ? 0 : z[i]) + w sum_k prod_ax <V_ax[i, :], y_ax[:, k]>   (b_prim_column, tei.cpp:33-44,
// and the contraction-weighted accumulation of tei.cpp:166-170), rows split over CTAs, the K columns of
// each row over thread groups; products summed in k order.
constexpr int kCD_COLS = 48;  // K <= 48 kernel columns: six n8 tiles
__device__ __forceinline__ void dmma_cd(double (&c)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b0));
}

// The same column on the FP64 tensor cores (mma.sync m16n8k4 f64): one m16
// row tile per CTA, the three axes on separate warps (warp w: axis w / 2, n8
// tiles 3 (w & 1) .. + 2, K zero-padded to 48).  A and B fragments come
// straight from L2/L1 — no shared-memory staging round trips, no barrier
// before the MMAs (a 32-row CTA staging V and y in shared memory measured 44
// vs 14.5 us per column at config 3); the axis products meet in shared
// memory and the row sums reduce in a fixed order (lanes t, tiles, warps).
constexpr int kCD2_THREADS = 192;
// One 16-row tile (rows i0 .. i0 + 15) of the column; COHERENT: y was written
// earlier in the same (cooperative) grid, so it is read through L2 only.
template <bool COHERENT>
__device__ __forceinline__ void col_dmma_tile(int64_t np2, int K, const int* __restrict__ rr,
                                              const double* const* __restrict__ V, const double* const* Y,
                                              int64_t i0, int init, double w, double* __restrict__ z,
                                              double (&part)[2][16][kCD_COLS + 1], double (&red)[2][16][2]) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int ax = warp >> 1, nt0 = (warp & 1) * 3;
  const int r = rr[ax];
  const double* __restrict__ Va = V[ax];
  const double* Ya = Y[ax];
  const bool in0 = i0 + g < np2, in1 = i0 + g + 8 < np2;
  const double* va = Va + i0 + g;
  int64_t yb[3];
  bool cin[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int col = (nt0 + j) * 8 + g;
    cin[j] = col < K;
    yb[j] = static_cast<int64_t>(r) * col;
  }
  double acc[3][4];
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[j][c] = 0.0;
#pragma unroll 4
  for (int k4 = 0; k4 < r; k4 += 4) {
    const int q = k4 + t;
    const bool qin = q < r;
    const int64_t vq = np2 * q;
    const double a0 = (qin && in0) ? __ldg(va + vq) : 0.0;
    const double a1 = (qin && in1) ? __ldg(va + vq + 8) : 0.0;
    double b[3];
#pragma unroll
    for (int j = 0; j < 3; ++j)
      b[j] = (qin && cin[j]) ? (COHERENT ? __ldcg(Ya + q + yb[j]) : __ldg(Ya + q + yb[j])) : 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) dmma_cd(acc[j], a0, a1, b[j]);
  }
  // fragment (j, c): row g + 8 (c >= 2), column (nt0 + j) 8 + 2t + (c & 1)
  if (ax > 0) {
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) part[ax - 1][g + 8 * (c >> 1)][(nt0 + j) * 8 + 2 * t + (c & 1)] = acc[j][c];
  }
  __syncthreads();
  if (ax == 0) {
    double rs[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int row = g + 8 * h, col = (nt0 + j) * 8 + 2 * t;
        const double p0 = acc[j][2 * h] * part[0][row][col] * part[1][row][col];
        const double p1 = acc[j][2 * h + 1] * part[0][row][col + 1] * part[1][row][col + 1];
        v += p0 + p1;
      }
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      rs[h] = v;
    }
    if (t == 0) {
      red[warp][g][0] = rs[0];
      red[warp][g][1] = rs[1];
    }
  }
  __syncthreads();
  if (tid < 16) {
    const int hh = tid >> 3, gg = tid & 7;
    const double sum = red[0][gg][hh] + red[1][gg][hh];  // n tiles 0-2, then 3-5
    const int64_t i = i0 + tid;
    if (i < np2) z[i] = init ? w * sum : (w != 0.0 ? (COHERENT ? __ldcg(z + i) : z[i]) + w * sum : z[i]);
  }
  __syncthreads();  // part / red reusable
}

__global__ void __launch_bounds__(kCD2_THREADS) chol_col_dmma_kernel(int64_t np2, int K, const int* __restrict__ rr,
                                                                     const double* const* __restrict__ V,
                                                                     const double* const* __restrict__ Y,
                                                                     const CholState* st, int init,
                                                                     double* __restrict__ z) {
  if (st->done) return;
  __shared__ double part[2][16][kCD_COLS + 1];  // axes 1 and 2: [row][col] of the 16 x 48 tile
  __shared__ double red[2][16][2];
  col_dmma_tile<false>(np2, K, rr, V, Y, blockIdx.x * 16LL, init, st->w, z, part, red);
}

// ---- The whole TEI pivoted Cholesky (tei.cpp:198-204 with pivoted_cholesky
// :48-90) as ONE cooperative grid: per step, every CTA reduces the previous
// step's (argmax, flags) partials itself in a fixed order (identical pivot and
// stop decisions everywhere), the grid gathers y_k (rows of the stored
// V M_k^T), forms the column with the DMMA tiles, then downdates its rows of
// L and the diagonal with the contraction inline — three grid barriers per
// step and no host or graph launches in the loop.  The per-row arithmetic is
// chol_col_dmma_kernel's and chol_step_dev_kernel's, in the same order, so L,
// the pivots and R_B are those of the graph-replayed loop.
struct TeiCoopArgs {
  int64_t np2;
  int nb, np, K, cap, max_terms;
  int r[3];
  const double* V[3];
  const double* Pk[3];
  double* Y[3];
  const int* fstart;
  const double* pw;
  double *z, *L, *diag;
  int64_t* piv_list;
  double target, max0, neg_tol;
  double4* part;  // [2][gridDim]
  CholState* st;  // out: rank, done, flags[1]
  unsigned long long* phase;  // analysis (TGB_PHASE_CLK): CTA 0's cycles in gather / column / downdate / reduce
};
constexpr int kTC_ROWS = kCD2_THREADS / kCholParts;  // 24 downdate rows per pass
__global__ void __launch_bounds__(kCD2_THREADS, 3) tei_chol_coop_kernel(TeiCoopArgs A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double tpart[2][16][kCD_COLS + 1];
  __shared__ double tred[2][16][2];
  __shared__ double dpart[kCholParts][kTC_ROWS];
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ int s_rank, s_p, s_done, s_err, s_j;
  __shared__ double s_dm, s_w;
  const int tid = threadIdx.x, nblk = gridDim.x;
  const int64_t n = A.nb * static_cast<int64_t>(A.nb);
  const int64_t np2 = A.np2;
  const int ntiles = static_cast<int>((np2 + 15) / 16);
  const int64_t gthreads = static_cast<int64_t>(nblk) * blockDim.x;
  // partial argmax of the initial diagonal
  {
    double lm = -INFINITY;
    int li = 0x7fffffff;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + tid; i < n; i += gthreads)
      argmax_combine(lm, li, A.diag[i], static_cast<int>(i));
    block_argmax(lm, li, sv, si);
    if (tid == 0) A.part[blockIdx.x] = make_double4(lm, static_cast<double>(li), 0.0, 0.0);
  }
  grid.sync();
  if (tid < 32) {
    double dm, ds;
    int p, fl;
    coop_reduce(A.part, nblk, dm, p, ds, fl);
    if (tid == 0) {
      s_rank = 0;
      s_err = 0;
      s_dm = dm;
      s_p = p;
      s_done = A.cap <= 0 || dm <= A.target || dm <= 0.0;  // chol_pivot_kernel's stop rule
    }
  }
  __syncthreads();
  for (int step = 1;; ++step) {
    if (s_done) break;
    const int buf = step & 1;
    const int rank = s_rank, pp = s_p;
    if (blockIdx.x == 0 && tid == 0) A.piv_list[rank] = pp;
    for (int t = 0; t < A.max_terms; ++t) {
      __syncthreads();  // s_w / s_j of the previous term read
      if (tid == 0) {  // chol_term
        const int kappa = pp % A.nb, lambda = pp / A.nb;
        const int nk = A.fstart[kappa + 1] - A.fstart[kappa], nl = A.fstart[lambda + 1] - A.fstart[lambda];
        if (t >= nk * nl) {
          s_w = 0.0;
        } else {
          const int p = A.fstart[kappa] + t % nk, q = A.fstart[lambda] + t / nk;
          s_j = p + A.np * q;
          s_w = A.pw[p] * A.pw[q];
        }
      }
      __syncthreads();
      const double w = s_w;
      if (w == 0.0) continue;  // grid-uniform: no term, z unchanged
      const int64_t j = s_j;
      long long c0 = A.phase ? clock64() : 0;
      // y_ax[e] = Pk_ax[j + np2 e], e < r_ax K, spread over the grid
      for (int ax = 0; ax < 3; ++ax) {
        const int64_t cnt = static_cast<int64_t>(A.r[ax]) * A.K;
        const double* src = A.Pk[ax] + j;
        for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + tid; e < cnt; e += gthreads)
          A.Y[ax][e] = __ldg(src + np2 * e);
      }
      grid.sync();
      long long c1 = A.phase ? clock64() : 0;
      for (int mt = blockIdx.x; mt < ntiles; mt += nblk)
        col_dmma_tile<true>(np2, A.K, A.r, A.V, A.Y, mt * 16LL, t == 0 ? 1 : 0, w, A.z, tpart, tred);
      grid.sync();
      if (A.phase && blockIdx.x == 0 && tid == 0) {
        A.phase[0] += static_cast<unsigned long long>(c1 - c0);
        A.phase[1] += static_cast<unsigned long long>(clock64() - c1);
      }
    }
    long long c2 = A.phase ? clock64() : 0;
    // downdate (chol_step_dev_kernel's arithmetic): rows in passes of kTC_ROWS, kCholParts partial sums each
    const double piv = sqrt(s_dm);
    double lm = -INFINITY;
    int li = 0x7fffffff, bad = 0, cl = 0;
    const int row = tid % kTC_ROWS, grp = tid / kTC_ROWS;
    for (int64_t r0 = blockIdx.x * static_cast<int64_t>(kTC_ROWS); r0 < n; r0 += static_cast<int64_t>(nblk) * kTC_ROWS) {
      const int64_t i = r0 + row;
      double acc = 0.0;
      if (i < n) {
        // the same r order as chol_step_dev_kernel; loads issued 8 terms at a time
        int r = grp;
        for (; r + 7 * kCholParts < rank; r += 8 * kCholParts) {
          double lv[8], pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            lv[u] = __ldcg(A.L + i + n * (r + u * kCholParts));
            pv[u] = __ldcg(A.L + pp + n * (r + u * kCholParts));
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) acc += lv[u] * pv[u];
        }
        for (; r < rank; r += kCholParts) acc += __ldcg(A.L + i + n * r) * __ldcg(A.L + pp + n * r);
      }
      dpart[grp][row] = acc;
      __syncthreads();
      if (grp == 0 && i < n) {
        double dd = 0.0;
        for (int g2 = 0; g2 < kCholParts; ++g2) dd += dpart[g2][row];
        const double c = contract_at<true>(static_cast<int>(i), A.nb, A.np, A.fstart, A.pw, A.z) - dd;
        double l = c / piv;
        if (i == pp) l = piv;
        A.L[i + n * rank] = l;
        double d = A.diag[i] - l * l;
        if (i == pp) d = 0.0;
        if (d < 0.0) {
          if (d < -A.neg_tol * A.max0) bad = 1;
          d = 0.0;
          cl = 1;
        }
        A.diag[i] = d;
        argmax_combine(lm, li, d, static_cast<int>(i));
      }
      __syncthreads();
    }
    bad = __syncthreads_or(bad);
    cl = __syncthreads_or(cl);
    block_argmax(lm, li, sv, si);
    if (tid == 0) A.part[buf * nblk + blockIdx.x] = make_double4(lm, static_cast<double>(li), 0.0, 2.0 * bad + cl);
    long long c3 = A.phase ? clock64() : 0;
    grid.sync();
    if (A.phase && blockIdx.x == 0 && tid == 0) {
      A.phase[2] += static_cast<unsigned long long>(c3 - c2);
      A.phase[3] += static_cast<unsigned long long>(clock64() - c3);
      A.phase[4] += 1;
    }
    if (tid < 32) {
      double dm, ds;
      int p, fl;
      coop_reduce(A.part + buf * nblk, nblk, dm, p, ds, fl);
      if (tid == 0) {
        s_rank = rank + 1;
        if (fl & 2) {
          s_err = 1;
          s_done = 1;
        } else {
          s_dm = dm;
          s_p = p;
          s_done = s_rank >= A.cap || dm <= A.target || dm <= 0.0;
        }
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) {
    A.st->rank = s_rank;
    A.st->done = 1;
    A.st->flags[1] = s_err;
  }
}

__global__ void chol_col_kernel(int64_t np2, int K, int rows, const int* __restrict__ rr,
                                const double* const* __restrict__ V, const double* const* __restrict__ Y,
                                const CholState* st, int init, double* __restrict__ z) {
  if (st->done) return;
  extern __shared__ double csh[];
  const int r0 = rr[0], r1 = rr[1], r2 = rr[2];
  double* ys[3] = {csh, csh + static_cast<int64_t>(r0) * K, csh + static_cast<int64_t>(r0 + r1) * K};
  double* prod = csh + static_cast<int64_t>(r0 + r1 + r2) * K;  // rows x K
  double* vt = prod + static_cast<int64_t>(rows) * K;              // rows x r_ax tile of V_ax
  const int rax[3] = {r0, r1, r2};
  for (int ax = 0; ax < 3; ++ax)
    for (int e = threadIdx.x; e < rax[ax] * K; e += blockDim.x) ys[ax][e] = Y[ax][e];
  __syncthreads();
  const int groups = blockDim.x / rows;
  const int row = threadIdx.x % rows, grp = threadIdx.x / rows;
  const int64_t i0 = blockIdx.x * static_cast<int64_t>(rows);
  const int64_t i = i0 + row;
  constexpr int kMaxK = 8;  // K <= groups * kMaxK (host-checked)
  double p[kMaxK];
#pragma unroll
  for (int u = 0; u < kMaxK; ++u) p[u] = 1.0;
  for (int ax = 0; ax < 3; ++ax) {
    const int r = rax[ax];
    __syncthreads();  // the previous axis' tile is consumed
    for (int e = threadIdx.x; e < rows * r; e += blockDim.x) {  // coalesced: rows are contiguous in V
      const int rw = e % rows, q = e / rows;
      vt[rw + rows * q] = i0 + rw < np2 ? V[ax][i0 + rw + np2 * q] : 0.0;
    }
    __syncthreads();
    double acc[kMaxK];
#pragma unroll
    for (int u = 0; u < kMaxK; ++u) acc[u] = 0.0;
    const double* y = ys[ax];
    if (grp < groups) {
      for (int q = 0; q < r; ++q) {
        const double v = vt[row + rows * q];
#pragma unroll
        for (int u = 0; u < kMaxK; ++u) {
          const int k = grp + u * groups;
          if (k < K) acc[u] += v * y[q + r * k];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kMaxK; ++u) p[u] = ax == 0 ? acc[u] : p[u] * acc[u];
  }
  if (grp < groups && i < np2) {
#pragma unroll
    for (int u = 0; u < kMaxK; ++u) {
      const int k = grp + u * groups;
      if (k < K) prod[row + rows * k] = p[u];
    }
  }
  __syncthreads();
  if (grp == 0 && i < np2) {
    double sum = 0.0;
    for (int k = 0; k < K; ++k) sum += prod[row + rows * k];
    const double w = st->w;
    z[i] = init ? w * sum : (w != 0.0 ? z[i] + w * sum : z[i]);
  }
}

// y_ax[q + r k] = Pk_ax[j + np2 (q + r k)] = (M_k V_ax[j, :]^T)[q]   (grid: 3 axes)
__global__ void chol_ygather_kernel(int64_t np2, int K, const int* __restrict__ rr,
                                    const double* const* __restrict__ Pk, const CholState* st,
                                    double* const* __restrict__ Y) {
  if (st->done) return;
  const int ax = blockIdx.y;
  const int64_t cnt = static_cast<int64_t>(rr[ax]) * K;
  const double* src = Pk[ax] + st->j;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < cnt;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    Y[ax][e] = src[np2 * e];
}


}  // namespace

// ---------------------------------------------------------------- host orchestration

struct TEI {
  int64_t nb = 0, np = 0;
  std::vector<int> fstart;  // primitives of function f: fstart[f] .. fstart[f+1]-1
  std::vector<double> pw;   // primitive weights
  std::array<int64_t, 3> n{};
  std::array<double, 3> h{};
  std::array<int64_t, 3> R{};
  std::array<DevBuf, 3> U, V, M, Mst;  // M: R x (R K) = [M_0 | M_1 | ...]; Mst: (R K) x R stacked
  int64_t K = 0;
  std::array<double, 3> fit_res{};
  bool fit_clamped = false;
  DevBuf L, diag;
  int64_t RB = 0;
  std::vector<int64_t> chol_piv;
  DevBuf d_fstart, d_pw, d_cstart, d_cpairs, d_cw;
  // pivoted-Cholesky column engine: Pk[ax] = [V M_0^T | ... | V M_{K-1}^T] (np^2 x r K),
  // formed by the diagonal pass and kept when it fits (row j gives y_k = M_k V[j, :]^T)
  std::array<DevBuf, 3> Pk;
  bool have_pk = false;
};

}  // namespace tgb

struct tgb_tei {
  tgb::TEI t;
};

namespace tgb {

static double* dptr(DevBuf& b) { return static_cast<double*>(b.p); }

void tei_fit(tgb_ctx* ctx, TEI& f, const tgb_cp& basis_dev, const int64_t* fn_offset, int64_t nb, const double h[3],
             double eps_fit) {
  f.nb = nb;
  f.np = basis_dev.rank;
  f.fstart.assign(fn_offset, fn_offset + nb + 1);
  f.pw.resize(f.np);
  if (f.np) TGB_CUDA(cudaMemcpy(f.pw.data(), basis_dev.weight, f.np * sizeof(double), cudaMemcpyDeviceToHost));
  const int64_t np = f.np, np2 = np * np;
  // phase 1: per axis G (n x np^2, column p + np q = g_p .* g_q) and its Gram GG^T as the elementwise
  // square of F F^T (n x n x np instead of n x n x np^2 flops; tei.cpp:118-124)
  std::array<DevBuf, 3>& gbuf = ctx_buf3(ctx, "tei1110.gbuf");
  std::array<DevBuf, 3>& grambuf = ctx_buf3(ctx, "tei1110.grambuf");
  std::array<DevBuf, 3>& lbuf = ctx_buf3(ctx, "tei1110.lbuf");
  std::array<DevBuf, 3>& smallbuf = ctx_buf3(ctx, "tei1110.smallbuf");  // per context
  std::array<double*, 3> G{}, gram{}, Lw{}, dg{}, resid{};
  std::array<int*, 3> piv{}, info{};
  std::array<int64_t, 3> cap{};
  PivBatch pb{};
  for (int ax = 0; ax < 3; ++ax) {
    const int64_t n = basis_dev.n[ax];
    f.n[ax] = n;
    f.h[ax] = h[ax];
    G[ax] = static_cast<double*>(gbuf[ax].get(std::max<int64_t>(1, n * np2) * sizeof(double)));
    dim3 g1(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 64)), static_cast<unsigned>(np2));
    gprod_kernel<<<g1, 256, 0, ctx->stream>>>(n, static_cast<int>(np), basis_dev.factor[ax], G[ax]);
    TGB_LAUNCHED(ctx);
    gram[ax] = static_cast<double*>(grambuf[ax].get(std::max<int64_t>(1, n * n) * sizeof(double)));
    dgemm(ctx, false, true, n, n, np, 1.0, basis_dev.factor[ax], n, basis_dev.factor[ax], n, 0.0, gram[ax], n);
    square_kernel<<<static_cast<unsigned>(std::min<int64_t>((n * n + 255) / 256, 4096)), 256, 0, ctx->stream>>>(
        n * n, gram[ax]);
    TGB_LAUNCHED(ctx);
    cap[ax] = std::min(n, np2);
    Lw[ax] = static_cast<double*>(lbuf[ax].get(static_cast<size_t>(n) * std::max<int64_t>(cap[ax], 1) * sizeof(double)));
    auto* sm = static_cast<double*>(smallbuf[ax].get((n + 64 + std::max<int64_t>(cap[ax], 1)) * sizeof(double)));
    dg[ax] = sm;
    info[ax] = reinterpret_cast<int*>(sm + n);
    resid[ax] = sm + n + 4;
    piv[ax] = reinterpret_cast<int*>(sm + n + 8);
    pb.ax[ax] = PivAxis{static_cast<int>(n), static_cast<int>(cap[ax]), gram[ax], dg[ax], Lw[ax], resid[ax], piv[ax],
                        info[ax]};
  }
  // phase 2: the three pivoted Choleskys (tei.cpp:125-129, trace stop at eps_fit^2) concurrently
  {
    int nmax = 1, capmax = 1;
    for (int ax = 0; ax < 3; ++ax) {
      nmax = std::max(nmax, pb.ax[ax].n);
      capmax = std::max(capmax, pb.ax[ax].cap);
    }
    const size_t lp_bytes = static_cast<size_t>(capmax) * sizeof(double);
    int per_sm = 0;
    TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pivchol_coop3_kernel, kCoopThreads, lp_bytes));
    int G = std::min<int>(ctx->num_sms / 3, (nmax + 63) / 64);
    if (lp_bytes <= 48 * 1024 && per_sm >= 1 && G >= 2 && !getenv("TGB_FIT_SINGLE_CTA")) {
      auto* part = static_cast<double4*>(ctx->ws_misc2.get(static_cast<size_t>(2 * 3 * G) * sizeof(double4)));
      double tol2 = eps_fit * eps_fit, neg = 1e-12;
      int trace = 1;
      void* args[] = {&pb, &G, &tol2, &trace, &neg, &part};
      TGB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(pivchol_coop3_kernel), dim3(3 * G),
                                           dim3(kCoopThreads), args, lp_bytes, ctx->stream));
    } else {
      pivchol_explicit3_kernel<<<3, kRedThreads, 0, ctx->stream>>>(pb, eps_fit * eps_fit, 1, 1e-12);
    }
    TGB_LAUNCHED(ctx);
  }
  int hinfo[3][4];
  for (int ax = 0; ax < 3; ++ax)
    TGB_CUDA(cudaMemcpyAsync(hinfo[ax], info[ax], 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int ax = 0; ax < 3; ++ax)
    if (hinfo[ax][2]) throw Error(TGB_NUMERICAL_ERROR, "tei_density_fitting: Gram matrix indefinite beyond tolerance");
  // phase 3: per axis U = Q of the factor, V = G^T U, residual (tei.cpp:130-142)
  for (int ax = 0; ax < 3; ++ax) {
    const int64_t n = f.n[ax];
    f.fit_clamped = f.fit_clamped || hinfo[ax][1];
    const int64_t r = hinfo[ax][0];
    f.R[ax] = r;
    f.U[ax].get(std::max<int64_t>(1, n * r) * sizeof(double));
    f.V[ax].get(std::max<int64_t>(1, np2 * r) * sizeof(double));
    if (r > 0) {
      // U = orthonormal basis of span(L) (tei.cpp:136-138), GEMM-based Cholesky-QR
      TGB_CUDA(cudaMemcpyAsync(dptr(f.U[ax]), Lw[ax], static_cast<size_t>(n) * r * sizeof(double),
                               cudaMemcpyDeviceToDevice, ctx->stream));
      orthonormalize_columns(ctx, n, static_cast<int>(r), dptr(f.U[ax]));
      dgemm(ctx, true, false, np2, r, n, 1.0, G[ax], n, dptr(f.U[ax]), n, 0.0, dptr(f.V[ax]), np2);
    }
    // residual ||G - U V^T|| / ||G||  (T reuses the Gram buffer when large enough)
    auto* T = static_cast<double*>(grambuf[ax].get(std::max(static_cast<size_t>(n) * n, static_cast<size_t>(n) * np2) *
                                                   sizeof(double)));
    if (r > 0)
      dgemm(ctx, false, true, n, np2, r, 1.0, dptr(f.U[ax]), n, dptr(f.V[ax]), np2, 0.0, T, n);
    else
      TGB_CUDA(cudaMemsetAsync(T, 0, static_cast<size_t>(n) * np2 * sizeof(double), ctx->stream));
    const int nblk = 256;
    auto* part = static_cast<double*>(ctx->ws_misc2.get(2 * nblk * sizeof(double)));
    resid_kernel<<<nblk, 256, 0, ctx->stream>>>(n * np2, G[ax], T, part);
    TGB_LAUNCHED(ctx);
    std::vector<double> hp(2 * nblk);
    TGB_CUDA(cudaMemcpyAsync(hp.data(), part, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    double a = 0, b = 0;
    for (int i = 0; i < nblk; ++i) {
      a += hp[2 * i];
      b += hp[2 * i + 1];
    }
    f.fit_res[ax] = std::sqrt(a) / std::max(std::sqrt(b), 1e-300);
  }
}

void tei_conv(tgb_ctx* ctx, TEI& f, const tgb_cp& kernel_dev) {
  f.K = kernel_dev.rank;
  for (int ax = 0; ax < 3; ++ax) {
    require(kernel_dev.n[ax] == f.n[ax], "tei_convolution_matrices: kernel grid mismatch");
    const int64_t n = f.n[ax], r = f.R[ax], K = f.K;
    f.M[ax].get(std::max<int64_t>(1, r * r * K) * sizeof(double));
    if (r == 0 || K == 0) continue;
    // conv columns: column i + r k = h * window(conv(U_i, p_k))   (tei.cpp:153-154)
    auto* co = static_cast<double*>(ctx->ws_out.get(static_cast<size_t>(n) * r * K * sizeof(double)));
    if (ctx->comm_size > 1) {
      // multi-GPU: this rank convolves its block of kernel-term PAIRS {j, K-1-j} (the +-t
      // sinc nodes stay together, so duplicates are still convolved once); the other
      // terms' columns are zero, the full-size GEMM below then gives this rank's M_k
      // blocks bit-identical to one process and zeros elsewhere, and one all-reduce of
      // M completes it
      const int64_t npair = (K + 1) / 2;
      int64_t p0 = 0, p1 = 0;
      shard_range(npair, ctx->comm_rank, ctx->comm_size, &p0, &p1);
      std::vector<int64_t> ks;
      for (int64_t j = p0; j < p1; ++j) {
        ks.push_back(j);
        if (K - 1 - j != j) ks.push_back(K - 1 - j);
      }
      std::sort(ks.begin(), ks.end());
      TGB_CUDA(cudaMemsetAsync(co, 0, static_cast<size_t>(n) * r * K * sizeof(double), ctx->stream));
      if (!ks.empty()) {
        const int64_t S = static_cast<int64_t>(ks.size());
        auto* ksub = static_cast<double*>(ctx_buf(ctx, "tei.conv.ksub").get(static_cast<size_t>(n) * S * sizeof(double)));
        auto* csub = static_cast<double*>(ctx_buf(ctx, "tei.conv.csub").get(static_cast<size_t>(n) * r * S * sizeof(double)));
        for (int64_t s2 = 0; s2 < S; ++s2)
          TGB_CUDA(cudaMemcpyAsync(ksub + n * s2, kernel_dev.factor[ax] + n * ks[s2], n * sizeof(double),
                                   cudaMemcpyDeviceToDevice, ctx->stream));
        convolve_axis(ctx, n, r, dptr(f.U[ax]), S, ksub, f.h[ax], csub);
        for (int64_t s2 = 0; s2 < S; ++s2)
          TGB_CUDA(cudaMemcpyAsync(co + n * r * ks[s2], csub + n * r * s2, static_cast<size_t>(n) * r * sizeof(double),
                                   cudaMemcpyDeviceToDevice, ctx->stream));
      }
    } else {
      convolve_axis(ctx, n, r, dptr(f.U[ax]), K, kernel_dev.factor[ax], f.h[ax], co);
    }
    // [M_0 | ... | M_{K-1}] = U^T [conv_0 | ...]   (tei.cpp:155)
    dgemm(ctx, true, false, r, r * K, n, 1.0, dptr(f.U[ax]), n, co, n, 0.0, dptr(f.M[ax]), r);
    if (ctx->comm_size > 1) comm_allreduce(ctx, dptr(f.M[ax]), r * r * K, true);
    f.Mst[ax].get(std::max<int64_t>(1, r * r * K) * sizeof(double));
    stack_kernel<<<static_cast<unsigned>((r * r * K + 255) / 256), 256, 0, ctx->stream>>>(
        static_cast<int>(r), static_cast<int>(K), dptr(f.M[ax]), dptr(f.Mst[ax]));
    TGB_LAUNCHED(ctx);
  }
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
}

static void ensure_contraction_tables(tgb_ctx* ctx, TEI& f) {
  // contracted pair c = mu + nb nu -> primitive pairs (p + np q) with weights pw[p] pw[q]
  if (f.d_cstart.p) return;
  const int64_t nb = f.nb, np = f.np;
  std::vector<int> cstart(nb * nb + 1, 0), cpairs;
  std::vector<double> cw;
  // (mu, nu) with mu > nu lists the mirrored primitive pairs of (nu, mu) in the
  // same order, so symmetric entries are bitwise equal and exact ties in the
  // pivot search resolve to the first index (tei.cpp:66 semantics).
  for (int64_t nu = 0; nu < nb; ++nu)
    for (int64_t mu = 0; mu < nb; ++mu) {
      const int64_t c = mu + nb * nu;
      const int64_t a = std::min(mu, nu), b = std::max(mu, nu);
      for (int p = f.fstart[a]; p < f.fstart[a + 1]; ++p)
        for (int q = f.fstart[b]; q < f.fstart[b + 1]; ++q) {
          cpairs.push_back(static_cast<int>(mu <= nu ? p + np * q : q + np * p));
          cw.push_back(f.pw[p] * f.pw[q]);
        }
      cstart[c + 1] = static_cast<int>(cpairs.size());
    }
  auto up = [&](DevBuf& b, const void* src, size_t bytes) {
    b.get(std::max<size_t>(bytes, 16));
    if (bytes) TGB_CUDA(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  };
  up(f.d_cstart, cstart.data(), cstart.size() * sizeof(int));
  up(f.d_cpairs, cpairs.data(), cpairs.size() * sizeof(int));
  up(f.d_cw, cw.data(), cw.size() * sizeof(double));
  std::vector<int> fs(f.fstart.begin(), f.fstart.end());
  up(f.d_fstart, fs.data(), fs.size() * sizeof(int));
  up(f.d_pw, f.pw.data(), f.pw.size() * sizeof(double));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
}

// diag[c], c = mu + nb nu (device output, nb^2 entries)
void tei_diagonal_dev(tgb_ctx* ctx, TEI& f, double* diag) {
  ensure_contraction_tables(ctx, f);
  const int64_t nb = f.nb, np2 = f.np * f.np;
  const int nc = static_cast<int>(nb * nb);
  TGB_CUDA(cudaMemsetAsync(diag, 0, nc * sizeof(double), ctx->stream));
  std::array<double*, 3> Y{};
  std::array<DevBuf, 3>& ybuf = ctx_buf3(ctx, "tei1265.ybuf");  // per context
  // keep every V M_k^T for the Cholesky columns when it fits a modest budget (config 3: 0.8 GB)
  size_t pk_bytes = 0;
  for (int ax = 0; ax < 3; ++ax) pk_bytes += static_cast<size_t>(np2) * f.R[ax] * f.K * sizeof(double);
  f.have_pk = pk_bytes <= (size_t(8) << 30) && f.K > 0 && !getenv("TGB_TEI_NO_PK");
  for (int ax = 0; ax < 3; ++ax) {
    Y[ax] = static_cast<double*>(ybuf[ax].get(std::max<int64_t>(1, np2 * f.R[ax]) * sizeof(double)));
    if (f.have_pk) f.Pk[ax].get(std::max<size_t>(8, static_cast<size_t>(np2) * f.R[ax] * f.K * sizeof(double)));
  }
  if (f.have_pk) {  // every Y_k first, then all terms in one launch and a k-ordered sum
    // [Y_0 | Y_1 | ...] = V [M_0^T | M_1^T | ...] = V Mst^T: one GEMM per axis (same per-element k order
    // as one GEMM per term)
    for (int ax = 0; ax < 3; ++ax) {
      const int64_t r = f.R[ax];
      if (r == 0) continue;
      dgemm(ctx, false, true, np2, r * f.K, r, 1.0, dptr(f.V[ax]), np2, dptr(f.Mst[ax]), r * f.K, 0.0,
            dptr(f.Pk[ax]), np2);
    }
    DevBuf& sbuf = ctx_buf(ctx, "tei1283.sbuf");  // per context
    auto* sk = static_cast<double*>(sbuf.get(std::max<size_t>(8, static_cast<size_t>(f.K) * nc * sizeof(double))));
    // multi-GPU: this rank's block of pair rows, zeros elsewhere, one all-reduce (x + 0 is exact,
    // so the diagonal is bit-identical to the single-process one); Pk stays replicated (the
    // Cholesky column engine reads every row of it)
    int64_t c0 = 0, c1 = nc;
    if (ctx->comm_size > 1) shard_range(nc, ctx->comm_rank, ctx->comm_size, &c0, &c1);
    const int nrow = static_cast<int>(c1 - c0);
    if (nrow > 0) {
      tei_diag_terms_kernel<<<dim3((nrow + 127) / 128, static_cast<unsigned>(f.K)), 128, 0, ctx->stream>>>(
          nc, static_cast<int>(c0), static_cast<int>(c1), static_cast<const int*>(f.d_cstart.p),
          static_cast<const int*>(f.d_cpairs.p), static_cast<const double*>(f.d_cw.p), np2, dptr(f.V[0]),
          dptr(f.V[1]), dptr(f.V[2]), static_cast<int>(f.R[0]), static_cast<int>(f.R[1]), static_cast<int>(f.R[2]),
          dptr(f.Pk[0]), dptr(f.Pk[1]), dptr(f.Pk[2]), sk);
      TGB_LAUNCHED(ctx);
      tei_diag_sum_kernel<<<(nrow + 255) / 256, 256, 0, ctx->stream>>>(
          nc, static_cast<int>(c0), static_cast<int>(c1), static_cast<int>(f.K), sk, diag);
      TGB_LAUNCHED(ctx);
    }
    if (ctx->comm_size > 1) comm_allreduce(ctx, diag, nc, true);
    return;
  }
  for (int64_t k = 0; k < f.K; ++k) {
    for (int ax = 0; ax < 3; ++ax) {
      const int64_t r = f.R[ax];
      if (r == 0) continue;
      // Y = V M_k^T
      dgemm(ctx, false, true, np2, r, r, 1.0, dptr(f.V[ax]), np2, dptr(f.M[ax]) + r * r * k, r, 0.0, Y[ax], np2);
    }
    tei_diag_term_kernel<<<(nc + 127) / 128, 128, 0, ctx->stream>>>(
        nc, static_cast<const int*>(f.d_cstart.p), static_cast<const int*>(f.d_cpairs.p),
        static_cast<const double*>(f.d_cw.p), np2, dptr(f.V[0]), dptr(f.V[1]), dptr(f.V[2]),
        static_cast<int>(f.R[0]), static_cast<int>(f.R[1]), static_cast<int>(f.R[2]), Y[0], Y[1], Y[2], diag);
    TGB_LAUNCHED(ctx);
  }
}

// primitive-level column b_prim_column(j) (np^2, device) via three GEMMs + combine
static void b_prim_column_dev(tgb_ctx* ctx, TEI& f, int64_t j, double* col) {
  const int64_t np2 = f.np * f.np, K = f.K;
  std::array<DevBuf, 3>& wbuf = ctx_buf3(ctx, "tei1313.wbuf");
  std::array<DevBuf, 3>& ybuf = ctx_buf3(ctx, "tei1313.ybuf");
  std::array<DevBuf, 3>& vrow = ctx_buf3(ctx, "tei1313.vrow");  // per context
  std::array<double*, 3> W{};
  for (int ax = 0; ax < 3; ++ax) {
    const int64_t r = f.R[ax];
    W[ax] = static_cast<double*>(wbuf[ax].get(std::max<int64_t>(1, np2 * K) * sizeof(double)));
    auto* y = static_cast<double*>(ybuf[ax].get(std::max<int64_t>(1, r * K) * sizeof(double)));
    auto* vr = static_cast<double*>(vrow[ax].get(std::max<int64_t>(1, r) * sizeof(double)));
    if (r == 0) {
      TGB_CUDA(cudaMemsetAsync(W[ax], 0, np2 * K * sizeof(double), ctx->stream));
      continue;
    }
    gather_row_kernel<<<static_cast<unsigned>((r + 127) / 128), 128, 0, ctx->stream>>>(dptr(f.V[ax]), np2,
                                                                                      static_cast<int>(r),
                                                                                      static_cast<int>(j), vr);
    TGB_LAUNCHED(ctx);
    // Y (r x K, column k = M_k V[j, :]^T) = stacked [M_0; ...; M_{K-1}] (rK x r) * vr
    dgemm(ctx, false, false, r * K, 1, r, 1.0, dptr(f.Mst[ax]), r * K, vr, r, 0.0, y, r * K);
    // W_ax (np2 x K) = V_ax (np2 x r) Y (r x K)
    dgemm(ctx, false, false, np2, K, r, 1.0, dptr(f.V[ax]), np2, y, r, 0.0, W[ax], np2);
  }
  tei_col_combine_kernel<<<static_cast<unsigned>((np2 + 255) / 256), 256, 0, ctx->stream>>>(np2, static_cast<int>(K),
                                                                                           W[0], W[1], W[2], col);
  TGB_LAUNCHED(ctx);
}

// tei_column(pair) (nb^2, device)
void tei_column_dev(tgb_ctx* ctx, TEI& f, int64_t pair, double* out) {
  ensure_contraction_tables(ctx, f);
  const int64_t nb = f.nb, np = f.np, np2 = np * np;
  const int64_t kappa = pair % nb, lambda = pair / nb;
  DevBuf& zbuf = ctx_buf(ctx, "tei1343.zbuf");
  DevBuf& cbuf = ctx_buf(ctx, "tei1343.cbuf");  // per context
  auto* z = static_cast<double*>(zbuf.get(std::max<int64_t>(1, np2) * sizeof(double)));
  auto* c = static_cast<double*>(cbuf.get(std::max<int64_t>(1, np2) * sizeof(double)));
  // z = sum over primitive pairs (p, q) of (kappa, lambda) of w_p w_q b_prim_column(p + np q)
  bool first = true;
  for (int q = f.fstart[lambda]; q < f.fstart[lambda + 1]; ++q)
    for (int p = f.fstart[kappa]; p < f.fstart[kappa + 1]; ++p) {
      const double w = f.pw[p] * f.pw[q];
      b_prim_column_dev(ctx, f, p + np * q, c);
      axpy_kernel<<<static_cast<unsigned>((np2 + 255) / 256), 256, 0, ctx->stream>>>(np2, w, c, z, first ? 1 : 0);
      TGB_LAUNCHED(ctx);
      first = false;
    }
  // the contraction weights are applied in contract_kernel (pw[p] pw[q] on both sides)
  contract_kernel<<<static_cast<unsigned>((nb * nb + 127) / 128), 128, 0, ctx->stream>>>(
      static_cast<int>(nb), static_cast<int>(np), static_cast<const int*>(f.d_fstart.p),
      static_cast<const double*>(f.d_pw.p), z, out);
  TGB_LAUNCHED(ctx);
}

void tei_cholesky(tgb_ctx* ctx, TEI& f, double eps_chol) {
  ensure_contraction_tables(ctx, f);
  const int64_t nb = f.nb, np = f.np, nb2 = nb * nb, np2 = np * np, K = f.K;
  auto* dg = static_cast<double*>(f.diag.get(std::max<int64_t>(1, nb2) * sizeof(double)));
  tei_diagonal_dev(ctx, f, dg);
  f.L.get(std::max<int64_t>(1, nb2 * nb2) * sizeof(double));
  double* L = dptr(f.L);
  DevBuf& zbuf = ctx_buf(ctx, "tei1370.zbuf");
  DevBuf& cbuf = ctx_buf(ctx, "tei1370.cbuf");
  DevBuf& stbuf = ctx_buf(ctx, "tei1370.stbuf");
  DevBuf& pivbuf = ctx_buf(ctx, "tei1370.pivbuf");  // per context
  std::array<DevBuf, 3>& wbuf = ctx_buf3(ctx, "tei1371.wbuf");
  std::array<DevBuf, 3>& ybuf = ctx_buf3(ctx, "tei1371.ybuf");
  std::array<DevBuf, 3>& vrow = ctx_buf3(ctx, "tei1371.vrow");  // per context
  auto* z = static_cast<double*>(zbuf.get(std::max<int64_t>(1, np2) * sizeof(double)));
  auto* cc = static_cast<double*>(cbuf.get(std::max<int64_t>(1, np2) * sizeof(double)));
  auto* st = static_cast<CholState*>(stbuf.get(sizeof(CholState)));
  auto* piv = static_cast<int64_t*>(pivbuf.get(std::max<int64_t>(1, nb2) * sizeof(int64_t)));
  std::array<double*, 3> W{}, Y{}, VR{};
  for (int ax = 0; ax < 3; ++ax) {
    W[ax] = static_cast<double*>(wbuf[ax].get(std::max<int64_t>(1, np2 * K) * sizeof(double)));
    Y[ax] = static_cast<double*>(ybuf[ax].get(std::max<int64_t>(1, f.R[ax] * K) * sizeof(double)));
    VR[ax] = static_cast<double*>(vrow[ax].get(std::max<int64_t>(1, f.R[ax]) * sizeof(double)));
  }
  // max0 of the initial diagonal (host: it fixes the stop target)
  double hv[2];
  {
    auto* sm = static_cast<double*>(cbuf.p);
    argmax_kernel<<<1, kRedThreads, 0, ctx->stream>>>(static_cast<int>(nb2), dg, sm, reinterpret_cast<int*>(sm + 1));
    TGB_LAUNCHED(ctx);
    TGB_CUDA(cudaMemcpyAsync(hv, sm, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  const double max0 = hv[0];
  f.chol_piv.clear();
  f.RB = 0;
  if (!(max0 > 0.0)) return;
  const double target = eps_chol * max0;  // max-diagonal stop (tei.cpp:202)
  const int cap = static_cast<int>(nb2);
  int max_terms = 1;  // primitive pairs per contracted pair, at most
  for (int64_t a = 0; a < nb; ++a)
    for (int64_t b = 0; b < nb; ++b)
      max_terms = std::max<int>(max_terms, (f.fstart[a + 1] - f.fstart[a]) * (f.fstart[b + 1] - f.fstart[b]));
  CholState h0{};
  TGB_CUDA(cudaMemcpyAsync(st, &h0, sizeof(CholState), cudaMemcpyHostToDevice, ctx->stream));
  // fused column path: the three y_ax (r_ax x K) and a rows x K product tile in shared memory
  DevBuf& ptrbuf = ctx_buf(ctx, "tei1404.ptrbuf");  // per context
  const int64_t rmax = std::max({f.R[0], f.R[1], f.R[2], int64_t(1)});
  int col_rows = static_cast<int>(std::min<int64_t>(96, std::max<int64_t>(8, (np2 + ctx->num_sms - 1) / ctx->num_sms)));
  const int col_groups = std::max(1, std::min(8, 1024 / col_rows));
  const size_t col_smem =
      static_cast<size_t>((f.R[0] + f.R[1] + f.R[2] + col_rows) * K + col_rows * rmax) * sizeof(double);
  const bool fused_col = col_smem <= ctx->smem_optin - 1024 && K <= 8 * col_groups &&
                         !getenv("TGB_TEI_GEMM_COLUMN") && K > 0;
  // DMMA column kernel for K <= 48 kernel columns (config 3: 14.5 us per column vs 64 us SIMT)
  const bool dmma_col = fused_col && K <= kCD_COLS && !getenv("TGB_TEI_SIMT_COLUMN");
  const double** dV = nullptr;
  const double** dM = nullptr;
  double** dY = nullptr;
  const double* const* dYc = nullptr;
  const int* dr = nullptr;
  const double* const* dPk = nullptr;
  if (fused_col) {
    static bool attr[kTgbMaxDevices] = {};  // per device
    if (!attr[ctx->device]) {
      TGB_CUDA(cudaFuncSetAttribute(chol_col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(ctx->smem_optin - 1024)));
      attr[ctx->device] = true;
    }
    struct Ptrs {
      const double* V[3];
      const double* M[3];
      double* Y[3];
      const double* P[3];
      int r[4];
    } hp{};
    for (int ax = 0; ax < 3; ++ax) {
      hp.V[ax] = dptr(f.V[ax]);
      hp.M[ax] = dptr(f.Mst[ax]);
      hp.Y[ax] = Y[ax];
      hp.P[ax] = f.have_pk ? dptr(f.Pk[ax]) : nullptr;
      hp.r[ax] = static_cast<int>(f.R[ax]);
    }
    auto* dp = static_cast<Ptrs*>(ptrbuf.get(sizeof(Ptrs)));
    TGB_CUDA(cudaMemcpyAsync(dp, &hp, sizeof(Ptrs), cudaMemcpyHostToDevice, ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));  // hp leaves scope
    dV = const_cast<const double**>(dp->V);
    dM = const_cast<const double**>(dp->M);
    dY = dp->Y;
    dYc = dp->Y;
    dr = dp->r;
    dPk = const_cast<const double**>(dp->P);
  }
  const unsigned gnp = static_cast<unsigned>((np2 + 255) / 256);
  auto step = [&]() {
    chol_pivot_kernel<<<1, kRedThreads, 0, ctx->stream>>>(static_cast<int>(nb2), dg, target, cap, st, piv,
                                                          static_cast<int>(nb), static_cast<int>(np),
                                                          static_cast<const int*>(f.d_fstart.p),
                                                          static_cast<const double*>(f.d_pw.p));
    TGB_LAUNCHED(ctx);
    for (int t = 0; t < max_terms; ++t) {
      if (t > 0) {  // the pivot kernel formed term 0
        chol_term_kernel<<<1, 1, 0, ctx->stream>>>(static_cast<int>(nb), static_cast<int>(np), t,
                                                   static_cast<const int*>(f.d_fstart.p),
                                                   static_cast<const double*>(f.d_pw.p), st);
        TGB_LAUNCHED(ctx);
      }
      if (fused_col) {
        if (f.have_pk) {  // y_k = row j of the stored V M_k^T (the diagonal pass formed them): a gather
          chol_ygather_kernel<<<dim3(16, 3), 256, 0, ctx->stream>>>(np2, static_cast<int>(K), dr, dPk, st, dY);
          TGB_LAUNCHED(ctx);
        } else {  // y_k = M_k v
          chol_y_kernel<<<dim3(static_cast<unsigned>(K), 3), 128, rmax * sizeof(double), ctx->stream>>>(
              np2, static_cast<int>(K), dr, dV, dM, st, dY);
          TGB_LAUNCHED(ctx);
        }
        if (dmma_col) {
          chol_col_dmma_kernel<<<static_cast<unsigned>((np2 + 15) / 16), kCD2_THREADS, 0, ctx->stream>>>(
              np2, static_cast<int>(K), dr, dV, dYc, st, t == 0 ? 1 : 0, z);
        } else {
          chol_col_kernel<<<static_cast<unsigned>((np2 + col_rows - 1) / col_rows), col_rows * col_groups, col_smem,
                            ctx->stream>>>(np2, static_cast<int>(K), col_rows, dr, dV, dYc, st, t == 0 ? 1 : 0, z);
        }
        TGB_LAUNCHED(ctx);
        continue;
      }
      for (int ax = 0; ax < 3; ++ax) {  // b_prim_column (tei.cpp:33-44) for the current primitive pair
        const int64_t r = f.R[ax];
        if (r == 0) {
          TGB_CUDA(cudaMemsetAsync(W[ax], 0, np2 * K * sizeof(double), ctx->stream));
          continue;
        }
        gather_row_dev_kernel<<<static_cast<unsigned>((r + 127) / 128), 128, 0, ctx->stream>>>(
            dptr(f.V[ax]), np2, static_cast<int>(r), st, VR[ax]);
        TGB_LAUNCHED(ctx);
        dgemm(ctx, false, false, r * K, 1, r, 1.0, dptr(f.Mst[ax]), r * K, VR[ax], r, 0.0, Y[ax], r * K);
        dgemm(ctx, false, false, np2, K, r, 1.0, dptr(f.V[ax]), np2, Y[ax], r, 0.0, W[ax], np2);
      }
      tei_col_combine_kernel<<<gnp, 256, 0, ctx->stream>>>(np2, static_cast<int>(K), W[0], W[1], W[2], cc);
      TGB_LAUNCHED(ctx);
      axpy_dev_kernel<<<gnp, 256, 0, ctx->stream>>>(np2, st, cc, z, t == 0 ? 1 : 0);
      TGB_LAUNCHED(ctx);
    }
    chol_step_dev_kernel<<<static_cast<unsigned>((nb2 + kCholRows - 1) / kCholRows), kCholRows * kCholParts, 0,
                           ctx->stream>>>(nb2, max0, 1e-10, static_cast<int>(nb), static_cast<int>(np),
                                          static_cast<const int*>(f.d_fstart.p),
                                          static_cast<const double*>(f.d_pw.p), z, L, dg, st);
    TGB_LAUNCHED(ctx);
  };
  // the whole loop as one cooperative grid when the y_k come from the stored V M_k^T and the column fits
  // the DMMA tile (config 3); otherwise the graph-replayed step below
  if (dmma_col && f.have_pk && !getenv("TGB_TEI_GRAPH")) {
    int per_sm = 0;
    TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tei_chol_coop_kernel, kCD2_THREADS, 0));
    if (per_sm >= 1) {
      const int nblk = ctx->num_sms * std::min(per_sm, 3);
      TeiCoopArgs a{};
      a.np2 = np2;
      a.nb = static_cast<int>(nb);
      a.np = static_cast<int>(np);
      a.K = static_cast<int>(K);
      a.cap = cap;
      a.max_terms = max_terms;
      for (int ax = 0; ax < 3; ++ax) {
        a.r[ax] = static_cast<int>(f.R[ax]);
        a.V[ax] = dptr(f.V[ax]);
        a.Pk[ax] = dptr(f.Pk[ax]);
        a.Y[ax] = Y[ax];
      }
      a.fstart = static_cast<const int*>(f.d_fstart.p);
      a.pw = static_cast<const double*>(f.d_pw.p);
      a.z = z;
      a.L = L;
      a.diag = dg;
      a.piv_list = piv;
      a.target = target;
      a.max0 = max0;
      a.neg_tol = 1e-10;  // tei.cpp:202
      a.part = static_cast<double4*>(ctx->ws_misc3.get(static_cast<size_t>(2 * nblk) * sizeof(double4)));
      a.st = st;
      a.phase = nullptr;
      DevBuf& phbuf = ctx_buf(ctx, "tei1539.phbuf");  // per context
      if (getenv("TGB_PHASE_CLK")) {
        a.phase = static_cast<unsigned long long*>(phbuf.get(8 * sizeof(unsigned long long)));
        TGB_CUDA(cudaMemsetAsync(a.phase, 0, 8 * sizeof(unsigned long long), ctx->stream));
      }
      void* args[] = {&a};
      TGB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tei_chol_coop_kernel), dim3(nblk),
                                           dim3(kCD2_THREADS), args, 0, ctx->stream));
      TGB_LAUNCHED(ctx);
      CholState hs{};
      TGB_CUDA(cudaMemcpyAsync(&hs, st, sizeof(CholState), cudaMemcpyDeviceToHost, ctx->stream));
      TGB_CUDA(cudaStreamSynchronize(ctx->stream));
      if (a.phase) {  // analysis only
        unsigned long long h[8];
        TGB_CUDA(cudaMemcpy(h, a.phase, sizeof(h), cudaMemcpyDeviceToHost));
        const double ns = static_cast<double>(h[4] ? h[4] : 1);
        fprintf(stderr, "tei coop cycles/step (CTA 0): gather+barrier %.0f column+barrier %.0f downdate %.0f "
                "barrier+reduce wait %.0f (steps %llu)\n", h[0] / ns, h[1] / ns, h[2] / ns, h[3] / ns, h[4]);
      }
      if (hs.flags[1])
        throw Error(TGB_NUMERICAL_ERROR, "pivoted_cholesky: negative diagonal beyond tolerance; matrix not PSD");
      f.RB = hs.rank;
      f.chol_piv.resize(hs.rank);
      if (hs.rank)
        TGB_CUDA(cudaMemcpy(f.chol_piv.data(), piv, hs.rank * sizeof(int64_t), cudaMemcpyDeviceToHost));
      return;
    }
  }
  // one eager step sizes every workspace (no allocation may happen under capture)
  step();
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  const bool use_graph = !getenv("TGB_TEI_NO_GRAPH");
  int64_t per_step = 0;  // kernel launches in one step (captured, so counted per replay)
  if (use_graph) {
    const int64_t before = ctx->launches;
    TGB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    try {
      step();
    } catch (...) {
      cudaStreamEndCapture(ctx->stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    TGB_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
    TGB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    per_step = ctx->launches - before;
    ctx->launches = before;
  }
  CholState hs{};
  const int batch = 16;
  for (;;) {
    TGB_CUDA(cudaMemcpyAsync(&hs, st, sizeof(CholState), cudaMemcpyDeviceToHost, ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hs.flags[1]) {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
      throw Error(TGB_NUMERICAL_ERROR, "pivoted_cholesky: negative diagonal beyond tolerance; matrix not PSD");
    }
    if (hs.done) break;
    // a batch never needs more steps than the remaining cap
    for (int b = 0; b < batch; ++b) {
      if (exec) {
        TGB_CUDA(cudaGraphLaunch(exec, ctx->stream));
        ctx->launches += per_step;
      } else {
        step();
      }
    }
  }
  if (exec) TGB_CUDA(cudaGraphExecDestroy(exec));
  if (graph) TGB_CUDA(cudaGraphDestroy(graph));
  f.RB = hs.rank;
  f.chol_piv.resize(hs.rank);
  if (hs.rank)
    TGB_CUDA(cudaMemcpy(f.chol_piv.data(), piv, hs.rank * sizeof(int64_t), cudaMemcpyDeviceToHost));
}

// tg::pivoted_cholesky (tei.cpp:48-90) of an explicit PSD matrix on the device
// (the column callback of the reference reads columns of A).  Returns rank;
// L (n x min(n, max_rank)) and pivots device-side / host-side as documented
// in tgb.h.
int64_t pivoted_cholesky_dev(tgb_ctx* ctx, int64_t n, const double* A, double tol, bool trace_stop,
                             int64_t max_rank, double neg_tol, double* L, int64_t* pivots_host, double* residual,
                             bool* clamped) {
  const int64_t cap = std::min(n, max_rank);
  DevBuf& wbuf = ctx_buf(ctx, "tei1625.wbuf");  // per context
  auto* w = static_cast<double*>(wbuf.get((n + 64 + std::max<int64_t>(cap, 1)) * sizeof(double)));
  double* dg = w;
  int* piv = reinterpret_cast<int*>(w + n + 8);
  int* info = reinterpret_cast<int*>(w + n);
  double* res = w + n + 4;
  pivchol_explicit_kernel<<<1, kRedThreads, 0, ctx->stream>>>(static_cast<int>(n), A, tol, trace_stop ? 1 : 0,
                                                              static_cast<int>(cap), neg_tol, dg, L, piv, info, res);
  TGB_LAUNCHED(ctx);
  int hinfo[3];
  TGB_CUDA(cudaMemcpyAsync(hinfo, info, 3 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaMemcpyAsync(residual, res, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hinfo[2]) throw Error(TGB_NUMERICAL_ERROR, "pivoted_cholesky: negative diagonal beyond tolerance; matrix not PSD");
  std::vector<int> hp(std::max(hinfo[0], 1));
  if (hinfo[0]) TGB_CUDA(cudaMemcpy(hp.data(), piv, hinfo[0] * sizeof(int), cudaMemcpyDeviceToHost));
  for (int i = 0; i < hinfo[0]; ++i) pivots_host[i] = hp[i];
  *clamped = hinfo[1] != 0;
  return hinfo[0];
}

}  // namespace tgb

// ---------------------------------------------------------------- C-ABI

namespace {
struct DevCopy {
  tgb_cp t{};
  std::vector<double*> bufs;
  DevCopy(const tgb_cp* h, bool on_device) {
    t = *h;
    if (on_device) return;
    for (int ax = 0; ax < 3; ++ax) {
      double* p = nullptr;
      const size_t bytes = h->n[ax] * h->rank * sizeof(double);
      if (bytes) {
        TGB_CUDA(cudaMalloc(&p, bytes));
        TGB_CUDA(cudaMemcpy(p, h->factor[ax], bytes, cudaMemcpyHostToDevice));
      }
      t.factor[ax] = p;
      bufs.push_back(p);
    }
    double* w = nullptr;
    if (h->rank) {
      TGB_CUDA(cudaMalloc(&w, h->rank * sizeof(double)));
      TGB_CUDA(cudaMemcpy(w, h->weight, h->rank * sizeof(double), cudaMemcpyHostToDevice));
    }
    t.weight = w;
    bufs.push_back(w);
  }
  ~DevCopy() {
    for (double* p : bufs)
      if (p) cudaFree(p);
  }
};

void copy_out(double* dst, const void* src, size_t bytes, int mem) {
  if (!bytes) return;
  TGB_CUDA(cudaMemcpy(dst, src, bytes, mem == TGB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
}
}  // namespace

extern "C" {

int tgb_tei_create(tgb_tei** out) {
  return tgb::guarded_call([&] { *out = new tgb_tei(); });
}

int tgb_tei_destroy(tgb_tei* t) {
  return tgb::guarded_call([&] { delete t; });
}

int tgb_tei_density_fitting(tgb_ctx* ctx, tgb_tei* t, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb,
                            const double h[3], double eps_fit, int mem) {
  return tgb::guarded_call([&] {
    tgb::DevStreamScope scope(ctx);
    tgb::require(basis && fn_offset && nb >= 1, "tei_density_fitting: empty basis");
    tgb::require(fn_offset[0] == 0 && fn_offset[nb] == basis->rank, "tei_density_fitting: bad function offsets");
    TGB_CUDA(cudaSetDevice(ctx->device));
    DevCopy d(basis, mem == TGB_MEM_DEVICE);
    tgb::tei_fit(ctx, t->t, d.t, fn_offset, nb, h, eps_fit);
  });
}

int tgb_tei_convolution_matrices(tgb_ctx* ctx, tgb_tei* t, const tgb_cp* kernel, int mem) {
  return tgb::guarded_call([&] {
    tgb::DevStreamScope scope(ctx);
    TGB_CUDA(cudaSetDevice(ctx->device));
    DevCopy d(kernel, mem == TGB_MEM_DEVICE);
    tgb::tei_conv(ctx, t->t, d.t);
  });
}

int tgb_tei_diagonal(tgb_ctx* ctx, tgb_tei* t, double* out, int mem) {
  return tgb::guarded_call([&] {
    tgb::DevStreamScope scope(ctx);
    const int64_t nb2 = t->t.nb * t->t.nb;
    tgb::DevBuf& buf = tgb::ctx_buf(ctx, "tei1722.buf");  // per context
    auto* d = static_cast<double*>(buf.get(std::max<int64_t>(1, nb2) * sizeof(double)));
    tgb::tei_diagonal_dev(ctx, t->t, d);
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    copy_out(out, d, nb2 * sizeof(double), mem);
  });
}

int tgb_tei_column(tgb_ctx* ctx, tgb_tei* t, int64_t pair, double* out, int mem) {
  return tgb::guarded_call([&] {
    tgb::DevStreamScope scope(ctx);
    tgb::require(pair >= 0 && pair < t->t.nb * t->t.nb, "tei_column: index out of range");
    const int64_t nb2 = t->t.nb * t->t.nb;
    tgb::DevBuf& buf = tgb::ctx_buf(ctx, "tei1735.buf");  // per context
    auto* d = static_cast<double*>(buf.get(std::max<int64_t>(1, nb2) * sizeof(double)));
    tgb::tei_column_dev(ctx, t->t, pair, d);
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    copy_out(out, d, nb2 * sizeof(double), mem);
  });
}

int tgb_tei_cholesky(tgb_ctx* ctx, tgb_tei* t, double eps_chol) {
  return tgb::guarded_call([&] {
    tgb::DevStreamScope scope(ctx);
    TGB_CUDA(cudaSetDevice(ctx->device));
    tgb::tei_cholesky(ctx, t->t, eps_chol);
  });
}

int tgb_tei_info(tgb_tei* t, int64_t* info, double* fit_residual) {
  return tgb::guarded_call([&] {
    const auto& f = t->t;
    for (int ax = 0; ax < 3; ++ax) {
      info[ax] = f.R[ax];
      fit_residual[ax] = f.fit_res[ax];
    }
    info[3] = f.np;
    info[4] = f.nb;
    info[5] = f.RB;
    info[6] = f.fit_clamped;
    info[7] = f.K;
  });
}

int tgb_tei_get_fit(tgb_tei* t, int ax, double* U, double* V, int mem) {
  return tgb::guarded_call([&] {
    auto& f = t->t;
    copy_out(U, f.U[ax].p, f.n[ax] * f.R[ax] * sizeof(double), mem);
    copy_out(V, f.V[ax].p, f.np * f.np * f.R[ax] * sizeof(double), mem);
  });
}

int tgb_tei_get_conv(tgb_tei* t, int64_t k, int ax, double* M, int mem) {
  return tgb::guarded_call([&] {
    auto& f = t->t;
    tgb::require(k >= 0 && k < f.K, "tei: kernel term out of range");
    const int64_t r = f.R[ax];
    copy_out(M, static_cast<double*>(f.M[ax].p) + r * r * k, r * r * sizeof(double), mem);
  });
}

int tgb_tei_get_cholesky(tgb_tei* t, double* L, int64_t* pivots, int mem) {
  return tgb::guarded_call([&] {
    auto& f = t->t;
    const int64_t nb2 = f.nb * f.nb;
    copy_out(L, f.L.p, nb2 * f.RB * sizeof(double), mem);
    for (size_t i = 0; i < f.chol_piv.size(); ++i) pivots[i] = f.chol_piv[i];
  });
}

}  // extern "C"

// Rank reduction of canonical tensors on sm_100a (reference
// proj/src/reduction.cpp:34-273): RHOSVD, canonical-to-Tucker ALS sweeps and
// Tucker-to-canonical, with every dense product (Gram matrices, projections
// Z^T F, the ALS unfolding F C, the core projection) on the DMMA GEMM.
//
// Left singular subspaces (thin_svd_left, reduction.cpp:85-138) come from a
// two-sided blocked subspace iteration on the unfolding itself with a small
// Rayleigh-Ritz SVD per step — only the leading singular pairs the rank rule
// needs, plus the exact Frobenius norm for the tail sum.  Not forming a Gram
// matrix keeps small singular values accurate (as the reference's JacobiSVD
// branch); the reference's Gram branches have an accuracy floor ~sqrt(eps)
// (reduction.cpp:91-92), which bounds the parity of the reduced tensors.
// Rank selection (select_rank, reduction.cpp:34-59), the ALS mode order,
// early exit and the T2C unfolding rule are the reference's.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "tgb_internal.hpp"

namespace tgb {

namespace {

// ---------------------------------------------------------------- kernels

// normalize (tensor.cpp:18-31): per column k, per axis in order 0,1,2:
// nrm = ||col||; nrm > 0 ? (col /= nrm, w *= nrm) : w = 0
__global__ void normalize_kernel(int64_t n0, int64_t n1, int64_t n2, double* __restrict__ f0, double* __restrict__ f1,
                                 double* __restrict__ f2, double* __restrict__ w) {
  __shared__ double sv[32];
  const int64_t k = blockIdx.x;
  double* fs[3] = {f0 + n0 * k, f1 + n1 * k, f2 + n2 * k};
  const int64_t ns[3] = {n0, n1, n2};
  double wk = w[k];
  for (int ax = 0; ax < 3; ++ax) {
    double part = 0.0;
    for (int64_t i = threadIdx.x; i < ns[ax]; i += blockDim.x) part += fs[ax][i] * fs[ax][i];
    // block reduce
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
    if (nrm > 0.0) {
      for (int64_t i = threadIdx.x; i < ns[ax]; i += blockDim.x) fs[ax][i] /= nrm;
      wk *= nrm;
    } else {
      wk = 0.0;
    }
  }
  if (threadIdx.x == 0) w[k] = wk;
}

// out(:, k) = f(:, k) * s[k]
__global__ void scale_cols_kernel(int64_t n, int64_t R, const double* __restrict__ f, const double* __restrict__ s,
                                  double* __restrict__ out) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= n * R) return;
  out[idx] = f[idx] * s[idx / n];
}

// ALS coefficient matrix (reduction.cpp:207-216): C[k, l rm + i] = (w_k pp[l,k]) pm[i,k]   (R x rm rp)
__global__ void als_coef_kernel(int64_t R, int rm, int rp, const double* __restrict__ w, const double* __restrict__ pm,
                                const double* __restrict__ pp, double* __restrict__ C) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t tot = R * rm * rp;
  if (idx >= tot) return;
  const int64_t k = idx % R, col = idx / R;
  const int i = static_cast<int>(col % rm), l = static_cast<int>(col / rm);
  C[idx] = (w[k] * pp[l + static_cast<int64_t>(rp) * k]) * pm[i + static_cast<int64_t>(rm) * k];
}

// Khatri-Rao rows for the core projection: K[(j + r1 l), k] = w_k P1[j,k] P2[l,k]   (r1 r2 x R)
__global__ void khatri_rao_kernel(int64_t R, int r1, int r2, const double* __restrict__ w, const double* __restrict__ P1,
                                  const double* __restrict__ P2, double* __restrict__ K) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t rows = static_cast<int64_t>(r1) * r2;
  if (idx >= rows * R) return;
  const int64_t row = idx % rows, k = idx / rows;
  const int j = static_cast<int>(row % r1), l = static_cast<int>(row / r1);
  K[idx] = (w[k] * P2[l + static_cast<int64_t>(r2) * k]) * P1[j + static_cast<int64_t>(r1) * k];
}

// T2C fibres (reduction.cpp:251-264): S[i, q] = core(idx with ax = i, m1 = j1, m2 = j2), q = j1 + r_m1 j2
__global__ void t2c_slices_kernel(int r0, int r1, int r2, int ax, int m1, int m2, const double* __restrict__ core,
                                  double* __restrict__ S) {
  const int rr[3] = {r0, r1, r2};
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t tot = static_cast<int64_t>(rr[ax]) * rr[m1] * rr[m2];
  if (idx >= tot) return;
  const int i = static_cast<int>(idx % rr[ax]);
  const int64_t q = idx / rr[ax];
  const int j1 = static_cast<int>(q % rr[m1]), j2 = static_cast<int>(q / rr[m1]);
  int id[3];
  id[ax] = i;
  id[m1] = j1;
  id[m2] = j2;
  S[idx] = core[id[0] + static_cast<int64_t>(r0) * (id[1] + static_cast<int64_t>(r1) * id[2])];
}

// out(:, q) = side(:, sel(q))
__global__ void gather_cols_kernel(int64_t n, int64_t ncols, const double* __restrict__ side, int mod, int div,
                                   double* __restrict__ out) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= n * ncols) return;
  const int64_t i = idx % n, q = idx / n;
  const int64_t c = (q / div) % mod;
  out[idx] = side[i + n * c];
}

// scale every column of X (d x p) to unit norm (zero columns left as is)
__global__ void colnormalize_kernel(int64_t d, double* __restrict__ X) {
  __shared__ double sv[32];
  double* x = X + d * blockIdx.x;
  double part = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) part += x[i] * x[i];
  for (int o = 16; o; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ss = 0.0;
    for (int i = 0; i < (blockDim.x + 31) / 32; ++i) ss += sv[i];
    sv[0] = ss;
  }
  __syncthreads();
  const double nrm = sqrt(sv[0]);
  if (nrm > 0.0)
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) x[i] /= nrm;
}

__global__ void sumsq_kernel(int64_t total, const double* __restrict__ a, double* __restrict__ out) {
  __shared__ double sv[32];
  double part = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    part += a[i] * a[i];
  for (int o = 16; o; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double ss = 0.0;
    for (int i = 0; i < (blockDim.x + 31) / 32; ++i) ss += sv[i];
    out[blockIdx.x] = ss;
  }
}

// H (p x p Gram of column-normalised X, global) -> R^{-1} with H = R^T R
// (R upper), single CTA.  A column whose component orthogonal to the previous
// ones is below 1e-13 of its norm is numerically dependent (the unfolding has
// lower rank than the block): it is retired — its column of R^{-1} is zero, so
// it comes out as an exact zero column that adds no spurious singular value.
constexpr int kMaxBlock = 1024;
__global__ void chol_inv_kernel(int p, double* __restrict__ H, double* __restrict__ Wk) {
  __shared__ double s_mx;
  __shared__ unsigned char dead[kMaxBlock];
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int i = 0; i < p; ++i) mx = fmax(mx, H[i + static_cast<int64_t>(p) * i]);
    s_mx = mx;
  }
  for (int idx = threadIdx.x; idx < p * p; idx += blockDim.x) Wk[idx] = H[idx];
  __syncthreads();
  const double tiny = 1e-26 * s_mx;
  for (int j = 0; j < p; ++j) {
    if (threadIdx.x == 0) {
      const double d = Wk[j + p * j];
      dead[j] = !(d > tiny);
      Wk[j + p * j] = dead[j] ? 1.0 : sqrt(d);
    }
    __syncthreads();
    const bool dj = dead[j];
    const double djj = Wk[j + p * j];
    for (int i = j + 1 + threadIdx.x; i < p; i += blockDim.x) Wk[i + p * j] = dj ? 0.0 : Wk[i + p * j] / djj;
    __syncthreads();
    if (!dj) {
      const int m = p - j - 1;
      for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int i = j + 1 + e % m, k = j + 1 + e / m;
        if (i >= k) Wk[i + p * k] -= Wk[i + p * j] * Wk[k + p * j];
      }
    }
    __syncthreads();
  }
  // R = L^T upper; R^{-1} column c by back substitution (one thread per column)
  for (int c = threadIdx.x; c < p; c += blockDim.x) {
    for (int i = p - 1; i >= 0; --i) {
      double sum = (i == c) ? 1.0 : 0.0;
      for (int k = i + 1; k <= c; ++k) sum -= Wk[k + p * i] * H[k + p * c];
      H[i + p * c] = (i > c || dead[c]) ? 0.0 : sum / Wk[i + p * i];
    }
  }
}

// Same factorisation when L and L^{-1} both fit in shared memory (2 p^2
// doubles): right-looking Cholesky (one barrier pair per column), then
// R^{-1} = (L^{-1})^T by right-looking forward substitution over the rows of
// L^{-1}; the retired-column rule is the global-memory version's.
constexpr int kCholSmem = 128;
constexpr int kCholSmemBytes = 200 * 1024;  // L (+ L^{-1} when 2 p^2 doubles fit)
__global__ void __launch_bounds__(1024) chol_inv_smem_kernel(int p, double* __restrict__ H) {
  extern __shared__ double Ls[];  // p x p, column-major; then X = L^{-1} (p x p) when it fits
  __shared__ double s_mx;
  __shared__ unsigned char dead[kCholSmem];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int idx = threadIdx.x; idx < p * p; idx += blockDim.x) Ls[idx] = H[idx];
  __syncthreads();
  if (threadIdx.x < 32) {
    double mx = 0.0;
    for (int i = threadIdx.x; i < p; i += 32) mx = fmax(mx, Ls[i + p * i]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) s_mx = mx;
  }
  __syncthreads();
  const double tiny = 1e-26 * s_mx;
  for (int j = 0; j < p; ++j) {
    __syncthreads();                 // previous trailing update complete
    const double d = Ls[j + p * j];  // every thread reads the pivot
    const bool dj = !(d > tiny);
    const double djj = dj ? 1.0 : sqrt(d);
    const double inv = 1.0 / djj;
    for (int i = j + 1 + threadIdx.x; i < p; i += blockDim.x) Ls[i + p * j] = dj ? 0.0 : Ls[i + p * j] * inv;
    __syncthreads();  // column j scaled; the pivot slot is rewritten only after every read of it
    if (threadIdx.x == 0) {
      dead[j] = dj;
      Ls[j + p * j] = djj;
    }
    if (!dj) {  // trailing update, column k per warp, rows i >= k per lane
      for (int k = j + 1 + warp; k < p; k += nw) {
        const double lkj = Ls[k + p * j];
        for (int i = k + lane; i < p; i += 32) Ls[i + p * k] -= Ls[i + p * j] * lkj;
      }
    }
  }
  __syncthreads();
  // X = L^{-1} by right-looking forward substitution over rows (all columns at
  // once); R^{-1} = X^T, retired columns of R^{-1} (rows of X) are zero.
  // launched only when 2 p^2 doubles fit (cholqr2); larger p: chol_inv_fast_kernel
  double* X = Ls + p * p;
  {
    for (int idx = threadIdx.x; idx < p * p; idx += blockDim.x) X[idx] = (idx % p == idx / p) ? 1.0 : 0.0;
    __syncthreads();
    for (int i = 0; i < p; ++i) {
      // row i final: x_i(c) = acc_i(c) / L_ii for c <= i
      const double rl = dead[i] ? 0.0 : 1.0 / Ls[i + p * i];
      for (int c = threadIdx.x; c <= i; c += blockDim.x) X[i + p * c] *= rl;
      __syncthreads();
      // rows r > i: acc_r(c) -= L_ri x_i(c)
      for (int c = warp; c <= i; c += nw) {
        const double xic = X[i + p * c];
        if (xic != 0.0)
          for (int r = i + 1 + lane; r < p; r += 32) X[r + p * c] -= Ls[r + p * i] * xic;
      }
      __syncthreads();
    }
    for (int idx = threadIdx.x; idx < p * p; idx += blockDim.x) {
      const int r = idx % p, c = idx / p;  // H(r, c) = R^{-1}(r, c) = X(c, r)
      H[idx] = X[c + p * r];
    }
  }
}

// The same factorisation for p <= kCholSmem, tuned for latency: 512 threads
// as (row i, group g) pairs, so the right-looking Cholesky update of column j
// splits each row's trailing columns k = j+1+g, j+5+g, ... over four groups
// (element-wise the same operations in the same j order as the kernels
// above); then L^{-1} in place column by column from the last (LAPACK trti2
// order: column j = -(inverted trailing block) x / l_jj, the row sums split
// over the groups and combined in a fixed order).  R^{-1} = (D L^{-1})^T with
// D zeroing the retired rows (their L columns are zero below a unit pivot, so
// every other row of L^{-1} is unaffected).  Two barriers per column in each
// phase instead of the row-at-a-time forward substitution.
constexpr int kCF_ROWS = 128, kCF_GRP = 4;
__global__ void __launch_bounds__(kCF_ROWS * kCF_GRP) chol_inv_fast_kernel(int p, double* __restrict__ H) {
  extern __shared__ double Lf[];  // p x p, column-major
  __shared__ double xs[kCF_ROWS];
  __shared__ double part[kCF_GRP][kCF_ROWS];
  __shared__ unsigned char dead[kCF_ROWS];
  __shared__ double s_mx;
  const int i = threadIdx.x % kCF_ROWS, grp = threadIdx.x / kCF_ROWS;
  for (int idx = threadIdx.x; idx < p * p; idx += blockDim.x) Lf[idx] = H[idx];
  __syncthreads();
  if (threadIdx.x < 32) {
    double mx = 0.0;
    for (int q = threadIdx.x; q < p; q += 32) mx = fmax(mx, Lf[q + p * q]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) s_mx = mx;
  }
  __syncthreads();
  const double tiny = 1e-26 * s_mx;
  const bool row = i < p;
  for (int j = 0; j < p; ++j) {
    __syncthreads();  // previous trailing update complete
    const double d = Lf[j + p * j];
    const bool dj = !(d > tiny);
    const double djj = dj ? 1.0 : sqrt(d);
    const double inv = 1.0 / djj;
    if (grp == 0 && row && i > j) Lf[i + p * j] = dj ? 0.0 : Lf[i + p * j] * inv;
    __syncthreads();  // column j scaled; every read of the pivot done
    if (threadIdx.x == 0) {
      dead[j] = dj;
      Lf[j + p * j] = djj;
    }
    if (!dj && row && i > j) {
      // loads of a batch issued before its stores (the compiler cannot prove
      // the column-j reads and the row-i writes disjoint)
      const double lij = Lf[i + p * j];
      int k = j + 1 + grp;
      for (; k + 3 * kCF_GRP <= i; k += 4 * kCF_GRP) {
        double c[4], r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          c[u] = Lf[k + u * kCF_GRP + p * j];
          r[u] = Lf[i + p * (k + u * kCF_GRP)];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) Lf[i + p * (k + u * kCF_GRP)] = r[u] - lij * c[u];
      }
      for (; k <= i; k += kCF_GRP) Lf[i + p * k] -= lij * Lf[k + p * j];
    }
  }
  for (int j = p - 1; j >= 0; --j) {
    __syncthreads();  // column j + 1 of the inverse written
    const double ljj = Lf[j + p * j];
    if (grp == 0 && row && i > j) xs[i] = Lf[i + p * j];
    __syncthreads();
    double acc = 0.0;
    if (row && i > j) {
#pragma unroll 4
      for (int k = j + 1 + grp; k <= i; k += kCF_GRP) acc += Lf[i + p * k] * xs[k];
    }
    part[grp][i] = acc;
    __syncthreads();
    if (grp == 0 && row && i >= j)
      Lf[i + p * j] = i == j ? 1.0 / ljj : -((part[0][i] + part[1][i]) + (part[2][i] + part[3][i])) / ljj;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < p * p; idx += blockDim.x) {
    const int r = idx % p, c = idx / p;  // H(r, c) = R^{-1}(r, c) = (D L^{-1})(c, r)
    H[idx] = (c >= r && !dead[c]) ? Lf[c + p * r] : 0.0;
  }
}

// One-sided (Hestenes) Jacobi SVD of an m x p matrix X held in global memory
// (L2-resident for the sizes thin_svd_left sends here), one CTA: X <- X V with
// orthogonal columns; V (p x p, optional) accumulates the rotations.  The
// rotation formula, the tournament ordering and the stopping test are those
// of jacobi_svd_kernel; accurate singular values down to ~eps sigma_max
// (no Gram squaring), as the reference's JacobiSVD.  Epilogue: sg = column
// norms sorted descending (stable), perm[c] = source column of rank c.
__global__ void __launch_bounds__(1024) jacobi_onesided_kernel(int64_t m, int p, double* __restrict__ X,
                                                                double* __restrict__ V, double* __restrict__ sg,
                                                                int* __restrict__ perm) {
  __shared__ int rot_any;
  extern __shared__ double nr_sh[];  // p column norms (dynamic)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int pe = p + (p & 1), half = pe / 2;
  const double tol = fmax(1e-16, p * 1.1102230246251565e-16);
  const double tol2 = tol * tol;
  if (V)
    for (int i = threadIdx.x; i < p * p; i += blockDim.x) V[i] = (i % p == i / p) ? 1.0 : 0.0;
  __syncthreads();
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) rot_any = 0;
    __syncthreads();
    int any = 0;
    for (int round = 0; round < pe - 1; ++round) {
      for (int q = warp; q < half; q += nw) {
        int a = (q == 0) ? pe - 1 : (round + q) % (pe - 1);
        int b = (round + pe - 1 - q) % (pe - 1);
        if (q == 0) b = round % (pe - 1);
        const int i = min(a, b), j = max(a, b);
        if (j >= p) continue;  // the padding column of odd p
        double* ci = X + m * i;
        double* cj = X + m * j;
        double al = 0, be = 0, ga = 0;
        for (int64_t r = lane; r < m; r += 32) {
          const double x = ci[r], y = cj[r];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga == 0.0 || ga * ga <= tol2 * (al * be)) continue;
        any = 1;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = rsqrt(1.0 + t * t), sn = c * t;
        for (int64_t r = lane; r < m; r += 32) {
          const double x = ci[r], y = cj[r];
          ci[r] = c * x - sn * y;
          cj[r] = sn * x + c * y;
        }
        if (V) {
          double* vi = V + static_cast<int64_t>(p) * i;
          double* vj = V + static_cast<int64_t>(p) * j;
          for (int r = lane; r < p; r += 32) {
            const double x = vi[r], y = vj[r];
            vi[r] = c * x - sn * y;
            vj[r] = sn * x + c * y;
          }
        }
      }
      __syncthreads();
    }
    if (any && lane == 0) rot_any = 1;
    __syncthreads();
    if (!rot_any) break;
    __syncthreads();
  }
  for (int j = warp; j < p; j += nw) {
    double ss = 0;
    for (int64_t r = lane; r < m; r += 32) ss += X[r + m * j] * X[r + m * j];
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) nr_sh[j] = sqrt(ss);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    int rk = 0;
    for (int k = 0; k < p; ++k) rk += (nr_sh[k] > nr_sh[j]) || (nr_sh[k] == nr_sh[j] && k < j);
    perm[rk] = j;
    sg[rk] = nr_sh[j];
  }
}

// U(:, c) = X(:, perm[c]) / sg[c] (left vectors of a tall matrix; a zero
// column gives 0, or e_c with normalize == 2), or U(:, c) = V(:, perm[c])
// (left vectors of a wide one, from A^T's rotations)
__global__ void jacobi_gather_kernel(int64_t m, int p, const double* __restrict__ src, const int* __restrict__ perm,
                                     const double* __restrict__ sg, int normalize, double* __restrict__ U) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= m * p) return;
  const int64_t r = idx % m;
  const int c = static_cast<int>(idx / m);
  const double v = src[r + m * perm[c]];
  U[idx] = normalize ? (sg[c] > 0.0 ? v / sg[c] : (normalize == 2 && r == c ? 1.0 : 0.0)) : v;
}

__global__ void sqrt_kernel(int64_t n, double* __restrict__ x) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = sqrt(fmax(0.0, x[i]));
}

__global__ void transpose_kernel(int64_t rows, int64_t cols, const double* __restrict__ a, double* __restrict__ t) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * cols) return;
  t[idx / rows + cols * (idx % rows)] = a[idx];  // t (cols x rows) = a^T
}

__global__ void fill_kernel(int64_t n, double v, double* __restrict__ x) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) x[i] = v;
}

// One-sided Jacobi SVD on the device for p <= kJacMax: one CTA,
// columns in shared memory, round-robin (tournament) ordering so the p/2
// rotations of a round are disjoint and run on separate warps; the rotation
// formula and the stopping test are jacobi_onesided_kernel's.  Output: U (sorted
// columns, in place of S) and sg, descending, stable in the column index.
constexpr int kJacMax = 128;
constexpr int kJacThreads = 1024;

__global__ void __launch_bounds__(kJacThreads) jacobi_svd_kernel(int p, double* __restrict__ S,
                                                                 double* __restrict__ sg_out) {
  extern __shared__ double js[];
  const int pe = p + (p & 1);  // even column count (a zero column pads odd p)
  double* col = js;            // pe columns of length p
  __shared__ int rot_any;
  __shared__ int perm_sh[kJacMax + 1];
  __shared__ double nr_sh[kJacMax + 1];
  for (int i = threadIdx.x; i < p * pe; i += blockDim.x) col[i] = i < p * p ? S[i] : 0.0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int half = pe / 2;
  // convergence |c_i . c_j| <= tol |c_i| |c_j| with tol = p eps: below the
  // rounding level of the dot products a stricter test never settles
  const double tol = fmax(1e-16, p * 1.1102230246251565e-16);
  const double tol2 = tol * tol;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) rot_any = 0;
    __syncthreads();
    int any = 0;
    for (int round = 0; round < pe - 1; ++round) {
      for (int q = warp; q < half; q += nw) {
        // tournament pairing: fixed element pe-1, the rest rotate
        int a = (q == 0) ? pe - 1 : (round + q) % (pe - 1);
        int b = (round + pe - 1 - q) % (pe - 1);
        if (q == 0) b = round % (pe - 1);
        int i = min(a, b), j = max(a, b);
        double* ci = col + static_cast<size_t>(p) * i;
        double* cj = col + static_cast<size_t>(p) * j;
        double al = 0, be = 0, ga = 0;
        for (int r = lane; r < p; r += 32) {
          const double x = ci[r], y = cj[r];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga == 0.0 || ga * ga <= tol2 * (al * be)) continue;
        any = 1;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = rsqrt(1.0 + t * t), sn = c * t;
        for (int r = lane; r < p; r += 32) {
          const double x = ci[r], y = cj[r];
          ci[r] = c * x - sn * y;
          cj[r] = sn * x + c * y;
        }
      }
      __syncthreads();
    }
    if (any && lane == 0) rot_any = 1;
    __syncthreads();
    if (!rot_any) break;
    __syncthreads();
  }
  for (int j = warp; j < p; j += nw) {
    double ss = 0;
    for (int r = lane; r < p; r += 32) ss += col[r + static_cast<size_t>(p) * j] * col[r + static_cast<size_t>(p) * j];
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) nr_sh[j] = sqrt(ss);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < p; j += blockDim.x) {  // stable descending rank
    int rk = 0;
    for (int k = 0; k < p; ++k) rk += (nr_sh[k] > nr_sh[j]) || (nr_sh[k] == nr_sh[j] && k < j);
    perm_sh[rk] = j;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < p * p; i += blockDim.x) {
    const int r = i % p, c = i / p;
    const int j = perm_sh[c];
    const double nj = nr_sh[j];
    S[i] = nj > 0 ? col[r + static_cast<size_t>(p) * j] / nj : (r == c ? 1.0 : 0.0);
  }
  for (int c = threadIdx.x; c < p; c += blockDim.x) sg_out[c] = nr_sh[perm_sh[c]];
}

// Scratch of the reduction / TEI drivers: while a DevStreamScope is alive,
// blocks come from the context's cache (best fit) and go back to it, so the
// many short-lived buffers of the iterations cost neither cudaMalloc latency
// nor the device-wide synchronisation of cudaFree.  All users run on
// ctx->stream, so reuse is stream-ordered.
thread_local tgb_ctx* g_dev_ctx = nullptr;

struct Dev {
  double* p = nullptr;
  size_t n = 0;
  size_t bytes = 0;
  tgb_ctx* c = nullptr;
  explicit Dev(size_t count = 0) { resize(count); }
  void resize(size_t count) {
    if (count <= n) return;
    release();
    c = g_dev_ctx;
    if (count) {
      if (c) {
        p = static_cast<double*>(scratch_alloc(c, count * sizeof(double), &bytes));
      } else {
        TGB_CUDA(cudaMalloc(&p, count * sizeof(double)));
        bytes = count * sizeof(double);
      }
    }
    n = count;
  }
  void release() {
    if (p) {
      if (c)
        scratch_free(c, p, bytes);
      else
        cudaFree(p);
    }
    p = nullptr;
    n = 0;
    bytes = 0;
  }
  ~Dev() { release(); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

// analysis only (TGB_RED_TIME): host-side stage timer, synchronising the stream
struct StageTimer {
  tgb_ctx* ctx;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit StageTimer(tgb_ctx* c) : ctx(c), on(getenv("TGB_RED_TIME") != nullptr), t(std::chrono::steady_clock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(ctx->stream);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[tgb-time] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

std::vector<double> to_host(tgb_ctx* ctx, const double* d, size_t count) {
  std::vector<double> h(count);
  if (count) {
    TGB_CUDA(cudaMemcpyAsync(h.data(), d, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return h;
}

void to_dev(tgb_ctx* ctx, double* d, const std::vector<double>& h) {
  if (!h.empty()) TGB_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
}

// Orthonormalise the columns of X (d x p) in place: Cholesky-QR, twice.
// Columns that are numerically dependent are replaced deterministically.
void cholqr2(tgb_ctx* ctx, int64_t d, int p, double* X, Dev& tmp) {
  tmp.resize(static_cast<size_t>(d) * p + 2 * static_cast<size_t>(p) * p);
  double* H = tmp.p + static_cast<size_t>(d) * p;
  double* Wk = H + static_cast<size_t>(p) * p;
  for (int rep = 0; rep < 2; ++rep) {
    if (rep) {
      colnormalize_kernel<<<p, 256, 0, ctx->stream>>>(d, X);
      TGB_LAUNCHED(ctx);
    }
    dgemm(ctx, true, false, p, p, d, 1.0, X, d, X, d, 0.0, H, p);
    // H is written in place with R^{-1}; back substitution reads H's upper part as it goes,
    // so each column c only reads entries (k, c) with k > i that it already produced.
    const size_t l_bytes = static_cast<size_t>(p) * p * sizeof(double);
    if (p <= kCholSmem && 2 * l_bytes <= static_cast<size_t>(kCholSmemBytes)) {
      // L and L^{-1} both in shared memory: the row-at-a-time kernel (96 vs 101 us at config 1's blocks)
      static bool cattr[kTgbMaxDevices] = {};  // per device
      if (!cattr[ctx->device]) {
        TGB_CUDA(cudaFuncSetAttribute(chol_inv_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kCholSmemBytes));
        cattr[ctx->device] = true;
      }
      chol_inv_smem_kernel<<<1, p > 64 ? 1024 : 512, 2 * l_bytes, ctx->stream>>>(p, H);
    } else if (p <= kCF_ROWS) {
      // in-place inverse (0.21 vs 0.38 ms at p = 110-128, the TEI fit's ranks)
      static bool fattr[kTgbMaxDevices] = {};  // per device
      if (!fattr[ctx->device]) {
        TGB_CUDA(cudaFuncSetAttribute(chol_inv_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kCF_ROWS * kCF_ROWS * static_cast<int>(sizeof(double))));
        fattr[ctx->device] = true;
      }
      chol_inv_fast_kernel<<<1, kCF_ROWS * kCF_GRP, l_bytes, ctx->stream>>>(p, H);
    } else {
      chol_inv_kernel<<<1, 256, 0, ctx->stream>>>(p, H, Wk);
    }
    TGB_LAUNCHED(ctx);
    TGB_CUDA(cudaMemcpyAsync(tmp.p, X, static_cast<size_t>(d) * p * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    dgemm(ctx, false, false, d, p, p, 1.0, tmp.p, d, H, p, 0.0, X, d);
  }
}

// deterministic pseudo-random start block
void random_block(tgb_ctx* ctx, int64_t d, int p, double* X, uint64_t seed) {
  std::vector<double> h(static_cast<size_t>(d) * p);
  uint64_t s = seed;
  for (auto& x : h) {
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    x = static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
  to_dev(ctx, X, h);
}

}  // namespace

// thin_svd_left (reduction.cpp:85-138) for min(rows, cols) <= 128 on the
// device: Cholesky-QR2 of the taller side, then the one-CTA Jacobi SVD of the
// small triangular-shaped factor (tall: A = Q R, SVD(R); wide: A^T = Q R, so
// A = R^T Q^T and SVD(A Q)).  The reference's branch picks only the OUTPUT
// shape here: the wide Gram branch (cols >= 4 rows, cols > 8192) and the
// Jacobi branch return min(rows, cols) pairs; the tall Gram branch (rows >=
// 4 cols, cols >= 8) keeps the leading pairs with sigma^2 > sigma_0^2 1e-24.
// U (rows x min) and sigma (min) are device outputs; returns the kept count.
void jacobi_svd_dev(tgb_ctx* ctx, int p, double* S, double* sg);
// One CTA, any p the column-norm scratch fits (p doubles of shared memory).
static void launch_jacobi_onesided(tgb_ctx* ctx, int64_t m, int64_t p, double* X, double* V, double* sg, int* perm) {
  const size_t sm = static_cast<size_t>(p) * sizeof(double);
  if (sm + 1024 > ctx->smem_optin) throw Error(TGB_INVALID_ARGUMENT, "one-sided Jacobi: too many columns");
  static bool attr[kTgbMaxDevices] = {};  // per device
  if (!attr[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(jacobi_onesided_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ctx->smem_optin - 1024)));
    attr[ctx->device] = true;
  }
  jacobi_onesided_kernel<<<1, 1024, sm, ctx->stream>>>(m, static_cast<int>(p), X, V, sg, perm);
  TGB_LAUNCHED(ctx);
}
static void dgemm_transpose(tgb_ctx* ctx, int64_t rows, int64_t cols, const double* a, double* t) {
  const int64_t tot = rows * cols;
  transpose_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, ctx->stream>>>(rows, cols, a, t);
  TGB_LAUNCHED(ctx);
}
int64_t thin_svd_left_dev(tgb_ctx* ctx, int64_t rows, int64_t cols, const double* A, double* U, double* sigma) {
  const int64_t p = std::min(rows, cols);
  if (p == 0) return 0;
  DevStreamScope scope(ctx);
  const bool gram_wide = cols >= 4 * rows && cols > 8192;               // reduction.cpp:93-104
  const bool jacobi_branch = !gram_wide && (rows < 4 * cols || cols < 8);  // reduction.cpp:105-108
  Dev perm_d(static_cast<size_t>(p)), V(static_cast<size_t>(p) * p);
  int* perm = reinterpret_cast<int*>(perm_d.p);
  const unsigned gb = static_cast<unsigned>((rows * p + 255) / 256);
  if (rows >= cols) {  // tall: one-sided Jacobi on A itself, U = normalised rotated columns
    Dev X(static_cast<size_t>(rows) * cols);
    TGB_CUDA(cudaMemcpyAsync(X.p, A, static_cast<size_t>(rows) * cols * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    launch_jacobi_onesided(ctx, rows, p, X.p, nullptr, sigma, perm);
    jacobi_gather_kernel<<<gb, 256, 0, ctx->stream>>>(rows, static_cast<int>(p), X.p, perm, sigma, 1, U);
    TGB_LAUNCHED(ctx);
  } else if (gram_wide) {  // the reference's Gram branch: eigenpairs of A A^T (rows x rows)
    Dev G(static_cast<size_t>(rows) * rows);
    dgemm(ctx, false, true, rows, rows, cols, 1.0, A, rows, A, rows, 0.0, G.p, rows);
    launch_jacobi_onesided(ctx, rows, p, G.p, nullptr, sigma, perm);
    jacobi_gather_kernel<<<gb, 256, 0, ctx->stream>>>(rows, static_cast<int>(p), G.p, perm, sigma, 1, U);
    TGB_LAUNCHED(ctx);
    sqrt_kernel<<<static_cast<unsigned>((p + 255) / 256), 256, 0, ctx->stream>>>(p, sigma);  // sigma = sqrt(lambda)
    TGB_LAUNCHED(ctx);
  } else {  // wide: Jacobi on A^T with the rotations accumulated; U = V
    Dev X(static_cast<size_t>(rows) * cols);
    dgemm_transpose(ctx, rows, cols, A, X.p);
    launch_jacobi_onesided(ctx, cols, p, X.p, V.p, sigma, perm);
    jacobi_gather_kernel<<<gb, 256, 0, ctx->stream>>>(rows, static_cast<int>(p), V.p, perm, sigma, 0, U);
    TGB_LAUNCHED(ctx);
  }
  int64_t kept = p;
  if (!gram_wide && !jacobi_branch) {  // tall Gram branch: drop lambda <= lambda_max 1e-24 (reduction.cpp:119-122)
    std::vector<double> hs(p);
    TGB_CUDA(cudaMemcpyAsync(hs.data(), sigma, p * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    const double lmax = hs[0] * hs[0];
    kept = 0;
    while (kept < p && hs[kept] * hs[kept] > lmax * 1e-24 && hs[kept] > 0.0) ++kept;
  }
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  return kept;
}

// One-CTA one-sided Jacobi SVD of a p x p device matrix: U replaces S in
// place (columns sorted by descending singular value; a zero column -> e_c),
// sg gets the p singular values.  p <= 128: columns in shared memory;
// larger p: the global-memory sweep, then the sorted gather.  Used by the
// Rayleigh-Ritz step of the rank reduction and the generalized eigensolver.
void jacobi_svd_dev(tgb_ctx* ctx, int p, double* S, double* sg) {
  if (p <= 0) return;
  if (p > kJacMax) {
    Dev perm_d(static_cast<size_t>(p)), U(static_cast<size_t>(p) * p);
    int* perm = reinterpret_cast<int*>(perm_d.p);
    launch_jacobi_onesided(ctx, p, p, S, nullptr, sg, perm);
    const int64_t tot = static_cast<int64_t>(p) * p;
    jacobi_gather_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, ctx->stream>>>(p, p, S, perm, sg, 2, U.p);
    TGB_LAUNCHED(ctx);
    TGB_CUDA(cudaMemcpyAsync(S, U.p, static_cast<size_t>(tot) * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));  // the scratch is released on return
    return;
  }
  const size_t jsm = static_cast<size_t>(p) * (p + (p & 1)) * sizeof(double);
  static bool jattr[kTgbMaxDevices] = {};  // per device
  if (!jattr[ctx->device]) {
    cudaFuncAttributes fa{};
    TGB_CUDA(cudaFuncGetAttributes(&fa, jacobi_svd_kernel));
    TGB_CUDA(cudaFuncSetAttribute(jacobi_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ctx->smem_optin - fa.sharedSizeBytes)));
    jattr[ctx->device] = true;
  }
  jacobi_svd_kernel<<<1, kJacThreads, jsm, ctx->stream>>>(p, S, sg);
  TGB_LAUNCHED(ctx);
}

DevStreamScope::DevStreamScope(tgb_ctx* ctx) : prev(g_dev_ctx) {
  if (!getenv("TGB_NO_SCRATCH_CACHE")) g_dev_ctx = ctx;
}
DevStreamScope::~DevStreamScope() { g_dev_ctx = prev; }

void* scratch_alloc(tgb_ctx* ctx, size_t bytes, size_t* got) {
  auto it = ctx->scratch_free.lower_bound(bytes);
  if (it != ctx->scratch_free.end() && it->first <= 2 * bytes + (1 << 20)) {  // best fit, bounded waste
    void* p = it->second;
    *got = it->first;
    ctx->scratch_free.erase(it);
    return p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {  // release the cache and retry once
    cudaGetLastError();
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (auto& kv : ctx->scratch_free) cudaFree(kv.second);
    ctx->scratch_free.clear();
    TGB_CUDA(cudaMalloc(&p, bytes));
  }
  *got = bytes;
  return p;
}

void scratch_free(tgb_ctx* ctx, void* p, size_t bytes) { ctx->scratch_free.emplace(bytes, p); }

// Column-normalise then Cholesky-QR twice: orthonormal basis of the columns of
// X (d x p, device, in place).  Used by the TEI fit (Q of the pivoted Cholesky
// factor, tei.cpp:136-138: the column space is what matters there; column
// signs may differ from a Householder Q, which B = V M V^T does not see).
void orthonormalize_columns(tgb_ctx* ctx, int64_t d, int p, double* X) {
  if (d == 0 || p == 0) return;
  colnormalize_kernel<<<p, 256, 0, ctx->stream>>>(d, X);
  TGB_LAUNCHED(ctx);
  Dev tmp;
  cholqr2(ctx, d, p, X, tmp);
}

// ---------------------------------------------------------------- reduction driver

struct RedCfgC {
  bool use_eps;
  double eps;
  int64_t ranks[3];
  int max_sweeps;
  bool full_spectra = false;  // also the whole spectrum of each RHOSVD mode matrix (spectrum.cu)
};

struct RedState {
  std::array<int64_t, 3> n{};
  int64_t R = 0;
  std::array<double*, 3> f{};  // normalized factors (device, owned by bufs)
  double* w = nullptr;
  std::array<Dev, 3> fbuf;
  Dev wbuf;
  std::array<Dev, 3> Z;        // n_ax x r_ax
  std::array<int64_t, 3> r{};
  Dev core;
  bool rank_clamped = false, fallback = false;
  std::vector<double> sweep_fits;
  std::array<std::vector<double>, 3> sigma;
  std::array<std::vector<double>, 3> sigma_full;  // mode_singular_values when requested
  bool has_full = false;
  // rank-selection margins of the initializing SVDs (tgb_tucker_margins)
  std::array<double, 3> total{};  // sum of ALL squared singular values of the mode's side matrix
  bool use_eps = false;
  double eps = 0.0;
};

// select_rank (reduction.cpp:34-59) on the leading singular values sg (descending);
// `total` = sum of ALL squared singular values (the Gram trace), `d` = their count.
static int64_t select_rank_host(const std::vector<double>& sg, double total, int64_t d, const RedCfgC& c, int mode,
                                bool* clamped, bool* need_more) {
  *need_more = false;
  if (sg.empty()) return 0;
  const double cut = sg[0] * 1e-15 * std::sqrt(static_cast<double>(d));
  int64_t numeric = 0;
  while (numeric < static_cast<int64_t>(sg.size()) && sg[numeric] > cut) ++numeric;
  const bool numeric_known = numeric < static_cast<int64_t>(sg.size()) || static_cast<int64_t>(sg.size()) == d;
  if (!c.use_eps) {
    const int64_t want = c.ranks[mode];
    if (!numeric_known && want > numeric) {
      *need_more = true;
      return want;
    }
    if (want > numeric && clamped) *clamped = true;
    return std::min(want, numeric);
  }
  if (total == 0.0) return 0;
  const double budget = c.eps * c.eps * total;
  double tail = total;
  int64_t r = 0;
  while (r < numeric && tail > budget) {
    tail -= sg[r] * sg[r];
    ++r;
  }
  if (tail > budget && !numeric_known) *need_more = true;
  return r;
}

// thin_svd_left of a (n x k, device) truncated to the selected/needed rank.
// sel < 0: select with the config (rhosvd); sel >= 0: keep min(sel, available).
//
// Two-sided subspace iteration on a itself (never forming a Gram matrix, so
// small singular values keep ~eps * sigma_0 absolute accuracy, as the
// reference's JacobiSVD branch): X <- orth(a Y), Y <- orth(a^T X), with a
// small SVD of S = X^T a Y (host, one-sided Jacobi) rotating the blocks to
// the singular directions every iteration.  Columns are normalised before
// the Cholesky-QR so the blocks stay well conditioned.
static int64_t left_subspace(tgb_ctx* ctx, int64_t n, int64_t k, const double* a, const RedCfgC* cfg, int mode,
                             int64_t sel, bool* clamped, Dev& Zout, std::vector<double>* sigma_out,
                             const double* warm = nullptr, int64_t warm_cols = 0, double* total_out = nullptr) {
  if (n == 0 || k == 0) {
    if (sigma_out) sigma_out->clear();
    return 0;
  }
  const int64_t dmin = std::min(n, k);
  // ||a||_F^2 = sum of all squared singular values (the tail-rule total)
  Dev part(256);
  sumsq_kernel<<<256, 256, 0, ctx->stream>>>(n * k, a, part.p);
  TGB_LAUNCHED(ctx);
  double total = 0.0;
  for (double x : to_host(ctx, part.p, 256)) total += x;
  int p = static_cast<int>(std::min<int64_t>(std::min<int64_t>(dmin, kMaxBlock), sel >= 0 ? std::max<int64_t>(sel + 8, 16) : 48));
  Dev X, Y, T, tmp, Sd, sgd;
  std::vector<double> sg;
  int64_t r = 0;
  int pcur = 0;  // columns of X already holding a (partially converged) subspace
  bool have_x = false;
  if (warm && warm_cols > 0) {
    pcur = static_cast<int>(std::min<int64_t>(warm_cols, p));
    X.resize(static_cast<size_t>(n) * p);
    TGB_CUDA(cudaMemcpyAsync(X.p, warm, static_cast<size_t>(n) * pcur * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    have_x = true;
  }
  int iters = 0;
  while (true) {
    X.resize(static_cast<size_t>(n) * p);
    Y.resize(static_cast<size_t>(k) * p);
    T.resize(static_cast<size_t>(std::max(n, k)) * p);
    Sd.resize(static_cast<size_t>(p) * p);
    if (have_x) {
      // keep the current subspace, fill the new columns at random, Y = orth(a^T X)
      if (pcur < p) random_block(ctx, n, p - pcur, X.p + static_cast<size_t>(n) * pcur, 0x5EEDULL + pcur);
      colnormalize_kernel<<<p, 256, 0, ctx->stream>>>(n, X.p);
      TGB_LAUNCHED(ctx);
      cholqr2(ctx, n, p, X.p, tmp);
      dgemm(ctx, true, false, k, p, n, 1.0, a, n, X.p, n, 0.0, Y.p, k);
    } else {
      random_block(ctx, k, p, Y.p, 0x1504062890ULL + static_cast<uint64_t>(p));
    }
    colnormalize_kernel<<<p, 256, 0, ctx->stream>>>(k, Y.p);
    TGB_LAUNCHED(ctx);
    cholqr2(ctx, k, p, Y.p, tmp);
    std::vector<double> prev(p, -1.0);
    bool done = false, grow = false;
    for (int it = 0; it < 400 && !done; ++it, ++iters) {
      dgemm(ctx, false, false, n, p, k, 1.0, a, n, Y.p, k, 0.0, T.p, n);  // T = a Y
      TGB_CUDA(cudaMemcpyAsync(X.p, T.p, static_cast<size_t>(n) * p * sizeof(double), cudaMemcpyDeviceToDevice,
                               ctx->stream));
      colnormalize_kernel<<<p, 256, 0, ctx->stream>>>(n, X.p);
      TGB_LAUNCHED(ctx);
      cholqr2(ctx, n, p, X.p, tmp);
      have_x = true;
      pcur = p;
      if (it % 2 == 1 || it >= 40) {
        // Rayleigh-Ritz: S = X^T a Y, rotate X to the singular directions
        dgemm(ctx, true, false, p, p, n, 1.0, X.p, n, T.p, n, 0.0, Sd.p, p);
        // device Jacobi: U replaces S in place, only the p singular values come back
        sgd.resize(p);
        jacobi_svd_dev(ctx, p, Sd.p, sgd.p);
        sg = to_host(ctx, sgd.p, p);
        dgemm(ctx, false, false, n, p, p, 1.0, X.p, n, Sd.p, p, 0.0, T.p, n);
        TGB_CUDA(cudaMemcpyAsync(X.p, T.p, static_cast<size_t>(n) * p * sizeof(double), cudaMemcpyDeviceToDevice,
                                 ctx->stream));
        int conv = 0;
        while (conv < p && std::fabs(sg[conv] - prev[conv]) <= 1e-14 * std::max(sg[0], 1e-300)) ++conv;
        prev = sg;
        // rank estimate from the whole (possibly unconverged) block
        int64_t r_est;
        if (sel >= 0) {
          r_est = std::min<int64_t>(sel, dmin);
        } else {
          bool more = false, cl = false;
          r_est = select_rank_host(sg, total, dmin, *cfg, mode, &cl, &more);
          if (more) r_est = p;  // tail rule not met inside this block
        }
        if (getenv("TGB_RED_DEBUG") && getenv("TGB_RED_DEBUG")[0] == '2')
          fprintf(stderr, "[tgb]   it=%d p=%d conv=%d r_est=%lld s0=%.3e s_last=%.3e\n", it, p, conv,
                  static_cast<long long>(r_est), sg[0], sg[p - 1]);
        if (r_est + 4 > p && p < dmin) {
          if (p >= kMaxBlock)  // the block cannot grow past kMaxBlock columns: fail instead of looping
            throw Error(TGB_NUMERICAL_ERROR,
                        "reduce: more than " + std::to_string(kMaxBlock - 4) +
                            " singular vectors needed in one mode (device subspace block limit)");
          grow = true;
          break;
        }
        const int64_t need = std::min<int64_t>(r_est + 1, dmin);
        if (conv >= need || (p == dmin && conv == p)) {
          r = r_est;
          done = true;
          break;
        }
      }
      // Y <- orth(a^T X)
      dgemm(ctx, true, false, k, p, n, 1.0, a, n, X.p, n, 0.0, Y.p, k);
      colnormalize_kernel<<<p, 256, 0, ctx->stream>>>(k, Y.p);
      TGB_LAUNCHED(ctx);
      cholqr2(ctx, k, p, Y.p, tmp);
    }
    if (!done && !grow && !getenv("TGB_QUIET"))
      fprintf(stderr, "[tgb] warning: reduce: subspace iteration hit its 400-iteration cap (n=%lld k=%lld p=%d); "
                      "rank taken from the unconverged block\n", static_cast<long long>(n), static_cast<long long>(k), p);
    if (done || !grow) break;
    // grow the block: keep X, double p
    const int pn = static_cast<int>(std::min<int64_t>(std::min<int64_t>(dmin, 2 * p), kMaxBlock));
    Dev X2(static_cast<size_t>(n) * pn);
    TGB_CUDA(cudaMemcpyAsync(X2.p, X.p, static_cast<size_t>(n) * p * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    X.resize(static_cast<size_t>(n) * pn);
    TGB_CUDA(cudaMemcpyAsync(X.p, X2.p, static_cast<size_t>(n) * p * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
    pcur = p;
    p = pn;
  }
  if (getenv("TGB_RED_DEBUG"))
    fprintf(stderr, "[tgb] left_subspace n=%lld k=%lld p=%d iters=%d\n", static_cast<long long>(n),
            static_cast<long long>(k), p, iters);
  if (sel >= 0) {
    r = std::min<int64_t>(sel, static_cast<int64_t>(sg.size()));
  } else {
    bool more = false;
    r = select_rank_host(sg, total, dmin, *cfg, mode, clamped, &more);
  }
  if (sigma_out) *sigma_out = sg;
  if (total_out) *total_out = total;
  Zout.resize(std::max<int64_t>(1, n * r));
  if (r > 0)
    TGB_CUDA(cudaMemcpyAsync(Zout.p, X.p, static_cast<size_t>(n) * r * sizeof(double), cudaMemcpyDeviceToDevice,
                             ctx->stream));
  return r;
}

static void project_core(tgb_ctx* ctx, RedState& st) {
  const int64_t R = st.R;
  std::array<Dev, 3> P;
  for (int ax = 0; ax < 3; ++ax) {
    P[ax].resize(std::max<int64_t>(1, st.r[ax] * R));
    if (st.r[ax] && R) dgemm(ctx, true, false, st.r[ax], R, st.n[ax], 1.0, st.Z[ax].p, st.n[ax], st.f[ax], st.n[ax], 0.0,
                             P[ax].p, st.r[ax]);
  }
  const int64_t r0 = st.r[0], r12 = st.r[1] * st.r[2];
  st.core.resize(std::max<int64_t>(1, r0 * r12));
  if (r0 * r12 == 0) return;
  if (R == 0) {
    fill_kernel<<<static_cast<unsigned>((r0 * r12 + 255) / 256), 256, 0, ctx->stream>>>(r0 * r12, 0.0, st.core.p);
    TGB_LAUNCHED(ctx);
    return;
  }
  Dev K(static_cast<size_t>(r12) * R);
  khatri_rao_kernel<<<static_cast<unsigned>((r12 * R + 255) / 256), 256, 0, ctx->stream>>>(
      R, static_cast<int>(st.r[1]), static_cast<int>(st.r[2]), st.w, P[1].p, P[2].p, K.p);
  TGB_LAUNCHED(ctx);
  // core (r0 x r1 r2) = P0 (r0 x R) K^T (R x r1 r2)
  dgemm(ctx, false, true, r0, r12, R, 1.0, P[0].p, r0, K.p, r12, 0.0, st.core.p, r0);
}

static double fro_norm_dev(tgb_ctx* ctx, const double* x, int64_t count) {
  const std::vector<double> h = to_host(ctx, x, count);
  double s = 0.0;
  for (double v : h) s += v * v;
  return std::sqrt(s);
}

void reduce_dev(tgb_ctx* ctx, const tgb_cp& a, const RedCfgC& cfg, bool als, RedState& st) {
  StageTimer tm(ctx);
  st.R = a.rank;
  for (int ax = 0; ax < 3; ++ax) st.n[ax] = a.n[ax];
  // normalized copy (reduction.cpp:176-177)
  for (int ax = 0; ax < 3; ++ax) {
    st.fbuf[ax].resize(std::max<int64_t>(1, a.n[ax] * a.rank));
    if (a.rank)
      TGB_CUDA(cudaMemcpyAsync(st.fbuf[ax].p, a.factor[ax], a.n[ax] * a.rank * sizeof(double), cudaMemcpyDeviceToDevice,
                               ctx->stream));
    st.f[ax] = st.fbuf[ax].p;
  }
  st.wbuf.resize(std::max<int64_t>(1, a.rank));
  if (a.rank)
    TGB_CUDA(cudaMemcpyAsync(st.wbuf.p, a.weight, a.rank * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  st.w = st.wbuf.p;
  if (a.rank) {
    normalize_kernel<<<static_cast<unsigned>(a.rank), 256, 0, ctx->stream>>>(a.n[0], a.n[1], a.n[2], st.f[0], st.f[1],
                                                                             st.f[2], st.w);
    TGB_LAUNCHED(ctx);
  }
  // RHOSVD (reduction.cpp:172-190): per mode left subspace of f diag(w)
  for (int mode = 0; mode < 3; ++mode) {
    const int64_t n = a.n[mode], R = a.rank;
    Dev W(std::max<int64_t>(1, n * R));
    if (R) {
      scale_cols_kernel<<<static_cast<unsigned>((n * R + 255) / 256), 256, 0, ctx->stream>>>(n, R, st.f[mode], st.w, W.p);
      TGB_LAUNCHED(ctx);
    }
    st.r[mode] = left_subspace(ctx, n, R, W.p, &cfg, mode, -1, &st.rank_clamped, st.Z[mode], &st.sigma[mode],
                               nullptr, 0, &st.total[mode]);
    if (cfg.full_spectra) {
      st.sigma_full[mode] = mode_spectrum_dev(ctx, n, R, W.p);
      st.has_full = true;
    }
    st.use_eps = cfg.use_eps;
    st.eps = cfg.eps;
    tm.mark("rhosvd left subspace");
  }
  project_core(ctx, st);
  tm.mark("project core");
  if (!als || a.rank == 0 || st.r[0] * st.r[1] * st.r[2] == 0) return;
  // ALS sweeps (reduction.cpp:205-232)
  double prev = -1.0;
  for (int sweep = 0; sweep < cfg.max_sweeps; ++sweep) {
    double fit = 0.0;
    for (int ax = 0; ax < 3; ++ax) {
      const int m = (ax + 1) % 3, p = (ax + 2) % 3;
      const int64_t R = st.R, rm = st.r[m], rp = st.r[p], n = st.n[ax];
      Dev pm(std::max<int64_t>(1, rm * R)), pp(std::max<int64_t>(1, rp * R));
      dgemm(ctx, true, false, rm, R, st.n[m], 1.0, st.Z[m].p, st.n[m], st.f[m], st.n[m], 0.0, pm.p, rm);
      dgemm(ctx, true, false, rp, R, st.n[p], 1.0, st.Z[p].p, st.n[p], st.f[p], st.n[p], 0.0, pp.p, rp);
      Dev Cm(static_cast<size_t>(R) * rm * rp);
      als_coef_kernel<<<static_cast<unsigned>((R * rm * rp + 255) / 256), 256, 0, ctx->stream>>>(
          R, static_cast<int>(rm), static_cast<int>(rp), st.w, pm.p, pp.p, Cm.p);
      TGB_LAUNCHED(ctx);
      Dev mat(static_cast<size_t>(n) * rm * rp);
      dgemm(ctx, false, false, n, rm * rp, R, 1.0, st.f[ax], n, Cm.p, R, 0.0, mat.p, n);
      tm.mark("als unfolding");
      Dev Znew;
      const int64_t r = left_subspace(ctx, n, rm * rp, mat.p, nullptr, ax, st.r[ax], nullptr, Znew, nullptr,
                                      st.Z[ax].p, st.r[ax]);
      if (r == 0) {
        st.fallback = true;
        return;
      }
      st.r[ax] = std::min<int64_t>(st.r[ax], r);
      st.Z[ax].resize(static_cast<size_t>(n) * st.r[ax]);
      TGB_CUDA(cudaMemcpyAsync(st.Z[ax].p, Znew.p, static_cast<size_t>(n) * st.r[ax] * sizeof(double),
                               cudaMemcpyDeviceToDevice, ctx->stream));
      Dev proj(static_cast<size_t>(st.r[ax]) * rm * rp);
      dgemm(ctx, true, false, st.r[ax], rm * rp, n, 1.0, st.Z[ax].p, n, mat.p, n, 0.0, proj.p, st.r[ax]);
      fit = fro_norm_dev(ctx, proj.p, st.r[ax] * rm * rp);
      tm.mark("als subspace + fit");
    }
    st.sweep_fits.push_back(fit);
    if (prev >= 0.0 && std::fabs(fit - prev) < 1e-14 * std::max(1.0, fit)) break;
    prev = fit;
  }
  project_core(ctx, st);
  tm.mark("final core");
}

// tucker_to_canonical (reduction.cpp:238-269) into caller-sized device buffers
int64_t t2c_rank(const RedState& st) {
  const auto& r = st.r;
  if (r[0] * r[1] * r[2] == 0) return 0;
  int ax = 0;
  for (int m = 1; m < 3; ++m)
    if (r[m] > r[ax]) ax = m;
  return r[(ax + 1) % 3] * r[(ax + 2) % 3];
}

void t2c_dev(tgb_ctx* ctx, RedState& st, double* out_f[3], double* out_w) {
  const auto& r = st.r;
  const int64_t rank = t2c_rank(st);
  if (rank == 0) return;
  int ax = 0;
  for (int m = 1; m < 3; ++m)
    if (r[m] > r[ax]) ax = m;
  const int m1 = (ax + 1) % 3, m2 = (ax + 2) % 3;
  Dev S(static_cast<size_t>(r[ax]) * rank);
  t2c_slices_kernel<<<static_cast<unsigned>((r[ax] * rank + 255) / 256), 256, 0, ctx->stream>>>(
      static_cast<int>(r[0]), static_cast<int>(r[1]), static_cast<int>(r[2]), ax, m1, m2, st.core.p, S.p);
  TGB_LAUNCHED(ctx);
  dgemm(ctx, false, false, st.n[ax], rank, r[ax], 1.0, st.Z[ax].p, st.n[ax], S.p, r[ax], 0.0, out_f[ax], st.n[ax]);
  gather_cols_kernel<<<static_cast<unsigned>((st.n[m1] * rank + 255) / 256), 256, 0, ctx->stream>>>(
      st.n[m1], rank, st.Z[m1].p, static_cast<int>(r[m1]), 1, out_f[m1]);
  TGB_LAUNCHED(ctx);
  gather_cols_kernel<<<static_cast<unsigned>((st.n[m2] * rank + 255) / 256), 256, 0, ctx->stream>>>(
      st.n[m2], rank, st.Z[m2].p, static_cast<int>(r[m2]), static_cast<int>(r[m1]), out_f[m2]);
  TGB_LAUNCHED(ctx);
  fill_kernel<<<static_cast<unsigned>((rank + 255) / 256), 256, 0, ctx->stream>>>(rank, 1.0, out_w);
  TGB_LAUNCHED(ctx);
  normalize_kernel<<<static_cast<unsigned>(rank), 256, 0, ctx->stream>>>(st.n[0], st.n[1], st.n[2], out_f[0], out_f[1],
                                                                         out_f[2], out_w);
  TGB_LAUNCHED(ctx);
}

}  // namespace tgb

// ---------------------------------------------------------------- C-ABI

struct tgb_tucker {
  tgb::RedState st;
};

extern "C" {

// mode: 0 rhosvd, 1 canonical_to_tucker (RHOSVD + ALS); + 2: also the full
// spectra of the RHOSVD mode matrices (mode_singular_values).  a: device or host (mem).
int tgb_reduce_tucker(tgb_ctx* ctx, const tgb_cp* a, int use_eps, double eps, const int64_t* ranks, int max_sweeps,
                      int mode, int mem, tgb_tucker** out) {
  return tgb::guarded_call([&] {
    tgb::require(a != nullptr && out != nullptr, "reduce: null argument");
    tgb::require(use_eps ? eps > 0.0 : (ranks != nullptr), "ReductionConfig: set exactly one of {ranks, epsilon}");
    tgb::require(max_sweeps >= 1, "ReductionConfig: need at least one sweep");
    if (!use_eps)
      for (int i = 0; i < 3; ++i) tgb::require(ranks[i] >= 0, "select_rank: negative rank request");
    TGB_CUDA(cudaSetDevice(ctx->device));
    tgb::DevStreamScope scope(ctx);
    tgb::StageTimer tm(ctx);
    tgb::require(mode >= 0 && mode <= 3, "reduce: bad mode");
    tgb::RedCfgC cfg{use_eps != 0, eps, {0, 0, 0}, max_sweeps, (mode & 2) != 0};
    if (!use_eps)
      for (int i = 0; i < 3; ++i) cfg.ranks[i] = ranks[i];
    tgb_cp dev = *a;
    std::array<tgb::Dev, 4> bufs;
    if (mem == TGB_MEM_HOST) {
      for (int ax = 0; ax < 3; ++ax) {
        bufs[ax].resize(std::max<int64_t>(1, a->n[ax] * a->rank));
        if (a->rank) tgb::h2d(ctx, bufs[ax].p, a->factor[ax], a->n[ax] * a->rank * sizeof(double), ctx->stream);
        dev.factor[ax] = bufs[ax].p;
      }
      bufs[3].resize(std::max<int64_t>(1, a->rank));
      if (a->rank) tgb::h2d(ctx, bufs[3].p, a->weight, a->rank * sizeof(double), ctx->stream);
      dev.weight = bufs[3].p;
    }
    tm.mark("input to device");
    auto* t = new tgb_tucker();
    try {
      tgb::reduce_dev(ctx, dev, cfg, (mode & 1) != 0, t->st);
      TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

int tgb_tucker_destroy(tgb_tucker* t) {
  return tgb::guarded_call([&] { delete t; });
}

// info[0..2] Tucker ranks, [3] rank_clamped, [4] rhosvd_fallback, [5] sweeps, [6] t2c rank
int tgb_tucker_info(tgb_tucker* t, int64_t* info) {
  return tgb::guarded_call([&] {
    for (int ax = 0; ax < 3; ++ax) info[ax] = t->st.r[ax];
    info[3] = t->st.rank_clamped;
    info[4] = t->st.fallback;
    info[5] = static_cast<int64_t>(t->st.sweep_fits.size());
    info[6] = tgb::t2c_rank(t->st);
  });
}

// core (r0 r1 r2), sides n_ax x r_ax, sweep fits, leading singular values per mode (count in nsig[ax])
int tgb_tucker_get(tgb_tucker* t, double* core, double* side0, double* side1, double* side2, double* sweep_fits,
                   int mem) {
  return tgb::guarded_call([&] {
    auto& st = t->st;
    const auto kind = mem == TGB_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    const int64_t cs = st.r[0] * st.r[1] * st.r[2];
    if (core && cs) TGB_CUDA(cudaMemcpy(core, st.core.p, cs * sizeof(double), kind));
    double* sides[3] = {side0, side1, side2};
    for (int ax = 0; ax < 3; ++ax)
      if (sides[ax] && st.r[ax]) TGB_CUDA(cudaMemcpy(sides[ax], st.Z[ax].p, st.n[ax] * st.r[ax] * sizeof(double), kind));
    if (sweep_fits)
      for (size_t i = 0; i < st.sweep_fits.size(); ++i) sweep_fits[i] = st.sweep_fits[i];
  });
}

int tgb_tucker_sigma(tgb_tucker* t, int axis, int64_t* count, double* sigma) {
  return tgb::guarded_call([&] {
    tgb::require(t && count && axis >= 0 && axis < 3, "tucker_sigma: bad argument");
    const auto& s = t->st.has_full ? t->st.sigma_full[axis] : t->st.sigma[axis];
    *count = static_cast<int64_t>(s.size());
    if (sigma)
      for (size_t i = 0; i < s.size(); ++i) sigma[i] = s[i];
  });
}

// Rank-selection margins of mode `axis` (the RHOSVD initializing SVD,
// select_rank reduction.cpp:34-59), for judging whether a rank is robust:
// out = {r, sigma_{r-1} (last kept), sigma_r (first dropped; -1 if not formed),
//        sigma_{r-1} / sigma_r, tail(r-1) / budget (> 1), tail(r) / budget (<= 1)}
// with tail(j) = sum_{i >= j} sigma_i^2 and budget = eps^2 * total (eps mode;
// the two tail ratios are -1 in fixed-rank mode).
int tgb_tucker_margins(tgb_tucker* t, int axis, double* out) {
  return tgb::guarded_call([&] {
    tgb::require(t && out && axis >= 0 && axis < 3, "tucker_margins: bad argument");
    const auto& st = t->st;
    const auto& sg = st.sigma[axis];
    const int64_t r = st.r[axis];
    out[0] = static_cast<double>(r);
    out[1] = r >= 1 && r - 1 < static_cast<int64_t>(sg.size()) ? sg[r - 1] : -1.0;
    out[2] = r < static_cast<int64_t>(sg.size()) ? sg[r] : -1.0;
    out[3] = out[1] > 0 && out[2] > 0 ? out[1] / out[2] : -1.0;
    out[4] = out[5] = -1.0;
    if (st.use_eps && st.total[axis] > 0.0) {
      const double budget = st.eps * st.eps * st.total[axis];
      double tail = st.total[axis];
      for (int64_t i = 0; i + 1 < r && i < static_cast<int64_t>(sg.size()); ++i) tail -= sg[i] * sg[i];
      out[4] = tail / budget;  // before dropping sigma_{r-1}
      if (r >= 1 && r - 1 < static_cast<int64_t>(sg.size())) tail -= sg[r - 1] * sg[r - 1];
      out[5] = tail / budget;
    }
  });
}

// tucker_to_canonical into a caller-allocated CP (rank = info[6])
int tgb_tucker_to_canonical(tgb_ctx* ctx, tgb_tucker* t, tgb_cp* out, int mem) {
  return tgb::guarded_call([&] {
    const int64_t rank = tgb::t2c_rank(t->st);
    tgb::require(out->rank == rank, "tucker_to_canonical: output rank mismatch");
    TGB_CUDA(cudaSetDevice(ctx->device));
    tgb::DevStreamScope scope(ctx);
    if (mem == TGB_MEM_DEVICE) {
      tgb::t2c_dev(ctx, t->st, out->factor, out->weight);
      TGB_CUDA(cudaStreamSynchronize(ctx->stream));
      return;
    }
    std::array<tgb::Dev, 4> bufs;
    double* f[3];
    for (int ax = 0; ax < 3; ++ax) {
      bufs[ax].resize(std::max<int64_t>(1, t->st.n[ax] * rank));
      f[ax] = bufs[ax].p;
    }
    bufs[3].resize(std::max<int64_t>(1, rank));
    tgb::t2c_dev(ctx, t->st, f, bufs[3].p);
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int ax = 0; ax < 3; ++ax)
      if (rank) tgb::d2h(ctx, out->factor[ax], f[ax], t->st.n[ax] * rank * sizeof(double), ctx->stream);
    if (rank) tgb::d2h(ctx, out->weight, bufs[3].p, rank * sizeof(double), ctx->stream);
  });
}

}  // extern "C"

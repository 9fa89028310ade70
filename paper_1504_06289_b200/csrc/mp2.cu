// MP2 on the factorised TEI: the MO congruence transform
// of the Cholesky columns (reference proj/src/mp2.cpp:7-24) and the
// second-order energy by direct summation (mp2.cpp:40-56) or through the
// exponential-sum denominator (mp2.cpp:58-93).
//
// Device layout: V = L_V L_V^T (N_ov x N_ov) by one DGEMM, then one CTA per
// occupied pair (i, j) sums v_iajb (2 v_iajb - v_ibja) g(e_a + e_b - e_i - e_j)
// over (a, b) with g = 1/x (direct) or sum_k w_k d_k(ia) d_k(jb),
// d_k(ia) = exp(-lambda_k (e_a - e_i)) (factorised: the same separable
// denominator the reference's Gram route contracts, mp2.cpp:66-90).  Partial
// sums are combined in a fixed order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "tgb_host.h"
#include "tgb_internal.hpp"

namespace tgb {
namespace {

struct Buf {
  tgb_ctx* c;
  double* p = nullptr;
  size_t bytes = 0;
  Buf(tgb_ctx* ctx, size_t count) : c(ctx) {
    if (count) p = static_cast<double*>(scratch_alloc(c, count * sizeof(double), &bytes));
  }
  ~Buf() {
    if (p) scratch_free(c, p, bytes);
  }
};

// out[(i n_vir + a) + N_ov s] = sum_nu W[i, nu + nb s] C[nu, n_occ + a]   (mp2.cpp:17-21)
__global__ void mo_vir_kernel(int64_t nb, int64_t n_occ, int64_t n_vir, int64_t R, const double* __restrict__ W,
                              const double* __restrict__ C, double* __restrict__ out) {
  const int64_t nov = n_occ * n_vir, tot = nov * R;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < tot;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = idx / nov, ia = idx % nov, i = ia / n_vir, a = ia % n_vir;
    const double* w = W + i + n_occ * nb * s;
    const double* c = C + nb * (n_occ + a);
    double acc = 0.0;
    for (int64_t nu = 0; nu < nb; ++nu) acc += w[n_occ * nu] * c[nu];
    out[idx] = acc;
  }
}

// d[k * N_ov + ia] = exp(-rate_k (e_{n_occ + a} - e_i))
__global__ void denom_factor_kernel(int64_t n_occ, int64_t n_vir, int64_t K, const double* __restrict__ e,
                                    const double* __restrict__ rates, double* __restrict__ d) {
  const int64_t nov = n_occ * n_vir;
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= nov * K) return;
  const int64_t k = idx / nov, ia = idx % nov, i = ia / n_vir, a = ia % n_vir;
  d[idx] = exp(-rates[k] * (e[n_occ + a] - e[i]));
}

// part[i + n_occ j] = sum_{a,b} v_iajb (2 v_iajb - v_ibja) g_iajb
__global__ void __launch_bounds__(256) mp2_pair_kernel(int64_t n_occ, int64_t n_vir, const double* __restrict__ V,
                                                       const double* __restrict__ e, int64_t K,
                                                       const double* __restrict__ d, const double* __restrict__ w,
                                                       double* __restrict__ part) {
  const int64_t i = blockIdx.x, j = blockIdx.y, nov = n_occ * n_vir;
  double acc = 0.0;
  for (int64_t ab = threadIdx.x; ab < n_vir * n_vir; ab += blockDim.x) {
    const int64_t a = ab / n_vir, b = ab % n_vir;
    const int64_t ia = i * n_vir + a, jb = j * n_vir + b, ib = i * n_vir + b, ja = j * n_vir + a;
    const double v1 = V[ia + nov * jb], v2 = V[ib + nov * ja];
    double g;
    if (K == 0) {
      g = 1.0 / (e[n_occ + a] + e[n_occ + b] - e[i] - e[j]);
    } else {
      g = 0.0;
      for (int64_t k = 0; k < K; ++k) g += w[k] * (d[k * nov + ia] * d[k * nov + jb]);
    }
    acc += v1 * (2.0 * v1 - v2) * g;
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int st = 128; st; st >>= 1) {
    if (threadIdx.x < st) sh[threadIdx.x] += sh[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[i + n_occ * j] = sh[0];
}

}  // namespace

void mo_transform_dev(tgb_ctx* ctx, int64_t nb, int64_t R, const double* chol, int64_t n_occ, const double* C,
                      double* out) {
  const int64_t n_vir = nb - n_occ;
  if (R == 0 || n_occ == 0 || n_vir == 0) return;
  Buf W(ctx, n_occ * nb * R);
  // W = C_occ^T [M_1 ... M_R]  (chol viewed nb x nb R)
  dgemm(ctx, true, false, n_occ, nb * R, nb, 1.0, C, nb, chol, nb, 0.0, W.p, n_occ);
  const int64_t tot = n_occ * n_vir * R;
  mo_vir_kernel<<<static_cast<unsigned>(std::min<int64_t>((tot + 255) / 256, 32 * ctx->num_sms)), 256, 0,
                  ctx->stream>>>(nb, n_occ, n_vir, R, W.p, C, out);
  TGB_LAUNCHED(ctx);
}

double mp2_energy_dev(tgb_ctx* ctx, int64_t n_occ, int64_t n_vir, int64_t R, const double* F, const double* e_host,
                      int mode, double expsum_eps) {
  const int64_t nb = n_occ + n_vir, nov = n_occ * n_vir;
  require(n_occ >= 1 && n_vir >= 1, "MOSpace: need occupied and virtual orbitals");
  const double gap = e_host[n_occ] - e_host[n_occ - 1];
  if (gap <= 0.0) throw Error(TGB_NUMERICAL_ERROR, "mp2_energy: non-positive homo-lumo gap, denominator may vanish");
  std::vector<double> rates, weights;
  if (mode == 1) {  // energy_denominator_expsum (mp2.cpp:26-36)
    const double spread = e_host[nb - 1] - e_host[0];
    const double lo = 2.0 * gap, hi = std::max(2.0 * spread, lo);
    rates.assign(256, 0.0);
    weights.assign(256, 0.0);
    int64_t terms = 0;
    double achieved = 0.0;
    int ok = 0;
    const int rc = tgb_reciprocal_expsum(lo, hi, expsum_eps, 256, &terms, rates.data(), weights.data(), &achieved, &ok);
    if (rc != TGB_OK) throw Error(rc, tgb_host_last_error());
    if (!ok) throw Error(TGB_NUMERICAL_ERROR, "energy_denominator_expsum: tolerance unattainable within the term cap");
    rates.resize(terms);
    weights.resize(terms);
  }
  const int64_t K = static_cast<int64_t>(rates.size());
  Buf V(ctx, nov * nov), de(ctx, nb), dr(ctx, std::max<int64_t>(K, 1)), dw(ctx, std::max<int64_t>(K, 1)),
      dd(ctx, std::max<int64_t>(K * nov, 1)), part(ctx, n_occ * n_occ);
  if (R > 0) {
    dgemm(ctx, false, true, nov, nov, R, 1.0, F, nov, F, nov, 0.0, V.p, nov);
  } else {
    TGB_CUDA(cudaMemsetAsync(V.p, 0, nov * nov * sizeof(double), ctx->stream));
  }
  TGB_CUDA(cudaMemcpyAsync(de.p, e_host, nb * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  if (K) {
    TGB_CUDA(cudaMemcpyAsync(dr.p, rates.data(), K * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    TGB_CUDA(cudaMemcpyAsync(dw.p, weights.data(), K * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    denom_factor_kernel<<<static_cast<unsigned>((K * nov + 255) / 256), 256, 0, ctx->stream>>>(n_occ, n_vir, K, de.p,
                                                                                            dr.p, dd.p);
    TGB_LAUNCHED(ctx);
  }
  mp2_pair_kernel<<<dim3(static_cast<unsigned>(n_occ), static_cast<unsigned>(n_occ)), 256, 0, ctx->stream>>>(
      n_occ, n_vir, V.p, de.p, K, dd.p, dw.p, part.p);
  TGB_LAUNCHED(ctx);
  std::vector<double> hp(n_occ * n_occ);
  TGB_CUDA(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  double e = 0.0;
  for (double x : hp) e -= x;
  return e;
}

}  // namespace tgb

// Hartree-Fock operators that sit on the convolution / assembly path
// (SURVEY.md §8f): the nuclear potential tensor and matrix
// (reference proj/src/hf.cpp:89-116), the exchange matrix by one batched
// convolution per occupied orbital (hf.cpp:153-170), the Cholesky-factor
// Coulomb / exchange / Fock builders (proj/src/tei.cpp:215-238) and the
// overlap / kinetic matrices (hf.cpp:48-87).
//
// Every O(n) or O(n^2) step runs on the device (window gathers, Hadamard
// columns, FFT convolutions, DMMA GEMMs, fixed-order reductions); the host
// only folds the few per-primitive-pair numbers into nb x nb matrices, in a
// fixed order (results are deterministic run to run).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <vector>

#include "tgb_internal.hpp"

namespace tgb {
namespace {

// Context-cached device scratch (stream-ordered reuse on ctx->stream).
struct Scratch {
  tgb_ctx* c;
  double* p = nullptr;
  size_t bytes = 0;
  Scratch(tgb_ctx* ctx, size_t count) : c(ctx) {
    if (count) p = static_cast<double*>(scratch_alloc(c, count * sizeof(double), &bytes));
  }
  ~Scratch() {
    if (p) scratch_free(c, p, bytes);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
};

template <class T>
T* upload(tgb_ctx* ctx, Scratch& s, const std::vector<T>& v) {
  static_assert(sizeof(T) <= sizeof(double) && sizeof(double) % sizeof(T) == 0, "scratch element size");
  if (v.empty()) return nullptr;
  TGB_CUDA(cudaMemcpyAsync(s.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  return reinterpret_cast<T*>(s.p);
}

// out(:, a R + q) = ref(ofs[a] : ofs[a] + n, q)   (hf.cpp:94-98, WindowMap::apply grid.hpp:66-69)
__global__ void window_gather_kernel(int64_t n, int64_t R, const double* __restrict__ ref,
                                     const int64_t* __restrict__ ofs, int64_t cols, double* __restrict__ out) {
  for (int64_t col = blockIdx.y; col < cols; col += gridDim.y) {
    const int64_t a = col / R, q = col % R;
    const double* src = ref + q * 2 * n + ofs[a];
    double* dst = out + col * n;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
      dst[i] = __ldg(src + i);
  }
}

// out[a R + q] = charge[a] * w[q]   (hf.cpp:95: nuc.charge * reference.tensor.weight)
__global__ void charge_weights_kernel(int64_t R, int64_t nnuc, const double* __restrict__ w,
                                      const double* __restrict__ charge, double* __restrict__ out) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= R * nnuc) return;
  out[idx] = charge[idx / R] * w[idx % R];
}

// out(:, c) = F(:, gi[c]) .* F(:, gj[c])   (hadamard column, tensor.cpp:153)
__global__ void hadamard_pairs_kernel(int64_t n, const double* __restrict__ F, const int* __restrict__ gi,
                                      const int* __restrict__ gj, int64_t cols, double* __restrict__ out) {
  for (int64_t c = blockIdx.y; c < cols; c += gridDim.y) {
    const double* u = F + static_cast<int64_t>(gi[c]) * n;
    const double* v = F + static_cast<int64_t>(gj[c]) * n;
    double* o = out + c * n;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
      o[i] = __ldg(u + i) * __ldg(v + i);
  }
}

// s[g * P + p] = sum_{r in segment g} w[r] T0[r, p] T1[r, p] T2[r, p]  (T* rows x P,
// column-major; segments are contiguous row ranges seg[g] .. seg[g + 1]).
// One CTA per (p, g), fixed-order tree reduction.
__global__ void __launch_bounds__(256) seg_triple_dot_kernel(int64_t rows, int P, const double* __restrict__ T0,
                                                             const double* __restrict__ T1,
                                                             const double* __restrict__ T2,
                                                             const double* __restrict__ w,
                                                             const int64_t* __restrict__ seg, double* __restrict__ s) {
  const int p = blockIdx.x, g = blockIdx.y;
  const int64_t o = static_cast<int64_t>(p) * rows;
  double acc = 0.0;
  for (int64_t r = seg[g] + threadIdx.x; r < seg[g + 1]; r += blockDim.x)
    acc += w[r] * T0[o + r] * T1[o + r] * T2[o + r];
  __shared__ double sh[256];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int st = 128; st; st >>= 1) {
    if (threadIdx.x < st) sh[threadIdx.x] += sh[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) s[static_cast<int64_t>(g) * P + p] = sh[0];
}

// Z(:, l + n s) = M_s D(:, l) with M_s = chol(:, s) viewed n x n (tei.cpp:229-230)
__global__ void block_times_d_kernel(int64_t n, int64_t R, const double* __restrict__ chol,
                                     const double* __restrict__ D, double* __restrict__ Z) {
  const int64_t tot = n * n * R;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < tot;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t mu = idx % n, l = (idx / n) % n, s = idx / (n * n);
    const double* m = chol + s * n * n + mu;
    const double* d = D + l * n;
    double acc = 0.0;
    for (int64_t nu = 0; nu < n; ++nu) acc += m[nu * n] * d[nu];
    Z[idx] = acc;
  }
}

// out = alpha (A + A^T) [+ H]: exactly symmetric (tei.cpp:224, 233).
__global__ void symmetrize_kernel(int64_t n, double alpha, const double* __restrict__ A, const double* __restrict__ H,
                                  const double* __restrict__ J, double* __restrict__ out) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= n * n) return;
  const int64_t i = idx % n, j = idx / n;
  const double v = alpha * (A[i + n * j] + A[j + n * i]);
  // fock_from_factors: (h_core + J) + K, in the reference's evaluation order (tei.cpp:237)
  out[idx] = H ? (H[idx] + J[idx]) + v : v;
}

// Per primitive pair (pi[p], pj[p]) on one axis: <u, v>, u^T tridiag{-1,2,-1} v,
// u^T tridiag{1,4,1} v / 6   (hf.cpp:13-37, 71-76).  One CTA per pair.
__global__ void __launch_bounds__(256) pair_forms_kernel(int64_t n, const double* __restrict__ F,
                                                         const int* __restrict__ pi, const int* __restrict__ pj,
                                                         double* __restrict__ out) {
  const int p = blockIdx.x;
  const double* u = F + static_cast<int64_t>(pi[p]) * n;
  const double* v = F + static_cast<int64_t>(pj[p]) * n;
  double d = 0.0, st = 0.0, ms = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double vi = v[i], vm = i > 0 ? v[i - 1] : 0.0, vp = i + 1 < n ? v[i + 1] : 0.0;
    double av = 2.0 * vi;
    if (i > 0) av -= vm;
    if (i + 1 < n) av -= vp;
    double bv = 4.0 * vi;
    if (i > 0) bv += vm;
    if (i + 1 < n) bv += vp;
    d += u[i] * vi;
    st += u[i] * av;
    ms += u[i] * bv;
  }
  __shared__ double sh[3][256];
  sh[0][threadIdx.x] = d;
  sh[1][threadIdx.x] = st;
  sh[2][threadIdx.x] = ms;
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < 3; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[3 * p + 0] = sh[0][0];
    out[3 * p + 1] = sh[1][0];
    out[3 * p + 2] = sh[2][0] / 6.0;
  }
}

// ---- generalized symmetric eigenproblem F C = S C diag(e) (hf.cpp:187-199),
// one CTA: Cholesky S = L L^T, F~ = L^-1 F^T L^-T (the reference's two
// triangular solves), B = (F~ + F~^T)/2 + sigma I with sigma = 1.5 ||B||_F so
// B is positive definite and its one-sided Jacobi SVD is its eigen-
// decomposition; e = s - sigma ascending, C = L^-T V.
// Up to kGenMax the two n x n work tiles live in shared memory; beyond it
// they are a global workspace (wk, 2 n^2 doubles) and the same code runs.
constexpr int kGenMax = 112;

__global__ void __launch_bounds__(1024) gen_eig_prep_kernel(int n, const double* __restrict__ F,
                                                            const double* __restrict__ S, double* __restrict__ Lg,
                                                            double* __restrict__ B, double* __restrict__ sigma,
                                                            int* __restrict__ fail, double* __restrict__ wk) {
  extern __shared__ double gsm[];
  double* L = wk ? wk : gsm;  // n x n, column-major, lower
  double* Y = L + n * n;      // n x n work
  __shared__ int bad;
  __shared__ double red[32];
  if (threadIdx.x == 0) bad = 0;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) L[i] = S[i];
  __syncthreads();
  for (int j = 0; j < n; ++j) {  // right-looking Cholesky (LLT of S)
    const double d = L[j + n * j];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) bad = 1;
      break;
    }
    const double r = sqrt(d);
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) L[i + n * j] /= r;
    if (threadIdx.x == 0) L[j + n * j] = r;
    __syncthreads();
    const int m = n - j - 1;
    for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
      const int i = j + 1 + t % m, k = j + 1 + t / m;
      if (i >= k) L[i + n * k] -= L[i + n * j] * L[k + n * j];
    }
    __syncthreads();
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) *fail = 1;
    return;
  }
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int r = i % n, c = i / n;
    if (r < c) L[i] = 0.0;
    Lg[i] = r < c ? 0.0 : L[i];
  }
  __syncthreads();
  // Y = L^-1 F^T (column c of F^T = row c of F), one thread per column
  for (int c = threadIdx.x; c < n; c += blockDim.x)
    for (int i = 0; i < n; ++i) {
      double s = F[c + n * i];
      for (int k = 0; k < i; ++k) s -= L[i + n * k] * Y[k + n * c];
      Y[i + n * c] = s / L[i + n * i];
    }
  __syncthreads();
  // F~ = L^-1 Y^T, written to B (global) column by column
  for (int c = threadIdx.x; c < n; c += blockDim.x)
    for (int i = 0; i < n; ++i) {
      double s = Y[c + n * i];
      for (int k = 0; k < i; ++k) s -= L[i + n * k] * B[k + n * c];
      B[i + n * c] = s / L[i + n * i];
    }
  __syncthreads();
  __threadfence_block();
  // symmetrise into Y, Frobenius norm
  double ss = 0.0;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int r = i % n, c = i / n;
    const double v = 0.5 * (B[r + n * c] + B[c + n * r]);
    Y[i] = v;
    ss += v * v;
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = 1.5 * sqrt(v) + 1e-300;
  }
  __syncthreads();
  const double sg = red[0];
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) B[i] = Y[i] + ((i % n) == (i / n) ? sg : 0.0);
  if (threadIdx.x == 0) {
    *sigma = sg;
    *fail = 0;
  }
}

// e[i] = s[n-1-i] - sigma (ascending); C(:, i) = L^-T U(:, n-1-i)
__global__ void __launch_bounds__(1024) gen_eig_finish_kernel(int n, const double* __restrict__ Lg,
                                                              const double* __restrict__ U,
                                                              const double* __restrict__ s,
                                                              const double* __restrict__ sigma, double* __restrict__ C,
                                                              double* __restrict__ e, int staged) {
  extern __shared__ double gsm[];
  const double* L = Lg;
  if (staged) {
    for (int i = threadIdx.x; i < n * n; i += blockDim.x) gsm[i] = Lg[i];
    __syncthreads();
    L = gsm;
  }
  const double sg = *sigma;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const double* u = U + static_cast<int64_t>(n - 1 - c) * n;
    e[c] = s[n - 1 - c] - sg;
    for (int i = n - 1; i >= 0; --i) {  // L^T x = u (back substitution)
      double acc = u[i];
      for (int k = i + 1; k < n; ++k) acc -= L[k + n * i] * C[k + n * c];
      C[i + n * c] = acc / L[i + n * i];
    }
  }
}

dim3 col_grid(int64_t n, int64_t cols) {
  return dim3(static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 16)),
              static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(cols, 65535))));
}

}  // namespace

// ---------------------------------------------------------------- nuclear

void nuclear_potential_dev(tgb_ctx* ctx, const tgb_cp& ref, const int64_t n[3], const int64_t* offsets,
                           const double* charges, int64_t nnuc, tgb_cp& out) {
  const int64_t R = ref.rank, cols = R * nnuc;
  if (cols == 0) return;
  Scratch so(ctx, nnuc * 3), sq(ctx, nnuc);
  std::vector<int64_t> o(3 * nnuc);
  for (int ax = 0; ax < 3; ++ax)
    for (int64_t a = 0; a < nnuc; ++a) o[ax * nnuc + a] = offsets[3 * a + ax];
  const int64_t* dofs = upload(ctx, so, o);
  const double* dq = upload(ctx, sq, std::vector<double>(charges, charges + nnuc));
  for (int ax = 0; ax < 3; ++ax) {
    window_gather_kernel<<<col_grid(n[ax], cols), 256, 0, ctx->stream>>>(n[ax], R, ref.factor[ax],
                                                                        dofs + ax * nnuc, cols, out.factor[ax]);
    TGB_LAUNCHED(ctx);
  }
  charge_weights_kernel<<<static_cast<unsigned>((cols + 255) / 256), 256, 0, ctx->stream>>>(R, nnuc, ref.weight, dq,
                                                                                          out.weight);
  TGB_LAUNCHED(ctx);
}

// ---------------------------------------------------------------- exchange

// K_km = sum_a h^3 <G_k . phi_a, (G_m . phi_a) * (P / h^3)>, then (K + K^T) / 2
// (hf.cpp:153-170).  Per orbital a, all nb Hadamard tensors g_phi[m] are one
// batch of columns (block m = the primitives of G_m x the columns of phi_a,
// column i + n_pm j as in hadamard, tensor.cpp:151); ONE batched convolution
// with the kernel writes v_m for every m, each block's columns contiguous in
// the reference's own order (local column + s_m q, tensor.cpp:191), so that
// <g_phi[k], v_m> for all k is a GEMM against block m followed by a weighted
// triple-product reduction (tensor.cpp:94-97).
void exchange_matrix_dev(tgb_ctx* ctx, const tgb_cp& basis, const int64_t* fn_offset, int64_t nb, const double* c_occ,
                         int64_t nocc, const tgb_cp& kernel, const double h[3], double* K) {
  const int64_t P = basis.rank, RN = kernel.rank;
  const double vol = h[0] * h[1] * h[2], inv_vol = 1.0 / vol;
  std::vector<double> kacc(nb * nb, 0.0);
  std::vector<double> wprim(P), wk(RN);
  if (P) TGB_CUDA(cudaMemcpy(wprim.data(), basis.weight, P * sizeof(double), cudaMemcpyDeviceToHost));
  if (RN) TGB_CUDA(cudaMemcpy(wk.data(), kernel.weight, RN * sizeof(double), cudaMemcpyDeviceToHost));
  // Mirror-symmetric kernel columns (p[i] == p[n-1-i] on every axis: every sinc column,
  // kernel.cpp:194) make the windowed convolution a symmetric Toeplitz operator, so
  // <g_c, g_c' * p> = <g_c', g_c * p>: only the blocks k <= m of K are formed and the
  // other triangle is their mirror (the reference forms both and averages, hf.cpp:169).
  bool sym_kernel = RN > 0 && !getenv("TGB_EXCHANGE_FULL");
  std::array<std::vector<double>, 3> kfh;
  for (int ax = 0; ax < 3; ++ax) {
    const int64_t n = kernel.n[ax];
    kfh[ax].resize(n * RN);
    if (n * RN)
      TGB_CUDA(cudaMemcpy(kfh[ax].data(), kernel.factor[ax], kfh[ax].size() * sizeof(double), cudaMemcpyDeviceToHost));
    const std::vector<double>& kf = kfh[ax];
    for (int64_t q = 0; q < RN && sym_kernel; ++q)
      for (int64_t i = 0; i < n / 2; ++i)
        if (kf[i + n * q] != kf[n - 1 - i + n * q]) {
          sym_kernel = false;
          break;
        }
  }
  // Bitwise-twin kernel columns (the +-t sinc nodes, kernel.cpp:194) produce identical convolved
  // columns, and K is linear in the kernel's weighted columns: convolve with the distinct columns
  // only, each weighted by the sum of its twins' weights (config-1 basis: 41 -> 21 columns, the
  // GEMM rows halve).
  std::vector<int64_t> reps;
  std::vector<double> wrep;
  for (int64_t q = 0; q < RN; ++q) {
    int64_t r = -1;
    for (size_t i = 0; i < reps.size() && r < 0; ++i) {
      bool eq = true;
      for (int ax = 0; ax < 3 && eq; ++ax) {
        const int64_t n = kernel.n[ax];
        eq = std::memcmp(kfh[ax].data() + n * reps[i], kfh[ax].data() + n * q, n * sizeof(double)) == 0;
      }
      if (eq) r = static_cast<int64_t>(i);
    }
    if (r < 0 || getenv("TGB_EXCHANGE_NO_DEDUP")) {
      reps.push_back(q);
      wrep.push_back(wk[q]);
    } else {
      wrep[r] += wk[q];
    }
  }
  const int64_t RD = static_cast<int64_t>(reps.size());
  Scratch skd(ctx, (kernel.n[0] + kernel.n[1] + kernel.n[2]) * std::max<int64_t>(RD, 1));
  const double* kfd[3];
  {
    int64_t off = 0;
    for (int ax = 0; ax < 3; ++ax) {
      double* dst = skd.p + off * RD;
      for (int64_t i = 0; i < RD; ++i)
        TGB_CUDA(cudaMemcpyAsync(dst + kernel.n[ax] * i, kernel.factor[ax] + kernel.n[ax] * reps[i],
                                 kernel.n[ax] * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
      kfd[ax] = dst;
      off += kernel.n[ax];
    }
  }
  wk = wrep;
  for (int64_t a = 0; a < nocc && RD > 0; ++a) {
    // phi_a = sum_k c_ka G_k (orbital_tensor, hf.cpp:39-46): columns = primitives of G_k, c_k != 0
    std::vector<int> phic;
    std::vector<double> wphi;
    for (int64_t k = 0; k < nb; ++k) {
      const double c = c_occ[k + nb * a];
      if (c == 0.0) continue;
      for (int64_t p = fn_offset[k]; p < fn_offset[k + 1]; ++p) {
        phic.push_back(static_cast<int>(p));
        wphi.push_back(wprim[p] * c);  // scale(): weight *= alpha (tensor.cpp:176)
      }
    }
    const int64_t rphi = static_cast<int64_t>(phic.size());
    if (rphi == 0) continue;
    // Hadamard columns of all blocks m (block m: [c0[m], c0[m + 1]))
    const int64_t G = P * rphi;
    std::vector<int> gi(G), gj(G);
    std::vector<double> wg(G);
    std::vector<int64_t> c0(nb + 1), cmap(2 * G);
    for (int64_t m = 0; m < nb; ++m) {
      c0[m] = fn_offset[m] * rphi;
      const int64_t npm = fn_offset[m + 1] - fn_offset[m];
      for (int64_t j = 0; j < rphi; ++j)
        for (int64_t i = 0; i < npm; ++i) {
          const int64_t c = c0[m] + i + npm * j;
          gi[c] = static_cast<int>(fn_offset[m] + i);
          gj[c] = phic[j];
          wg[c] = wprim[fn_offset[m] + i] * wphi[j];
          cmap[c] = RD * c0[m] + (c - c0[m]);  // v_m columns [RD c0[m], RD c0[m+1]), local col + s_m q
          cmap[G + c] = npm * rphi;
        }
    }
    c0[nb] = G;
    std::vector<double> wy(G * RD);  // weights of the convolved columns: w_g * (w_q / h^3)
    for (int64_t c = 0; c < G; ++c)
      for (int64_t q = 0; q < RD; ++q) wy[cmap[c] + cmap[G + c] * q] = wg[c] * (wk[q] * inv_vol);
    Scratch sgi(ctx, (G + 1) / 2), sgj(ctx, (G + 1) / 2), smap(ctx, 2 * G), swy(ctx, G * RD);
    const int* dgi = upload(ctx, sgi, gi);
    const int* dgj = upload(ctx, sgj, gj);
    const int64_t* dmap = upload(ctx, smap, cmap);
    const double* dwy = upload(ctx, swy, wy);
    Scratch sgp(ctx, (basis.n[0] + basis.n[1] + basis.n[2]) * G);
    Scratch sy(ctx, (basis.n[0] + basis.n[1] + basis.n[2]) * G * RD);
    double *gp[3], *y[3];
    int64_t off = 0;
    for (int ax = 0; ax < 3; ++ax) {
      gp[ax] = sgp.p + off * G;
      y[ax] = sy.p + off * G * RD;
      off += basis.n[ax];
      hadamard_pairs_kernel<<<col_grid(basis.n[ax], G), 256, 0, ctx->stream>>>(basis.n[ax], basis.factor[ax], dgi,
                                                                               dgj, G, gp[ax]);
      TGB_LAUNCHED(ctx);
    }
    const double* gpc[3] = {gp[0], gp[1], gp[2]};
    convolve_axes(ctx, 3, basis.n, G, gpc, RD, kfd, h, y, dmap);
    // groups of consecutive blocks m -> one GEMM per axis + the segmented reduction
    // symmetric kernel: small groups keep the GEMM width c0[m1] (blocks k <= m) tight
    const int64_t row_cap = sym_kernel ? std::max<int64_t>(2048, RD * (c0[nb] / std::max<int64_t>(nb, 1)) * 4)
                                       : std::max<int64_t>(8192, (int64_t(1) << 26) / std::max<int64_t>(G, 1));
    std::vector<double> s_all(nb * G);
    int64_t m0 = 0;
    while (m0 < nb) {
      int64_t m1 = m0 + 1;
      while (m1 < nb && RD * (c0[m1 + 1] - c0[m0]) <= row_cap) ++m1;
      const int64_t r0 = RD * c0[m0], rows = RD * (c0[m1] - c0[m0]);
      const int64_t Gc = sym_kernel ? c0[m1] : G;  // left columns needed: blocks k <= m (symmetric) or all
      Scratch st(ctx, 3 * rows * Gc), sseg(ctx, m1 - m0 + 1), ss(ctx, (m1 - m0) * Gc);
      std::vector<int64_t> seg(m1 - m0 + 1);
      for (int64_t m = m0; m <= m1; ++m) seg[m - m0] = RD * c0[m] - r0;
      const int64_t* dseg = upload(ctx, sseg, seg);
      double* T[3];
      // the three axis GEMMs are independent: axis 2 runs on the aux stream so its wave tail
      // overlaps axes 0-1 (only without split-K, whose workspace is shared)
      const bool fork = ((rows + 63) / 64) * ((Gc + 63) / 64) >= ctx->num_sms && !getenv("TGB_EXCHANGE_SERIAL");
      if (fork) {
        TGB_CUDA(cudaEventRecord(ctx->aux_in, ctx->stream));
        TGB_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ctx->aux_in, 0));
      }
      for (int ax = 0; ax < 3; ++ax) {
        T[ax] = st.p + ax * rows * Gc;
        StreamSwap on_aux(ctx, fork && ax == 2, ctx->aux_stream);  // restored on every exit path
        // T_ax (rows x Gc) = Y_ax(:, r0 : r0 + rows)^T GP_ax(:, 0 : Gc)
        dgemm(ctx, true, false, rows, Gc, basis.n[ax], 1.0, y[ax] + r0 * basis.n[ax], basis.n[ax], gp[ax],
              basis.n[ax], 0.0, T[ax], rows);
      }
      if (fork) {
        TGB_CUDA(cudaEventRecord(ctx->aux_done, ctx->aux_stream));
        TGB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_done, 0));
      }
      seg_triple_dot_kernel<<<dim3(static_cast<unsigned>(Gc), static_cast<unsigned>(m1 - m0)), 256, 0, ctx->stream>>>(
          rows, static_cast<int>(Gc), T[0], T[1], T[2], dwy + r0, dseg, ss.p);
      TGB_LAUNCHED(ctx);
      for (int64_t m = m0; m < m1; ++m)
        TGB_CUDA(cudaMemcpyAsync(s_all.data() + m * G, ss.p + (m - m0) * Gc, Gc * sizeof(double),
                                 cudaMemcpyDeviceToHost, ctx->stream));
      TGB_CUDA(cudaStreamSynchronize(ctx->stream));
      m0 = m1;
    }
    // K(k, m) += h^3 sum_{c in block k} w_g[c] s[m][c]   (vol * scalar_product, hf.cpp:166)
    for (int64_t m = 0; m < nb; ++m)
      for (int64_t k = 0; k < (sym_kernel ? m + 1 : nb); ++k) {
        double sp = 0.0;
        for (int64_t c = c0[k]; c < c0[k + 1]; ++c) sp += wg[c] * s_all[m * G + c];
        kacc[k + nb * m] += vol * sp;
        if (sym_kernel && k != m) kacc[m + nb * k] += vol * sp;
      }
  }
  for (int64_t m = 0; m < nb; ++m)
    for (int64_t k = 0; k < nb; ++k) K[k + nb * m] = 0.5 * (kacc[k + nb * m] + kacc[m + nb * k]);
}

// ---------------------------------------------------------------- Cholesky-factor J / K / Fock

// which: 0 Coulomb (tei.cpp:215-223), 1 exchange (tei.cpp:225-234), 2 Fock (tei.cpp:236-238).
void factor_operator_dev(tgb_ctx* ctx, int which, int64_t nb, int64_t R, const double* h_core, const double* chol,
                         const double* D, double* out) {
  const int64_t nn = nb * nb;
  if (nn == 0) return;
  // sj: raw vec_j [0, nn), symmetrised J [nn, 2 nn), L^T vec_d [2 nn, 2 nn + R)
  Scratch sj(ctx, which != 1 ? 2 * nn + std::max<int64_t>(R, 1) : 0), sk(ctx, which != 0 ? nn + nn * R : 0);
  const unsigned gb = static_cast<unsigned>((nn + 255) / 256);
  double* Js = nullptr;
  if (which != 1) {  // vec_j = L (L^T vec_d); J = (j + j^T) / 2
    double* J = sj.p;
    double* t = sj.p + 2 * nn;
    Js = which == 0 ? out : sj.p + nn;
    if (R > 0) {
      dgemm(ctx, true, false, R, 1, nn, 1.0, chol, nn, D, nn, 0.0, t, R);
      dgemm(ctx, false, false, nn, 1, R, 1.0, chol, nn, t, R, 0.0, J, nn);
    } else {
      TGB_CUDA(cudaMemsetAsync(J, 0, nn * sizeof(double), ctx->stream));
    }
    symmetrize_kernel<<<gb, 256, 0, ctx->stream>>>(nb, 0.5, J, nullptr, nullptr, Js);
    TGB_LAUNCHED(ctx);
    if (which == 0) return;
  }
  // K0 = sum_s M_s D M_s^T = Z L^T over the n R columns (Z_s = M_s D); k = -K0 / 2; K = (k + k^T) / 2
  double* K0 = sk.p;
  double* Z = sk.p + nn;
  if (R > 0) {
    const int64_t tot = nn * R;
    block_times_d_kernel<<<static_cast<unsigned>(std::min<int64_t>((tot + 255) / 256, 16 * ctx->num_sms)), 256, 0,
                           ctx->stream>>>(nb, R, chol, D, Z);
    TGB_LAUNCHED(ctx);
    dgemm(ctx, false, true, nb, nb, nb * R, -0.5, Z, nb, chol, nb, 0.0, K0, nb);
  } else {
    TGB_CUDA(cudaMemsetAsync(K0, 0, nn * sizeof(double), ctx->stream));
  }
  symmetrize_kernel<<<gb, 256, 0, ctx->stream>>>(nb, 0.5, K0, which == 2 ? h_core : nullptr, Js, out);
  TGB_LAUNCHED(ctx);
}

// ---------------------------------------------------------------- overlap / kinetic

// which: 0 overlap S_km = h^3 <G_k, G_m> (hf.cpp:48-58); 1/2 kinetic with lumped /
// exact P1 mass (hf.cpp:60-87).  Output nb x nb on the host.
void one_electron_dev(tgb_ctx* ctx, int which, const tgb_cp& basis, const int64_t* fn_offset, int64_t nb,
                      const double h[3], double* M) {
  std::vector<int> pi, pj;
  for (int64_t k = 0; k < nb; ++k)
    for (int64_t m = k; m < nb; ++m)
      for (int64_t i = fn_offset[k]; i < fn_offset[k + 1]; ++i)
        for (int64_t j = fn_offset[m]; j < fn_offset[m + 1]; ++j) {
          pi.push_back(static_cast<int>(i));
          pj.push_back(static_cast<int>(j));
        }
  const int64_t np = static_cast<int64_t>(pi.size());
  std::vector<double> w(basis.rank);
  if (basis.rank) TGB_CUDA(cudaMemcpy(w.data(), basis.weight, basis.rank * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<double> forms(3 * 3 * np);
  if (np) {
    Scratch si(ctx, (np + 1) / 2), sj(ctx, (np + 1) / 2), sf(ctx, 9 * np);
    const int* dpi = upload(ctx, si, pi);
    const int* dpj = upload(ctx, sj, pj);
    for (int ax = 0; ax < 3; ++ax) {
      pair_forms_kernel<<<static_cast<unsigned>(np), 256, 0, ctx->stream>>>(basis.n[ax], basis.factor[ax], dpi, dpj,
                                                                           sf.p + ax * 3 * np);
      TGB_LAUNCHED(ctx);
    }
    TGB_CUDA(cudaMemcpyAsync(forms.data(), sf.p, forms.size() * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  const double vol = h[0] * h[1] * h[2];
  int64_t p = 0;
  for (int64_t k = 0; k < nb; ++k)
    for (int64_t m = k; m < nb; ++m) {
      double sum = 0.0;
      for (int64_t i = fn_offset[k]; i < fn_offset[k + 1]; ++i)
        for (int64_t j = fn_offset[m]; j < fn_offset[m + 1]; ++j, ++p) {
          const double wij = w[i] * w[j];
          const double* f[3] = {&forms[0 * 3 * np + 3 * p], &forms[1 * 3 * np + 3 * p], &forms[2 * 3 * np + 3 * p]};
          if (which == 0) {  // scalar_product (tensor.cpp:94-97): w_i w_j prod_ax <u, v>
            sum += wij * (f[0][0] * f[1][0] * f[2][0]);
          } else {  // hf.cpp:71-81
            double stiff[3], mass[3];
            for (int ax = 0; ax < 3; ++ax) {
              stiff[ax] = f[ax][1] / h[ax];
              mass[ax] = which == 2 ? h[ax] * f[ax][2] : h[ax] * f[ax][0];
            }
            for (int ax = 0; ax < 3; ++ax) sum += wij * stiff[ax] * mass[(ax + 1) % 3] * mass[(ax + 2) % 3];
          }
        }
      const double v = which == 0 ? vol * sum : 0.5 * sum;
      M[k + nb * m] = v;
      M[m + nb * k] = v;
    }
}

// ---------------------------------------------------------------- density tensor

// Theta = sum_a 2 phi_a . phi_a (hf.cpp:118-127): phi_a = concatenation of
// scale(G_k, c_ka) over c_ka != 0 (orbital_tensor, hf.cpp:39-46); the
// Hadamard square has column i + R_phi j = F(:, p_i) .* F(:, p_j) and weight
// (w_i c_i)(w_j c_j) * 2 (tensor.cpp:151-153, 176), orbitals concatenated in
// order (add, tensor.cpp:159-171).  Builds the factors into `out` (device,
// rank = density_rank()) without touching the host.
int64_t density_rank(const int64_t* fn_offset, int64_t nb, const double* c_occ, int64_t nocc) {
  int64_t tot = 0;
  for (int64_t a = 0; a < nocc; ++a) {
    int64_t r = 0;
    for (int64_t k = 0; k < nb; ++k)
      if (c_occ[k + nb * a] != 0.0) r += fn_offset[k + 1] - fn_offset[k];
    tot += r * r;
  }
  return tot;
}

void density_build_dev(tgb_ctx* ctx, const tgb_cp& basis, const int64_t* fn_offset, int64_t nb, const double* c_occ,
                       int64_t nocc, tgb_cp& out) {
  const int64_t P = basis.rank;
  std::vector<double> wprim(P);
  if (P) TGB_CUDA(cudaMemcpy(wprim.data(), basis.weight, P * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<int> gi, gj;
  std::vector<double> w;
  for (int64_t a = 0; a < nocc; ++a) {
    std::vector<int> pc;
    std::vector<double> wphi;
    for (int64_t k = 0; k < nb; ++k) {
      const double c = c_occ[k + nb * a];
      if (c == 0.0) continue;
      for (int64_t p = fn_offset[k]; p < fn_offset[k + 1]; ++p) {
        pc.push_back(static_cast<int>(p));
        wphi.push_back(wprim[p] * c);
      }
    }
    const size_t r = pc.size();
    for (size_t j = 0; j < r; ++j)
      for (size_t i = 0; i < r; ++i) {
        gi.push_back(pc[i]);
        gj.push_back(pc[j]);
        w.push_back((wphi[i] * wphi[j]) * 2.0);
      }
  }
  const int64_t cols = static_cast<int64_t>(w.size());
  require(cols == out.rank, "density_tensor: output rank mismatch");
  if (cols == 0) return;
  Scratch sgi(ctx, (cols + 1) / 2), sgj(ctx, (cols + 1) / 2);
  const int* dgi = upload(ctx, sgi, gi);
  const int* dgj = upload(ctx, sgj, gj);
  TGB_CUDA(cudaMemcpyAsync(out.weight, w.data(), cols * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  for (int ax = 0; ax < 3; ++ax) {
    hadamard_pairs_kernel<<<col_grid(basis.n[ax], cols), 256, 0, ctx->stream>>>(basis.n[ax], basis.factor[ax], dgi,
                                                                                dgj, cols, out.factor[ax]);
    TGB_LAUNCHED(ctx);
  }
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));  // host index/weight vectors leave scope
}

// ---------------------------------------------------------------- generalized eigensolver

void generalized_eigensolve_dev(tgb_ctx* ctx, int64_t nb, const double* F, const double* S, double* C, double* e) {
  if (nb == 0) return;
  const int n = static_cast<int>(nb);
  const bool staged = nb <= kGenMax;
  Scratch sl(ctx, nb * nb), sb(ctx, nb * nb), ss(ctx, nb + 2), sw(ctx, staged ? 1 : 2 * nb * nb);
  const size_t smem = staged ? 2 * static_cast<size_t>(nb * nb) * sizeof(double) : 0;
  static bool attr[kTgbMaxDevices] = {};  // per device
  if (!attr[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(gen_eig_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(2 * kGenMax * kGenMax * sizeof(double))));
    TGB_CUDA(cudaFuncSetAttribute(gen_eig_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kGenMax * kGenMax * sizeof(double))));
    attr[ctx->device] = true;
  }
  double* sigma = ss.p + nb;
  int* fail = reinterpret_cast<int*>(ss.p + nb + 1);
  gen_eig_prep_kernel<<<1, 1024, smem, ctx->stream>>>(n, F, S, sl.p, sb.p, sigma, fail, staged ? nullptr : sw.p);
  TGB_LAUNCHED(ctx);
  int hfail = 0;
  TGB_CUDA(cudaMemcpyAsync(&hfail, fail, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hfail)
    throw Error(TGB_NUMERICAL_ERROR, "generalized_eigensolve: overlap not positive definite (basis near-dependence)");
  jacobi_svd_dev(ctx, n, sb.p, ss.p);
  gen_eig_finish_kernel<<<1, 1024, smem / 2, ctx->stream>>>(n, sl.p, sb.p, ss.p, sigma, C, e, staged ? 1 : 0);
  TGB_LAUNCHED(ctx);
}

}  // namespace tgb

// Internal plumbing of libtgb: context, error mapping, device workspace.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tgb.h"

namespace tgb {

// cudaFuncSetAttribute is per device: one-time flags are kept per device id
constexpr int kTgbMaxDevices = 64;

// Exceptions carry the C-ABI return code (tgb.h) and map 1:1 to the
// reference's exception types (common.hpp:11-25).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void require(bool c, const std::string& m) {
  if (!c) throw Error(TGB_INVALID_ARGUMENT, m);
}

#define TGB_CUDA(expr)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (expr);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      throw ::tgb::Error(TGB_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define TGB_LAUNCHED(ctx)                                                                           \
  do {                                                                                              \
    cudaError_t e_ = cudaGetLastError();                                                            \
    if (e_ != cudaSuccess) throw ::tgb::Error(TGB_CUDA_ERROR, std::string("launch: ") + cudaGetErrorString(e_)); \
    (ctx)->launches++;                                                                              \
  } while (0)

// Device buffer that only grows.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      if (need) {
        cudaError_t e = cudaMalloc(&p, need);
        if (e != cudaSuccess) throw Error(TGB_CUDA_ERROR, std::string("cudaMalloc: ") + cudaGetErrorString(e));
      }
      bytes = need;
    }
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct ConvPlan;  // fftconv.cu

void set_last_error(const std::string& msg);  // capi.cpp

// Scratch allocations of the reduction / TEI drivers become stream-ordered
// (pooled) on ctx->stream while one of these is alive (reduction.cu).
struct DevStreamScope {
  tgb_ctx* prev;
  explicit DevStreamScope(tgb_ctx* ctx);
  ~DevStreamScope();
};
void* scratch_alloc(tgb_ctx* ctx, size_t bytes, size_t* got);
// host <-> device copies; pageable host memory is staged through pinned chunks (hostcopy.cpp)
void h2d(tgb_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t stream);
void d2h(tgb_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t stream);
bool is_pageable(const void* p);
void par_memcpy(void* dst, const void* src, size_t bytes);  // host threads
// replication of freshly landed D2H pieces: spinning threads, non-temporal stores (hostcopy.cpp)
void stream_copy_begin();
void stream_copy(void* dst, const void* src, size_t bytes);
void stream_copy_end();
void scratch_free(tgb_ctx* ctx, void* p, size_t bytes);

// Run f, mapping exceptions to the C-ABI return codes (tgb.h).
template <class F>
int guarded_call(F&& f) {
  try {
    f();
    return TGB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return TGB_CUDA_ERROR;
  }
}

}  // namespace tgb

struct tgb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;
  cudaStream_t aux_stream = nullptr;  // kernel-column grouping, overlapped with the spectra
  cudaEvent_t aux_in = nullptr, aux_done = nullptr;
  void* pinned_flags = nullptr;
  size_t pinned_flags_bytes = 0;
  bool own_stream = false;
  int64_t launches = 0;
  int64_t direct_max = 64;
  int num_sms = 148;
  size_t smem_optin = 232448;
  // workspaces (named so independent stages never alias)
  tgb::DevBuf ws_spec_a, ws_spec_b, ws_pairs, ws_flags, ws_in, ws_out, ws_misc, ws_misc2, ws_misc3, ws_gemm;
  std::vector<cudaEvent_t> events;
  bool profiling = false;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  cudaEvent_t pinned_event = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
  size_t prof_used = 0;
  std::map<int64_t, std::shared_ptr<tgb::ConvPlan>> plans;
  std::multimap<size_t, void*> scratch_free;  // cached Dev blocks (reduction.cu)
  void* stage_pin[2] = {nullptr, nullptr};     // pinned chunks for pageable host copies (hostcopy.cpp)
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  // per-context named device workspaces of the TEI / HF drivers (device
  // pointers are never shared across contexts or devices)
  std::map<std::string, tgb::DevBuf> named;
  std::map<std::string, std::array<tgb::DevBuf, 3>> named3;
  // multi-GPU (comm.cpp): a libtgb-owned NCCL communicator or a caller's tgb_comm
  void* nccl_comm = nullptr;  // ncclComm_t (tgb_ctx_init_nccl)
  bool own_nccl = false;
  tgb_comm user_comm{};
  int comm_rank = 0, comm_size = 1;
  // bytes moved between host and device by host-memory calls (tgb_ctx_transfer_bytes)
  int64_t bytes_h2d = 0, bytes_d2h = 0;
};

namespace tgb {
// comm.cpp: sums over the context's ranks (no-ops on a single process)
void comm_allreduce(tgb_ctx* ctx, double* buf, int64_t count, bool on_device);
void symmetric_allreduce_host(const tgb_comm* c, tgb_ctx* ctx, double* J, int64_t nb);
void shard_range(int64_t total, int rank, int world, int64_t* lo, int64_t* hi);
void comm_release(tgb_ctx* ctx);
// assembly.cu: bitwise equality of two device double arrays (synchronises the context stream)
bool device_equal(tgb_ctx* ctx, const double* x, const double* y, int64_t count);
// a named per-context workspace (replaces function-static buffers)
inline DevBuf& ctx_buf(tgb_ctx* ctx, const std::string& name) { return ctx->named[name]; }
inline std::array<DevBuf, 3>& ctx_buf3(tgb_ctx* ctx, const std::string& name) { return ctx->named3[name]; }

// Runs a section of work on another stream of the context and restores
// ctx->stream on every exit path (exceptions included).
struct StreamSwap {
  tgb_ctx* ctx;
  cudaStream_t saved;
  StreamSwap(tgb_ctx* c, bool on, cudaStream_t s) : ctx(c), saved(c->stream) {
    if (on) ctx->stream = s;
  }
  ~StreamSwap() { ctx->stream = saved; }
};

// bracket a hot-kernel launch with timing events when profiling is enabled
inline void prof_begin(tgb_ctx* ctx) {
  if (!ctx->profiling) return;
  if (ctx->prof_used == ctx->prof_events.size()) {
    cudaEvent_t a, b;
    TGB_CUDA(cudaEventCreate(&a));
    TGB_CUDA(cudaEventCreate(&b));
    ctx->prof_events.push_back({a, b});
  }
  TGB_CUDA(cudaEventRecord(ctx->prof_events[ctx->prof_used].first, ctx->stream));
}
inline void prof_end(tgb_ctx* ctx) {
  if (!ctx->profiling) return;
  TGB_CUDA(cudaEventRecord(ctx->prof_events[ctx->prof_used].second, ctx->stream));
  ctx->prof_used++;
}
void convolve_axis(tgb_ctx* ctx, int64_t n, int64_t ra, const double* A, int64_t rb, const double* B, double h,
                   double* out);
// colmap (device, optional): 2 ra entries; density column i's result for
// kernel column j goes to output column colmap[i] + colmap[ra + i] * j
// instead of i + ra * j.
// wout (optional): the output weights wout[i + ra j] = wa[i] * (wscale != 1 ? wb[j] * wscale : wb[j]),
// as weights_outer, computed inside the first launch where the small plan fuses it.
void convolve_axes(tgb_ctx* ctx, int naxes, const int64_t* n, int64_t ra, const double* const* A, int64_t rb,
                   const double* const* B, const double* h, double* const* out, const int64_t* colmap = nullptr,
                   const double* wa = nullptr, const double* wb = nullptr, double wscale = 1.0,
                   double* wout = nullptr);
void conv_central_many_dev(tgb_ctx* ctx, int64_t n, int64_t cols, const double* U, const double* v, double* out);
void weights_outer(tgb_ctx* ctx, int64_t ra, const double* wa, int64_t rb, const double* wb, double scale, double* out);
double scalar_product_dev(tgb_ctx* ctx, const tgb_cp& a, const tgb_cp& b);
void coulomb_matrix_dev(tgb_ctx* ctx, const tgb_cp& basis, const int64_t* fn_offset, int64_t nb, const tgb_cp& vh,
                        double vol, double* J);
// spectrum.cu: full spectra of RHOSVD mode matrices (mode_singular_values)
void sym_eigvals_dev(tgb_ctx* ctx, int64_t m, double* G, double* lam);
std::vector<double> mode_spectrum_dev(tgb_ctx* ctx, int64_t n, int64_t R, const double* W);
std::vector<double> cp_mode_spectrum(tgb_ctx* ctx, const tgb_cp& a, int axis);
void dgemm(tgb_ctx* ctx, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
           int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc);
void orthonormalize_columns(tgb_ctx* ctx, int64_t d, int p, double* X);
void value_at_dev(tgb_ctx* ctx, const tgb_cp& t, int64_t npts, const int64_t* ijk, double* out);
void lattice_assemble_dev(tgb_ctx* ctx, int64_t n, int64_t R, const double* ref, const int64_t* offsets, int64_t L,
                          double* out);
// reduction.cu
void jacobi_svd_dev(tgb_ctx* ctx, int p, double* S, double* sg);
int64_t thin_svd_left_dev(tgb_ctx* ctx, int64_t rows, int64_t cols, const double* A, double* U, double* sigma);
// tei.cu
int64_t pivoted_cholesky_dev(tgb_ctx* ctx, int64_t n, const double* A, double tol, bool trace_stop,
                             int64_t max_rank, double neg_tol, double* L, int64_t* pivots_host, double* residual,
                             bool* clamped);
// mp2.cu
void mo_transform_dev(tgb_ctx* ctx, int64_t nb, int64_t R, const double* chol, int64_t n_occ, const double* C,
                      double* out);
double mp2_energy_dev(tgb_ctx* ctx, int64_t n_occ, int64_t n_vir, int64_t R, const double* F, const double* e_host,
                      int mode, double expsum_eps);
// hf.cu
int64_t density_rank(const int64_t* fn_offset, int64_t nb, const double* c_occ, int64_t nocc);
void density_build_dev(tgb_ctx* ctx, const tgb_cp& basis, const int64_t* fn_offset, int64_t nb, const double* c_occ,
                       int64_t nocc, tgb_cp& out);
void generalized_eigensolve_dev(tgb_ctx* ctx, int64_t nb, const double* F, const double* S, double* C, double* e);
void nuclear_potential_dev(tgb_ctx* ctx, const tgb_cp& ref, const int64_t n[3], const int64_t* offsets,
                           const double* charges, int64_t nnuc, tgb_cp& out);
void exchange_matrix_dev(tgb_ctx* ctx, const tgb_cp& basis, const int64_t* fn_offset, int64_t nb, const double* c_occ,
                         int64_t nocc, const tgb_cp& kernel, const double h[3], double* K);
void factor_operator_dev(tgb_ctx* ctx, int which, int64_t nb, int64_t R, const double* h_core, const double* chol,
                         const double* D, double* out);
void one_electron_dev(tgb_ctx* ctx, int which, const tgb_cp& basis, const int64_t* fn_offset, int64_t nb,
                      const double h[3], double* M);
}  // namespace tgb

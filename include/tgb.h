/* tgb.h — C ABI of the B200-native tengrid hot path.
 *
 * Drop-in boundary for the canonical/Tucker Newton-kernel convolution path of
 * the reference library `tengrid` (/root/reference/proj).  Each entry point
 * names the reference function it replaces.  All matrices are column-major
 * (Eigen's default layout: entry (i, j) at p[i + rows * j]) so an
 * Eigen::MatrixXd::data() pointer can be passed straight through.
 *
 * Memory: every call takes `mem` = TGB_MEM_HOST or TGB_MEM_DEVICE and ALL
 * pointers of that call live in that space.  Host calls stage through the
 * context's device workspace (host<->device copies are part of the call);
 * device calls are stream-ordered on the context stream and return without a
 * device synchronisation unless a result is a host scalar.  Buffers are
 * caller-allocated and nothing is retained past the call.
 *
 * Errors: return code 0 ok, 1 invalid_argument, 2 domain_error, 3 snap error,
 * 4 numerical error, 5 CUDA/NCCL error; tgb_last_error() gives a per-thread
 * message.  The C++ wrapper (include/tengrid_b200/tengrid.hpp) rethrows the
 * reference's exception types (common.hpp:11-25).
 */
#ifndef TGB_H
#define TGB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TGB_OK 0
#define TGB_INVALID_ARGUMENT 1
#define TGB_DOMAIN_ERROR 2
#define TGB_SNAP_ERROR 3
#define TGB_NUMERICAL_ERROR 4
#define TGB_CUDA_ERROR 5

#define TGB_MEM_HOST 0
#define TGB_MEM_DEVICE 1

typedef struct tgb_ctx tgb_ctx;
typedef struct tgb_tucker tgb_tucker; /* device-resident Tucker result (rank reduction, below) */

/* Rank-R canonical tensor sum_k w_k u_k^(1) x u_k^(2) x u_k^(3)
 * (reference CanonicalTensor3, proj/include/tengrid/tensor.hpp:119-150). */
typedef struct tgb_cp {
  int64_t n[3];      /* extent per axis */
  int64_t rank;      /* R */
  double* factor[3]; /* n[ax] x R, column-major */
  double* weight;    /* R */
} tgb_cp;

/* A communicator for the multi-GPU path (one process per GPU):
 * allreduce_sum sums `count` doubles in place over all ranks (device memory on
 * the cudaStream_t `stream` when on_device, else host memory) and returns 0 on
 * success.  libtgb also owns an NCCL communicator itself (tgb_ctx_init_nccl);
 * a tgb_comm lets any other backend (MPI, torch.distributed, gloo) stand in. */
typedef struct tgb_comm {
  int rank;
  int world;
  int (*allreduce_sum)(double* buf, int64_t count, int on_device, void* stream, void* user);
  void* user;
} tgb_comm;

/* ---- context -------------------------------------------------------------
 * One CUDA stream per context (`stream` = a cudaStream_t, or NULL for a
 * context-owned stream).  Calls are reentrant across contexts. */
int tgb_ctx_create(int device, void* stream, tgb_ctx** out);
int tgb_ctx_destroy(tgb_ctx* ctx);
void* tgb_ctx_stream(tgb_ctx* ctx);
int tgb_ctx_synchronize(tgb_ctx* ctx);
const char* tgb_last_error(void);
/* Kernel launches issued by this context since creation (or the last reset). */
int64_t tgb_ctx_launch_count(tgb_ctx* ctx);
void tgb_ctx_reset_launch_count(tgb_ctx* ctx);
/* Live kernel timing for bench.py: when enabled, every launch of the pair
 * (inverse FFT) convolution kernel is bracketed by CUDA events on the context
 * stream; tgb_ctx_profile_read synchronises, returns the summed device time
 * (ms) and launch count since the last read, and resets them. */
int tgb_ctx_set_profiling(tgb_ctx* ctx, int enabled);
int tgb_ctx_profile_read(tgb_ctx* ctx, double* total_ms, int64_t* launches);
/* Bytes host-memory calls moved host->device and device->host since the last
 * read (then reset).  Bitwise-twin output blocks of tgb_convolve /
 * tgb_hartree_potential cross PCIe once and are replicated on the host. */
int tgb_ctx_transfer_bytes(tgb_ctx* ctx, int64_t* h2d, int64_t* d2h);
/* Tuning / testing knob: 1D convolutions with n <= direct_max use direct
 * summation (reference: kFftConvThreshold = 128, fft.hpp:13).  Default 64;
 * 0 forces the FFT path wherever it exists. */
int tgb_ctx_set_direct_max(tgb_ctx* ctx, int64_t direct_max);

/* ---- multi-GPU ---------------------------------------------------------------
 * No reference counterpart (the reference is one CPU process).  The mode
 * convolutions shard by density column: rank r owns columns [lo, hi) of
 * tgb_shard_range(theta.rank, r, world) and produces its (hi - lo) * R_b output
 * columns with no exchange.  Sums over all pairs (V_H at points, J) take ONE
 * all-reduce over the context's communicator; the TEI convolution matrices
 * (by kernel term) and diagonal (by pair row) likewise.
 * tgb_ctx_init_nccl: rank 0 calls tgb_nccl_get_unique_id and distributes the
 * 128 bytes; every rank then creates the libtgb-owned NCCL communicator.
 * tgb_ctx_set_comm: a caller-provided communicator (NULL detaches). */
int tgb_shard_range(int64_t total, int rank, int world, int64_t* lo, int64_t* hi);
int tgb_nccl_get_unique_id(unsigned char id[128]);
int tgb_ctx_init_nccl(tgb_ctx* ctx, int rank, int world, const unsigned char id[128]);
int tgb_ctx_set_comm(tgb_ctx* ctx, const tgb_comm* comm);
int tgb_ctx_comm_info(tgb_ctx* ctx, int* rank, int* world);
/* Context-free helpers (host buffers): the sum, and the sum followed by the
 * exact mirror of the upper triangle that keeps J symmetric (hf.cpp:145-149)
 * whatever order the all-reduce summed J_km and J_mk in. */
int tgb_comm_allreduce_host(const tgb_comm* comm, double* buf, int64_t count);
int tgb_symmetric_allreduce_host(const tgb_comm* comm, double* J, int64_t nb);

/* ---- mode convolutions -----------------------------------------------------
 * replaces tg::conv_central_many (proj/include/tengrid/fft.hpp:30,
 * proj/src/fft.cpp:97-122): out(:, c) = central_window(conv_full(U(:, c), v)). */
int tgb_conv_central_many(tgb_ctx* ctx, int64_t n, int64_t cols, const double* U, const double* v, double* out,
                          int mem);

/* replaces tg::convolve(a, b, h) (tensor.hpp:185-186, tensor.cpp:179-198).
 * `out` must have rank a.rank * b.rank; column i + a.rank * j of every factor
 * is h[ax] * conv_central(a_i, b_j); weight = a.w[i] * b.w[j].
 * Device memory: axes of b that point at the SAME factor matrix (the Newton kernel on a cubic
 * grid) with the same h share one set of kernel spectra. */
int tgb_convolve(tgb_ctx* ctx, const tgb_cp* a, const tgb_cp* b, const double h[3], tgb_cp* out, int mem);

/* replaces tg::hartree_potential (hf.hpp:34-39, hf.cpp:131-138):
 * convolve(theta, kernel with weights / (h0 h1 h2), h).  `kernel` must be a
 * primary-grid kernel tensor (doubled kernels are rejected by the caller). */
int tgb_hartree_potential(tgb_ctx* ctx, const tgb_cp* theta, const tgb_cp* kernel, const double h[3], tgb_cp* out,
                          int mem);

/* Multi-GPU tg::hartree_potential: this rank's density-column block [lo, hi)
 * (tgb_shard_range over theta->rank with the context's rank / world) convolved
 * with the whole kernel; `out` has rank (hi - lo) * kernel->rank, column
 * (i - lo) + (hi - lo) j.  No communication; a single process gets the full
 * result (identical to tgb_hartree_potential). */
int tgb_hartree_potential_shard(tgb_ctx* ctx, const tgb_cp* theta, const tgb_cp* kernel, const double h[3],
                                tgb_cp* out, int mem);

/* replaces CanonicalTensor3::value_at (tensor.hpp:135-140) for a batch of
 * grid points: out[p] = sum_k w_k f0(i_p,k) f1(j_p,k) f2(l_p,k); ijk is
 * npts x 3 (row-major triples), both in the space given by `mem`. */
int tgb_value_at(tgb_ctx* ctx, const tgb_cp* t, int64_t npts, const int64_t* ijk, double* out, int mem);

/* value_at of a sharded tensor: each rank evaluates its own columns, then one
 * all-reduce (the sum over all rank pairs) leaves the full values on every rank. */
int tgb_value_at_allreduce(tgb_ctx* ctx, const tgb_cp* t_shard, int64_t npts, const int64_t* ijk, double* out,
                           int mem);

/* ---- canonical-tensor algebra (tensor.hpp:173-177, tensor.cpp:141-177) -------
 * replaces tg::hadamard: out rank a.rank * b.rank, column i + a.rank j =
 * a_i .* b_j per axis, weight a.w[i] b.w[j];  tg::add: out rank a.rank + b.rank,
 * [a | b];  tg::scale: weights times alpha.  `out` caller-allocated; all
 * element-wise, bit-identical to the reference. */
int tgb_hadamard(tgb_ctx* ctx, const tgb_cp* a, const tgb_cp* b, tgb_cp* out, int mem);
int tgb_add(tgb_ctx* ctx, const tgb_cp* a, const tgb_cp* b, tgb_cp* out, int mem);
int tgb_scale(tgb_ctx* ctx, const tgb_cp* a, double alpha, tgb_cp* out, int mem);

/* ---- assembly --------------------------------------------------------------
 * replaces tg::scalar_product(CanonicalTensor3, CanonicalTensor3)
 * (tensor.hpp:173, tensor.cpp:88-98).  Result written to *result (host). */
int tgb_scalar_product(tgb_ctx* ctx, const tgb_cp* a, const tgb_cp* b, double* result, int mem);

/* replaces tg::coulomb_matrix (hf.hpp:41-44, hf.cpp:140-151):
 * J_km = h0 h1 h2 <G_k . G_m, V_H> for k <= m, mirrored.  The basis is given
 * flattened: `basis` holds all primitives of all functions as one CP tensor
 * (rank = total primitives, weights = contraction coeff * primitive norm),
 * fn_offset[k] .. fn_offset[k+1]-1 are the primitives of function k
 * (nb + 1 entries, host memory).  J is nb x nb (space given by `mem`). */
int tgb_coulomb_matrix(tgb_ctx* ctx, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb, const tgb_cp* vh,
                       const double h[3], double* J, int mem);
/* Multi-GPU coulomb_matrix: the partial J over this rank's V_H columns, one
 * all-reduce of the N_b x N_b partials, then the exact mirror. */
int tgb_coulomb_matrix_allreduce(tgb_ctx* ctx, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb,
                                 const tgb_cp* vh_shard, const double h[3], double* J, int mem);

/* ---- Hartree-Fock operators on the same path -------------------
 * replaces tg::nuclear_potential_tensor (hf.hpp:29-30, hf.cpp:89-101):
 * P_c = sum_a Z_a W_a Ptilde.  `reference` is the DOUBLED-grid kernel tensor
 * (2 n[ax] x R per axis); `offsets` (nnuc x 3, row-major, host memory) are
 * tg::window_for_center(grid, center_a).offset and `charges` (nnuc, host) the
 * nuclear charges.  `out` has extents n[ax] = reference.n[ax] / 2 and rank
 * nnuc R: columns a R + q = reference(offset_a : offset_a + n, q), weights
 * charge_a * reference.w[q] (the reference's add() order). */
int tgb_nuclear_potential_tensor(tgb_ctx* ctx, const tgb_cp* reference, const int64_t* offsets,
                                 const double* charges, int64_t nnuc, tgb_cp* out, int mem);

/* replaces tg::nuclear_matrix (hf.hpp:25-26, hf.cpp:103-116):
 * V_km = -<G_k . G_m, P_c> for k <= m, mirrored.  Basis flattened as for
 * tgb_coulomb_matrix; `pc` from tgb_nuclear_potential_tensor. */
int tgb_nuclear_matrix(tgb_ctx* ctx, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb, const tgb_cp* pc,
                       double* V, int mem);

/* replaces tg::exchange_matrix (hf.hpp:49-50, hf.cpp:153-170):
 * K_km = sum_a h^3 <G_k . phi_a, (G_m . phi_a) * (P / h^3)>, returned as
 * (K + K^T) / 2.  c_occ is nb x nocc (column-major, space given by `mem`);
 * `kernel` is a PRIMARY-grid kernel tensor (doubled kernels are rejected by
 * the caller, hf.cpp:155). */
int tgb_exchange_matrix(tgb_ctx* ctx, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb,
                        const double* c_occ, int64_t nocc, const tgb_cp* kernel, const double h[3], double* K,
                        int mem);

/* replace tg::coulomb_from_factors / exchange_from_factors / fock_from_factors
 * (tei.hpp:76-79, tei.cpp:215-238).  chol is the TEI Cholesky factor
 * (nb^2 x rank, column-major), density and h_core nb x nb; the result is nb x nb
 * and exactly symmetric.  All pointers in the space given by `mem`. */
int tgb_coulomb_from_factors(tgb_ctx* ctx, int64_t nb, int64_t rank, const double* chol, const double* density,
                             double* J, int mem);
int tgb_exchange_from_factors(tgb_ctx* ctx, int64_t nb, int64_t rank, const double* chol, const double* density,
                              double* K, int mem);
int tgb_fock_from_factors(tgb_ctx* ctx, int64_t nb, int64_t rank, const double* h_core, const double* chol,
                          const double* density, double* F, int mem);

/* replaces tg::generalized_eigensolve (hf.hpp:94-95, hf.cpp:187-199):
 * F C = S C diag(e) by the Cholesky congruence of S; e ascending, columns of C
 * S-orthonormal (eigenvector signs are not fixed, as in the reference).
 * One CTA (work tiles in shared memory up to nb = 112, global beyond).
 * NUMERICAL_ERROR when S is not positive definite. */
int tgb_generalized_eigensolve(tgb_ctx* ctx, int64_t nb, const double* F, const double* S, double* C, double* e,
                               int mem);

/* ---- restricted closed-shell SCF on the grid (hf.hpp:54-91, hf.cpp:172-270) ----
 * replaces tg::scf_solve: snapped nuclei, overlap / kinetic / nuclear matrices,
 * Newton kernel from tg::expsum_for_interval(1.5 h_min, r_max, kernel_eps), the
 * factorised TEI (build_tei), then the Roothaan iterations with
 * fock_from_factors / generalized_eigensolve / linear density mixing, all on
 * the device.  Inputs and outputs are HOST memory. */
typedef struct tgb_scf_config { /* SCFConfig, hf.hpp:54-64 (same defaults) */
  int max_iterations;           /* 60 */
  double energy_tol;            /* 1e-9 */
  double mixing;                /* 0.7 */
  double eps_fit;               /* 1e-8 */
  double eps_chol;              /* 1e-10 */
  double kernel_eps;            /* 1e-6 */
  double kernel_r_max;          /* 0: the box diagonal */
  double density_reduce_eps;    /* 1e-7 (unused by the SCF loop, as in the reference) */
  int exact_mass_kinetic;       /* 0 */
} tgb_scf_config;

typedef struct tgb_basis_spec { /* BasisSet, basis.hpp:18-35 */
  double b_half[3];
  int64_t n[3];
  int64_t nfn;
  const double* centers;      /* nfn x 3, row-major */
  const int* degrees;         /* nfn x 3, row-major, each 0 or 1 */
  const int64_t* prim_offset; /* nfn + 1 */
  const double* exponents;    /* prim_offset[nfn] */
  const double* coeffs;
} tgb_basis_spec;

typedef struct tgb_molecule { /* Molecule, basis.hpp:37-52 */
  int64_t nnuc;
  const double* charges; /* nnuc */
  const double* centers; /* nnuc x 3, row-major */
  int64_t n_electrons;
} tgb_molecule;

typedef struct tgb_scf_state { /* SCFState, hf.hpp:66-88; arrays caller-allocated (NULL: not returned) */
  double energy, nuclear_energy;
  int converged, iterations, n_occupied;
  int64_t tei_rank_b;             /* 0 for one electron */
  int64_t kernel_m;               /* quadrature M from expsum_for_interval */
  double kernel_c0;
  double* coefficients;           /* nb x nb */
  double* orbital_energies;       /* nb */
  double* density;                /* nb x nb */
  double* overlap, *kinetic, *nuclear, *core_hamiltonian; /* nb x nb each */
  double* energy_history;         /* max_iterations */
  double* residual_history;       /* max_iterations */
  double* orthonormality_defects; /* max_iterations */
  double* snapped_centers;        /* nnuc x 3 */
} tgb_scf_state;

void tgb_scf_config_default(tgb_scf_config* cfg);
int tgb_scf_solve(tgb_ctx* ctx, const tgb_molecule* mol, const tgb_basis_spec* basis, const tgb_scf_config* cfg,
                  tgb_scf_state* out);

/* ---- MP2 on the factorised TEI (mp2.hpp:8-57, mp2.cpp:7-105) ----------------
 * replaces tg::mo_transform_cholesky: out (N_ov x rank, row i n_vir + a) holds
 * C_occ^T mat(L_s) C_vir for every Cholesky column s; coefficients nb x nb
 * (occupied columns first).  chol is nb^2 x rank. */
int tgb_mo_transform_cholesky(tgb_ctx* ctx, int64_t nb, int64_t rank, const double* chol, int64_t n_occ,
                              const double* coefficients, double* out, int mem);
/* replaces tg::mp2_energy: mode 0 = MP2Mode::oracle (exact denominators), 1 =
 * MP2Mode::factorized (exponential-sum denominators at expsum_eps).  mo_factor
 * N_ov x rank (space given by `mem`); energies nb ascending (HOST memory);
 * result in *energy (host). */
int tgb_mp2_energy(tgb_ctx* ctx, int64_t n_occ, int64_t n_vir, int64_t rank, const double* mo_factor,
                   const double* energies, int mode, double expsum_eps, double* energy, int mem);

/* replaces tg::overlap_matrix (hf.hpp:14, hf.cpp:48-58): S_km = h^3 <G_k, G_m>. */
int tgb_overlap_matrix(tgb_ctx* ctx, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb, const double h[3],
                       double* S, int mem);
/* replaces tg::kinetic_matrix (hf.hpp:19-20, hf.cpp:60-87): Kronecker FEM
 * Laplacian, lumped (exact_mass = 0) or P1 (exact_mass = 1) mass on the
 * non-derivative axes. */
int tgb_kinetic_matrix(tgb_ctx* ctx, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb, const double h[3],
                       int exact_mass, double* T, int mem);

/* replaces tg::density_tensor (hf.hpp:34-35, hf.cpp:118-129) with the tensor
 * built on the device: Theta = sum_a 2 phi_a . phi_a from the flattened basis
 * and c_occ (nb x nocc, HOST memory), then reduce_rank(reduce_eps) (RHOSVD +
 * ALS + T2C) on the device when rank > 1 and reduce_eps > 0.
 *  - tgb_density_rank: the unreduced rank sum_a R_phi_a^2;
 *  - tgb_density_build: the unreduced Theta into `out` (rank = that value);
 *  - tgb_density_reduce: build + canonical_to_tucker; *out receives the
 *    Tucker handle (tgb_tucker_info / tgb_tucker_to_canonical as for
 *    tgb_reduce_tucker, max_sweeps 3 as ReductionConfig::tolerance). */
int tgb_density_rank(const int64_t* fn_offset, int64_t nb, const double* c_occ, int64_t nocc, int64_t* rank);
int tgb_density_build(tgb_ctx* ctx, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb, const double* c_occ,
                      int64_t nocc, tgb_cp* out, int mem);
int tgb_density_reduce(tgb_ctx* ctx, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb, const double* c_occ,
                       int64_t nocc, double reduce_eps, int mem, tgb_tucker** out);

/* ---- factorised two-electron integrals (proj/include/tengrid/tei.hpp:38-72) ----
 * A tgb_tei holds the device-resident factorisation (TEIFactorization,
 * tei.hpp:38-57).  The basis is given flattened as for tgb_coulomb_matrix
 * (all primitives of all functions as one CP tensor, weights = contraction
 * coefficient x primitive norm; fn_offset has nb + 1 entries, host memory).
 * Pair indices: primitive (p, q) -> p + n_prim q; contracted (mu, nu) -> mu + nb nu. */
typedef struct tgb_tei tgb_tei;
int tgb_tei_create(tgb_tei** out);
int tgb_tei_destroy(tgb_tei* t);
/* replaces tg::tei_density_fitting (tei.hpp:60-61, tei.cpp:92-143) */
int tgb_tei_density_fitting(tgb_ctx* ctx, tgb_tei* t, const tgb_cp* basis, const int64_t* fn_offset, int64_t nb,
                            const double h[3], double eps_fit, int mem);
/* replaces tg::tei_convolution_matrices (tei.hpp:62, tei.cpp:145-158); primary-grid kernel */
int tgb_tei_convolution_matrices(tgb_ctx* ctx, tgb_tei* t, const tgb_cp* kernel, int mem);
/* replaces tg::tei_diagonal (tei.hpp:66, tei.cpp:182-196): nb^2 entries */
int tgb_tei_diagonal(tgb_ctx* ctx, tgb_tei* t, double* out, int mem);
/* replaces tg::tei_column (tei.hpp:65, tei.cpp:160-174): nb^2 entries */
int tgb_tei_column(tgb_ctx* ctx, tgb_tei* t, int64_t pair_index, double* out, int mem);
/* replaces tg::tei_cholesky (tei.hpp:67, tei.cpp:198-204): max-diagonal stop at eps_chol */
int tgb_tei_cholesky(tgb_ctx* ctx, tgb_tei* t, double eps_chol);
/* info[0..2] fit ranks R_l, [3] n_prim, [4] nb, [5] R_B, [6] fit_clamped_negative, [7] kernel terms */
int tgb_tei_info(tgb_tei* t, int64_t* info, double* fit_residual);
int tgb_tei_get_fit(tgb_tei* t, int axis, double* U, double* V, int mem);  /* U n x R_l, V n_prim^2 x R_l */
int tgb_tei_get_conv(tgb_tei* t, int64_t k, int axis, double* M, int mem); /* R_l x R_l */
int tgb_tei_get_cholesky(tgb_tei* t, double* L, int64_t* pivots, int mem); /* nb^2 x R_B; pivots host */

/* ---- rank reduction (proj/include/tengrid/reduction.hpp:12-67) --------------
 * tgb_reduce_tucker runs rhosvd (mode 0) or canonical_to_tucker = RHOSVD + ALS
 * (mode 1) on the device; ReductionConfig is (use_eps, eps) or ranks[3], plus
 * max_sweeps.  The result (TuckerResult) stays on the device; read it with
 * tgb_tucker_info / _get / _sigma, or convert it with tgb_tucker_to_canonical
 * (tucker_to_canonical, reduction.cpp:238-269; reduce_rank = mode 1 + T2C).
 * Singular values are the leading ones the rank rule needed; mode + 2 also
 * computes each RHOSVD mode matrix's FULL spectrum (TuckerResult::
 * mode_singular_values, reduction.hpp:42), which tgb_tucker_sigma then returns. */
typedef struct tgb_tucker tgb_tucker;
int tgb_reduce_tucker(tgb_ctx* ctx, const tgb_cp* a, int use_eps, double eps, const int64_t* ranks, int max_sweeps,
                      int mode, int mem, tgb_tucker** out);
int tgb_tucker_destroy(tgb_tucker* t);
/* info[0..2] Tucker ranks, [3] rank_clamped, [4] rhosvd_fallback, [5] ALS sweeps run, [6] T2C canonical rank */
int tgb_tucker_info(tgb_tucker* t, int64_t* info);
int tgb_tucker_get(tgb_tucker* t, double* core, double* side0, double* side1, double* side2, double* sweep_fits,
                   int mem);
int tgb_tucker_sigma(tgb_tucker* t, int axis, int64_t* count, double* sigma);
/* Rank-selection margins of mode `axis` (RHOSVD's initializing SVD, the
 * reference's select_rank, reduction.cpp:34-59): out[6] = {r, sigma_{r-1},
 * sigma_r (-1: not formed), sigma_{r-1}/sigma_r, tail(r-1)/budget,
 * tail(r)/budget} with budget = eps^2 sum sigma^2 (tail ratios -1 in
 * fixed-rank mode).  A rank is robust when the last ratio is well below 1 and
 * the one before well above it. */
int tgb_tucker_margins(tgb_tucker* t, int axis, double* out);
int tgb_tucker_to_canonical(tgb_ctx* ctx, tgb_tucker* t, tgb_cp* out, int mem);

/* TuckerResult::mode_singular_values of rhosvd(a) for one mode (reduction.hpp:42,
 * reduction.cpp:172-190 with thin_svd_left's branches, :85-138): the singular
 * values of W = f_axis diag(w) of normalize(a), descending; min(n_axis, rank)
 * of them, except the tall Gram branch (n >= 4 R, R >= 8), which keeps
 * lambda > lambda_max 1e-24.  sigma: min(n_axis, rank) doubles, host; *count =
 * values written.  Device Gram + Householder tridiagonalisation (one
 * cooperative grid) + bisection; sigma_i carries ~eps m sigma_0^2 / sigma_i
 * absolute error (Gram spectrum).  a in space `mem`. */
int tgb_mode_spectrum(tgb_ctx* ctx, const tgb_cp* a, int axis, int mem, int64_t* count, double* sigma);

/* replaces tg::thin_svd_left (reduction.hpp:67, reduction.cpp:85-138):
 * left singular pairs of a rows x cols matrix A (column-major, space `mem`),
 * sigma descending.  U needs rows x min(rows, cols), sigma min(rows, cols)
 * entries; *kept = the pairs returned under the reference's branch rule
 * (all min(rows, cols) except the tall Gram branch, which keeps sigma^2 >
 * sigma_0^2 1e-24).  Device one-sided Jacobi, any size.  Singular-vector
 * signs are not fixed (as in the reference). */
int tgb_thin_svd_left(tgb_ctx* ctx, int64_t rows, int64_t cols, const double* A, double* U, double* sigma,
                      int64_t* kept, int mem);

/* replaces tg::pivoted_cholesky (tei.hpp:27-30, tei.cpp:48-90) for an explicit
 * PSD matrix A (n x n; the reference's column callback reads A's columns and
 * its diagonal argument is diag(A)).  stop: 0 max-diagonal, 1 trace.  L needs
 * n x min(n, max_rank) doubles (space `mem`), pivots min(n, max_rank) entries
 * (HOST); *rank, *residual (the stop measure ratio), *clamped_negative on the
 * host.  NUMERICAL_ERROR when a diagonal goes below -neg_tol * max0. */
int tgb_pivoted_cholesky(tgb_ctx* ctx, int64_t n, const double* A, double tol, int stop, int64_t max_rank,
                         double neg_tol, double* L, int64_t* pivots, int64_t* rank, double* residual,
                         int* clamped_negative, int mem);

/* ---- dense FP64 building block -------------------------------------------
 * C = alpha op(A) op(B) + beta C on the FP64 tensor cores (DMMA), column-major
 * DEVICE pointers, stream-ordered on the context stream.  The dense products
 * of reduction.cpp / tei.cpp (Gram matrices, projections, unfoldings) run on
 * it; exported for tests and callers that hold device matrices. */
int tgb_dgemm(tgb_ctx* ctx, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc);
/* Measured FP64 issue rate of this device (independent DFMA chains on every SM, best of three
 * ~5 ms runs): the FP64 roofline denominator bench.py reports against, taken in the same run. */
int tgb_probe_fp64_peak(tgb_ctx* ctx, double* tflops);

/* ---- lattice sums ------------------------------------------------------------
 * replaces the per-axis assembly of tg::lattice_sum_canonical / _tucker /
 * _composite (lattice.hpp:56-69, lattice.cpp:50-61,116-165):
 * out(:, q) = sum_{l < L} ref(offsets[l] : offsets[l] + n, q), summed in
 * lattice-index order l = 0..L-1 (bit-identical to the reference).
 * ref is (2n) x R; offsets (host memory) come from tg::window_offset. */
int tgb_lattice_assemble_axis(tgb_ctx* ctx, int64_t n, int64_t R, const double* ref, const int64_t* offsets,
                              int64_t L, double* out, int mem);
/* All three axes of lattice_sum_canonical (lattice.cpp:116-129) in one call:
 * axis arrays n[3], ref[3] (2 n[ax] x R), offsets[3] (L[ax] entries, host),
 * out[3] (n[ax] x R).  An axis whose extent, offsets and reference factor equal
 * an earlier axis's (cubic lattice, cubic grid) gets that axis's result copied,
 * which is bit-identical to assembling it again (host memory: the factors are
 * compared bitwise; device memory: the same reference pointer). */
int tgb_lattice_assemble(tgb_ctx* ctx, const int64_t* n, int64_t R, const double* const* ref,
                         const int64_t* const* offsets, const int64_t* L, double* const* out, int mem);

#ifdef __cplusplus
}
#endif

#endif /* TGB_H */

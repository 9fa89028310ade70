// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference `tengrid` hot path (arXiv 1504.06289,
// /root/reference/proj) used as the parity checker for the B200 kernels.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load it; the product path never does.
//
// Pinning: the reference's own translation units (fft, tensor, grid, kernel,
// basis, lattice, parallel, hf, tei, reduction, mp2 .cpp) are compiled in
// place from /root/reference against oracle/eigen_shim into oracle/_ref/
// (paper_1504_06289_b200/build.py build_ref).  The shim's dense
// decompositions (SelfAdjointEigenSolver, HouseholderQR, JacobiSVD, LLT)
// delegate to THIS restatement's LA, so oracle/_ref runs the reference's own
// control flow (thresholds, pivots, rank rules, loop orders) on a stand-in LA.
// The restatement is checked against oracle/_ref and the committed fixtures in
// tests/golden/ (reference_conv_path.npz, reference_hf.npz, reference_scf.npz).
//
// Every function names the reference file:line it restates.  Matrices are
// column-major (Eigen's default), entry (i, j) at data[i + rows * j].
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using idx = std::int64_t;

struct Mat {
  idx rows = 0, cols = 0;
  std::vector<double> d;
  Mat() = default;
  Mat(idx r, idx c, double fill = 0.0) : rows(r), cols(c), d(static_cast<size_t>(r * c), fill) {}
  double& operator()(idx i, idx j) { return d[static_cast<size_t>(i + rows * j)]; }
  double operator()(idx i, idx j) const { return d[static_cast<size_t>(i + rows * j)]; }
  double* col(idx j) { return d.data() + rows * j; }
  const double* col(idx j) const { return d.data() + rows * j; }
};

using Vec = std::vector<double>;

struct CP3 {  // proj/include/tengrid/tensor.hpp:119-150 (CanonicalTensor3)
  std::array<Mat, 3> f;
  Vec w;
  idx rank() const { return static_cast<idx>(w.size()); }
  idx extent(int ax) const { return f[ax].rows; }
};

struct Tucker3 {  // proj/include/tengrid/tensor.hpp:154-164
  std::array<Mat, 3> side;
  std::array<idx, 3> r{0, 0, 0};
  Vec core;  // r0 x r1 x r2 column-major
};

struct Grid {  // proj/include/tengrid/grid.hpp:18-52
  std::array<idx, 3> n{};
  std::array<double, 3> b{};
  std::array<double, 3> h{};
  double coord(int ax, idx i) const { return (static_cast<double>(i) - 0.5 * static_cast<double>(n[ax] - 1)) * h[ax]; }
  double ref_coord(int ax, idx j) const { return (static_cast<double>(j) - static_cast<double>(n[ax] - 1)) * h[ax]; }
};

struct invalid_argument : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct numerical_error : std::runtime_error { using std::runtime_error::runtime_error; };
struct snap_error : std::runtime_error { using std::runtime_error::runtime_error; };
inline void req(bool c, const char* m) { if (!c) throw invalid_argument(m); }

// grid.cpp
Grid make_grid(const std::array<double, 3>& b, const std::array<idx, 3>& n);
idx snap_to_node(const Grid& g, int ax, double x);
idx window_offset(const Grid& g, int ax, double center);

// fft.cpp
void fft_radix2(std::vector<double>& re, std::vector<double>& im, bool inverse);
Vec conv_full_direct(const double* u, idx nu, const double* v, idx nv);
Vec conv_full_fft(const double* u, idx nu, const double* v, idx nv);
Vec central_window(const Vec& full, idx n);
Mat conv_central_many(const Mat& U, const double* v, idx n);

// tensor.cpp
void normalize(CP3& t);
CP3 convolve(const CP3& a, const CP3& b, const std::array<double, 3>& h);
CP3 hadamard(const CP3& a, const CP3& b);
CP3 add(const CP3& a, const CP3& b);
double scalar_product(const CP3& a, const CP3& b);
double value_at(const CP3& t, idx i, idx j, idx k);

// kernel.cpp
struct ExpSum { idx m = 0; double c0 = 1, mesh = 0, scale = 1; Vec nodes, weights; };
ExpSum make_expsum(idx m, double c0, double fit_lo, double fit_hi);
double gauss_cell_integral(double t, double c, double h);
CP3 kernel_tensor(const Grid& g, const ExpSum& es, bool doubled);

// basis.cpp
struct BasisFn { std::array<double, 3> center{}; std::array<int, 3> deg{}; Vec exps, coefs; };
double primitive_norm(double alpha, int l);
std::vector<CP3> discretize_basis(const Grid& g, const std::vector<BasisFn>& fns);

// reduction.cpp
struct RedCfg { bool use_eps = true; double eps = 1e-7; std::array<idx, 3> ranks{}; int max_sweeps = 3; };
struct TuckerRes { Tucker3 t; bool rank_clamped = false, rhosvd_fallback = false; Vec sweep_fits; std::array<Vec, 3> sigma; };
void thin_svd_left(const Mat& a, Mat& u, Vec& s);
TuckerRes rhosvd(const CP3& a, const RedCfg& c);
TuckerRes canonical_to_tucker(const CP3& a, const RedCfg& c);
CP3 tucker_to_canonical(const Tucker3& t);
CP3 reduce_rank(const CP3& a, const RedCfg& c);

// hf.cpp
CP3 density_tensor(const std::vector<CP3>& disc, const Mat& c_occ, double eps);
CP3 hartree_potential(const CP3& theta, const CP3& kernel, const std::array<double, 3>& h);
Mat coulomb_matrix(const Grid& g, const std::vector<CP3>& disc, const CP3& vh);
Mat overlap_matrix(const Grid& g, const std::vector<CP3>& disc);
Mat kinetic_matrix(const Grid& g, const std::vector<CP3>& disc, bool exact_mass);
CP3 nuclear_potential_tensor(const Grid& g, const std::vector<std::array<double, 3>>& centers, const Vec& charges,
                             const CP3& ref);
Mat nuclear_matrix(const std::vector<CP3>& disc, const CP3& pc);
Mat exchange_matrix(const Grid& g, const std::vector<CP3>& disc, const Mat& c_occ, const CP3& kernel);
Mat coulomb_from_factors(const Mat& chol, const Mat& d);
Mat exchange_from_factors(const Mat& chol, const Mat& d);
Mat fock_from_factors(const Mat& h_core, const Mat& chol, const Mat& d);

// lattice.cpp
Mat assemble_axis(const Grid& g, const Mat& ref, int ax, const std::vector<double>& centers, idx* ops);

// tei.cpp
struct PivChol { Mat L; std::vector<idx> piv; double residual = 0; bool clamped = false; };
PivChol pivoted_cholesky(const std::function<Vec(idx)>& column, Vec diag, double tol, bool trace_stop,
                         idx max_rank, double neg_tol);
struct TEI {
  idx nb = 0, np = 0;
  std::vector<idx> owner;
  Vec pw;
  std::array<double, 3> h{};
  std::array<Mat, 3> U, V;
  std::array<double, 3> fit_res{};
  std::vector<std::array<Mat, 3>> M;
  Mat L;
  std::vector<idx> chol_piv;
  bool fit_clamped = false;
};
void tei_density_fitting(TEI& f, const Grid& g, const std::vector<CP3>& disc, double eps_fit);
void tei_convolution_matrices(TEI& f, const CP3& kernel);
Vec tei_column(const TEI& f, idx pair);
Vec tei_diagonal(const TEI& f);
void tei_cholesky(TEI& f, double eps_chol);

// dense LA used by the restatement (own code; the reference uses Eigen)
Mat matmul(const Mat& a, bool ta, const Mat& b, bool tb);
void sym_eigen(const Mat& a, Vec& evals_ascending, Mat& evecs);
void householder_qr_thin(const Mat& a, Mat& q, Mat& r);
void jacobi_svd_thin(const Mat& a, Mat& u, Vec& s);

}  // namespace orc

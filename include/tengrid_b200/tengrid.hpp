// tengrid_b200/tengrid.hpp — header-only C++ mirror of the reference's
// hot-path API over the libtgb C-ABI (include/tgb.h).
//
// A reference build switches to the B200 path by replacing the bodies of
// tg::convolve / tg::hartree_potential / tg::scalar_product /
// tg::coulomb_matrix / tg::conv_central_many / the HF operators
// (overlap, kinetic, exchange, *_from_factors, generalized_eigensolve) with
// calls into this header
// (INTEGRATION.md).  It is templated on the matrix type so it works with
// Eigen::MatrixXd / Eigen::VectorXd (column-major, data()/rows()/cols()/
// size()) without including Eigen here.
//
// Errors are rethrown as the reference's own exception classes
// (proj/include/tengrid/common.hpp:11-25): std::invalid_argument,
// std::domain_error, tg::SnapError, tg::NumericalError.  The two tg:: types
// are taken from the including translation unit:
//   * a reference build has proj/include on its include path, so
//     <tengrid/common.hpp> is found and tg::SnapError / tg::NumericalError
//     are thrown directly;
//   * or the includer names them before including this header:
//       #define TGB_SNAP_ERROR_T tg::SnapError
//       #define TGB_NUMERICAL_ERROR_T tg::NumericalError
//   * otherwise (standalone use) the tgb_cpp fallbacks below are thrown.
// Both types must be constructible from a std::string, as the reference's are.
#pragma once

#include <array>
#include <stdexcept>
#include <string>
#include <vector>

#include "tgb.h"
#include "tgb_host.h"

#if !defined(TGB_SNAP_ERROR_T) && !defined(TGB_NUMERICAL_ERROR_T) && defined(__has_include)
#if __has_include(<tengrid/common.hpp>)
#include <tengrid/common.hpp>
#define TGB_SNAP_ERROR_T ::tg::SnapError
#define TGB_NUMERICAL_ERROR_T ::tg::NumericalError
#endif
#endif

namespace tgb_cpp {

// standalone fallbacks (used only when the reference's classes are not visible)
struct SnapError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#ifdef TGB_SNAP_ERROR_T
using snap_error_t = TGB_SNAP_ERROR_T;
#else
using snap_error_t = SnapError;
#endif
#ifdef TGB_NUMERICAL_ERROR_T
using numerical_error_t = TGB_NUMERICAL_ERROR_T;
#else
using numerical_error_t = NumericalError;
#endif

inline void throw_code(int rc, const std::string& msg) {
  switch (rc) {
    case TGB_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case TGB_DOMAIN_ERROR: throw std::domain_error(msg);
    case TGB_SNAP_ERROR: throw snap_error_t(msg);
    case TGB_NUMERICAL_ERROR: throw numerical_error_t(msg);
    default: throw CudaError(msg);
  }
}

// device entry points (tgb.h): message from tgb_last_error()
inline void check(int rc) {
  if (rc != TGB_OK) throw_code(rc, tgb_last_error());
}
// host input producers (tgb_host.h): message from tgb_host_last_error()
inline void check_host(int rc) {
  if (rc != TGB_OK) throw_code(rc, tgb_host_last_error());
}

// One context per thread per device (contexts are not shared across threads).
inline tgb_ctx* context(int device = 0) {
  struct Holder {
    tgb_ctx* c = nullptr;
    ~Holder() {
      if (c) tgb_ctx_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.c) check(tgb_ctx_create(device, nullptr, &h.c));
  return h.c;
}

// Canonical tensor with the reference's layout: factor[ax] n_ax x R
// column-major, weight R.  Works for tg::CanonicalTensor3 (Eigen members).
template <class Cp>
tgb_cp view(const Cp& t) {
  tgb_cp c{};
  c.rank = static_cast<int64_t>(t.weight.size());
  for (int ax = 0; ax < 3; ++ax) {
    c.n[ax] = static_cast<int64_t>(t.factor[ax].rows());
    c.factor[ax] = const_cast<double*>(t.factor[ax].data());
  }
  c.weight = const_cast<double*>(t.weight.data());
  return c;
}

// tg::convolve (tensor.cpp:179-198).  Cp must be default-constructible with
// resizable Eigen-like members (factor[ax] = Matrix(n, r); weight = Vector(r)).
template <class Cp, class Matrix, class Vector>
Cp convolve(const Cp& a, const Cp& b, const std::array<double, 3>& h) {
  Cp out;
  const auto r = a.weight.size() * b.weight.size();
  for (int ax = 0; ax < 3; ++ax) out.factor[ax] = Matrix(a.factor[ax].rows(), r);
  out.weight = Vector(r);
  tgb_cp ca = view(a), cb = view(b), co = view(out);
  check(tgb_convolve(context(), &ca, &cb, h.data(), &co, TGB_MEM_HOST));
  return out;
}

// tg::hartree_potential (hf.cpp:131-138) on a primary-grid kernel tensor.
template <class Cp, class Matrix, class Vector>
Cp hartree_potential(const Cp& theta, const Cp& kernel, const std::array<double, 3>& h) {
  Cp out;
  const auto r = theta.weight.size() * kernel.weight.size();
  for (int ax = 0; ax < 3; ++ax) out.factor[ax] = Matrix(theta.factor[ax].rows(), r);
  out.weight = Vector(r);
  tgb_cp ct = view(theta), ck = view(kernel), co = view(out);
  check(tgb_hartree_potential(context(), &ct, &ck, h.data(), &co, TGB_MEM_HOST));
  return out;
}

// tg::conv_central_many (fft.cpp:97-122).
template <class Matrix, class Vec>
Matrix conv_central_many(const Matrix& U, const Vec& v) {
  Matrix out(U.rows(), U.cols());
  check(tgb_conv_central_many(context(), U.rows(), U.cols(), U.data(), v.data(), out.data(), TGB_MEM_HOST));
  return out;
}

// tg::scalar_product (tensor.cpp:88-98).
template <class Cp>
double scalar_product(const Cp& a, const Cp& b) {
  tgb_cp ca = view(a), cb = view(b);
  double r = 0.0;
  check(tgb_scalar_product(context(), &ca, &cb, &r, TGB_MEM_HOST));
  return r;
}

// The discretised basis (one canonical tensor per function, discretize_basis)
// flattened into one tensor of all primitives + function offsets, the form
// every basis-level tgb_* entry point takes (host copy, small).
struct FlatBasis {
  std::array<std::vector<double>, 3> f;
  std::vector<double> w;
  std::vector<int64_t> off;
  tgb_cp cp{};
  int64_t nb = 0;
  template <class Cp>
  explicit FlatBasis(const std::vector<Cp>& disc) : off(disc.size() + 1, 0), nb(static_cast<int64_t>(disc.size())) {
    for (int64_t k = 0; k < nb; ++k) off[k + 1] = off[k] + static_cast<int64_t>(disc[k].weight.size());
    for (const auto& d : disc) {
      for (int ax = 0; ax < 3; ++ax)
        f[ax].insert(f[ax].end(), d.factor[ax].data(), d.factor[ax].data() + d.factor[ax].size());
      w.insert(w.end(), d.weight.data(), d.weight.data() + d.weight.size());
    }
    cp.rank = off[nb];
    for (int ax = 0; ax < 3; ++ax) {
      cp.n[ax] = disc.empty() ? 0 : static_cast<int64_t>(disc[0].factor[ax].rows());
      cp.factor[ax] = f[ax].data();
    }
    cp.weight = w.data();
  }
};

// tg::coulomb_matrix (hf.cpp:140-151): disc = discretize_basis(bs).
template <class Cp, class Matrix>
Matrix coulomb_matrix(const std::vector<Cp>& disc, const Cp& vh, const std::array<double, 3>& h) {
  FlatBasis fb(disc);
  tgb_cp cv = view(vh);
  Matrix J(fb.nb, fb.nb);
  check(tgb_coulomb_matrix(context(), &fb.cp, fb.off.data(), fb.nb, &cv, h.data(), J.data(), TGB_MEM_HOST));
  return J;
}

// tg::overlap_matrix / tg::kinetic_matrix (hf.cpp:48-87).
template <class Cp, class Matrix>
Matrix overlap_matrix(const std::vector<Cp>& disc, const std::array<double, 3>& h) {
  FlatBasis fb(disc);
  Matrix S(fb.nb, fb.nb);
  check(tgb_overlap_matrix(context(), &fb.cp, fb.off.data(), fb.nb, h.data(), S.data(), TGB_MEM_HOST));
  return S;
}
template <class Cp, class Matrix>
Matrix kinetic_matrix(const std::vector<Cp>& disc, const std::array<double, 3>& h, bool exact_mass = false) {
  FlatBasis fb(disc);
  Matrix T(fb.nb, fb.nb);
  check(tgb_kinetic_matrix(context(), &fb.cp, fb.off.data(), fb.nb, h.data(), exact_mass ? 1 : 0, T.data(),
                           TGB_MEM_HOST));
  return T;
}

// tg::exchange_matrix (hf.cpp:153-170) with a primary-grid kernel tensor.
template <class Cp, class Matrix>
Matrix exchange_matrix(const std::vector<Cp>& disc, const Matrix& c_occ, const Cp& kernel,
                       const std::array<double, 3>& h) {
  FlatBasis fb(disc);
  tgb_cp ck = view(kernel);
  Matrix K(fb.nb, fb.nb);
  check(tgb_exchange_matrix(context(), &fb.cp, fb.off.data(), fb.nb, c_occ.data(), c_occ.cols(), &ck, h.data(),
                            K.data(), TGB_MEM_HOST));
  return K;
}

// tg::coulomb_from_factors / exchange_from_factors / fock_from_factors (tei.cpp:215-238).
template <class Matrix>
Matrix coulomb_from_factors(const Matrix& chol, const Matrix& density) {
  Matrix J(density.rows(), density.rows());
  check(tgb_coulomb_from_factors(context(), density.rows(), chol.cols(), chol.data(), density.data(), J.data(),
                                 TGB_MEM_HOST));
  return J;
}
template <class Matrix>
Matrix exchange_from_factors(const Matrix& chol, const Matrix& density) {
  Matrix K(density.rows(), density.rows());
  check(tgb_exchange_from_factors(context(), density.rows(), chol.cols(), chol.data(), density.data(), K.data(),
                                  TGB_MEM_HOST));
  return K;
}
template <class Matrix>
Matrix fock_from_factors(const Matrix& h_core, const Matrix& chol, const Matrix& density) {
  Matrix F(density.rows(), density.rows());
  check(tgb_fock_from_factors(context(), density.rows(), chol.cols(), h_core.data(), chol.data(), density.data(),
                              F.data(), TGB_MEM_HOST));
  return F;
}

// tg::generalized_eigensolve (hf.cpp:187-199): F C = S C diag(e).
template <class Matrix, class Vector>
void generalized_eigensolve(const Matrix& f, const Matrix& s, Matrix& c, Vector& e) {
  c = Matrix(f.rows(), f.rows());
  e = Vector(f.rows());
  check(tgb_generalized_eigensolve(context(), f.rows(), f.data(), s.data(), c.data(), e.data(), TGB_MEM_HOST));
}

// ---- host input producers (tgb_host.h) ------------------------------------

// tg::snap_to_node (grid.cpp:23-30): std::domain_error outside the box,
// the reference's SnapError farther than h/2 from every node.
template <class Grid>
int64_t snap_to_node(const Grid& g, int axis, double x) {
  int64_t node = 0;
  check_host(tgb_snap_to_node(g.b_half[axis], static_cast<int64_t>(g.n[axis]), x, &node));
  return node;
}

// tg::expsum_for_interval (kernel.cpp:131-165): the Newton quadrature (M, C0)
// meeting eps on [r_min, r_max]; the reference's NumericalError when m_cap
// is exceeded.
struct ExpSumChoice {
  int64_t m;
  double c0;
};
inline ExpSumChoice expsum_for_interval(double r_min, double r_max, double eps, int64_t m_cap = 2048) {
  ExpSumChoice c{0, 0.0};
  check_host(tgb_expsum_for_interval(r_min, r_max, eps, m_cap, &c.m, &c.c0));
  return c;
}

// ---- SCF / MP2 (tgb.h) ------------------------------------------------------

// tg::scf_solve (hf.cpp:201-270) for a reference-shaped Molecule / BasisSet /
// SCFConfig (members as in basis.hpp:10-52 and hf.hpp:54-64).  Returns the
// scalar results and the orbital energies / density (column-major nb x nb).
struct ScfResult {
  double energy = 0.0, nuclear_energy = 0.0;
  bool converged = false;
  int iterations = 0, n_occupied = 0;
  int64_t tei_rank_b = 0;
  std::vector<double> orbital_energies, density;
};
template <class Mol, class Basis, class Cfg>
ScfResult scf_solve(const Mol& mol, const Basis& bs, const Cfg& cfg) {
  std::vector<double> centers, exps, coefs, charges, ncent;
  std::vector<int> degs;
  std::vector<int64_t> off(1, 0);
  for (const auto& f : bs.functions) {
    for (int ax = 0; ax < 3; ++ax) {
      centers.push_back(f.center[ax]);
      degs.push_back(f.degree[ax]);
    }
    for (const auto& p : f.primitives) {
      exps.push_back(p.exponent);
      coefs.push_back(p.coeff);
    }
    off.push_back(static_cast<int64_t>(exps.size()));
  }
  for (const auto& nu : mol.nuclei) {
    charges.push_back(nu.charge);
    for (int ax = 0; ax < 3; ++ax) ncent.push_back(nu.center[ax]);
  }
  tgb_basis_spec spec{};
  for (int ax = 0; ax < 3; ++ax) {
    spec.b_half[ax] = bs.grid.b_half[ax];
    spec.n[ax] = static_cast<int64_t>(bs.grid.n[ax]);
  }
  spec.nfn = static_cast<int64_t>(bs.functions.size());
  spec.centers = centers.data();
  spec.degrees = degs.data();
  spec.prim_offset = off.data();
  spec.exponents = exps.data();
  spec.coeffs = coefs.data();
  tgb_molecule m{static_cast<int64_t>(mol.nuclei.size()), charges.data(), ncent.data(),
                 static_cast<int64_t>(mol.n_electrons)};
  tgb_scf_config c{};
  c.max_iterations = cfg.max_iterations;
  c.energy_tol = cfg.energy_tol;
  c.mixing = cfg.mixing;
  c.eps_fit = cfg.eps_fit;
  c.eps_chol = cfg.eps_chol;
  c.kernel_eps = cfg.kernel_eps;
  c.kernel_r_max = cfg.kernel_r_max;
  c.density_reduce_eps = cfg.density_reduce_eps;
  c.exact_mass_kinetic = cfg.exact_mass_kinetic ? 1 : 0;
  ScfResult r;
  const size_t nb = bs.functions.size();
  r.orbital_energies.assign(nb, 0.0);
  r.density.assign(nb * nb, 0.0);
  tgb_scf_state st{};
  st.orbital_energies = r.orbital_energies.data();
  st.density = r.density.data();
  check(tgb_scf_solve(context(), &m, &spec, &c, &st));
  r.energy = st.energy;
  r.nuclear_energy = st.nuclear_energy;
  r.converged = st.converged != 0;
  r.iterations = st.iterations;
  r.n_occupied = st.n_occupied;
  r.tei_rank_b = st.tei_rank_b;
  return r;
}

// tg::mp2_energy (mp2.cpp:60-105): mode 0 = MP2Mode::oracle, 1 = factorized.
// factor is the MOCholesky factor (N_ov x R_B, column-major); energies the
// MOSpace orbital energies (ascending).  The reference's NumericalError for a
// non-positive denominator gap.
template <class Matrix, class Vector>
double mp2_energy(const Matrix& factor, int64_t n_occ, int64_t n_vir, const Vector& energies, int mode = 0,
                  double expsum_eps = 1e-9) {
  double e = 0.0;
  check(tgb_mp2_energy(context(), n_occ, n_vir, static_cast<int64_t>(factor.cols()), factor.data(), energies.data(),
                       mode, expsum_eps, &e, TGB_MEM_HOST));
  return e;
}

}  // namespace tgb_cpp

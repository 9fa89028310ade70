// C++ drop-in check: the header-only mirror include/tengrid_b200/tengrid.hpp
// driven with Eigen-layout containers (oracle/eigen_shim stands in for Eigen,
// which is absent from the image).  Exit code = number of failures.
#include <Eigen/Core>
#include <cmath>
#include <cstdio>
#include <cstring>

#ifndef TGB_TEST_REFERENCE_HEADERS
// The reference's include tree is not on the GPU box: these stand-ins play
// tg::SnapError / tg::NumericalError (common.hpp:11-21 declares both as
// std::runtime_error subclasses with a string constructor) and are handed to
// the mirror the way a reference build does it.
namespace tg {
class SnapError : public std::runtime_error {
 public:
  explicit SnapError(const std::string& m) : std::runtime_error(m) {}
};
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};
}  // namespace tg
#define TGB_SNAP_ERROR_T tg::SnapError
#define TGB_NUMERICAL_ERROR_T tg::NumericalError
#endif
// (with -DTGB_TEST_REFERENCE_HEADERS -I proj/include the header finds
// <tengrid/common.hpp> itself and throws the reference's classes)
#include "tengrid_b200/tengrid.hpp"

static_assert(std::is_same_v<tgb_cpp::snap_error_t, tg::SnapError>, "mirror must throw tg::SnapError");
static_assert(std::is_same_v<tgb_cpp::numerical_error_t, tg::NumericalError>, "mirror must throw tg::NumericalError");

// Host-side error mapping (no GPU needed): the reference tests
// test_kernel.cpp:88 (expsum_for_interval -> NumericalError) and
// test_grid.cpp:100-106 (out of box -> domain_error, between nodes -> SnapError).
struct G {
  std::array<long long, 3> n{10, 10, 10};
  std::array<double, 3> b_half{5.0, 5.0, 5.0};
};
static int host_checks() {
  int fails = 0;
  try {
    tgb_cpp::expsum_for_interval(1e-6, 1e6, 1e-10, 64);
    std::printf("expsum_for_interval: no NumericalError\n");
    ++fails;
  } catch (const tg::NumericalError&) {
  }
  const G g;
  try {
    tgb_cpp::snap_to_node(g, 0, 6.0);
    std::printf("snap_to_node: no domain_error\n");
    ++fails;
  } catch (const std::domain_error&) {
  }
  const double h = 10.0 / 11.0, wall_gap = (9 - 4.5) * h + 0.9 * h;
  try {
    tgb_cpp::snap_to_node(g, 0, wall_gap);
    std::printf("snap_to_node: no SnapError\n");
    ++fails;
  } catch (const tg::SnapError&) {
  }
  const auto es = tgb_cpp::expsum_for_interval(0.8, 10.0, 1e-5);
  if (es.m <= 0) { std::printf("expsum_for_interval: bad M\n"); ++fails; }
  return fails;
}

// reference-shaped SCF inputs (basis.hpp:10-52, hf.hpp:54-64)
struct Prim { double exponent = 1.0, coeff = 1.0; };
struct Fn { std::array<double, 3> center{0, 0, 0}; std::array<int, 3> degree{0, 0, 0}; std::vector<Prim> primitives; };
struct Grid { std::array<long long, 3> n{}; std::array<double, 3> b_half{}; };
struct Basis { Grid grid; std::vector<Fn> functions; };
struct Nuc { double charge = 1.0; std::array<double, 3> center{0, 0, 0}; };
struct Mol { std::vector<Nuc> nuclei; int n_electrons = 0; };
struct Cfg {
  int max_iterations = 60;
  double energy_tol = 1e-9, mixing = 0.7, eps_fit = 1e-8, eps_chol = 1e-10, kernel_eps = 1e-6, kernel_r_max = 0.0,
         density_reduce_eps = 1e-7;
  bool exact_mass_kinetic = false;
};

// Device-side error mapping: test_hf.cpp:609-622 (duplicate basis function ->
// singular overlap -> NumericalError) and test_mp2.cpp:164-173 (zero
// denominator gap -> NumericalError).
static int device_error_checks() {
  int fails = 0;
  {
    Basis bs;
    bs.grid.n = {32, 32, 32};
    bs.grid.b_half = {6.0, 6.0, 6.0};
    Fn f;
    f.primitives.push_back({0.8, 1.0});
    bs.functions = {f, f};
    Mol mol;
    mol.nuclei = {Nuc{}};
    mol.n_electrons = 2;
    try {
      tgb_cpp::scf_solve(mol, bs, Cfg{});
      std::printf("scf_solve (duplicate basis): no NumericalError\n");
      ++fails;
    } catch (const tg::NumericalError&) {
    }
  }
  {
    Eigen::MatrixXd factor = Eigen::MatrixXd::Ones(1, 1);
    Eigen::VectorXd e(2);
    e[0] = -0.1;
    e[1] = -0.1;
    try {
      tgb_cpp::mp2_energy(factor, 1, 1, e);
      std::printf("mp2_energy (zero gap): no NumericalError\n");
      ++fails;
    } catch (const tg::NumericalError&) {
    }
  }
  return fails;
}

struct CP {  // same members as tg::CanonicalTensor3 (tensor.hpp:119-122)
  std::array<Eigen::MatrixXd, 3> factor;
  Eigen::VectorXd weight;
};

int main(int argc, char** argv) {
  int fails = host_checks();
  if (argc > 1 && std::strcmp(argv[1], "--host-only") == 0) {
    std::printf("cpp api (host): %d failures\n", fails);
    return fails;
  }
  fails += device_error_checks();
  const long n = 33;
  CP a, b;
  for (int ax = 0; ax < 3; ++ax) {
    a.factor[ax] = Eigen::MatrixXd(n, 2);
    b.factor[ax] = Eigen::MatrixXd(n, 1);
    for (long i = 0; i < n; ++i) {
      const double x = (i - 0.5 * (n - 1)) * 0.3;
      a.factor[ax](i, 0) = std::exp(-0.5 * x * x);
      a.factor[ax](i, 1) = std::exp(-2.0 * (x - 0.4) * (x - 0.4));
      b.factor[ax](i, 0) = (i == (n - 1) / 2) ? 1.0 / 0.3 : 0.0;  // delta with h removed
    }
  }
  a.weight = Eigen::VectorXd(2);
  a.weight[0] = 1.5;
  a.weight[1] = -0.5;
  b.weight = Eigen::VectorXd::Ones(1);
  CP c = tgb_cpp::convolve<CP, Eigen::MatrixXd, Eigen::VectorXd>(a, b, {0.3, 0.3, 0.3});
  double err = 0;
  for (int ax = 0; ax < 3; ++ax)
    for (long i = 0; i < n; ++i)
      for (long k = 0; k < 2; ++k) err = std::max(err, std::abs(c.factor[ax](i, k) - a.factor[ax](i, k)));
  if (err > 1e-13) { std::printf("delta identity failed: %g\n", err); ++fails; }
  if (c.weight[0] != 1.5 || c.weight[1] != -0.5) { std::printf("weights failed\n"); ++fails; }
  const double sp = tgb_cpp::scalar_product(a, a);
  double ref = 0;
  for (long p = 0; p < 2; ++p)
    for (long q = 0; q < 2; ++q) {
      double g = a.weight[p] * a.weight[q];
      for (int ax = 0; ax < 3; ++ax) g *= a.factor[ax].col(p).dot(a.factor[ax].col(q));
      ref += g;
    }
  if (std::abs(sp - ref) > 1e-12 * std::abs(ref)) { std::printf("scalar_product failed %g %g\n", sp, ref); ++fails; }
  try {
    CP bad = b;
    bad.factor[2] = Eigen::MatrixXd(n + 1, 1);
    tgb_cpp::convolve<CP, Eigen::MatrixXd, Eigen::VectorXd>(a, bad, {0.3, 0.3, 0.3});
    std::printf("extent mismatch not rejected\n");
    ++fails;
  } catch (const std::invalid_argument&) {
  }
  // fock_from_factors (tei.cpp:215-238) against the defining loops
  {
    const long nb = 5, R = 3;
    Eigen::MatrixXd L(nb * nb, R), D(nb, nb), H(nb, nb);
    for (long i = 0; i < L.size(); ++i) L(i) = std::sin(0.37 * i + 0.1);
    for (long i = 0; i < nb; ++i)
      for (long j = 0; j < nb; ++j) {
        D(i, j) = std::cos(0.5 * (i + j)) + (i == j ? 2.0 : 0.0);
        H(i, j) = 0.1 * (i + 1) * (j + 1);
      }
    Eigen::MatrixXd F = tgb_cpp::fock_from_factors(H, L, D);
    double ferr = 0.0;
    for (long mu = 0; mu < nb; ++mu)
      for (long nu = 0; nu < nb; ++nu) {
        double j = 0.0, k = 0.0;
        for (long s = 0; s < R; ++s)
          for (long a = 0; a < nb; ++a)
            for (long b = 0; b < nb; ++b) {
              j += 0.5 * (L(mu + nb * nu, s) + L(nu + nb * mu, s)) * L(a + nb * b, s) * D(a, b);
              k -= 0.25 * (L(mu + nb * a, s) * D(a, b) * L(nu + nb * b, s) + L(nu + nb * a, s) * D(a, b) * L(mu + nb * b, s));
            }
        ferr = std::max(ferr, std::abs(F(mu, nu) - (H(mu, nu) + j + k)));
      }
    if (ferr > 1e-12) { std::printf("fock_from_factors failed: %g\n", ferr); ++fails; }
    for (long i = 0; i < nb; ++i)
      for (long j = 0; j < nb; ++j)
        if (F(i, j) != F(j, i)) { std::printf("fock not exactly symmetric\n"); ++fails; i = nb; break; }
  }
  std::printf("cpp api: %d failures\n", fails);
  return fails;
}

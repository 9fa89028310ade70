// C++ drop-in check: the header-only mirror include/tengrid_b200/tengrid.hpp
// driven with Eigen-layout containers (oracle/eigen_shim stands in for Eigen,
// which is absent from the image).  Exit code = number of failures.
#include <Eigen/Core>
#include <cmath>
#include <cstdio>

#include "tengrid_b200/tengrid.hpp"

struct CP {  // same members as tg::CanonicalTensor3 (tensor.hpp:119-122)
  std::array<Eigen::MatrixXd, 3> factor;
  Eigen::VectorXd weight;
};

int main() {
  int fails = 0;
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

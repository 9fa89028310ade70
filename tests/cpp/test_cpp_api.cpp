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
  std::printf("cpp api: %d failures\n", fails);
  return fails;
}

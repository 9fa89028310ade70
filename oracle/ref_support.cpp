// ORACLE — TEST INFRASTRUCTURE ONLY.
// Dense decompositions behind oracle/eigen_shim/Eigen/Dense for the
// reference translation units compiled into oracle/_ref (hf.cpp, tei.cpp,
// reduction.cpp, mp2.cpp).  Eigen is absent from the image; these hooks route
// SelfAdjointEigenSolver / HouseholderQR / JacobiSVD / LLT to the
// restatement's own LA (tengrid_oracle.cpp), so oracle/_ref runs the
// reference's control flow (pivots, thresholds, rank rules, loop orders) on a
// stand-in LA.  Eigen- and singular-vector signs may differ from Eigen's.
#include <cmath>
#include <cstring>
#include <stdexcept>

#include <Eigen/Dense>

#include "tengrid_oracle.hpp"

namespace {
orc::Mat to_orc(const Eigen::MatrixXd& a) {
  orc::Mat m(a.rows(), a.cols());
  for (Eigen::Index j = 0; j < a.cols(); ++j)
    for (Eigen::Index i = 0; i < a.rows(); ++i) m(i, j) = a(i, j);
  return m;
}
Eigen::MatrixXd from_orc(const orc::Mat& m) {
  Eigen::MatrixXd a(m.rows, m.cols);
  if (m.rows * m.cols) std::memcpy(a.data(), m.d.data(), sizeof(double) * m.rows * m.cols);
  return a;
}
Eigen::VectorXd from_vec(const orc::Vec& v) {
  Eigen::VectorXd a(static_cast<Eigen::Index>(v.size()));
  for (size_t i = 0; i < v.size(); ++i) a[static_cast<Eigen::Index>(i)] = v[i];
  return a;
}
}  // namespace

namespace Eigen::shim {

void sym_eigen(const MatrixXd& a, VectorXd& ev, MatrixXd& z) {
  orc::Vec e;
  orc::Mat zz;
  orc::sym_eigen(to_orc(a), e, zz);
  ev = from_vec(e);
  z = from_orc(zz);
}

void householder_qr(const MatrixXd& a, MatrixXd& q, MatrixXd& r) {
  orc::Mat qq, rr;
  orc::householder_qr_thin(to_orc(a), qq, rr);
  q = from_orc(qq);
  r = from_orc(rr);
}

void jacobi_svd(const MatrixXd& a, MatrixXd& u, VectorXd& s, MatrixXd* v) {
  if (v) throw std::logic_error("eigen_shim: JacobiSVD right vectors are not provided");
  orc::Mat uu;
  orc::Vec ss;
  orc::jacobi_svd_thin(to_orc(a), uu, ss);
  u = from_orc(uu);
  s = from_vec(ss);
}

// Cholesky-Banachiewicz, lower factor (the upper triangle is zero)
bool cholesky(const MatrixXd& a, MatrixXd& l) {
  const Index n = a.rows();
  l = MatrixXd(n, n);
  for (Index j = 0; j < n; ++j) {
    double d = a(j, j);
    for (Index k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
    if (!(d > 0.0)) return false;
    l(j, j) = std::sqrt(d);
    for (Index i = j + 1; i < n; ++i) {
      double s = a(i, j);
      for (Index k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
      l(i, j) = s / l(j, j);
    }
  }
  return true;
}

}  // namespace Eigen::shim

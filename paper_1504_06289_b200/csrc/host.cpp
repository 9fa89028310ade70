// Host-side input producers of the hot path (untimed, as in the reference):
// grid geometry, sinc-quadrature Gaussian sums for 1/r and their cell-integral
// factor columns, and sampled Gaussian basis factors.  Restated from
// proj/src/grid.cpp:7-38, proj/src/kernel.cpp:71-123,171-203 and
// proj/src/basis.cpp:8-46 so results are bit-identical to the reference's
// formulas evaluated with the same libm.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tgb_internal.hpp"
#include "tgb_host.h"

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kSqrtPi = 1.7724538509055160273;

thread_local std::string g_host_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TGB_OK;
  } catch (const tgb::Error& e) {
    g_host_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return TGB_INVALID_ARGUMENT;
  }
}

double coord(double h, int64_t n, int64_t i) { return (static_cast<double>(i) - 0.5 * static_cast<double>(n - 1)) * h; }
double ref_coord(double h, int64_t n, int64_t j) { return (static_cast<double>(j) - static_cast<double>(n - 1)) * h; }

double cell_integral(double t, double c, double h) {
  if (t == 0.0) return h;
  const double xl = c - 0.5 * h, xr = c + 0.5 * h;
  const double k = kSqrtPi / (2.0 * t);
  if (xl >= 0.0) return k * (std::erfc(t * xl) - std::erfc(t * xr));  // far-right cell: no cancellation
  if (xr <= 0.0) return k * (std::erfc(-t * xr) - std::erfc(-t * xl));
  return k * (std::erf(t * xr) - std::erf(t * xl));
}

}  // namespace

extern "C" {

const char* tgb_host_last_error(void) { return g_host_err.c_str(); }

double tgb_mesh_size(double b_half, int64_t n) { return 2.0 * b_half / static_cast<double>(n + 1); }

int tgb_snap_to_node(double b_half, int64_t n, double x, int64_t* node) {
  return guarded([&] {
    const double h = tgb_mesh_size(b_half, n);
    if (std::abs(x) > b_half) throw tgb::Error(TGB_DOMAIN_ERROR, "snap_to_node: point outside the computational box");
    const int64_t i = static_cast<int64_t>(std::llround(x / h + 0.5 * static_cast<double>(n - 1)));
    if (i < 0 || i >= n || std::abs(x - coord(h, n, i)) > 0.5 * h * (1.0 + 1e-12))
      throw tgb::Error(TGB_SNAP_ERROR, "snap_to_node: point farther than h/2 from every node; refine the grid");
    *node = i;
  });
}

int tgb_window_offset(double b_half, int64_t n, double center, int64_t* ofs) {
  return guarded([&] {
    int64_t i0 = 0;
    const int rc = tgb_snap_to_node(b_half, n, center, &i0);
    if (rc) throw tgb::Error(rc, g_host_err);
    const int64_t o = (n - 1) - i0;
    tgb::require(o >= 0 && o + n <= 2 * n, "window_offset: window escapes the doubled grid");
    *ofs = o;
  });
}

int tgb_make_expsum(int64_t m, double c0, double fit_lo, double fit_hi, double* nodes, double* weights,
                    double* scale_out, double* mesh_out) {
  return guarded([&] {
    tgb::require(m >= 1, "make_radial_expsum: need at least one quadrature point");
    tgb::require(c0 > 0.0, "make_radial_expsum: C0 must be positive");
    const double mesh = c0 * std::log(static_cast<double>(std::max<int64_t>(m, 2))) / static_cast<double>(m);
    const int64_t terms = 2 * m + 1;
    for (int64_t k = -m; k <= m; ++k) {
      nodes[k + m] = static_cast<double>(k) * mesh;
      weights[k + m] = 2.0 / kSqrtPi * mesh;  // Newton Laplace weight, t = 0 kept
    }
    const double t_max = c0 * std::log(static_cast<double>(std::max<int64_t>(m, 2)));
    double dlo = 3.0 / t_max, dhi = kPi / (3.0 * mesh);
    if (dhi < 2.0 * dlo) dhi = 2.0 * dlo;
    if (fit_lo <= 0.0 || fit_hi <= 0.0) {
      fit_lo = dlo;
      fit_hi = dhi;
    } else {
      fit_lo = std::max(fit_lo, dlo);
      fit_hi = std::min(fit_hi, dhi);
      if (fit_lo >= fit_hi) {
        fit_lo = dlo;
        fit_hi = dhi;
      }
    }
    double num = 0.0, den = 0.0;
    for (int i = 0; i < 200; ++i) {
      const double r = fit_lo * std::pow(fit_hi / fit_lo, static_cast<double>(i) / 199);
      double f = 0.0;
      for (int64_t k = 0; k < terms; ++k) f += weights[k] * std::exp(-nodes[k] * nodes[k] * r * r);
      num += f * (1.0 / r);
      den += f * f;
    }
    const double sc = den > 0.0 ? num / den : 1.0;
    for (int64_t k = 0; k < terms; ++k) weights[k] *= sc;
    *scale_out = sc;
    *mesh_out = mesh;
  });
}

int tgb_kernel_factors(double b_half, int64_t n, int64_t terms, const double* nodes, const double* weights,
                       int doubled, double* factor) {
  return guarded([&] {
    const double h = tgb_mesh_size(b_half, n);
    const int64_t len = doubled ? 2 * n : n;
    for (int64_t q = 0; q < terms; ++q) {
      const double tq = std::abs(nodes[q]);
      const double aq = std::cbrt(weights[q]);
      for (int64_t i = 0; i < len; ++i) {
        const double c = doubled ? ref_coord(h, n, i) : coord(h, n, i);
        factor[i + len * q] = aq * cell_integral(tq, c, h);
      }
    }
  });
}

// kernel.cpp:125-165 (Newton kernel): smallest M on the reference's schedule
// whose golden-section-optimal C0 meets eps on [r_min, r_max].
int tgb_expsum_for_interval(double r_min, double r_max, double eps, int64_t m_cap, int64_t* m_out, double* c0_out) {
  return guarded([&] {
    tgb::require(r_min > 0.0 && r_max >= r_min, "expsum_for_interval: bad interval");
    tgb::require(eps > 0.0, "expsum_for_interval: eps must be positive");
    std::vector<double> nodes, weights;
    auto build = [&](int64_t m, double c0) {
      nodes.assign(2 * m + 1, 0.0);
      weights.assign(2 * m + 1, 0.0);
      double sc, mesh;
      if (tgb_make_expsum(m, c0, r_min, r_max, nodes.data(), weights.data(), &sc, &mesh) != TGB_OK)
        throw tgb::Error(TGB_INVALID_ARGUMENT, g_host_err);
    };
    auto max_rel = [&](int samples) {  // ExpSum::max_relative_error (kernel.cpp:58-67), target 1/r
      double worst = 0.0;
      for (int i = 0; i < samples; ++i) {
        const double r = r_min * std::pow(r_max / r_min, samples == 1 ? 0.0 : static_cast<double>(i) / (samples - 1));
        double v = 0.0;
        for (size_t k = 0; k < weights.size(); ++k) v += weights[k] * std::exp(-nodes[k] * nodes[k] * r * r);
        const double f = 1.0 / r;
        worst = std::max(worst, std::abs(v - f) / std::abs(f));
      }
      return worst;
    };
    auto measured = [&](int64_t m, double c0) {
      build(m, c0);
      return max_rel(300);
    };
    // golden-section search of log c0 on [log 0.15, log 12] (22 shrinks, kernel.cpp:141-161); the
    // bracket and its two interior probes are updated with the reference's expressions, so c0
    // comes out bit-identical
    struct Probe {
      double x, err;
    };
    auto best_c0 = [&](int64_t m) {
      const double ratio = 0.5 * (std::sqrt(5.0) - 1.0);
      auto probe = [&](double x) { return Probe{x, measured(m, std::exp(x))}; };
      double left = std::log(0.15), right = std::log(12.0);
      Probe near = probe(right - ratio * (right - left));  // interior point closer to `left`
      Probe far = probe(left + ratio * (right - left));
      for (int shrink = 0; shrink < 22; ++shrink) {
        if (near.err <= far.err) {  // the minimum is left of `far`
          right = far.x;
          far = near;
          near = probe(right - ratio * (right - left));
        } else {
          left = near.x;
          near = far;
          far = probe(left + ratio * (right - left));
        }
      }
      return std::exp(0.5 * (left + right));
    };
    const double l = std::log(1.0 / std::min(eps * 1e3, 0.5));
    tgb::require(std::min(eps * 1e3, 0.5) > 0.0 && std::min(eps * 1e3, 0.5) < 1.0,
                 "expsum_terms_for_tolerance: eps in (0,1) required");
    for (int64_t m = std::max<int64_t>(6, static_cast<int64_t>(std::ceil(0.30 * l * l))); m <= m_cap;
         m = std::max<int64_t>(m + 4, static_cast<int64_t>(m * 1.3))) {
      const double c0 = best_c0(m);
      build(m, c0);
      if (max_rel(600) <= eps) {
        *m_out = m;
        *c0_out = c0;
        return;
      }
    }
    throw tgb::Error(TGB_NUMERICAL_ERROR, "expsum_for_interval: tolerance unattainable within the term cap");
  });
}

// kernel.cpp:205-250: 1/x ~ sum_j w_j exp(-r_j x) on [lo, hi] (sinc quadrature of
// 1/x = int exp(-x e^u + u) du, mesh shrunk by 0.8 until eps is met).  rates /
// weights need term_cap entries; *ok = 0 when the cap is hit (the reference's
// ReciprocalExpSum::ok).
int tgb_reciprocal_expsum(double lo, double hi, double eps, int64_t term_cap, int64_t* terms, double* rates,
                          double* weights, double* achieved, int* ok) {
  return guarded([&] {
    tgb::require(0.0 < lo && lo <= hi, "reciprocal_expsum: need 0 < lo <= hi");
    tgb::require(eps > 0.0, "reciprocal_expsum: eps must be positive");
    *ok = 0;
    *terms = 0;
    *achieved = 0.0;
    if (lo == hi) {
      tgb::require(term_cap >= 1, "reciprocal_expsum: term cap below one");
      rates[0] = 1.0 / lo;
      weights[0] = 2.71828182845904523536 / lo;  // std::numbers::e
      *terms = 1;
      *ok = 1;
      return;
    }
    // scaled problem 1/x on [1, q]; quadrature nodes u_j = u_min + j * mesh over [u_min, u_max]
    const double q = hi / lo;
    const double u_min = std::log(eps / (6.0 * q));
    const double u_max = std::log(std::log(6.0 * q / eps)) + 1.0;
    std::vector<double> rate, wt;
    auto worst_error = [&](int64_t n) {  // max relative error at 1000 log-spaced points of [1, q]
      double worst = 0.0;
      for (int i = 0; i < 1000; ++i) {
        const double x = std::pow(q, static_cast<double>(i) / 999);
        double sum = 0.0;
        for (int64_t j = 0; j < n; ++j) sum += wt[j] * std::exp(-rate[j] * x);
        worst = std::max(worst, std::abs(sum - 1.0 / x) * x);
      }
      return worst;
    };
    double mesh = 2.0 * kPi / (std::log(1.0 / eps) + 6.0);
    for (;;) {
      const int64_t n = static_cast<int64_t>(std::ceil((u_max - u_min) / mesh)) + 1;
      if (n > term_cap) return;  // *ok stays 0
      rate.resize(n);
      wt.resize(n);
      for (int64_t j = 0; j < n; ++j) {
        const double e = std::exp(u_min + static_cast<double>(j) * mesh);
        rate[j] = e;
        wt[j] = mesh * e;
      }
      const double worst = worst_error(n);
      if (worst <= eps) {
        for (int64_t j = 0; j < n; ++j) {  // back to [lo, hi]
          rates[j] = rate[j] / lo;
          weights[j] = wt[j] / lo;
        }
        *terms = n;
        *achieved = worst;
        *ok = 1;
        return;
      }
      mesh *= 0.8;
    }
  });
}

double tgb_gauss_cell_integral(double t, double c, double h) { return cell_integral(t, c, h); }

int tgb_primitive_norm(double alpha, int l, double* out) {
  return guarded([&] {
    tgb::require(alpha > 0.0, "primitive_norm: exponent must be positive");
    const double ns = std::pow(2.0 * alpha / kPi, 0.75);
    if (l == 0) *out = ns;
    else if (l == 1) *out = ns * 2.0 * std::sqrt(alpha);
    else throw tgb::Error(TGB_INVALID_ARGUMENT, "primitive_norm: only s and p supported");
  });
}

int tgb_gaussian_factor(double b_half, int64_t n, double center, double alpha, int degree, double* column) {
  return guarded([&] {
    if (std::abs(center) > b_half)
      throw tgb::Error(TGB_DOMAIN_ERROR, "discretize_basis: basis center outside the computational box");
    tgb::require(degree == 0 || degree == 1, "discretize_basis: per-axis degree must be 0 or 1");
    tgb::require(alpha > 0.0, "discretize_basis: primitive exponent must be positive");
    const double h = tgb_mesh_size(b_half, n);
    for (int64_t i = 0; i < n; ++i) {
      const double x = coord(h, n, i) - center;
      double v = std::exp(-alpha * x * x);
      if (degree == 1) v *= x;
      column[i] = v;
    }
  });
}

}  // extern "C"

// ORACLE — TEST INFRASTRUCTURE ONLY (see tengrid_oracle.hpp for the contract).
// Restatement of /root/reference/proj/src/{grid,fft,tensor,kernel,basis,
// reduction,hf,lattice,tei}.cpp without Eigen.  Line citations are to those
// files.  Arithmetic order follows the reference wherever it decides rounding
// (FFT butterflies, twiddle recurrence, window, lattice summation order).
#include "tengrid_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <thread>

namespace orc {

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kSqrtPi = 1.7724538509055160273;  // kernel.cpp:10

template <class F>
void par_for(idx n, F&& body) {
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 64 || nt == 1) {
    body(0, n);
    return;
  }
  std::vector<std::thread> ts;
  idx chunk = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    idx lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    ts.emplace_back([&, lo, hi] { body(lo, hi); });
  }
  for (auto& t : ts) t.join();
}

double fro(const Mat& a) {
  double s = 0;
  for (double x : a.d) s += x * x;
  return std::sqrt(s);
}

}  // namespace

// ---------------------------------------------------------------- dense LA

Mat matmul(const Mat& a, bool ta, const Mat& b, bool tb) {
  const idx m = ta ? a.cols : a.rows, k = ta ? a.rows : a.cols;
  const idx kb = tb ? b.cols : b.rows, n = tb ? b.rows : b.cols;
  req(k == kb, "matmul: inner dimension mismatch");
  Mat c(m, n);
  auto A = [&](idx i, idx l) { return ta ? a(l, i) : a(i, l); };
  auto B = [&](idx l, idx j) { return tb ? b(j, l) : b(l, j); };
  par_for(n, [&](idx j0, idx j1) {
    for (idx j = j0; j < j1; ++j) {
      double* cj = c.col(j);
      if (!ta) {
        for (idx l = 0; l < k; ++l) {
          const double blj = B(l, j);
          const double* al = a.col(l);
          for (idx i = 0; i < m; ++i) cj[i] += al[i] * blj;
        }
      } else {
        for (idx i = 0; i < m; ++i) {
          double s = 0;
          const double* ai = a.col(i);
          for (idx l = 0; l < k; ++l) s += ai[l] * B(l, j);
          cj[i] = s;
        }
      }
    }
  });
  (void)A;
  return c;
}

// Householder tridiagonalisation followed by implicit-shift QL; eigenvalues
// ascending, eigenvectors in columns.  (Replaces Eigen::SelfAdjointEigenSolver
// at reduction.cpp:95,110.)
void sym_eigen(const Mat& a_in, Vec& ev, Mat& z) {
  const idx n = a_in.rows;
  z = a_in;
  ev.assign(n, 0.0);
  Vec e(n, 0.0);
  if (n == 0) return;
  // matrix scale for the deflation test below (max |a_ij|, as the eigensolver the
  // reference links scales its input before tridiagonalising)
  double amax = 0.0;
  for (idx j = 0; j < n; ++j)
    for (idx i = 0; i < n; ++i) amax = std::max(amax, std::fabs(a_in(i, j)));
  // tridiagonalise (row i of the lower triangle eliminated from the bottom)
  for (idx i = n - 1; i > 0; --i) {
    const idx l = i - 1;
    double h = 0.0, scale = 0.0;
    if (l > 0) {
      for (idx k = 0; k <= l; ++k) scale += std::fabs(z(i, k));
      if (scale == 0.0) {
        e[i] = z(i, l);
      } else {
        for (idx k = 0; k <= l; ++k) {
          z(i, k) /= scale;
          h += z(i, k) * z(i, k);
        }
        double f = z(i, l);
        double g = f >= 0.0 ? -std::sqrt(h) : std::sqrt(h);
        e[i] = scale * g;
        h -= f * g;
        z(i, l) = f - g;
        f = 0.0;
        for (idx j = 0; j <= l; ++j) {
          z(j, i) = z(i, j) / h;
          g = 0.0;
          for (idx k = 0; k <= j; ++k) g += z(j, k) * z(i, k);
          for (idx k = j + 1; k <= l; ++k) g += z(k, j) * z(i, k);
          e[j] = g / h;
          f += e[j] * z(i, j);
        }
        const double hh = f / (h + h);
        for (idx j = 0; j <= l; ++j) {
          f = z(i, j);
          e[j] = g = e[j] - hh * f;
          for (idx k = 0; k <= j; ++k) z(j, k) -= (f * e[k] + g * z(i, k));
        }
      }
    } else {
      e[i] = z(i, l);
    }
    ev[i] = h;
  }
  ev[0] = 0.0;
  e[0] = 0.0;
  for (idx i = 0; i < n; ++i) {
    const idx l = i - 1;
    if (ev[i] != 0.0) {
      for (idx j = 0; j <= l; ++j) {
        double g = 0.0;
        for (idx k = 0; k <= l; ++k) g += z(i, k) * z(k, j);
        for (idx k = 0; k <= l; ++k) z(k, j) -= g * z(k, i);
      }
    }
    ev[i] = z(i, i);
    z(i, i) = 1.0;
    for (idx j = 0; j <= l; ++j) z(j, i) = z(i, j) = 0.0;
  }
  // implicit QL on the tridiagonal (ev diagonal, e sub-diagonal)
  for (idx i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  for (idx l = 0; l < n; ++l) {
    int iter = 0;
    idx m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::fabs(ev[m]) + std::fabs(ev[m + 1]);
        const double em = std::fabs(e[m]);
        // relative test, or |e|^2 <= eps^2 amax (|d_m| + |d_m+1|): deflates the
        // near-null block of a rank-deficient Gram matrix (RHOSVD's wide branch),
        // where both neighbouring diagonals are ~eps amax and the purely relative
        // test never fires
        if (em <= 1e-300 || em <= 2.220446049250313e-16 * dd ||
            (em / 2.220446049250313e-16) * (em / 2.220446049250313e-16) <= amax * dd)
          break;
      }
      if (m != l) {
        if (++iter > 200) throw numerical_error("sym_eigen: QL did not converge");
        double g = (ev[l + 1] - ev[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = ev[m] - ev[l] + e[l] / (g + (g >= 0 ? std::fabs(r) : -std::fabs(r)));
        double s = 1.0, c = 1.0, p = 0.0;
        idx i;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i], b = c * e[i];
          e[i + 1] = (r = std::hypot(f, g));
          if (r == 0.0) {
            ev[i + 1] -= p;
            e[m] = 0.0;
            break;
          }
          s = f / r;
          c = g / r;
          g = ev[i + 1] - p;
          r = (ev[i] - g) * s + 2.0 * c * b;
          ev[i + 1] = g + (p = s * r);
          g = c * r - b;
          for (idx k = 0; k < n; ++k) {
            f = z(k, i + 1);
            z(k, i + 1) = s * z(k, i) + c * f;
            z(k, i) = c * z(k, i) - s * f;
          }
        }
        if (r == 0.0 && i >= l) continue;
        ev[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  // sort ascending
  std::vector<idx> ord(n);
  for (idx i = 0; i < n; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](idx x, idx y) { return ev[x] < ev[y]; });
  Vec ev2(n);
  Mat z2(n, n);
  for (idx i = 0; i < n; ++i) {
    ev2[i] = ev[ord[i]];
    std::memcpy(z2.col(i), z.col(ord[i]), sizeof(double) * n);
  }
  ev.swap(ev2);
  z = std::move(z2);
}

// Householder QR with Eigen's reflector convention (beta = -sign(c0)*norm),
// returning the thin Q (m x k) and R (k x k).  (Replaces HouseholderQR at
// reduction.cpp:132 and tei.cpp:136.)
void householder_qr_thin(const Mat& a, Mat& q, Mat& r) {
  const idx m = a.rows, k = std::min(a.rows, a.cols);
  Mat w = a;
  Vec tau(k, 0.0);
  for (idx j = 0; j < k; ++j) {
    double c0 = w(j, j), tail = 0.0;
    for (idx i = j + 1; i < m; ++i) tail += w(i, j) * w(i, j);
    if (tail <= 2.2250738585072014e-308) {
      tau[j] = 0.0;
      for (idx i = j + 1; i < m; ++i) w(i, j) = 0.0;
      continue;
    }
    double beta = std::sqrt(c0 * c0 + tail);
    if (c0 >= 0.0) beta = -beta;
    for (idx i = j + 1; i < m; ++i) w(i, j) /= (c0 - beta);
    tau[j] = (beta - c0) / beta;
    w(j, j) = beta;
    // apply H = I - tau v v^T (v = [1; essential]) to the trailing columns
    for (idx c = j + 1; c < a.cols; ++c) {
      double s = w(j, c);
      for (idx i = j + 1; i < m; ++i) s += w(i, j) * w(i, c);
      s *= tau[j];
      w(j, c) -= s;
      for (idx i = j + 1; i < m; ++i) w(i, c) -= s * w(i, j);
    }
  }
  r = Mat(k, a.cols);
  for (idx c = 0; c < a.cols; ++c)
    for (idx i = 0; i <= std::min(c, k - 1); ++i) r(i, c) = w(i, c);
  q = Mat(m, k);
  for (idx i = 0; i < k; ++i) q(i, i) = 1.0;
  for (idx j = k - 1; j >= 0; --j) {
    if (tau[j] == 0.0) continue;
    for (idx c = 0; c < k; ++c) {
      double s = q(j, c);
      for (idx i = j + 1; i < m; ++i) s += w(i, j) * q(i, c);
      s *= tau[j];
      q(j, c) -= s;
      for (idx i = j + 1; i < m; ++i) q(i, c) -= s * w(i, j);
    }
  }
}

// One-sided Jacobi SVD, thin left vectors, singular values descending.
// (Replaces Eigen::JacobiSVD at reduction.cpp:29.)
void jacobi_svd_thin(const Mat& a, Mat& u, Vec& s) {
  const bool wide = a.rows < a.cols;
  // work on a tall matrix t (rows >= cols); left vectors of `a` are either
  // the normalised columns of t (tall) or the right rotation V (wide)
  Mat t = wide ? Mat(a.cols, a.rows) : a;
  if (wide)
    for (idx i = 0; i < a.rows; ++i)
      for (idx j = 0; j < a.cols; ++j) t(j, i) = a(i, j);
  const idx m = t.rows, k = t.cols;
  Mat v(k, k);
  for (idx i = 0; i < k; ++i) v(i, i) = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (idx p = 0; p < k; ++p)
      for (idx q2 = p + 1; q2 < k; ++q2) {
        double al = 0, be = 0, ga = 0;
        const double* tp = t.col(p);
        const double* tq = t.col(q2);
        for (idx i = 0; i < m; ++i) {
          al += tp[i] * tp[i];
          be += tq[i] * tq[i];
          ga += tp[i] * tq[i];
        }
        if (ga == 0.0 || std::fabs(ga) <= 1e-15 * std::sqrt(al * be)) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double tt = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + tt * tt), sn = c * tt;
        double* tpw = t.col(p);
        double* tqw = t.col(q2);
        for (idx i = 0; i < m; ++i) {
          const double x = tpw[i], y = tqw[i];
          tpw[i] = c * x - sn * y;
          tqw[i] = sn * x + c * y;
        }
        double* vp = v.col(p);
        double* vq = v.col(q2);
        for (idx i = 0; i < k; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = c * x - sn * y;
          vq[i] = sn * x + c * y;
        }
      }
    if (!rotated) break;
  }
  Vec sig(k);
  for (idx j = 0; j < k; ++j) {
    double ss = 0;
    for (idx i = 0; i < m; ++i) ss += t(i, j) * t(i, j);
    sig[j] = std::sqrt(ss);
  }
  std::vector<idx> ord(k);
  for (idx i = 0; i < k; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](idx x, idx y) { return sig[x] > sig[y]; });
  const idx r = std::min(a.rows, a.cols);
  s.assign(r, 0.0);
  u = Mat(a.rows, r);
  for (idx c = 0; c < r; ++c) {
    const idx j = ord[c];
    s[c] = sig[j];
    if (wide) {
      std::memcpy(u.col(c), v.col(j), sizeof(double) * a.rows);
    } else if (sig[j] > 0) {
      for (idx i = 0; i < m; ++i) u(i, c) = t(i, j) / sig[j];
    }
  }
  if (!wide) {
    // complete zero-singular columns with an orthonormal basis (Gram-Schmidt)
    for (idx c = 0; c < r; ++c) {
      if (s[c] > 0) continue;
      for (idx trial = 0; trial < a.rows; ++trial) {
        Vec x(a.rows, 0.0);
        x[(c + trial) % a.rows] = 1.0;
        for (int rep = 0; rep < 2; ++rep)
          for (idx c2 = 0; c2 < r; ++c2) {
            if (c2 == c || (s[c2] <= 0 && c2 > c)) continue;
            double d = 0;
            for (idx i = 0; i < a.rows; ++i) d += u(i, c2) * x[i];
            for (idx i = 0; i < a.rows; ++i) x[i] -= d * u(i, c2);
          }
        double nrm = 0;
        for (double y : x) nrm += y * y;
        nrm = std::sqrt(nrm);
        if (nrm > 0.5) {
          for (idx i = 0; i < a.rows; ++i) u(i, c) = x[i] / nrm;
          break;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- grid.cpp

Grid make_grid(const std::array<double, 3>& b, const std::array<idx, 3>& n) {  // grid.cpp:7-18
  Grid g;
  for (int ax = 0; ax < 3; ++ax) {
    req(b[ax] > 0.0, "make_grid: box half-width must be positive");
    req(n[ax] >= 2, "make_grid: need at least 2 grid points per axis");
    g.n[ax] = n[ax];
    g.b[ax] = b[ax];
    g.h[ax] = 2.0 * b[ax] / static_cast<double>(n[ax] + 1);
  }
  return g;
}

idx snap_to_node(const Grid& g, int ax, double x) {  // grid.cpp:23-30
  if (std::abs(x) > g.b[ax]) throw std::domain_error("snap_to_node: point outside the computational box");
  const idx i = static_cast<idx>(std::llround(x / g.h[ax] + 0.5 * static_cast<double>(g.n[ax] - 1)));
  if (i < 0 || i >= g.n[ax] || std::abs(x - g.coord(ax, i)) > 0.5 * g.h[ax] * (1.0 + 1e-12))
    throw snap_error("snap_to_node: point farther than h/2 from every node; refine the grid");
  return i;
}

idx window_offset(const Grid& g, int ax, double center) {  // grid.cpp:32-38
  const idx i0 = snap_to_node(g, ax, center);
  const idx ofs = (g.n[ax] - 1) - i0;
  req(ofs >= 0 && ofs + g.n[ax] <= 2 * g.n[ax], "window_offset: window escapes the doubled grid");
  return ofs;
}

// ---------------------------------------------------------------- fft.cpp

// fft.cpp:18-45 — bit reversal, radix-2 butterflies with the twiddle
// recurrence w *= wlen, 1/n scaling on the inverse.
static void fft_c(std::vector<std::complex<double>>& a, bool inverse) {
  const size_t n = a.size();
  req(n > 0 && (n & (n - 1)) == 0, "fft_inplace: size must be a power of two");
  size_t j = 0;
  for (size_t i = 1; i < n; ++i) {
    size_t bit = n >> 1;
    while (j & bit) {
      j ^= bit;
      bit >>= 1;
    }
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    const double ang = 2.0 * kPi / static_cast<double>(len) * (inverse ? 1.0 : -1.0);
    const std::complex<double> step(std::cos(ang), std::sin(ang));
    const size_t half = len / 2;
    for (size_t base = 0; base < n; base += len) {
      std::complex<double> w(1.0, 0.0);
      for (size_t k = 0; k < half; ++k) {
        const std::complex<double> top = a[base + k];
        const std::complex<double> bot = a[base + k + half] * w;
        a[base + k] = top + bot;
        a[base + k + half] = top - bot;
        w *= step;
      }
    }
  }
  if (inverse) {
    const double s = 1.0 / static_cast<double>(n);
    for (auto& z : a) z *= s;
  }
}

void fft_radix2(std::vector<double>& re, std::vector<double>& im, bool inverse) {
  std::vector<std::complex<double>> a(re.size());
  for (size_t i = 0; i < re.size(); ++i) a[i] = {re[i], im[i]};
  fft_c(a, inverse);
  for (size_t i = 0; i < re.size(); ++i) {
    re[i] = a[i].real();
    im[i] = a[i].imag();
  }
}

static size_t next_pow2(size_t n) {  // fft.cpp:12-16
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

Vec conv_full_direct(const double* u, idx nu, const double* v, idx nv) {  // fft.cpp:47-56
  Vec out(static_cast<size_t>(nu + nv - 1), 0.0);
  for (idx j = 0; j < nu; ++j) {
    const double uj = u[j];
    if (uj == 0.0) continue;
    for (idx k = 0; k < nv; ++k) out[j + k] += uj * v[k];
  }
  return out;
}

Vec conv_full_fft(const double* u, idx nu, const double* v, idx nv) {  // fft.cpp:58-71
  const size_t m = next_pow2(static_cast<size_t>(nu + nv - 1));
  std::vector<std::complex<double>> a(m), b(m);
  for (idx i = 0; i < nu; ++i) a[i] = u[i];
  for (idx i = 0; i < nv; ++i) b[i] = v[i];
  fft_c(a, false);
  fft_c(b, false);
  for (size_t i = 0; i < m; ++i) a[i] *= b[i];
  fft_c(a, true);
  Vec out(static_cast<size_t>(nu + nv - 1));
  for (idx i = 0; i < nu + nv - 1; ++i) out[i] = a[i].real();
  return out;
}

Vec central_window(const Vec& full, idx n) {  // fft.cpp:79-90
  req(static_cast<idx>(full.size()) == 2 * n - 1, "central_window: expected full convolution of two length-n vectors");
  Vec out(n);
  if (n % 2 == 1) {
    const idx ofs = (n - 1) / 2;
    for (idx i = 0; i < n; ++i) out[i] = full[i + ofs];
  } else {
    const idx ofs = n / 2 - 1;
    for (idx i = 0; i < n; ++i) out[i] = 0.5 * (full[i + ofs] + full[i + ofs + 1]);
  }
  return out;
}

Mat conv_central_many(const Mat& U, const double* v, idx n) {  // fft.cpp:97-122
  req(U.rows == n, "conv_central_many: column length mismatch");
  Mat out(n, U.cols);
  if (n < 128) {  // kFftConvThreshold, fft.hpp:13
    for (idx c = 0; c < U.cols; ++c) {
      Vec w = central_window(conv_full_direct(U.col(c), n, v, n), n);
      std::memcpy(out.col(c), w.data(), sizeof(double) * n);
    }
    return out;
  }
  const size_t m = next_pow2(static_cast<size_t>(2 * n - 1));
  std::vector<std::complex<double>> fv(m);
  for (idx i = 0; i < n; ++i) fv[i] = v[i];
  fft_c(fv, false);
  par_for(U.cols, [&](idx c0, idx c1) {
    std::vector<std::complex<double>> a(m);
    Vec full(static_cast<size_t>(2 * n - 1));
    for (idx c = c0; c < c1; ++c) {
      std::fill(a.begin(), a.end(), std::complex<double>(0.0, 0.0));
      for (idx i = 0; i < n; ++i) a[i] = U(i, c);
      fft_c(a, false);
      for (size_t i = 0; i < m; ++i) a[i] *= fv[i];
      fft_c(a, true);
      for (idx i = 0; i < 2 * n - 1; ++i) full[i] = a[i].real();
      Vec w = central_window(full, n);
      std::memcpy(out.col(c), w.data(), sizeof(double) * n);
    }
  });
  return out;
}

// ---------------------------------------------------------------- tensor.cpp

static void check_valid(const CP3& t) {  // tensor.hpp:145-149
  for (int ax = 0; ax < 3; ++ax) req(t.f[ax].cols == t.rank(), "CanonicalTensor3: factor/weight rank mismatch");
}

static void same_extents(const CP3& a, const CP3& b, const char* what) {
  for (int ax = 0; ax < 3; ++ax) req(a.extent(ax) == b.extent(ax), what);
}

void normalize(CP3& t) {  // tensor.cpp:18-31
  check_valid(t);
  for (idx k = 0; k < t.rank(); ++k)
    for (int ax = 0; ax < 3; ++ax) {
      double* c = t.f[ax].col(k);
      double ss = 0;
      for (idx i = 0; i < t.f[ax].rows; ++i) ss += c[i] * c[i];
      const double nrm = std::sqrt(ss);
      if (nrm > 0.0) {
        for (idx i = 0; i < t.f[ax].rows; ++i) c[i] /= nrm;
        t.w[k] *= nrm;
      } else {
        t.w[k] = 0.0;
      }
    }
}

CP3 convolve(const CP3& a, const CP3& b, const std::array<double, 3>& h) {  // tensor.cpp:179-198
  check_valid(a);
  check_valid(b);
  same_extents(a, b, "convolve: extent mismatch");
  req(h[0] > 0.0 && h[1] > 0.0 && h[2] > 0.0, "convolve: mesh size must be positive");
  const idx ra = a.rank(), rb = b.rank();
  CP3 out;
  out.w.resize(ra * rb);
  for (idx j = 0; j < rb; ++j)
    for (idx i = 0; i < ra; ++i) out.w[i + ra * j] = a.w[i] * b.w[j];
  for (int ax = 0; ax < 3; ++ax) {
    const idx n = a.extent(ax);
    out.f[ax] = Mat(n, ra * rb);
    for (idx j = 0; j < rb; ++j) {
      Mat cols = conv_central_many(a.f[ax], b.f[ax].col(j), n);
      for (idx i = 0; i < ra; ++i)
        for (idx r = 0; r < n; ++r) out.f[ax](r, j * ra + i) = h[ax] * cols(r, i);
    }
  }
  return out;
}

CP3 hadamard(const CP3& a, const CP3& b) {  // tensor.cpp:141-157
  check_valid(a);
  check_valid(b);
  same_extents(a, b, "hadamard: extent mismatch");
  const idx ra = a.rank(), rb = b.rank();
  CP3 out;
  out.w.resize(ra * rb);
  for (int ax = 0; ax < 3; ++ax) out.f[ax] = Mat(a.extent(ax), ra * rb);
  for (idx j = 0; j < rb; ++j)
    for (idx i = 0; i < ra; ++i) {
      const idx k = i + ra * j;
      out.w[k] = a.w[i] * b.w[j];
      for (int ax = 0; ax < 3; ++ax)
        for (idx r = 0; r < a.extent(ax); ++r) out.f[ax](r, k) = a.f[ax](r, i) * b.f[ax](r, j);
    }
  return out;
}

CP3 add(const CP3& a, const CP3& b) {  // tensor.cpp:159-171
  check_valid(a);
  check_valid(b);
  same_extents(a, b, "add: extent mismatch");
  CP3 out;
  out.w = a.w;
  out.w.insert(out.w.end(), b.w.begin(), b.w.end());
  for (int ax = 0; ax < 3; ++ax) {
    out.f[ax] = Mat(a.extent(ax), a.rank() + b.rank());
    std::copy(a.f[ax].d.begin(), a.f[ax].d.end(), out.f[ax].d.begin());
    std::copy(b.f[ax].d.begin(), b.f[ax].d.end(), out.f[ax].d.begin() + a.f[ax].d.size());
  }
  return out;
}

double scalar_product(const CP3& a, const CP3& b) {  // tensor.cpp:88-98
  check_valid(a);
  check_valid(b);
  same_extents(a, b, "scalar_product: extent mismatch");
  if (a.rank() == 0 || b.rank() == 0) return 0.0;
  Mat g(a.rank(), b.rank(), 1.0);
  for (int ax = 0; ax < 3; ++ax) {
    Mat p = matmul(a.f[ax], true, b.f[ax], false);
    for (size_t i = 0; i < g.d.size(); ++i) g.d[i] *= p.d[i];
  }
  double s = 0.0;
  for (idx j = 0; j < b.rank(); ++j) {
    double t = 0.0;
    for (idx i = 0; i < a.rank(); ++i) t += a.w[i] * g(i, j);
    s += t * b.w[j];
  }
  return s;
}

double value_at(const CP3& t, idx i, idx j, idx k) {  // tensor.hpp:135-140
  double s = 0.0;
  for (idx q = 0; q < t.rank(); ++q) s += t.w[q] * t.f[0](i, q) * t.f[1](j, q) * t.f[2](k, q);
  return s;
}

// ---------------------------------------------------------------- kernel.cpp

static double expsum_eval(const ExpSum& es, double r) {  // kernel.hpp:37-41
  double s = 0.0;
  for (size_t k = 0; k < es.weights.size(); ++k) s += es.weights[k] * std::exp(-es.nodes[k] * es.nodes[k] * r * r);
  return s;
}

ExpSum make_expsum(idx m, double c0, double fit_lo, double fit_hi) {  // kernel.cpp:71-123 (Newton kind)
  req(m >= 1, "make_radial_expsum: need at least one quadrature point");
  req(c0 > 0.0, "make_radial_expsum: C0 must be positive");
  ExpSum es;
  es.m = m;
  es.c0 = c0;
  es.mesh = c0 * std::log(static_cast<double>(std::max<idx>(m, 2))) / static_cast<double>(m);
  for (idx k = -m; k <= m; ++k) {
    const double t = static_cast<double>(k) * es.mesh;
    const double w = 2.0 / kSqrtPi * es.mesh;  // Newton integrand weight (kernel.cpp:18-19)
    if (w <= 0.0) continue;
    es.nodes.push_back(t);
    es.weights.push_back(w);
  }
  // default validity window (kernel.cpp:41-49)
  const double t_max = c0 * std::log(static_cast<double>(std::max<idx>(m, 2)));
  double dlo = 3.0 / t_max;
  double dhi = kPi / (3.0 * es.mesh);
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
  const int samples = 200;
  for (int i = 0; i < samples; ++i) {
    const double r = fit_lo * std::pow(fit_hi / fit_lo, static_cast<double>(i) / (samples - 1));
    const double f = expsum_eval(es, r);
    num += f * (1.0 / r);
    den += f * f;
  }
  es.scale = den > 0.0 ? num / den : 1.0;
  for (double& w : es.weights) w *= es.scale;
  return es;
}

double gauss_cell_integral(double t, double c, double h) {  // kernel.cpp:171-180
  if (t == 0.0) return h;
  const double xl = c - 0.5 * h;
  const double xr = c + 0.5 * h;
  const double k = kSqrtPi / (2.0 * t);
  if (xl >= 0.0) return k * (std::erfc(t * xl) - std::erfc(t * xr));
  if (xr <= 0.0) return k * (std::erfc(-t * xr) - std::erfc(-t * xl));
  return k * (std::erf(t * xr) - std::erf(t * xl));
}

CP3 kernel_tensor(const Grid& g, const ExpSum& es, bool doubled) {  // kernel.cpp:182-203
  const idx r = static_cast<idx>(es.weights.size());
  CP3 t;
  t.w.assign(r, 1.0);
  for (int ax = 0; ax < 3; ++ax) {
    const idx len = doubled ? 2 * g.n[ax] : g.n[ax];
    t.f[ax] = Mat(len, r);
    for (idx q = 0; q < r; ++q) {
      const double tq = std::abs(es.nodes[q]);
      const double aq = std::cbrt(es.weights[q]);
      for (idx i = 0; i < len; ++i) {
        const double c = doubled ? g.ref_coord(ax, i) : g.coord(ax, i);
        t.f[ax](i, q) = aq * gauss_cell_integral(tq, c, g.h[ax]);
      }
    }
  }
  return t;
}

// ---------------------------------------------------------------- basis.cpp

double primitive_norm(double alpha, int l) {  // basis.cpp:8-14
  req(alpha > 0.0, "primitive_norm: exponent must be positive");
  const double ns = std::pow(2.0 * alpha / kPi, 0.75);
  if (l == 0) return ns;
  if (l == 1) return ns * 2.0 * std::sqrt(alpha);
  throw invalid_argument("primitive_norm: only s and p supported");
}

std::vector<CP3> discretize_basis(const Grid& g, const std::vector<BasisFn>& fns) {  // basis.cpp:16-46
  std::vector<CP3> out;
  for (const auto& f : fns) {
    for (int ax = 0; ax < 3; ++ax) {
      if (std::abs(f.center[ax]) > g.b[ax])
        throw std::domain_error("discretize_basis: basis center outside the computational box");
      req(f.deg[ax] == 0 || f.deg[ax] == 1, "discretize_basis: per-axis degree must be 0 or 1");
    }
    req(!f.exps.empty(), "discretize_basis: contraction needs at least one primitive");
    const idx np = static_cast<idx>(f.exps.size());
    const int tot = f.deg[0] + f.deg[1] + f.deg[2];
    CP3 t;
    t.w.resize(np);
    for (int ax = 0; ax < 3; ++ax) t.f[ax] = Mat(g.n[ax], np);
    for (idx p = 0; p < np; ++p) {
      req(f.exps[p] > 0.0, "discretize_basis: primitive exponent must be positive");
      t.w[p] = f.coefs[p] * primitive_norm(f.exps[p], tot);
      for (int ax = 0; ax < 3; ++ax)
        for (idx i = 0; i < g.n[ax]; ++i) {
          const double x = g.coord(ax, i) - f.center[ax];
          double v = std::exp(-f.exps[p] * x * x);
          if (f.deg[ax] == 1) v *= x;
          t.f[ax](i, p) = v;
        }
    }
    out.push_back(std::move(t));
  }
  return out;
}

// ---------------------------------------------------------------- reduction.cpp

static idx select_rank(const Vec& s, const RedCfg& c, int mode, bool* clamped) {  // reduction.cpp:34-59
  idx numeric = 0;
  if (!s.empty()) {
    const double cut = s[0] * 1e-15 * std::sqrt(static_cast<double>(s.size()));
    while (numeric < static_cast<idx>(s.size()) && s[numeric] > cut) ++numeric;
  }
  if (!c.use_eps) {
    const idx want = c.ranks[mode];
    req(want >= 0, "select_rank: negative rank request");
    if (want > numeric && clamped) *clamped = true;
    return std::min(want, numeric);
  }
  double total = 0;
  for (double x : s) total += x * x;
  if (total == 0.0) return 0;
  const double budget = c.eps * c.eps * total;
  double tail = total;
  idx r = 0;
  while (r < numeric && tail > budget) {
    tail -= s[r] * s[r];
    ++r;
  }
  return r;
}

static Vec project_core(const CP3& a, const std::array<Mat, 3>& z, std::array<idx, 3>& rr) {  // reduction.cpp:63-81
  std::array<Mat, 3> p;
  for (int ax = 0; ax < 3; ++ax) p[ax] = matmul(z[ax], true, a.f[ax], false);
  const idx r0 = z[0].cols, r1 = z[1].cols, r2 = z[2].cols;
  rr = {r0, r1, r2};
  Vec core(static_cast<size_t>(r0 * r1 * r2), 0.0);
  for (idx k = 0; k < a.rank(); ++k) {
    const double w = a.w[k];
    if (w == 0.0) continue;
    for (idx l = 0; l < r2; ++l) {
      const double wl = w * p[2](l, k);
      for (idx j = 0; j < r1; ++j) {
        const double wjl = wl * p[1](j, k);
        double* col = core.data() + r0 * (j + r1 * l);
        for (idx i = 0; i < r0; ++i) col[i] += wjl * p[0](i, k);
      }
    }
  }
  return core;
}

static Mat left_cols(const Mat& u, idx r) {
  Mat o(u.rows, r);
  std::copy(u.d.begin(), u.d.begin() + u.rows * r, o.d.begin());
  return o;
}

void thin_svd_left(const Mat& a, Mat& u, Vec& s) {  // reduction.cpp:85-138
  if (a.cols == 0 || a.rows == 0) {
    u = Mat(a.rows, 0);
    s.clear();
    return;
  }
  if (a.cols >= 4 * a.rows && a.cols > 8192) {  // wide Gram branch, reduction.cpp:93-104
    Mat gram = matmul(a, false, a, true);
    Vec ev;
    Mat z;
    sym_eigen(gram, ev, z);
    const idx n = a.rows;
    u = Mat(n, n);
    s.assign(n, 0.0);
    for (idx i = 0; i < n; ++i) {
      std::memcpy(u.col(i), z.col(n - 1 - i), sizeof(double) * n);
      s[i] = std::sqrt(std::max(0.0, ev[n - 1 - i]));
    }
    return;
  }
  if (a.rows < 4 * a.cols || a.cols < 8) {  // reduction.cpp:105-108
    jacobi_svd_thin(a, u, s);
    return;
  }
  Mat gram = matmul(a, true, a, false);  // tall Gram branch, reduction.cpp:109-137
  Vec ev;
  Mat z;
  sym_eigen(gram, ev, z);
  const idx r = a.cols;
  double lmax = 0.0;
  for (double x : ev) lmax = std::max(lmax, x);
  s.clear();
  std::vector<Vec> cols;
  for (idx i = r - 1; i >= 0; --i) {
    const double lam = ev[i];
    if (lam <= lmax * 1e-24 || lam <= 0.0) break;
    const double sg = std::sqrt(lam);
    s.push_back(sg);
    Vec c(a.rows, 0.0);
    for (idx l = 0; l < r; ++l) {
      const double zl = z(l, i);
      const double* al = a.col(l);
      for (idx q = 0; q < a.rows; ++q) c[q] += al[q] * zl;
    }
    for (double& x : c) x /= sg;
    cols.push_back(std::move(c));
  }
  const idx kept = static_cast<idx>(s.size());
  Mat uu(a.rows, kept);
  for (idx c = 0; c < kept; ++c) std::memcpy(uu.col(c), cols[c].data(), sizeof(double) * a.rows);
  if (kept > 0) {
    Mat q, rr;
    householder_qr_thin(uu, q, rr);
    for (idx c = 0; c < kept; ++c)
      if (rr(c, c) < 0.0)
        for (idx i = 0; i < a.rows; ++i) q(i, c) = -q(i, c);
    u = q;
  } else {
    u = uu;
  }
}

TuckerRes rhosvd(const CP3& a, const RedCfg& c) {  // reduction.cpp:172-190
  check_valid(a);
  TuckerRes res;
  CP3 w = a;
  normalize(w);
  std::array<Mat, 3> z;
  for (int mode = 0; mode < 3; ++mode) {
    Mat aw = w.f[mode];
    for (idx k = 0; k < w.rank(); ++k)
      for (idx i = 0; i < aw.rows; ++i) aw(i, k) *= w.w[k];
    Mat u;
    Vec s;
    thin_svd_left(aw, u, s);
    const idx r = select_rank(s, c, mode, &res.rank_clamped);
    z[mode] = left_cols(u, r);
    res.sigma[mode] = s;
  }
  res.t.side = z;
  res.t.core = project_core(w, z, res.t.r);
  return res;
}

TuckerRes canonical_to_tucker(const CP3& a, const RedCfg& c) {  // reduction.cpp:192-236
  check_valid(a);
  TuckerRes init = rhosvd(a, c);
  if (a.rank() == 0 || init.t.core.empty()) return init;
  CP3 w = a;
  normalize(w);
  std::array<Mat, 3> z = init.t.side;
  TuckerRes res = init;
  res.sweep_fits.clear();
  double prev = -1.0;
  for (int sweep = 0; sweep < c.max_sweeps; ++sweep) {
    double fit = 0.0;
    for (int ax = 0; ax < 3; ++ax) {
      const int m = (ax + 1) % 3, p = (ax + 2) % 3;
      Mat pm = matmul(z[m], true, w.f[m], false);
      Mat pp = matmul(z[p], true, w.f[p], false);
      const idx rm = pm.rows, rp = pp.rows;
      Mat cm(w.rank(), rm * rp);
      for (idx k = 0; k < w.rank(); ++k)
        for (idx l = 0; l < rp; ++l) {
          const double s = w.w[k] * pp(l, k);
          for (idx i = 0; i < rm; ++i) cm(k, l * rm + i) = s * pm(i, k);
        }
      Mat mat = matmul(w.f[ax], false, cm, false);
      Mat u;
      Vec sg;
      thin_svd_left(mat, u, sg);
      bool finite = true;
      for (double x : u.d) finite = finite && std::isfinite(x);
      if (u.cols == 0 || !finite) {
        res.rhosvd_fallback = true;
        return res;
      }
      const idx r = std::min<idx>(z[ax].cols, u.cols);
      z[ax] = left_cols(u, r);
      fit = fro(matmul(z[ax], true, mat, false));
    }
    res.sweep_fits.push_back(fit);
    if (prev >= 0.0 && std::abs(fit - prev) < 1e-14 * std::max(1.0, fit)) break;
    prev = fit;
  }
  res.t.side = z;
  res.t.core = project_core(w, z, res.t.r);
  return res;
}

CP3 tucker_to_canonical(const Tucker3& t) {  // reduction.cpp:238-269
  const auto r = t.r;
  CP3 out;
  if (r[0] * r[1] * r[2] == 0) {
    for (int ax = 0; ax < 3; ++ax) out.f[ax] = Mat(t.side[ax].rows, 0);
    return out;
  }
  int ax = 0;
  for (int m = 1; m < 3; ++m)
    if (r[m] > r[ax]) ax = m;
  const int m1 = (ax + 1) % 3, m2 = (ax + 2) % 3;
  const idx rank = r[m1] * r[m2];
  out.w.assign(rank, 1.0);
  out.f[ax] = Mat(t.side[ax].rows, rank);
  out.f[m1] = Mat(t.side[m1].rows, rank);
  out.f[m2] = Mat(t.side[m2].rows, rank);
  Vec slice(r[ax]);
  for (idx j2 = 0; j2 < r[m2]; ++j2)
    for (idx j1 = 0; j1 < r[m1]; ++j1) {
      const idx q = j1 + r[m1] * j2;
      for (idx i = 0; i < r[ax]; ++i) {
        std::array<idx, 3> id{};
        id[ax] = i;
        id[m1] = j1;
        id[m2] = j2;
        slice[i] = t.core[id[0] + r[0] * (id[1] + r[1] * id[2])];
      }
      for (idx row = 0; row < t.side[ax].rows; ++row) {
        double s = 0;
        for (idx i = 0; i < r[ax]; ++i) s += t.side[ax](row, i) * slice[i];
        out.f[ax](row, q) = s;
      }
      std::memcpy(out.f[m1].col(q), t.side[m1].col(j1), sizeof(double) * t.side[m1].rows);
      std::memcpy(out.f[m2].col(q), t.side[m2].col(j2), sizeof(double) * t.side[m2].rows);
    }
  normalize(out);
  return out;
}

CP3 reduce_rank(const CP3& a, const RedCfg& c) {  // reduction.cpp:271-273
  return tucker_to_canonical(canonical_to_tucker(a, c).t);
}

// ---------------------------------------------------------------- hf.cpp

static CP3 zero_cp(const std::array<idx, 3>& d) {
  CP3 t;
  for (int ax = 0; ax < 3; ++ax) t.f[ax] = Mat(d[ax], 0);
  return t;
}

static CP3 scaled(const CP3& a, double s) {  // tensor.cpp:173-177
  CP3 o = a;
  for (double& x : o.w) x *= s;
  return o;
}

CP3 density_tensor(const std::vector<CP3>& disc, const Mat& c_occ, double eps) {  // hf.cpp:118-129, 39-46
  req(!disc.empty(), "density_tensor: empty basis");
  req(c_occ.rows == static_cast<idx>(disc.size()), "density_tensor: coefficient shape mismatch");
  const std::array<idx, 3> d{disc[0].extent(0), disc[0].extent(1), disc[0].extent(2)};
  CP3 theta = zero_cp(d);
  for (idx a = 0; a < c_occ.cols; ++a) {
    CP3 phi = zero_cp(d);
    for (idx k = 0; k < static_cast<idx>(disc.size()); ++k) {
      if (c_occ(k, a) == 0.0) continue;
      phi = add(phi, scaled(disc[k], c_occ(k, a)));
    }
    theta = add(theta, scaled(hadamard(phi, phi), 2.0));
  }
  if (theta.rank() <= 1 || eps <= 0.0) return theta;
  RedCfg c;
  c.use_eps = true;
  c.eps = eps;
  return reduce_rank(theta, c);
}

CP3 hartree_potential(const CP3& theta, const CP3& kernel, const std::array<double, 3>& h) {  // hf.cpp:131-138
  const double inv_vol = 1.0 / (h[0] * h[1] * h[2]);
  return convolve(theta, scaled(kernel, inv_vol), h);
}

Mat coulomb_matrix(const Grid& g, const std::vector<CP3>& disc, const CP3& vh) {  // hf.cpp:140-151
  const idx nb = static_cast<idx>(disc.size());
  const double vol = g.h[0] * g.h[1] * g.h[2];
  Mat j(nb, nb);
  for (idx k = 0; k < nb; ++k)
    for (idx m = k; m < nb; ++m) {
      j(k, m) = vol * scalar_product(hadamard(disc[k], disc[m]), vh);
      j(m, k) = j(k, m);
    }
  return j;
}

// S_km = h^3 <G_k, G_m>   (hf.cpp:48-58)
Mat overlap_matrix(const Grid& g, const std::vector<CP3>& disc) {
  const idx nb = static_cast<idx>(disc.size());
  const double vol = g.h[0] * g.h[1] * g.h[2];
  Mat s(nb, nb);
  for (idx k = 0; k < nb; ++k)
    for (idx m = k; m < nb; ++m) {
      s(k, m) = vol * scalar_product(disc[k], disc[m]);
      s(m, k) = s(k, m);
    }
  return s;
}

// u^T tridiag{-1,2,-1} v and u^T tridiag{1,4,1} v / 6   (hf.cpp:13-37)
static double stencil_form(const double* u, const double* v, idx n) {
  double s = 0.0;
  for (idx i = 0; i < n; ++i) {
    double av = 2.0 * v[i];
    if (i > 0) av -= v[i - 1];
    if (i + 1 < n) av -= v[i + 1];
    s += u[i] * av;
  }
  return s;
}
static double mass_form(const double* u, const double* v, idx n) {
  double s = 0.0;
  for (idx i = 0; i < n; ++i) {
    double av = 4.0 * v[i];
    if (i > 0) av += v[i - 1];
    if (i + 1 < n) av += v[i + 1];
    s += u[i] * av;
  }
  return s / 6.0;
}

// T_km = 1/2 sum_ij w_i w_j sum_ax stiff_ax mass_{ax+1} mass_{ax+2}   (hf.cpp:60-87)
Mat kinetic_matrix(const Grid& g, const std::vector<CP3>& disc, bool exact_mass) {
  const idx nb = static_cast<idx>(disc.size());
  Mat t(nb, nb);
  for (idx k = 0; k < nb; ++k)
    for (idx m = k; m < nb; ++m) {
      const CP3& a = disc[k];
      const CP3& b = disc[m];
      double sum = 0.0;
      for (idx i = 0; i < a.rank(); ++i)
        for (idx j = 0; j < b.rank(); ++j) {
          const double w = a.w[i] * b.w[j];
          double stiff[3], mass[3];
          for (int ax = 0; ax < 3; ++ax) {
            const idx n = a.f[ax].rows;
            const double* u = a.f[ax].col(i);
            const double* v = b.f[ax].col(j);
            stiff[ax] = stencil_form(u, v, n) / g.h[ax];
            double dot = 0.0;
            for (idx r = 0; r < n; ++r) dot += u[r] * v[r];
            mass[ax] = exact_mass ? g.h[ax] * mass_form(u, v, n) : g.h[ax] * dot;
          }
          for (int ax = 0; ax < 3; ++ax) sum += w * stiff[ax] * mass[(ax + 1) % 3] * mass[(ax + 2) % 3];
        }
      t(k, m) = 0.5 * sum;
      t(m, k) = t(k, m);
    }
  return t;
}

// P_c = sum_a Z_a W_a Ptilde: windows of the doubled reference   (hf.cpp:89-101)
CP3 nuclear_potential_tensor(const Grid& g, const std::vector<std::array<double, 3>>& centers, const Vec& charges,
                             const CP3& ref) {
  for (int ax = 0; ax < 3; ++ax)
    req(ref.extent(ax) == 2 * g.n[ax], "nuclear_potential_tensor: reference kernel must live on the doubled grid");
  CP3 pc = zero_cp(g.n);
  for (size_t a = 0; a < centers.size(); ++a) {
    CP3 sh;
    sh.w.resize(ref.w.size());
    for (size_t q = 0; q < ref.w.size(); ++q) sh.w[q] = charges[a] * ref.w[q];
    for (int ax = 0; ax < 3; ++ax) {
      const idx ofs = window_offset(g, ax, centers[a][ax]);
      sh.f[ax] = Mat(g.n[ax], ref.rank());
      for (idx q = 0; q < ref.rank(); ++q)
        for (idx i = 0; i < g.n[ax]; ++i) sh.f[ax](i, q) = ref.f[ax](ofs + i, q);
    }
    pc = add(pc, sh);
  }
  return pc;
}

// V_km = -<G_k . G_m, P_c>   (hf.cpp:103-116)
Mat nuclear_matrix(const std::vector<CP3>& disc, const CP3& pc) {
  const idx nb = static_cast<idx>(disc.size());
  Mat v(nb, nb);
  for (idx k = 0; k < nb; ++k)
    for (idx m = k; m < nb; ++m) {
      v(k, m) = -scalar_product(hadamard(disc[k], disc[m]), pc);
      v(m, k) = v(k, m);
    }
  return v;
}

// K_km = sum_a h^3 <G_k . phi_a, (G_m . phi_a) * P/h^3>, symmetrised   (hf.cpp:153-170)
Mat exchange_matrix(const Grid& g, const std::vector<CP3>& disc, const Mat& c_occ, const CP3& kernel) {
  const idx nb = static_cast<idx>(disc.size());
  const double vol = g.h[0] * g.h[1] * g.h[2];
  const double inv_vol = 1.0 / vol;
  Mat k_mat(nb, nb);
  const CP3 kscaled = scaled(kernel, inv_vol);
  for (idx a = 0; a < c_occ.cols; ++a) {
    CP3 phi = zero_cp(g.n);
    for (idx k = 0; k < nb; ++k) {
      if (c_occ(k, a) == 0.0) continue;
      phi = add(phi, scaled(disc[k], c_occ(k, a)));
    }
    std::vector<CP3> g_phi(nb);
    for (idx m = 0; m < nb; ++m) g_phi[m] = hadamard(disc[m], phi);
    for (idx m = 0; m < nb; ++m) {
      const CP3 v_m = convolve(g_phi[m], kscaled, g.h);
      for (idx k = 0; k < nb; ++k) k_mat(k, m) += vol * scalar_product(g_phi[k], v_m);
    }
  }
  Mat out(nb, nb);
  for (idx j = 0; j < nb; ++j)
    for (idx i = 0; i < nb; ++i) out(i, j) = 0.5 * (k_mat(i, j) + k_mat(j, i));
  return out;
}

// vec_j = L (L^T vec_d), J = (j + j^T) / 2   (tei.cpp:215-223)
Mat coulomb_from_factors(const Mat& chol, const Mat& d) {
  const idx n = d.rows;
  req(chol.rows == n * n && d.cols == n, "coulomb_from_factors: shape mismatch");
  Vec t(chol.cols, 0.0), vj(n * n, 0.0);
  for (idx s = 0; s < chol.cols; ++s) {
    double acc = 0.0;
    for (idx r = 0; r < n * n; ++r) acc += chol(r, s) * d.d[r];
    t[s] = acc;
  }
  for (idx s = 0; s < chol.cols; ++s)
    for (idx r = 0; r < n * n; ++r) vj[r] += chol(r, s) * t[s];
  Mat j(n, n);
  for (idx c = 0; c < n; ++c)
    for (idx r = 0; r < n; ++r) j(r, c) = 0.5 * (vj[r + n * c] + vj[c + n * r]);
  return j;
}

// k = -1/2 sum_s M_s D M_s^T, K = (k + k^T) / 2   (tei.cpp:225-234)
Mat exchange_from_factors(const Mat& chol, const Mat& d) {
  const idx n = d.rows;
  req(chol.rows == n * n && d.cols == n, "exchange_from_factors: shape mismatch");
  Mat k(n, n);
  for (idx s = 0; s < chol.cols; ++s) {
    Mat m(n, n);
    std::memcpy(m.d.data(), chol.col(s), sizeof(double) * n * n);
    const Mat md = matmul(m, false, d, false);
    const Mat mdm = matmul(md, false, m, true);
    for (idx r = 0; r < n * n; ++r) k.d[r] -= 0.5 * mdm.d[r];
  }
  Mat out(n, n);
  for (idx c = 0; c < n; ++c)
    for (idx r = 0; r < n; ++r) out(r, c) = 0.5 * (k(r, c) + k(c, r));
  return out;
}

// F = h_core + J + K   (tei.cpp:236-238)
Mat fock_from_factors(const Mat& h_core, const Mat& chol, const Mat& d) {
  const Mat j = coulomb_from_factors(chol, d), k = exchange_from_factors(chol, d);
  Mat f(h_core.rows, h_core.cols);
  for (size_t r = 0; r < f.d.size(); ++r) f.d[r] = (h_core.d[r] + j.d[r]) + k.d[r];
  return f;
}

// ---------------------------------------------------------------- lattice.cpp

Mat assemble_axis(const Grid& g, const Mat& ref, int ax, const std::vector<double>& centers, idx* ops) {  // lattice.cpp:50-61
  const idx n = g.n[ax];
  Mat out(n, ref.cols);
  for (double c : centers) {
    const idx ofs = window_offset(g, ax, c);
    for (idx q = 0; q < ref.cols; ++q)
      for (idx i = 0; i < n; ++i) out(i, q) += ref(ofs + i, q);
    if (ops) *ops += 1;
  }
  return out;
}

// ---------------------------------------------------------------- tei.cpp

PivChol pivoted_cholesky(const std::function<Vec(idx)>& column, Vec diag, double tol, bool trace_stop,
                         idx max_rank, double neg_tol) {  // tei.cpp:48-90
  const idx n = static_cast<idx>(diag.size());
  PivChol res;
  double max0 = -INFINITY, trace0 = 0.0;
  for (double x : diag) {
    max0 = std::max(max0, x);
    trace0 += x;
  }
  if (n == 0 || max0 <= 0.0) {
    res.L = Mat(n, 0);
    return res;
  }
  const idx cap = std::min(n, max_rank);
  Mat l(n, cap);
  idx rank = 0;
  auto dsum = [&] {
    double s = 0;
    for (double x : diag) s += x;
    return s;
  };
  const double target = tol * (trace_stop ? trace0 : max0);
  while (rank < cap) {
    idx p = 0;
    double dmax = diag[0];
    for (idx i = 1; i < n; ++i)
      if (diag[i] > dmax) {  // first maximal index, as Eigen's maxCoeff(&p)
        dmax = diag[i];
        p = i;
      }
    if ((trace_stop ? dsum() : dmax) <= target) break;
    if (dmax <= 0.0) break;
    Vec col = column(p);
    for (idx q = 0; q < rank; ++q) {
      const double lpq = l(p, q);
      const double* lq = l.col(q);
      for (idx i = 0; i < n; ++i) col[i] -= lq[i] * lpq;
    }
    const double piv = std::sqrt(dmax);
    double* lr = l.col(rank);
    for (idx i = 0; i < n; ++i) lr[i] = col[i] / piv;
    lr[p] = piv;
    for (idx i = 0; i < n; ++i) diag[i] -= lr[i] * lr[i];
    diag[p] = 0.0;
    for (idx i = 0; i < n; ++i)
      if (diag[i] < 0.0) {
        if (diag[i] < -neg_tol * max0) throw numerical_error("pivoted_cholesky: negative diagonal beyond tolerance; matrix not PSD");
        diag[i] = 0.0;
        res.clamped = true;
      }
    res.piv.push_back(p);
    ++rank;
  }
  res.L = left_cols(l, rank);
  double meas = 0;
  if (trace_stop) {
    meas = dsum();
  } else {
    meas = -INFINITY;
    for (double x : diag) meas = std::max(meas, x);
  }
  res.residual = meas / (trace_stop ? trace0 : max0);
  return res;
}

void tei_density_fitting(TEI& f, const Grid& g, const std::vector<CP3>& disc, double eps_fit) {  // tei.cpp:92-143
  req(!disc.empty(), "tei_density_fitting: empty basis");
  f.nb = static_cast<idx>(disc.size());
  for (int ax = 0; ax < 3; ++ax) f.h[ax] = g.h[ax];
  f.owner.clear();
  f.pw.clear();
  for (idx fn = 0; fn < f.nb; ++fn)
    for (idx p = 0; p < disc[fn].rank(); ++p) {
      f.owner.push_back(fn);
      f.pw.push_back(disc[fn].w[p]);
    }
  f.np = static_cast<idx>(f.owner.size());
  const idx np = f.np;
  for (int ax = 0; ax < 3; ++ax) {
    const idx n = g.n[ax];
    Mat prim(n, np);
    idx col = 0;
    for (idx fn = 0; fn < f.nb; ++fn)
      for (idx p = 0; p < disc[fn].rank(); ++p, ++col)
        std::memcpy(prim.col(col), disc[fn].f[ax].col(p), sizeof(double) * n);
    Mat G(n, np * np);
    for (idx q = 0; q < np; ++q)
      for (idx p = 0; p < np; ++p)
        for (idx i = 0; i < n; ++i) G(i, p + np * q) = prim(i, p) * prim(i, q);
    Mat gram = matmul(G, false, G, true);
    Vec dg(n);
    for (idx i = 0; i < n; ++i) dg[i] = gram(i, i);
    PivChol pc;
    try {
      pc = pivoted_cholesky([&](idx j) { return Vec(gram.col(j), gram.col(j) + n); }, dg, eps_fit * eps_fit, true,
                            std::min(n, np * np), 1e-12);
    } catch (const numerical_error&) {
      throw numerical_error("tei_density_fitting: Gram matrix indefinite beyond tolerance");
    }
    f.fit_clamped = f.fit_clamped || pc.clamped;
    Mat q, r;
    householder_qr_thin(pc.L, q, r);
    f.U[ax] = q;
    f.V[ax] = matmul(G, true, q, false);
    Mat uvt = matmul(f.U[ax], false, f.V[ax], true);
    double num = 0, den = 0;
    for (size_t i = 0; i < G.d.size(); ++i) {
      num += (G.d[i] - uvt.d[i]) * (G.d[i] - uvt.d[i]);
      den += G.d[i] * G.d[i];
    }
    f.fit_res[ax] = std::sqrt(num) / std::max(std::sqrt(den), 1e-300);
  }
}

void tei_convolution_matrices(TEI& f, const CP3& kernel) {  // tei.cpp:145-158
  const idx rk = kernel.rank();
  f.M.assign(rk, {});
  for (int ax = 0; ax < 3; ++ax) {
    req(kernel.extent(ax) == f.U[ax].rows, "tei_convolution_matrices: kernel grid mismatch");
    for (idx k = 0; k < rk; ++k) {
      Mat cols = conv_central_many(f.U[ax], kernel.f[ax].col(k), f.U[ax].rows);
      for (double& x : cols.d) x = f.h[ax] * x;
      f.M[k][ax] = matmul(f.U[ax], true, cols, false);
    }
  }
}

static Vec b_prim_column(const TEI& f, idx j) {  // tei.cpp:33-44
  const idx np2 = f.np * f.np;
  Vec out(np2, 0.0);
  std::array<Vec, 3> w;
  for (const auto& mk : f.M) {
    for (int ax = 0; ax < 3; ++ax) {
      const Mat& V = f.V[ax];
      const idx r = V.cols;
      Vec y(r, 0.0);  // M_k * V[j,:]^T
      for (idx c = 0; c < r; ++c) {
        const double vjc = V(j, c);
        for (idx i = 0; i < r; ++i) y[i] += mk[ax](i, c) * vjc;
      }
      w[ax].assign(np2, 0.0);
      for (idx c = 0; c < r; ++c)
        for (idx i = 0; i < np2; ++i) w[ax][i] += V(i, c) * y[c];
    }
    for (idx i = 0; i < np2; ++i) out[i] += w[0][i] * w[1][i] * w[2][i];
  }
  return out;
}

static std::vector<std::pair<idx, double>> contraction_column(const TEI& f, idx mu, idx nu) {  // tei.cpp:19-29
  std::vector<std::pair<idx, double>> out;
  for (idx p = 0; p < f.np; ++p) {
    if (f.owner[p] != mu) continue;
    for (idx q = 0; q < f.np; ++q) {
      if (f.owner[q] != nu) continue;
      out.push_back({p + f.np * q, f.pw[p] * f.pw[q]});
    }
  }
  return out;
}

Vec tei_column(const TEI& f, idx pair) {  // tei.cpp:160-174
  req(pair >= 0 && pair < f.nb * f.nb, "tei_column: index out of range");
  const idx kappa = pair % f.nb, lambda = pair / f.nb;
  const idx np2 = f.np * f.np;
  Vec z(np2, 0.0);
  for (const auto& [j, w] : contraction_column(f, kappa, lambda)) {
    Vec c = b_prim_column(f, j);
    for (idx i = 0; i < np2; ++i) z[i] += w * c[i];
  }
  Vec out(f.nb * f.nb, 0.0);
  for (idx q = 0; q < f.np; ++q)
    for (idx p = 0; p < f.np; ++p) out[f.owner[p] + f.nb * f.owner[q]] += f.pw[p] * f.pw[q] * z[p + f.np * q];
  return out;
}

Vec tei_diagonal(const TEI& f) {  // tei.cpp:182-196
  Vec d(f.nb * f.nb);
  for (idx nu = 0; nu < f.nb; ++nu)
    for (idx mu = 0; mu < f.nb; ++mu) {
      const auto pairs = contraction_column(f, mu, nu);
      double val = 0.0;
      for (const auto& [j, w] : pairs) {
        Vec col = b_prim_column(f, j);
        for (const auto& [j2, w2] : pairs) val += w * w2 * col[j2];
      }
      d[mu + f.nb * nu] = val;
    }
  return d;
}

void tei_cholesky(TEI& f, double eps_chol) {  // tei.cpp:198-204
  PivChol pc = pivoted_cholesky([&](idx j) { return tei_column(f, j); }, tei_diagonal(f), eps_chol, false,
                                f.nb * f.nb, 1e-10);
  f.L = pc.L;
  f.chol_piv = pc.piv;
}

}  // namespace orc

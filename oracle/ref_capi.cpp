// ORACLE — TEST INFRASTRUCTURE ONLY.
// extern "C" surface over the REFERENCE's own conv-path code (compiled in
// place from /root/reference/proj/src against oracle/eigen_shim) so tests can
// pin the restatement and generate golden fixtures, and bench.py can time the
// reference's CPU path (`--impl reference`).
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tengrid/basis.hpp"
#include "tengrid/fft.hpp"
#include "tengrid/grid.hpp"
#include "tengrid/kernel.hpp"
#include "tengrid/lattice.hpp"
#include "tengrid/tensor.hpp"

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const tg::SnapError& e) {
    g_err = e.what();
    return 3;
  } catch (const tg::NumericalError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}
Eigen::MatrixXd mat(const double* p, long long r, long long c) {
  Eigen::MatrixXd m(r, c);
  if (r * c) std::memcpy(m.data(), p, sizeof(double) * r * c);
  return m;
}
tg::Grid3 grid(const double* b, const long long* n) { return tg::make_grid({b[0], b[1], b[2]}, {n[0], n[1], n[2]}); }
}  // namespace

extern "C" {
const char* ref_last_error() { return g_err.c_str(); }
void* ref_cp_new() { return new tg::CanonicalTensor3(); }
void ref_cp_free(void* h) { delete static_cast<tg::CanonicalTensor3*>(h); }
long long ref_cp_rank(void* h) { return static_cast<tg::CanonicalTensor3*>(h)->rank(); }
long long ref_cp_extent(void* h, int ax) { return static_cast<tg::CanonicalTensor3*>(h)->extent(ax); }
void ref_cp_get(void* h, int ax, double* out) {
  auto& m = static_cast<tg::CanonicalTensor3*>(h)->factor[ax];
  if (m.size()) std::memcpy(out, m.data(), sizeof(double) * m.size());
}
void ref_cp_get_w(void* h, double* out) {
  auto& w = static_cast<tg::CanonicalTensor3*>(h)->weight;
  if (w.size()) std::memcpy(out, w.data(), sizeof(double) * w.size());
}
int ref_cp_set(void* h, const long long* n, long long r, const double* f0, const double* f1, const double* f2,
               const double* w) {
  return guard([&] {
    auto& t = *static_cast<tg::CanonicalTensor3*>(h);
    const double* fs[3] = {f0, f1, f2};
    for (int ax = 0; ax < 3; ++ax) t.factor[ax] = mat(fs[ax], n[ax], r);
    t.weight = Eigen::VectorXd(static_cast<Eigen::Index>(r));
    if (r) std::memcpy(t.weight.data(), w, sizeof(double) * r);
  });
}
int ref_conv_full(long long n, const double* u, const double* v, int use_fft, double* out) {
  return guard([&] {
    Eigen::VectorXd uu(static_cast<Eigen::Index>(n)), vv(static_cast<Eigen::Index>(n));
    std::memcpy(uu.data(), u, sizeof(double) * n);
    std::memcpy(vv.data(), v, sizeof(double) * n);
    Eigen::VectorXd r = use_fft ? tg::conv_full_fft(uu, vv) : tg::conv_full_direct(uu, vv);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}
// threads > 1 splits the column range across std::threads (the functions are
// pure) — used only by the CPU-baseline timing.
int ref_conv_central_many(long long n, long long c, const double* U, const double* v, double* out, int threads) {
  return guard([&] {
    Eigen::VectorXd vv(static_cast<Eigen::Index>(n));
    std::memcpy(vv.data(), v, sizeof(double) * n);
    if (threads <= 1 || c < 2) {
      Eigen::MatrixXd r = tg::conv_central_many(mat(U, n, c), vv);
      if (r.size()) std::memcpy(out, r.data(), sizeof(double) * r.size());
      return;
    }
    std::vector<std::thread> ts;
    const long long chunk = (c + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
      const long long lo = t * chunk, hi = std::min(c, lo + chunk);
      if (lo >= hi) break;
      ts.emplace_back([&, lo, hi] {
        Eigen::MatrixXd r = tg::conv_central_many(mat(U + lo * n, n, hi - lo), vv);
        std::memcpy(out + lo * n, r.data(), sizeof(double) * r.size());
      });
    }
    for (auto& t : ts) t.join();
  });
}
int ref_convolve(void* a, void* b, const double* h, void* out) {
  return guard([&] {
    *static_cast<tg::CanonicalTensor3*>(out) = tg::convolve(*static_cast<tg::CanonicalTensor3*>(a),
                                                            *static_cast<tg::CanonicalTensor3*>(b), {h[0], h[1], h[2]});
  });
}
int ref_hadamard(void* a, void* b, void* out) {
  return guard([&] {
    *static_cast<tg::CanonicalTensor3*>(out) =
        tg::hadamard(*static_cast<tg::CanonicalTensor3*>(a), *static_cast<tg::CanonicalTensor3*>(b));
  });
}
int ref_scalar_product(void* a, void* b, double* out) {
  return guard([&] {
    *out = tg::scalar_product(*static_cast<tg::CanonicalTensor3*>(a), *static_cast<tg::CanonicalTensor3*>(b));
  });
}
int ref_value_at(void* t, long long npts, const long long* ijk, double* out) {
  return guard([&] {
    auto& c = *static_cast<tg::CanonicalTensor3*>(t);
    for (long long p = 0; p < npts; ++p) out[p] = c.value_at(ijk[3 * p], ijk[3 * p + 1], ijk[3 * p + 2]);
  });
}
int ref_make_expsum(long long m, double c0, double lo, double hi, double* nodes, double* weights, double* scale,
                    double* mesh) {
  return guard([&] {
    tg::ExpSum es = tg::make_expsum(m, c0, lo, hi);
    std::memcpy(nodes, es.nodes.data(), sizeof(double) * es.nodes.size());
    std::memcpy(weights, es.weights.data(), sizeof(double) * es.weights.size());
    *scale = es.scale;
    *mesh = es.mesh;
  });
}
double ref_gauss_cell_integral(double t, double c, double h) { return tg::gauss_cell_integral(t, c, h); }
int ref_kernel_tensor(const double* b, const long long* n, long long m, double c0, int doubled, void* out) {
  return guard([&] {
    tg::ExpSum es = tg::make_expsum(m, c0);
    *static_cast<tg::CanonicalTensor3*>(out) = tg::kernel_tensor(grid(b, n), es, doubled != 0).tensor;
  });
}
int ref_window_offset(const double* b, const long long* n, int ax, double center, long long* ofs) {
  return guard([&] { *ofs = tg::window_offset(grid(b, n), ax, center); });
}
int ref_discretize_basis(const double* b, const long long* n, int nfn, const double* centers, const int* degs,
                         const int* nprim, const double* exps, const double* coefs, void** out_handles) {
  return guard([&] {
    tg::BasisSet bs;
    bs.grid = grid(b, n);
    int off = 0;
    for (int i = 0; i < nfn; ++i) {
      tg::SeparableBasisFunction f;
      for (int ax = 0; ax < 3; ++ax) {
        f.center[ax] = centers[3 * i + ax];
        f.degree[ax] = degs[3 * i + ax];
      }
      for (int p = 0; p < nprim[i]; ++p) f.primitives.push_back({exps[off + p], coefs[off + p]});
      off += nprim[i];
      bs.functions.push_back(f);
    }
    auto disc = tg::discretize_basis(bs);
    for (int i = 0; i < nfn; ++i) out_handles[i] = new tg::CanonicalTensor3(std::move(disc[i]));
  });
}
// lattice_sum_canonical with a doubled Newton reference built from (m, c0)
int ref_lattice_sum_canonical(const long long* counts, double spacing, double charge, const double* b,
                              const long long* n, long long m, double c0, void* out, long long* window_ops) {
  return guard([&] {
    tg::LatticeSpec spec;
    spec.counts = {counts[0], counts[1], counts[2]};
    spec.spacing = spacing;
    spec.charge = charge;
    const tg::Grid3 g = grid(b, n);
    const tg::KernelTensor ref = tg::kernel_tensor(g, tg::make_expsum(m, c0), true);
    tg::AssembledPotential ap = tg::lattice_sum_canonical(spec, g, ref);
    *static_cast<tg::CanonicalTensor3*>(out) = *ap.canonical;
    *window_ops = ap.window_ops;
  });
}
}  // extern "C"

// ORACLE — TEST INFRASTRUCTURE ONLY.
// extern "C" surface over the REFERENCE's own conv-path code (compiled in
// place from /root/reference/proj/src against oracle/eigen_shim) so tests can
// pin the restatement and generate golden fixtures, and bench.py can time the
// reference's CPU path (`--impl reference`).
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tengrid/basis.hpp"
#include "tengrid/fft.hpp"
#include "tengrid/hf.hpp"
#include "tengrid/mp2.hpp"
#include "tengrid/reduction.hpp"
#include "tengrid/tei.hpp"
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
// basis given as in ref_discretize_basis
struct BasisArgs {
  const double* b;
  const long long* n;
  int nfn;
  const double* centers;
  const int* degs;
  const int* nprim;
  const double* exps;
  const double* coefs;
};
tg::BasisSet basis_set(const BasisArgs& a) {
  tg::BasisSet bs;
  bs.grid = grid(a.b, a.n);
  int off = 0;
  for (int i = 0; i < a.nfn; ++i) {
    tg::SeparableBasisFunction f;
    for (int ax = 0; ax < 3; ++ax) {
      f.center[ax] = a.centers[3 * i + ax];
      f.degree[ax] = a.degs[3 * i + ax];
    }
    for (int p = 0; p < a.nprim[i]; ++p) f.primitives.push_back({a.exps[off + p], a.coefs[off + p]});
    off += a.nprim[i];
    bs.functions.push_back(f);
  }
  return bs;
}
void put(const Eigen::MatrixXd& m, double* out) {
  if (m.size()) std::memcpy(out, m.data(), sizeof(double) * m.size());
}
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
// CPU baseline shaped like tg::convolve's own loop (tensor.cpp:189-195): for
// each kernel column js[k], conv_central_many over ALL ra density columns
// (one kernel FFT per call, reused across the columns), times h.  `threads`
// std::threads split the k loop (the function is pure); each
// thread owns its result matrix.  checksum = sum over k of out(0, 0) (keeps
// the work observable).
int ref_convolve_axis_sample(long long n, long long ra, const double* U, const double* K, const long long* js,
                             long long njs, double h, int threads, double* checksum) {
  return guard([&] {
    const Eigen::MatrixXd Um = mat(U, n, ra);
    std::vector<double> first(static_cast<size_t>(njs), 0.0);
    auto work = [&](long long k0, long long k1) {
      for (long long k = k0; k < k1; ++k) {
        Eigen::VectorXd v(static_cast<Eigen::Index>(n));
        std::memcpy(v.data(), K + js[k] * n, sizeof(double) * n);
        Eigen::MatrixXd cols = h * tg::conv_central_many(Um, v);
        first[static_cast<size_t>(k)] = cols.size() ? cols(0, 0) : 0.0;
      }
    };
    if (threads <= 1 || njs < 2) {
      work(0, njs);
    } else {
      std::vector<std::thread> ts;
      for (int t = 0; t < threads; ++t) {
        const long long lo = njs * t / threads, hi = njs * (t + 1) / threads;
        if (lo < hi) ts.emplace_back(work, lo, hi);
      }
      for (auto& t : ts) t.join();
    }
    double s = 0.0;
    for (double x : first) s += x;
    *checksum = s;
  });
}

// Fixture generator (tools/make_golden_cfg2.py): V_H = hartree_potential(theta,
// kernel, h) (hf.cpp:131-138 -> convolve, tensor.cpp:179-198) evaluated at
// npts grid points (value_at, tensor.hpp:135-140) WITHOUT materialising the
// ra*rb-column factors: for each kernel column j, the three axes'
// conv_central_many(theta.factor[ax], kernel.factor[ax].col(j)) (the
// reference's own code), h-scaled as in convolve, then
// sum_i w_i w_j prod_ax F_ax(idx_ax, i) per point; per-j partials summed in j
// order, terms within a j in i order.
int ref_hartree_samples(void* theta_h, void* kernel_h, const double* h, long long npts, const long long* ijk,
                        int threads, double* out) {
  return guard([&] {
    const auto& th = *static_cast<tg::CanonicalTensor3*>(theta_h);
    const auto& kt = *static_cast<tg::CanonicalTensor3*>(kernel_h);
    const double inv_vol = 1.0 / (h[0] * h[1] * h[2]);
    const tg::CanonicalTensor3 ks = tg::scale(kt, inv_vol);
    const long long ra = th.rank(), rb = ks.rank();
    std::vector<std::vector<double>> part(static_cast<size_t>(rb), std::vector<double>(static_cast<size_t>(npts), 0.0));
    auto work = [&](long long j0, long long j1) {
      for (long long j = j0; j < j1; ++j) {
        Eigen::MatrixXd F[3];
        for (int ax = 0; ax < 3; ++ax) F[ax] = h[ax] * tg::conv_central_many(th.factor[ax], ks.factor[ax].col(j));
        auto& pj = part[static_cast<size_t>(j)];
        for (long long p = 0; p < npts; ++p) {
          double s = 0.0;
          for (long long i = 0; i < ra; ++i)
            s += (th.weight[i] * ks.weight[j]) * F[0](ijk[3 * p], i) * F[1](ijk[3 * p + 1], i) * F[2](ijk[3 * p + 2], i);
          pj[static_cast<size_t>(p)] = s;
        }
      }
    };
    std::vector<std::thread> ts;
    const int nt = std::max(1, threads);
    for (int t = 0; t < nt; ++t) {
      const long long lo = rb * t / nt, hi = rb * (t + 1) / nt;
      if (lo < hi) ts.emplace_back(work, lo, hi);
    }
    for (auto& t : ts) t.join();
    for (long long p = 0; p < npts; ++p) {
      double s = 0.0;
      for (long long j = 0; j < rb; ++j) s += part[static_cast<size_t>(j)][static_cast<size_t>(p)];
      out[p] = s;
    }
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

// ---- hf.cpp / tei.cpp / reduction.cpp (compiled against the shim's stand-in LA)
#define TG_BASIS_ARGS const double *b, const long long *n, int nfn, const double *centers, const int *degs, \
                      const int *nprim, const double *exps, const double *coefs
#define TG_BASIS BasisArgs{b, n, nfn, centers, degs, nprim, exps, coefs}

// which: 0 overlap_matrix, 1 kinetic_matrix (lumped), 2 kinetic_matrix (exact mass)   hf.cpp:48-87
int ref_one_electron(TG_BASIS_ARGS, int which, double* out) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    const auto disc = tg::discretize_basis(bs);
    put(which == 0 ? tg::overlap_matrix(bs, disc) : tg::kinetic_matrix(bs, disc, which == 2), out);
  });
}
// nuclear_potential_tensor + nuclear_matrix with the doubled Newton reference (m, c0)   hf.cpp:89-116
int ref_nuclear(TG_BASIS_ARGS, int nnuc, const double* charges, const double* ncenters, long long m, double c0,
                double* V, void* pc_out) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    const auto disc = tg::discretize_basis(bs);
    tg::Molecule mol;
    for (int a = 0; a < nnuc; ++a) mol.nuclei.push_back({charges[a], {ncenters[3 * a], ncenters[3 * a + 1], ncenters[3 * a + 2]}});
    const tg::KernelTensor ref = tg::kernel_tensor(bs.grid, tg::make_expsum(m, c0), true);
    if (pc_out) *static_cast<tg::CanonicalTensor3*>(pc_out) = tg::nuclear_potential_tensor(bs, mol, ref);
    if (V) put(tg::nuclear_matrix(bs, disc, mol, ref), V);
  });
}
int ref_coulomb_matrix(TG_BASIS_ARGS, void* vh, double* J) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    put(tg::coulomb_matrix(bs, tg::discretize_basis(bs), *static_cast<tg::CanonicalTensor3*>(vh)), J);
  });
}
int ref_exchange_matrix(TG_BASIS_ARGS, long long nocc, const double* c_occ, long long m, double c0, double* K) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    const tg::KernelTensor kern = tg::kernel_tensor(bs.grid, tg::make_expsum(m, c0), false);
    put(tg::exchange_matrix(bs, tg::discretize_basis(bs), mat(c_occ, nfn, nocc), kern), K);
  });
}
int ref_density_tensor(TG_BASIS_ARGS, long long nocc, const double* c_occ, double eps, void* out) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    *static_cast<tg::CanonicalTensor3*>(out) = tg::density_tensor(tg::discretize_basis(bs), mat(c_occ, nfn, nocc), eps);
  });
}
// which: 0 coulomb_from_factors, 1 exchange_from_factors, 2 fock_from_factors   tei.cpp:215-238
int ref_from_factors(int which, long long nb, long long rank, const double* h_core, const double* chol,
                     const double* density, double* out) {
  return guard([&] {
    const Eigen::MatrixXd l = mat(chol, nb * nb, rank), d = mat(density, nb, nb);
    if (which == 0) put(tg::coulomb_from_factors(l, d), out);
    if (which == 1) put(tg::exchange_from_factors(l, d), out);
    if (which == 2) put(tg::fock_from_factors(mat(h_core, nb, nb), l, d), out);
  });
}
int ref_generalized_eigensolve(long long nb, const double* f, const double* s, double* c, double* e) {
  return guard([&] {
    Eigen::MatrixXd cc;
    Eigen::VectorXd ee;
    tg::generalized_eigensolve(mat(f, nb, nb), mat(s, nb, nb), cc, ee);
    put(cc, c);
    put(ee, e);
  });
}
// build_tei with a primary Newton kernel (m, c0); info = {R_l[3], R_B, clamped}; chol / pivots optional
int ref_build_tei(TG_BASIS_ARGS, long long m, double c0, double eps_fit, double eps_chol, long long* info,
                  double* fit_residual, void** handle) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    const tg::KernelTensor kern = tg::kernel_tensor(bs.grid, tg::make_expsum(m, c0), false);
    auto* fac = new tg::TEIFactorization(tg::build_tei(bs, tg::discretize_basis(bs), kern, eps_fit, eps_chol));
    for (int ax = 0; ax < 3; ++ax) {
      info[ax] = fac->fit_ranks()[ax];
      fit_residual[ax] = fac->fit_residual[ax];
    }
    info[3] = fac->rank_b();
    info[4] = fac->fit_clamped_negative ? 1 : 0;
    *handle = fac;
  });
}
void ref_tei_free(void* h) { delete static_cast<tg::TEIFactorization*>(h); }
// what: 0 chol (nb^2 x R_B), 1 tei_diagonal (nb^2), 2 tei_column(j) (nb^2)
int ref_tei_get(void* h, int what, long long j, double* out) {
  return guard([&] {
    auto& f = *static_cast<tg::TEIFactorization*>(h);
    if (what == 0) put(f.chol, out);
    if (what == 1) put(tg::tei_diagonal(f), out);
    if (what == 2) put(tg::tei_column(f, j), out);
  });
}
// mode 0 rhosvd, 1 canonical_to_tucker, 2 reduce_rank (C2T + T2C); ranks used when use_eps == 0.
// info = {r0, r1, r2, rank_clamped, rhosvd_fallback, sweeps, canonical rank}
int ref_reduce(void* a, int use_eps, double eps, const long long* ranks, int sweeps, int mode, long long* info,
               void* out_cp) {
  return guard([&] {
    const auto& t = *static_cast<tg::CanonicalTensor3*>(a);
    const tg::ReductionConfig cfg = use_eps ? tg::ReductionConfig::tolerance(eps, sweeps)
                                            : tg::ReductionConfig::fixed(ranks[0], ranks[1], ranks[2], sweeps);
    if (mode == 2) {
      tg::CanonicalTensor3 c = tg::reduce_rank(t, cfg);
      info[6] = c.rank();
      if (out_cp) *static_cast<tg::CanonicalTensor3*>(out_cp) = std::move(c);
      return;
    }
    tg::TuckerResult r = mode == 0 ? tg::rhosvd(t, cfg) : tg::canonical_to_tucker(t, cfg);
    const auto rk = r.tucker.ranks();
    for (int ax = 0; ax < 3; ++ax) info[ax] = rk[ax];
    info[3] = r.rank_clamped;
    info[4] = r.rhosvd_fallback;
    info[5] = static_cast<long long>(r.sweep_fits.size());
    if (out_cp) {
      tg::CanonicalTensor3 c = tg::tucker_to_canonical(r.tucker);
      info[6] = c.rank();
      *static_cast<tg::CanonicalTensor3*>(out_cp) = std::move(c);
    }
  });
}

// TuckerResult::mode_singular_values[axis] of rhosvd (mode 0) / canonical_to_tucker (mode 1)
// (reduction.cpp:172-190); *count values into sigma (capacity cap).
int ref_mode_sigma(void* a, int use_eps, double eps, const long long* ranks, int mode, int axis, long long cap,
                   long long* count, double* sigma) {
  return guard([&] {
    const auto& t = *static_cast<tg::CanonicalTensor3*>(a);
    const tg::ReductionConfig cfg = use_eps ? tg::ReductionConfig::tolerance(eps)
                                            : tg::ReductionConfig::fixed(ranks[0], ranks[1], ranks[2]);
    const tg::TuckerResult r = mode == 0 ? tg::rhosvd(t, cfg) : tg::canonical_to_tucker(t, cfg);
    const auto& sv = r.mode_singular_values[axis];
    *count = static_cast<long long>(sv.size());
    for (size_t i = 0; i < sv.size() && static_cast<long long>(i) < cap; ++i) sigma[i] = sv[i];
  });
}

// kernel.cpp:131-165
int ref_expsum_for_interval(double r_min, double r_max, double eps, long long* m, double* c0) {
  return guard([&] {
    const tg::ExpSum es = tg::expsum_for_interval(r_min, r_max, eps);
    *m = es.m;
    *c0 = es.c0;
  });
}
// hf.cpp:201-270.  cfg = {max_iterations, energy_tol, mixing, eps_fit, eps_chol, kernel_eps, kernel_r_max};
// out = {energy, nuclear_energy, converged, iterations, n_occupied, tei_rank_b}; e (nb), density (nb x nb),
// energy_history (max_iterations)
int ref_scf_solve(TG_BASIS_ARGS, int nnuc, const double* charges, const double* ncenters, int n_electrons,
                  const double* cfg, double* out, double* e, double* density, double* energy_history) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    tg::Molecule mol;
    for (int a = 0; a < nnuc; ++a) mol.nuclei.push_back({charges[a], {ncenters[3 * a], ncenters[3 * a + 1], ncenters[3 * a + 2]}});
    mol.n_electrons = n_electrons;
    tg::SCFConfig c;
    c.max_iterations = static_cast<int>(cfg[0]);
    c.energy_tol = cfg[1];
    c.mixing = cfg[2];
    c.eps_fit = cfg[3];
    c.eps_chol = cfg[4];
    c.kernel_eps = cfg[5];
    c.kernel_r_max = cfg[6];
    const tg::SCFState st = tg::scf_solve(mol, bs, c);
    out[0] = st.energy;
    out[1] = st.nuclear_energy;
    out[2] = st.converged;
    out[3] = st.iterations;
    out[4] = st.n_occupied;
    out[5] = st.tei ? static_cast<double>(st.tei->rank_b()) : 0.0;
    put(st.orbital_energies, e);
    put(st.density, density);
    for (size_t i = 0; i < st.energy_history.size(); ++i) energy_history[i] = st.energy_history[i];
  });
}

// scf_solve then the MP2 chain of mp2.cpp on its MO space.  Returns the
// inputs the device path needs (chol, coefficients, energies) and the
// reference's outputs: the MO factor and both MP2 energies.
// sizes = {nb, R_B, n_occ}; call first with chol == nullptr to get sizes.
int ref_mp2_case(TG_BASIS_ARGS, int nnuc, const double* charges, const double* ncenters, int n_electrons,
                 const double* cfg, double expsum_eps, long long* sizes, double* chol, double* coef, double* energies,
                 double* mo_factor, double* e2) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    tg::Molecule mol;
    for (int a = 0; a < nnuc; ++a) mol.nuclei.push_back({charges[a], {ncenters[3 * a], ncenters[3 * a + 1], ncenters[3 * a + 2]}});
    mol.n_electrons = n_electrons;
    tg::SCFConfig c;
    c.max_iterations = static_cast<int>(cfg[0]);
    c.energy_tol = cfg[1];
    c.mixing = cfg[2];
    c.eps_fit = cfg[3];
    c.eps_chol = cfg[4];
    c.kernel_eps = cfg[5];
    const tg::SCFState st = tg::scf_solve(mol, bs, c);
    sizes[0] = bs.size();
    sizes[1] = st.tei->chol.cols();
    sizes[2] = st.n_occupied;
    if (!chol) return;
    put(st.tei->chol, chol);
    put(st.coefficients, coef);
    put(st.orbital_energies, energies);
    tg::MOSpace mos;
    mos.coefficients = st.coefficients;
    mos.energies = st.orbital_energies;
    mos.n_occ = st.n_occupied;
    const tg::MOCholesky mo = tg::mo_transform_cholesky(st.tei->chol, mos);
    put(mo.factor, mo_factor);
    e2[0] = tg::mp2_energy(mo, mos, tg::MP2Mode::oracle);
    e2[1] = tg::mp2_energy(mo, mos, tg::MP2Mode::factorized, expsum_eps);
  });
}
int ref_reciprocal_expsum(double lo, double hi, double eps, long long* terms, double* rates, double* weights,
                          double* achieved, int* ok) {
  return guard([&] {
    const tg::ReciprocalExpSum rs = tg::reciprocal_expsum(lo, hi, eps);
    *terms = rs.terms();
    put(rs.rates, rates);
    put(rs.weights, weights);
    *achieved = rs.achieved_error;
    *ok = rs.ok;
  });
}
// ---- full-size config fixtures (tools/make_golden_configs.py) -------------------
// density_tensor (hf.cpp:118-129) with reduce_rank split into its two steps
// (reduction.cpp:271-273) so the Tucker ranks can be reported.
// info = {r0, r1, r2, reduced canonical rank, unreduced rank}
int ref_density_tucker(TG_BASIS_ARGS, long long nocc, const double* c_occ, double eps, long long* info, void* out) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    const auto disc = tg::discretize_basis(bs);
    const tg::CanonicalTensor3 theta = tg::density_tensor(disc, mat(c_occ, nfn, nocc), 0.0);  // unreduced
    const tg::TuckerResult tr = tg::canonical_to_tucker(theta, tg::ReductionConfig::tolerance(eps));
    const auto rk = tr.tucker.ranks();
    for (int ax = 0; ax < 3; ++ax) info[ax] = rk[ax];
    tg::CanonicalTensor3 red = tg::tucker_to_canonical(tr.tucker);
    info[3] = red.rank();
    info[4] = theta.rank();
    *static_cast<tg::CanonicalTensor3*>(out) = std::move(red);
  });
}
// coulomb_matrix(bs, disc, hartree_potential(theta, kernel, h)) (hf.cpp:131-151) with
// V_H split by kernel column j (J is linear in V_H's columns): threads take blocks of
// j, each materialises only its V_H^(j); the partial J^(j) are summed in j order.
int ref_coulomb_from_theta(TG_BASIS_ARGS, void* theta_h, long long m, double c0, int threads, double* J) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    const auto disc = tg::discretize_basis(bs);
    const auto& th = *static_cast<tg::CanonicalTensor3*>(theta_h);
    const tg::KernelTensor kern = tg::kernel_tensor(bs.grid, tg::make_expsum(m, c0), false);
    const long long rb = kern.rank();
    std::vector<Eigen::MatrixXd> part(static_cast<size_t>(rb));
    auto work = [&](long long j0, long long j1) {
      for (long long j = j0; j < j1; ++j) {
        tg::KernelTensor kj = kern;
        for (int ax = 0; ax < 3; ++ax) kj.tensor.factor[ax] = Eigen::MatrixXd(kern.tensor.factor[ax].col(j));
        kj.tensor.weight = Eigen::VectorXd::Constant(1, kern.tensor.weight[j]);
        const tg::CanonicalTensor3 vh = tg::hartree_potential(th, kj, bs.grid.h);
        part[static_cast<size_t>(j)] = tg::coulomb_matrix(bs, disc, vh);
      }
    };
    std::vector<std::thread> ts;
    const int nt = std::max(1, threads);
    for (int t = 0; t < nt; ++t) {
      const long long lo = rb * t / nt, hi = rb * (t + 1) / nt;
      if (lo < hi) ts.emplace_back(work, lo, hi);
    }
    for (auto& t : ts) t.join();
    Eigen::MatrixXd acc = part[0];
    for (long long j = 1; j < rb; ++j) acc = acc + part[static_cast<size_t>(j)];
    put(acc, J);
  });
}
// build_tei (tei.cpp:206-213) with the pivot sequence of its Cholesky kept:
// tei_density_fitting + tei_convolution_matrices, then pivoted_cholesky with
// tei_cholesky's arguments (tei.cpp:198-204).  info = {R_l[3], R_B, clamped}
int ref_build_tei_pivots(TG_BASIS_ARGS, long long m, double c0, double eps_fit, double eps_chol, long long* info,
                         double* fit_residual, long long* pivots, void** handle) {
  return guard([&] {
    const tg::BasisSet bs = basis_set(TG_BASIS);
    const tg::KernelTensor kern = tg::kernel_tensor(bs.grid, tg::make_expsum(m, c0), false);
    auto* fac = new tg::TEIFactorization();
    tg::tei_density_fitting(*fac, bs, tg::discretize_basis(bs), eps_fit);
    tg::tei_convolution_matrices(*fac, kern);
    fac->eps_chol = eps_chol;
    const tg::PivotedCholesky pc = tg::pivoted_cholesky([&](tg::index_t j) { return tg::tei_column(*fac, j); },
                                                        tg::tei_diagonal(*fac), eps_chol, tg::CholeskyStop::max_diagonal,
                                                        fac->n_b * fac->n_b, 1e-10);
    fac->chol = pc.factor;
    for (int ax = 0; ax < 3; ++ax) {
      info[ax] = fac->fit_ranks()[ax];
      fit_residual[ax] = fac->fit_residual[ax];
    }
    info[3] = fac->rank_b();
    info[4] = fac->fit_clamped_negative ? 1 : 0;
    for (size_t r = 0; r < pc.pivots.size(); ++r) pivots[r] = pc.pivots[r];
    *handle = fac;
  });
}

}  // extern "C"

// ORACLE — TEST INFRASTRUCTURE ONLY.  extern "C" surface of the CPU
// restatement so that pytest (ctypes) and bench.py's cpu_baseline leg can
// drive it.  Results are returned through opaque handles so variable-rank
// outputs (reduce_rank, TEI) need no size negotiation.
#include <cstring>
#include <string>

#include "tengrid_oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const snap_error& e) {
    g_err = e.what();
    return 3;
  } catch (const numerical_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

Mat mat_from(const double* p, idx r, idx c) {
  Mat m(r, c);
  if (r * c) std::memcpy(m.d.data(), p, sizeof(double) * r * c);
  return m;
}

Grid grid_from(const double* b, const long long* n) {
  return make_grid({b[0], b[1], b[2]}, {n[0], n[1], n[2]});
}

std::vector<BasisFn> basis_from(int nfn, const double* centers, const int* degs, const int* nprim,
                                const double* exps, const double* coefs) {
  std::vector<BasisFn> fns(nfn);
  int off = 0;
  for (int i = 0; i < nfn; ++i) {
    for (int ax = 0; ax < 3; ++ax) {
      fns[i].center[ax] = centers[3 * i + ax];
      fns[i].deg[ax] = degs[3 * i + ax];
    }
    for (int p = 0; p < nprim[i]; ++p) {
      fns[i].exps.push_back(exps[off + p]);
      fns[i].coefs.push_back(coefs[off + p]);
    }
    off += nprim[i];
  }
  return fns;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// ---- CP handles
void* orc_cp_new() { return new CP3(); }
void orc_cp_free(void* h) { delete static_cast<CP3*>(h); }
long long orc_cp_rank(void* h) { return static_cast<CP3*>(h)->rank(); }
long long orc_cp_extent(void* h, int ax) { return static_cast<CP3*>(h)->extent(ax); }
void orc_cp_get(void* h, int ax, double* out) {
  auto& m = static_cast<CP3*>(h)->f[ax];
  if (!m.d.empty()) std::memcpy(out, m.d.data(), sizeof(double) * m.d.size());
}
void orc_cp_get_w(void* h, double* out) {
  auto& w = static_cast<CP3*>(h)->w;
  if (!w.empty()) std::memcpy(out, w.data(), sizeof(double) * w.size());
}
int orc_cp_set(void* h, const long long* n, long long r, const double* f0, const double* f1, const double* f2,
               const double* w) {
  return guard([&] {
    CP3& t = *static_cast<CP3*>(h);
    const double* fs[3] = {f0, f1, f2};
    for (int ax = 0; ax < 3; ++ax) t.f[ax] = mat_from(fs[ax], n[ax], r);
    t.w.assign(w, w + r);
  });
}

// ---- 1D
int orc_conv_central_many(long long n, long long c, const double* U, const double* v, double* out) {
  return guard([&] {
    Mat r = conv_central_many(mat_from(U, n, c), v, n);
    if (!r.d.empty()) std::memcpy(out, r.d.data(), sizeof(double) * r.d.size());
  });
}

int orc_conv_full(long long n, const double* u, const double* v, int use_fft, double* out) {
  return guard([&] {
    Vec r = use_fft ? conv_full_fft(u, n, v, n) : conv_full_direct(u, n, v, n);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

// ---- tensor algebra
int orc_convolve(void* a, void* b, const double* h, void* out) {
  return guard([&] { *static_cast<CP3*>(out) = convolve(*static_cast<CP3*>(a), *static_cast<CP3*>(b), {h[0], h[1], h[2]}); });
}
int orc_hartree_potential(void* theta, void* kernel, const double* h, void* out) {
  return guard([&] {
    *static_cast<CP3*>(out) = hartree_potential(*static_cast<CP3*>(theta), *static_cast<CP3*>(kernel), {h[0], h[1], h[2]});
  });
}
int orc_hadamard(void* a, void* b, void* out) {
  return guard([&] { *static_cast<CP3*>(out) = hadamard(*static_cast<CP3*>(a), *static_cast<CP3*>(b)); });
}
int orc_scalar_product(void* a, void* b, double* out) {
  return guard([&] { *out = scalar_product(*static_cast<CP3*>(a), *static_cast<CP3*>(b)); });
}
int orc_value_at(void* t, long long npts, const long long* ijk, double* out) {
  return guard([&] {
    const CP3& c = *static_cast<CP3*>(t);
    for (long long p = 0; p < npts; ++p) out[p] = value_at(c, ijk[3 * p], ijk[3 * p + 1], ijk[3 * p + 2]);
  });
}

// ---- kernel / grid / basis
int orc_make_expsum(long long m, double c0, double lo, double hi, double* nodes, double* weights, double* scale,
                    double* mesh) {
  return guard([&] {
    ExpSum es = make_expsum(m, c0, lo, hi);
    std::memcpy(nodes, es.nodes.data(), sizeof(double) * es.nodes.size());
    std::memcpy(weights, es.weights.data(), sizeof(double) * es.weights.size());
    *scale = es.scale;
    *mesh = es.mesh;
  });
}
double orc_gauss_cell_integral(double t, double c, double h) { return gauss_cell_integral(t, c, h); }
int orc_kernel_tensor(const double* b, const long long* n, long long terms, const double* nodes, const double* weights,
                      int doubled, void* out) {
  return guard([&] {
    ExpSum es;
    es.nodes.assign(nodes, nodes + terms);
    es.weights.assign(weights, weights + terms);
    *static_cast<CP3*>(out) = kernel_tensor(grid_from(b, n), es, doubled != 0);
  });
}
int orc_window_offset(const double* b, const long long* n, int ax, double center, long long* ofs) {
  return guard([&] { *ofs = window_offset(grid_from(b, n), ax, center); });
}
int orc_basis_handle(const double* b, const long long* n, int nfn, const double* centers, const int* degs,
                     const int* nprim, const double* exps, const double* coefs, void** out_handles) {
  return guard([&] {
    auto disc = discretize_basis(grid_from(b, n), basis_from(nfn, centers, degs, nprim, exps, coefs));
    for (int i = 0; i < nfn; ++i) out_handles[i] = new CP3(std::move(disc[i]));
  });
}

// ---- hf
int orc_coulomb_matrix(const double* b, const long long* n, int nb, void** disc_handles, void* vh, double* J) {
  return guard([&] {
    std::vector<CP3> disc;
    for (int i = 0; i < nb; ++i) disc.push_back(*static_cast<CP3*>(disc_handles[i]));
    Mat j = coulomb_matrix(grid_from(b, n), disc, *static_cast<CP3*>(vh));
    std::memcpy(J, j.d.data(), sizeof(double) * nb * nb);
  });
}
int orc_density_tensor(int nb, void** disc_handles, long long nocc, const double* c_occ, double eps, void* out) {
  return guard([&] {
    std::vector<CP3> disc;
    for (int i = 0; i < nb; ++i) disc.push_back(*static_cast<CP3*>(disc_handles[i]));
    *static_cast<CP3*>(out) = density_tensor(disc, mat_from(c_occ, nb, nocc), eps);
  });
}

// ---- hf.cpp / tei.cpp operators
static std::vector<CP3> disc_from(int nb, void** h) {
  std::vector<CP3> disc;
  for (int i = 0; i < nb; ++i) disc.push_back(*static_cast<CP3*>(h[i]));
  return disc;
}
int orc_one_electron(const double* b, const long long* n, int nb, void** disc_handles, int which, double* out) {
  return guard([&] {
    const auto disc = disc_from(nb, disc_handles);
    const Grid g = grid_from(b, n);
    Mat m = which == 0 ? overlap_matrix(g, disc) : kinetic_matrix(g, disc, which == 2);
    if (!m.d.empty()) std::memcpy(out, m.d.data(), sizeof(double) * m.d.size());
  });
}
int orc_nuclear_potential_tensor(const double* b, const long long* n, int nnuc, const double* centers,
                                 const double* charges, void* ref, void* out) {
  return guard([&] {
    std::vector<std::array<double, 3>> c(nnuc);
    for (int a = 0; a < nnuc; ++a) c[a] = {centers[3 * a], centers[3 * a + 1], centers[3 * a + 2]};
    *static_cast<CP3*>(out) =
        nuclear_potential_tensor(grid_from(b, n), c, Vec(charges, charges + nnuc), *static_cast<CP3*>(ref));
  });
}
int orc_nuclear_matrix(int nb, void** disc_handles, void* pc, double* V) {
  return guard([&] {
    Mat v = nuclear_matrix(disc_from(nb, disc_handles), *static_cast<CP3*>(pc));
    if (!v.d.empty()) std::memcpy(V, v.d.data(), sizeof(double) * v.d.size());
  });
}
int orc_exchange_matrix(const double* b, const long long* n, int nb, void** disc_handles, long long nocc,
                        const double* c_occ, void* kernel, double* K) {
  return guard([&] {
    Mat k = exchange_matrix(grid_from(b, n), disc_from(nb, disc_handles), mat_from(c_occ, nb, nocc),
                            *static_cast<CP3*>(kernel));
    if (!k.d.empty()) std::memcpy(K, k.d.data(), sizeof(double) * k.d.size());
  });
}
int orc_from_factors(int which, long long nb, long long rank, const double* h_core, const double* chol,
                     const double* density, double* out) {
  return guard([&] {
    const Mat l = mat_from(chol, nb * nb, rank), d = mat_from(density, nb, nb);
    Mat r = which == 0 ? coulomb_from_factors(l, d)
            : which == 1 ? exchange_from_factors(l, d)
                         : fock_from_factors(mat_from(h_core, nb, nb), l, d);
    if (!r.d.empty()) std::memcpy(out, r.d.data(), sizeof(double) * r.d.size());
  });
}

// ---- reduction
int orc_thin_svd_left(long long r, long long c, const double* a, double* u_out, double* s_out, long long* kept) {
  return guard([&] {
    Mat u;
    Vec s;
    thin_svd_left(mat_from(a, r, c), u, s);
    *kept = static_cast<long long>(s.size());
    if (!u.d.empty()) std::memcpy(u_out, u.d.data(), sizeof(double) * u.d.size());
    if (!s.empty()) std::memcpy(s_out, s.data(), sizeof(double) * s.size());
  });
}
int orc_sym_eigen(long long n, const double* a, double* ev, double* z) {
  return guard([&] {
    Vec e;
    Mat v;
    sym_eigen(mat_from(a, n, n), e, v);
    std::memcpy(ev, e.data(), sizeof(double) * n);
    std::memcpy(z, v.d.data(), sizeof(double) * n * n);
  });
}
int orc_householder_qr(long long m, long long k, const double* a, double* q, double* r) {
  return guard([&] {
    Mat qq, rr;
    householder_qr_thin(mat_from(a, m, k), qq, rr);
    std::memcpy(q, qq.d.data(), sizeof(double) * qq.d.size());
    std::memcpy(r, rr.d.data(), sizeof(double) * rr.d.size());
  });
}
int orc_jacobi_svd(long long m, long long k, const double* a, double* u, double* s) {
  return guard([&] {
    Mat uu;
    Vec ss;
    jacobi_svd_thin(mat_from(a, m, k), uu, ss);
    std::memcpy(u, uu.d.data(), sizeof(double) * uu.d.size());
    std::memcpy(s, ss.data(), sizeof(double) * ss.size());
  });
}
// mode: 0 rhosvd, 1 canonical_to_tucker, 2 reduce_rank (canonical out)
// info[0..2] tucker ranks, info[3] rank_clamped, info[4] fallback, info[5] n sweeps
int orc_reduce(void* a, int use_eps, double eps, const long long* ranks, int sweeps, int mode, void* out_cp,
               long long* info, double* core_out, double* side0, double* side1, double* side2, double* sweep_fits) {
  return guard([&] {
    RedCfg c;
    c.use_eps = use_eps != 0;
    c.eps = eps;
    if (ranks) c.ranks = {ranks[0], ranks[1], ranks[2]};
    c.max_sweeps = sweeps;
    const CP3& in = *static_cast<CP3*>(a);
    TuckerRes tr = mode == 0 ? rhosvd(in, c) : canonical_to_tucker(in, c);
    for (int ax = 0; ax < 3; ++ax) info[ax] = tr.t.r[ax];
    info[3] = tr.rank_clamped;
    info[4] = tr.rhosvd_fallback;
    info[5] = static_cast<long long>(tr.sweep_fits.size());
    if (core_out && !tr.t.core.empty()) std::memcpy(core_out, tr.t.core.data(), sizeof(double) * tr.t.core.size());
    double* sides[3] = {side0, side1, side2};
    for (int ax = 0; ax < 3; ++ax)
      if (sides[ax] && !tr.t.side[ax].d.empty())
        std::memcpy(sides[ax], tr.t.side[ax].d.data(), sizeof(double) * tr.t.side[ax].d.size());
    if (sweep_fits && !tr.sweep_fits.empty())
      std::memcpy(sweep_fits, tr.sweep_fits.data(), sizeof(double) * tr.sweep_fits.size());
    if (mode == 2) *static_cast<CP3*>(out_cp) = tucker_to_canonical(tr.t);
  });
}

// ---- lattice: one axis, centres = lattice positions along that axis
int orc_assemble_axis(const double* b, const long long* n, int ax, long long R, const double* ref, long long L,
                      const double* centers, double* out, long long* ops) {
  return guard([&] {
    Grid g = grid_from(b, n);
    std::vector<double> cs(centers, centers + L);
    idx cnt = 0;
    Mat o = assemble_axis(g, mat_from(ref, 2 * n[ax], R), ax, cs, &cnt);
    if (ops) *ops += cnt;
    std::memcpy(out, o.d.data(), sizeof(double) * o.d.size());
  });
}

// ---- TEI
void* orc_tei_new() { return new TEI(); }
void orc_tei_free(void* h) { delete static_cast<TEI*>(h); }
int orc_tei_fit(void* h, const double* b, const long long* n, int nb, void** disc_handles, double eps_fit) {
  return guard([&] {
    std::vector<CP3> disc;
    for (int i = 0; i < nb; ++i) disc.push_back(*static_cast<CP3*>(disc_handles[i]));
    tei_density_fitting(*static_cast<TEI*>(h), grid_from(b, n), disc, eps_fit);
  });
}
int orc_tei_conv(void* h, void* kernel) {
  return guard([&] { tei_convolution_matrices(*static_cast<TEI*>(h), *static_cast<CP3*>(kernel)); });
}
int orc_tei_cholesky(void* h, double eps) { return guard([&] { tei_cholesky(*static_cast<TEI*>(h), eps); }); }
// query: info[0..2] fit ranks, info[3] np, info[4] nb, info[5] R_B, info[6] fit_clamped
void orc_tei_info(void* h, long long* info, double* fit_res) {
  TEI& f = *static_cast<TEI*>(h);
  for (int ax = 0; ax < 3; ++ax) {
    info[ax] = f.U[ax].cols;
    fit_res[ax] = f.fit_res[ax];
  }
  info[3] = f.np;
  info[4] = f.nb;
  info[5] = f.L.cols;
  info[6] = f.fit_clamped;
}
void orc_tei_get_uv(void* h, int ax, double* u, double* v) {
  TEI& f = *static_cast<TEI*>(h);
  std::memcpy(u, f.U[ax].d.data(), sizeof(double) * f.U[ax].d.size());
  std::memcpy(v, f.V[ax].d.data(), sizeof(double) * f.V[ax].d.size());
}
void orc_tei_get_conv(void* h, long long k, int ax, double* m) {
  TEI& f = *static_cast<TEI*>(h);
  std::memcpy(m, f.M[k][ax].d.data(), sizeof(double) * f.M[k][ax].d.size());
}
void orc_tei_get_chol(void* h, double* L, long long* piv) {
  TEI& f = *static_cast<TEI*>(h);
  if (!f.L.d.empty()) std::memcpy(L, f.L.d.data(), sizeof(double) * f.L.d.size());
  for (size_t i = 0; i < f.chol_piv.size(); ++i) piv[i] = f.chol_piv[i];
}
int orc_tei_column(void* h, long long pair, double* out) {
  return guard([&] {
    Vec c = tei_column(*static_cast<TEI*>(h), pair);
    std::memcpy(out, c.data(), sizeof(double) * c.size());
  });
}
int orc_tei_diagonal(void* h, double* out) {
  return guard([&] {
    Vec d = tei_diagonal(*static_cast<TEI*>(h));
    std::memcpy(out, d.data(), sizeof(double) * d.size());
  });
}
// pivoted Cholesky of an explicit SPD matrix (tests)
int orc_pivoted_cholesky(long long n, const double* a, double tol, int trace_stop, long long max_rank, double neg_tol,
                         double* L, long long* piv, long long* rank, double* residual, int* clamped) {
  return guard([&] {
    Mat A = mat_from(a, n, n);
    Vec dg(n);
    for (idx i = 0; i < n; ++i) dg[i] = A(i, i);
    PivChol pc = pivoted_cholesky([&](idx j) { return Vec(A.col(j), A.col(j) + n); }, dg, tol, trace_stop != 0,
                                  max_rank, neg_tol);
    *rank = pc.L.cols;
    if (!pc.L.d.empty()) std::memcpy(L, pc.L.d.data(), sizeof(double) * pc.L.d.size());
    for (size_t i = 0; i < pc.piv.size(); ++i) piv[i] = pc.piv[i];
    *residual = pc.residual;
    *clamped = pc.clamped;
  });
}

}  // extern "C"

// Restricted closed-shell SCF on the grid: the driver of reference
// proj/src/hf.cpp:172-270 (nuclear_repulsion, scf_solve) over the device
// operators of this library.  Host code here only sequences device work and
// folds nb x nb scalars (energies, mixing) exactly as the reference's loop
// does; every grid-sized or O(nb^3) step (discretised basis upload, overlap /
// kinetic / nuclear assembly, TEI factorisation, Fock builds, the generalized
// eigensolver, C S C^T checks, commutator residuals) runs on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "tgb_host.h"
#include "tgb_internal.hpp"

namespace {

struct DevVec {
  double* p = nullptr;
  size_t n = 0;
  explicit DevVec(size_t count = 0) { resize(count); }
  void resize(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    if (count) TGB_CUDA(cudaMalloc(&p, count * sizeof(double)));
  }
  ~DevVec() {
    if (p) cudaFree(p);
  }
  DevVec(const DevVec&) = delete;
  DevVec& operator=(const DevVec&) = delete;
};

void host_check(int rc) {
  if (rc != TGB_OK) throw tgb::Error(rc, tgb_host_last_error());
}
void dev_check(int rc) {
  if (rc != TGB_OK) throw tgb::Error(rc, tgb_last_error());
}

void put(double* dst, const std::vector<double>& v) {
  if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
}

}  // namespace

extern "C" {

void tgb_scf_config_default(tgb_scf_config* c) {
  c->max_iterations = 60;
  c->energy_tol = 1e-9;
  c->mixing = 0.7;
  c->eps_fit = 1e-8;
  c->eps_chol = 1e-10;
  c->kernel_eps = 1e-6;
  c->kernel_r_max = 0.0;
  c->density_reduce_eps = 1e-7;
  c->exact_mass_kinetic = 0;
}

int tgb_scf_solve(tgb_ctx* ctx, const tgb_molecule* mol, const tgb_basis_spec* bs, const tgb_scf_config* cfg,
                  tgb_scf_state* st) {
  return tgb::guarded_call([&] {
    tgb::require(mol && bs && cfg && st, "scf_solve: null argument");
    tgb::require(mol->nnuc > 0, "scf_solve: no nuclei");
    tgb::require(mol->n_electrons >= 1, "scf_solve: no electrons");
    const int64_t nb = bs->nfn;
    int n_occ;  // Molecule::n_occupied (basis.hpp:46-51)
    if (mol->n_electrons == 1) {
      n_occ = 1;
    } else {
      tgb::require(mol->n_electrons >= 2 && mol->n_electrons % 2 == 0,
                   "Molecule: closed-shell treatment needs an even electron count (or exactly one)");
      n_occ = static_cast<int>(mol->n_electrons / 2);
    }
    tgb::require(n_occ <= nb, "scf_solve: more occupied orbitals than basis functions");
    TGB_CUDA(cudaSetDevice(ctx->device));
    st->n_occupied = n_occ;
    const bool one_electron = mol->n_electrons == 1;
    const double occ_scale = one_electron ? 1.0 : 2.0;
    double h[3];
    for (int ax = 0; ax < 3; ++ax) {
      tgb::require(bs->b_half[ax] > 0.0, "make_grid: box half-width must be positive");
      tgb::require(bs->n[ax] >= 2, "make_grid: need at least 2 grid points per axis");
      h[ax] = tgb_mesh_size(bs->b_half[ax], bs->n[ax]);
    }

    // snap nuclei to grid nodes (hf.cpp:219-223); repulsion of the snapped geometry (hf.cpp:172-185)
    const int64_t nn = mol->nnuc;
    std::vector<double> snapped(3 * nn);
    for (int64_t a = 0; a < nn; ++a)
      for (int ax = 0; ax < 3; ++ax) {
        int64_t node = 0;
        host_check(tgb_snap_to_node(bs->b_half[ax], bs->n[ax], mol->centers[3 * a + ax], &node));
        snapped[3 * a + ax] = (static_cast<double>(node) - 0.5 * static_cast<double>(bs->n[ax] - 1)) * h[ax];
      }
    double enuc = 0.0;
    if (nn > 1)
      for (int64_t a = 0; a < nn; ++a)
        for (int64_t b = a + 1; b < nn; ++b) {
          double r2 = 0.0;
          for (int ax = 0; ax < 3; ++ax) {
            const double d = snapped[3 * a + ax] - snapped[3 * b + ax];
            r2 += d * d;
          }
          tgb::require(r2 > 0.0, "nuclear_repulsion: coincident nuclei");
          enuc += mol->charges[a] * mol->charges[b] / std::sqrt(r2);
        }
    st->nuclear_energy = enuc;
    put(st->snapped_centers, snapped);

    // discretize_basis (basis.cpp:16-46): one column per primitive, weight coeff * norm
    std::vector<int64_t> fn_offset(nb + 1);
    for (int64_t k = 0; k <= nb; ++k) fn_offset[k] = bs->prim_offset[k];
    tgb::require(fn_offset[0] == 0, "discretize_basis: bad primitive offsets");
    for (int64_t k = 0; k < nb; ++k)
      tgb::require(fn_offset[k + 1] > fn_offset[k], "discretize_basis: contraction needs at least one primitive");
    const int64_t P = fn_offset[nb];
    std::vector<double> hf[3], wprim(P);
    for (int ax = 0; ax < 3; ++ax) hf[ax].assign(bs->n[ax] * P, 0.0);
    for (int64_t k = 0; k < nb; ++k) {
      const int* deg = bs->degrees + 3 * k;
      for (int ax = 0; ax < 3; ++ax)
        tgb::require(deg[ax] == 0 || deg[ax] == 1, "discretize_basis: per-axis degree must be 0 or 1");
      for (int64_t p = fn_offset[k]; p < fn_offset[k + 1]; ++p) {
        double nrm = 0.0;
        host_check(tgb_primitive_norm(bs->exponents[p], deg[0] + deg[1] + deg[2], &nrm));
        wprim[p] = bs->coeffs[p] * nrm;
        for (int ax = 0; ax < 3; ++ax)
          host_check(tgb_gaussian_factor(bs->b_half[ax], bs->n[ax], bs->centers[3 * k + ax], bs->exponents[p], deg[ax],
                                         hf[ax].data() + bs->n[ax] * p));
      }
    }
    DevVec dfac[3], dw(P);
    tgb_cp basis{};
    for (int ax = 0; ax < 3; ++ax) {
      basis.n[ax] = bs->n[ax];
      dfac[ax].resize(hf[ax].size());
      TGB_CUDA(cudaMemcpy(dfac[ax].p, hf[ax].data(), hf[ax].size() * sizeof(double), cudaMemcpyHostToDevice));
      basis.factor[ax] = dfac[ax].p;
    }
    TGB_CUDA(cudaMemcpy(dw.p, wprim.data(), P * sizeof(double), cudaMemcpyHostToDevice));
    basis.rank = P;
    basis.weight = dw.p;

    tgb::DevStreamScope scope(ctx);
    const int64_t n2 = nb * nb;
    std::vector<double> S(n2), T(n2), V(n2), H(n2);
    tgb::one_electron_dev(ctx, 0, basis, fn_offset.data(), nb, h, S.data());
    tgb::one_electron_dev(ctx, cfg->exact_mass_kinetic ? 2 : 1, basis, fn_offset.data(), nb, h, T.data());

    // Newton kernel (hf.cpp:230-236)
    const double h_min = std::min({h[0], h[1], h[2]});
    const double box_diag = 2.0 * std::sqrt(bs->b_half[0] * bs->b_half[0] + bs->b_half[1] * bs->b_half[1] +
                                            bs->b_half[2] * bs->b_half[2]);
    const double r_max = cfg->kernel_r_max > 0.0 ? cfg->kernel_r_max : box_diag;
    int64_t km = 0;
    double kc0 = 0.0;
    host_check(tgb_expsum_for_interval(1.5 * h_min, r_max, cfg->kernel_eps, 2048, &km, &kc0));
    st->kernel_m = km;
    st->kernel_c0 = kc0;
    const int64_t terms = 2 * km + 1;
    std::vector<double> nodes(terms), weights(terms);
    double sc = 0.0, mesh = 0.0;
    host_check(tgb_make_expsum(km, kc0, 1.5 * h_min, r_max, nodes.data(), weights.data(), &sc, &mesh));
    auto kernel_tensor = [&](bool doubled, DevVec* f, DevVec& w, tgb_cp& out) {
      out = tgb_cp{};
      for (int ax = 0; ax < 3; ++ax) {
        const int64_t len = doubled ? 2 * bs->n[ax] : bs->n[ax];
        std::vector<double> col(len * terms);
        host_check(tgb_kernel_factors(bs->b_half[ax], bs->n[ax], terms, nodes.data(), weights.data(), doubled ? 1 : 0,
                                      col.data()));
        f[ax].resize(col.size());
        TGB_CUDA(cudaMemcpy(f[ax].p, col.data(), col.size() * sizeof(double), cudaMemcpyHostToDevice));
        out.n[ax] = len;
        out.factor[ax] = f[ax].p;
      }
      std::vector<double> ones(terms, 1.0);  // kernel.cpp:189
      w.resize(terms);
      TGB_CUDA(cudaMemcpy(w.p, ones.data(), terms * sizeof(double), cudaMemcpyHostToDevice));
      out.rank = terms;
      out.weight = w.p;
    };
    {  // nuclear matrix with the doubled reference (hf.cpp:103-116)
      DevVec rf[3], rw;
      tgb_cp ref;
      kernel_tensor(true, rf, rw, ref);
      std::vector<int64_t> offs(3 * nn);
      for (int64_t a = 0; a < nn; ++a)
        for (int ax = 0; ax < 3; ++ax)
          host_check(tgb_window_offset(bs->b_half[ax], bs->n[ax], snapped[3 * a + ax], &offs[3 * a + ax]));
      DevVec pf[3], pw(nn * terms);
      tgb_cp pc{};
      for (int ax = 0; ax < 3; ++ax) {
        pc.n[ax] = bs->n[ax];
        pf[ax].resize(bs->n[ax] * nn * terms);
        pc.factor[ax] = pf[ax].p;
      }
      pc.rank = nn * terms;
      pc.weight = pw.p;
      const int64_t n3[3] = {bs->n[0], bs->n[1], bs->n[2]};
      std::vector<double> q(mol->charges, mol->charges + nn);
      tgb::nuclear_potential_dev(ctx, ref, n3, offs.data(), q.data(), nn, pc);
      tgb::coulomb_matrix_dev(ctx, basis, fn_offset.data(), nb, pc, -1.0, V.data());
    }
    for (int64_t i = 0; i < n2; ++i) H[i] = T[i] + V[i];
    put(st->overlap, S);
    put(st->kinetic, T);
    put(st->nuclear, V);
    put(st->core_hamiltonian, H);

    // factorised TEI (hf.cpp:238-241): build_tei on the device
    DevVec L;
    int64_t RB = 0;
    if (!one_electron) {
      DevVec kf[3], kw;
      tgb_cp kern;
      kernel_tensor(false, kf, kw, kern);
      tgb_tei* tei = nullptr;
      dev_check(tgb_tei_create(&tei));
      try {
        dev_check(tgb_tei_density_fitting(ctx, tei, &basis, fn_offset.data(), nb, h, cfg->eps_fit, TGB_MEM_DEVICE));
        dev_check(tgb_tei_convolution_matrices(ctx, tei, &kern, TGB_MEM_DEVICE));
        dev_check(tgb_tei_cholesky(ctx, tei, cfg->eps_chol));
        int64_t info[8];
        double res[3];
        dev_check(tgb_tei_info(tei, info, res));
        RB = info[5];
        L.resize(std::max<int64_t>(1, n2 * RB));
        std::vector<int64_t> piv(std::max<int64_t>(1, RB));
        dev_check(tgb_tei_get_cholesky(tei, L.p, piv.data(), TGB_MEM_DEVICE));
      } catch (...) {
        tgb_tei_destroy(tei);
        throw;
      }
      tgb_tei_destroy(tei);
    }
    st->tei_rank_b = RB;

    // Roothaan iterations (hf.cpp:243-268)
    DevVec dS(n2), dH(n2), dF(n2), dC(n2), de(nb), dD(n2), dDn(n2), dJ(n2), dK(n2), t1(n2), t2(n2), t3(n2);
    TGB_CUDA(cudaMemcpy(dS.p, S.data(), n2 * sizeof(double), cudaMemcpyHostToDevice));
    TGB_CUDA(cudaMemcpy(dH.p, H.data(), n2 * sizeof(double), cudaMemcpyHostToDevice));
    TGB_CUDA(cudaMemset(dD.p, 0, n2 * sizeof(double)));
    std::vector<double> d(n2, 0.0), dnew(n2), hj(n2), hk(n2), tmp(n2), C(n2), e(nb);
    double prev_energy = 0.0;
    st->converged = 0;
    st->iterations = 0;
    for (int it = 0; it < cfg->max_iterations; ++it) {
      const double* F = dH.p;
      if (!one_electron) {
        tgb::factor_operator_dev(ctx, 2, nb, RB, dH.p, L.p, dD.p, dF.p);
        F = dF.p;
      }
      tgb::generalized_eigensolve_dev(ctx, nb, F, dS.p, dC.p, de.p);
      // orthonormality defect max |C^T S C - I|
      tgb::dgemm(ctx, false, false, nb, nb, nb, 1.0, dS.p, nb, dC.p, nb, 0.0, t1.p, nb);
      tgb::dgemm(ctx, true, false, nb, nb, nb, 1.0, dC.p, nb, t1.p, nb, 0.0, t2.p, nb);
      TGB_CUDA(cudaMemcpyAsync(tmp.data(), t2.p, n2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      // D_new = occ_scale C_occ C_occ^T
      tgb::dgemm(ctx, false, true, nb, nb, n_occ, occ_scale, dC.p, nb, dC.p, nb, 0.0, dDn.p, nb);
      TGB_CUDA(cudaMemcpyAsync(dnew.data(), dDn.p, n2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      TGB_CUDA(cudaStreamSynchronize(ctx->stream));
      double defect = 0.0;
      for (int64_t j = 0; j < nb; ++j)
        for (int64_t i = 0; i < nb; ++i) defect = std::max(defect, std::abs(tmp[i + nb * j] - (i == j ? 1.0 : 0.0)));
      if (st->orthonormality_defects) st->orthonormality_defects[it] = defect;

      double energy = 0.0;
      for (int64_t i = 0; i < n2; ++i) energy += dnew[i] * H[i];
      energy += enuc;
      if (!one_electron) {
        tgb::factor_operator_dev(ctx, 0, nb, RB, nullptr, L.p, dDn.p, dJ.p);
        tgb::factor_operator_dev(ctx, 1, nb, RB, nullptr, L.p, dDn.p, dK.p);
        TGB_CUDA(cudaMemcpyAsync(hj.data(), dJ.p, n2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        TGB_CUDA(cudaMemcpyAsync(hk.data(), dK.p, n2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        TGB_CUDA(cudaStreamSynchronize(ctx->stream));
        double two = 0.0;
        for (int64_t i = 0; i < n2; ++i) two += dnew[i] * (hj[i] + hk[i]);
        energy += 0.5 * two;
      }
      if (st->energy_history) st->energy_history[it] = energy;
      // residual || F D S - S D F ||_F with the density F was built from
      tgb::dgemm(ctx, false, false, nb, nb, nb, 1.0, F, nb, dD.p, nb, 0.0, t1.p, nb);      // F D
      tgb::dgemm(ctx, false, false, nb, nb, nb, 1.0, t1.p, nb, dS.p, nb, 0.0, t3.p, nb);  // F D S
      tgb::dgemm(ctx, false, false, nb, nb, nb, 1.0, dS.p, nb, dD.p, nb, 0.0, t1.p, nb);  // S D
      tgb::dgemm(ctx, false, false, nb, nb, nb, -1.0, t1.p, nb, F, nb, 1.0, t3.p, nb);    // - S D F
      TGB_CUDA(cudaMemcpyAsync(tmp.data(), t3.p, n2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      TGB_CUDA(cudaStreamSynchronize(ctx->stream));
      double rn = 0.0;
      for (int64_t i = 0; i < n2; ++i) rn += tmp[i] * tmp[i];
      if (st->residual_history) st->residual_history[it] = std::sqrt(rn);

      for (int64_t i = 0; i < n2; ++i) d[i] = cfg->mixing * dnew[i] + (1.0 - cfg->mixing) * d[i];
      TGB_CUDA(cudaMemcpy(dD.p, d.data(), n2 * sizeof(double), cudaMemcpyHostToDevice));
      st->energy = energy;
      st->iterations = it + 1;
      if (it > 0 && std::abs(energy - prev_energy) <= cfg->energy_tol) {
        st->converged = 1;
        break;
      }
      prev_energy = energy;
    }
    TGB_CUDA(cudaMemcpy(C.data(), dC.p, n2 * sizeof(double), cudaMemcpyDeviceToHost));
    TGB_CUDA(cudaMemcpy(e.data(), de.p, nb * sizeof(double), cudaMemcpyDeviceToHost));
    put(st->coefficients, C);
    put(st->orbital_energies, e);
    put(st->density, dnew);
  });
}

}  // extern "C"

"""Per-config measurements of the §8 rows on one B200 (companion to bench.py,
which measures the headline config 2).  Prints one JSON object per config and
writes profiles/<tag>_configs.json.

  cfg0  Hartree convolution n=1025, R_f=50, R_N=31          (a-1..a-5)
  cfg1  J: density (rank 12,800) -> reduce_rank(1e-6) -> V_H (R_N=41) -> coulomb_matrix  (a-6..a-11)
  cfg3  TEI: fitting + conv matrices + pivoted Cholesky, N_b=80 s/p, n=4097  (a-12..a-16)
  cfg4  lattice sum L=32, n=32769, R_N=41 + 10^5 probes     (a-17)

Timings: CUDA-synchronised wall clock around each stage after one warm-up
(stages contain host-driven loops, so events on one stream would not cover
them all).  Parity checks run against the oracle on samples.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

HBM = 6527.5
FP64 = 36.6


def timed(fn, reps=1, sync=None):
    sync = sync or (lambda: None)
    fn()
    sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    sync()
    return (time.perf_counter() - t0) / reps, out


def cfg0(ctx):
    import torch

    import paper_1504_06289_b200 as tg
    from oracle import oracle as O
    from paper_1504_06289_b200.inputs import hartree_case

    case = hartree_case(0)
    dt, dk = tg.DeviceCP.from_host(case.theta), tg.DeviceCP.from_host(case.kernel.tensor)
    out = tg.DeviceCP.empty([1025] * 3, dt.rank() * dk.rank())
    t, _ = timed(lambda: tg.hartree_potential(dt, dk, case.grid.h, ctx, out=out), reps=20, sync=torch.cuda.synchronize)
    # device time per call (CUDA events on the context stream around 100 back-to-back calls)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.ExternalStream(ctx.stream)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(100):
        tg.hartree_potential(dt, dk, case.grid.h, ctx, out=out)
    e1.record(st)
    torch.cuda.synchronize()
    t_dev = e0.elapsed_time(e1) / 100 / 1e3
    ctx.reset_launch_count()
    tg.hartree_potential(dt, dk, case.grid.h, ctx, out=out)
    launches = ctx.launch_count()
    units = 3 * 50 * 31
    byts = 8.0 * 3 * 1025 * (50 * 31 + 50 + 31)
    vh = out.to_host()
    ovh = O.hartree_potential(O.OCP.from_cp(case.theta), O.OCP.from_cp(case.kernel.tensor), case.grid.h)
    err = max(float(np.abs(vh.factor[ax] - f).max() / np.abs(f).max()) for ax, f in enumerate(ovh.factors()))
    got = tg.value_at_points(vh, case.samples, ctx)
    ref = O.value_at(ovh, case.samples)
    # analytic Newton potential of the Gaussian density at 200 samples (reported, quadrature-limited)
    pts = case.samples[:200]
    xyz = np.stack([case.grid.coord(ax, pts[:, ax]) for ax in range(3)], 1)
    from paper_1504_06289_b200.inputs import analytic_potential

    ana = analytic_potential(xyz, case.a, case.centres, case.c)
    return {"config": 0, "what": "hartree_potential n=1025 R_f=50 R_N=31", "ms": t * 1e3, "convs_per_s": units / t,
            "device_ms_per_call": t_dev * 1e3, "launches_per_call": launches,
            "hbm_frac": byts / t / 1e9 / HBM, "parity_factor_relmax": err,
            "parity_samples_relmax": float(np.abs(got - ref).max() / np.abs(ref).max()),
            "analytic_relmax_200pts": float(np.abs(got[:200] - ana).max() / np.abs(ana).max())}


def cfg1(ctx):
    import torch

    import paper_1504_06289_b200 as tg
    from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, basis_case, occupied_coefficients

    bs, rng = basis_case(1)
    disc = tg.discretize_basis(bs)
    c_occ = occupied_coefficients(rng, len(disc), 8)
    # unreduced density (host tensor algebra, as the reference's add/hadamard)
    t_build0 = time.perf_counter()
    theta_full = tg.CanonicalTensor3.zero(disc[0].extents())
    for a in range(8):
        phi = tg.orbital_tensor(disc, c_occ[:, a])
        theta_full = tg.add(theta_full, tg.scale(tg.hadamard(phi, phi), 2.0))
    t_build = time.perf_counter() - t_build0
    cfgr = tg.ReductionConfig.tolerance(1e-6)
    t_red, red = timed(lambda: tg.reduce_rank(theta_full, cfgr, ctx), reps=1, sync=torch.cuda.synchronize)
    # the drop-in density_tensor: Theta built on the device from the basis, reduced there
    t_dens, red2 = timed(lambda: tg.density_tensor(disc, c_occ, 1e-6, ctx), reps=1, sync=torch.cuda.synchronize)
    res = tg.canonical_to_tucker(theta_full, cfgr, ctx)
    # opt-in full mode_singular_values (csrc/spectrum.cu): the three 2049-point spectra of Theta's mode matrices
    dth = tg.DeviceCP.from_host(theta_full)
    t_spec, spec = timed(lambda: [tg.mode_spectrum(dth, ax, ctx) for ax in range(3)], reps=1,
                         sync=torch.cuda.synchronize)
    kern = tg.kernel_tensor(bs.grid, tg.make_expsum(KERNEL_M[1], KERNEL_C0[1]), False)
    dt, dk = tg.DeviceCP.from_host(red), tg.DeviceCP.from_host(kern.tensor)
    vh = tg.DeviceCP.empty(list(bs.grid.n), dt.rank() * dk.rank())
    t_vh, _ = timed(lambda: tg.hartree_potential(dt, dk, bs.grid.h, ctx, out=vh), reps=3, sync=torch.cuda.synchronize)
    t_j, J = timed(lambda: tg.coulomb_matrix(bs, disc, vh, ctx), reps=3, sync=torch.cuda.synchronize)
    n, P, RV = bs.grid.n[0], len(disc) * (len(disc) + 1) // 2, vh.rank()
    # the +-t twin kernel columns give bitwise-equal V_H columns, merged before the GEMMs
    # (assembly.cu): the useful work runs over the distinct ones
    RVd = dt.rank() * ((dk.rank() + 1) // 2)
    flops_j = 2.0 * 3 * n * P * RVd
    return {"config": 1, "what": "density(12800)->reduce_rank(1e-6)->V_H->coulomb_matrix, n=2049, N_b=40",
            "density_build_host_s": t_build, "reduce_rank_ms": t_red * 1e3,
            "density_tensor_device_ms": t_dens * 1e3, "density_tensor_rank": red2.rank(), "tucker_ranks": list(res.tucker.ranks()),
            "reduced_rank": red.rank(), "rank_margins": res.rank_margins,
            "mode_spectra_ms": t_spec * 1e3, "mode_spectra_counts": [len(x) for x in spec],
            "hartree_ms": t_vh * 1e3, "R_V": RV, "R_V_distinct": RVd, "coulomb_ms": t_j * 1e3,
            "coulomb_tflops": flops_j / t_j / 1e12, "coulomb_fp64_frac": flops_j / t_j / 1e12 / FP64,
            "J_symmetric_exact": bool(np.array_equal(J, J.T)), "J_trace": float(np.trace(J))}


def cfg3(ctx):
    import torch

    import paper_1504_06289_b200 as tg
    from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, basis_case

    bs, _ = basis_case(3)
    disc = tg.discretize_basis(bs)
    kern = tg.kernel_tensor(bs.grid, tg.make_expsum(KERNEL_M[3], KERNEL_C0[3]), False)
    warm = tg.TEIFactorization(ctx)  # first use loads modules and builds plans; time the second build
    tg.tei_density_fitting(warm, bs, disc, 1e-6)
    tg.tei_convolution_matrices(warm, kern)
    tg.tei_cholesky(warm, 1e-6)
    torch.cuda.synchronize()
    # time the second build on the same factorisation object: its device buffers (L 328 MB, the stored
    # V M_k^T 0.8 GB, ...) are already allocated, so cudaMalloc/cudaFree (and Python GC of a previous
    # object) stay out of the timed region
    fac = warm
    t0 = time.perf_counter()
    tg.tei_density_fitting(fac, bs, disc, 1e-6)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tg.tei_convolution_matrices(fac, kern)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tg.tei_cholesky(fac, 1e-6)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    from paper_1504_06289_b200.tei import pivot_margins

    margins = pivot_margins(fac, tg.tei_diagonal(fac), 1e-6)
    n, np_ = bs.grid.n[0], fac.n_prim
    gram_flops = 3 * 2.0 * n * n * np_ * np_  # the reference's dense G G^T (ours forms (F F^T)^2: np x fewer)
    return {"config": 3, "what": "build_tei N_b=80 s/p, n=4097, eps_fit=eps_chol=1e-6", "fit_ms": (t1 - t0) * 1e3,
            "fit_dense_gram_equiv_tflops": gram_flops / (t1 - t0) / 1e12, "conv_ms": (t2 - t1) * 1e3,
            "cholesky_ms": (t3 - t2) * 1e3, "fit_ranks": list(fac.fit_ranks()), "R_B": fac.rank_b(),
            "pivot_margins": margins,
            "fit_residual": [float(x) for x in fac.fit_residual]}


def cfg4(ctx):
    import torch

    import paper_1504_06289_b200 as tg
    from paper_1504_06289_b200.inputs import Rng, lattice_case

    spec, grid, ref = lattice_case()
    offs = [tg.lattice_offsets(spec, grid, ax) for ax in range(3)]
    n, R = grid.n[0], ref.rank()
    dref = [torch.from_numpy(np.ascontiguousarray(ref.tensor.factor[ax].T)).cuda() for ax in range(3)]
    dout = [torch.empty((R, n), dtype=torch.float64, device="cuda") for _ in range(3)]
    import ctypes as C

    from paper_1504_06289_b200._lib import MEM_DEVICE, check, lib

    offs_c = [np.ascontiguousarray(o, dtype=np.int64) for o in offs]
    P3 = C.c_void_p * 3
    nn, LL = (C.c_int64 * 3)(n, n, n), (C.c_int64 * 3)(*[len(o) for o in offs_c])
    # equal host factors -> one device copy for every axis (tgb_lattice_assemble then assembles once)
    same = [ax == 0 or np.array_equal(ref.tensor.factor[ax], ref.tensor.factor[0]) for ax in range(3)]
    refp = P3(*[(dref[0] if same[ax] else dref[ax]).data_ptr() for ax in range(3)])
    offp = P3(*[o.ctypes.data for o in offs_c])
    outp = P3(*[d.data_ptr() for d in dout])

    def run():  # tgb_lattice_assemble: all three axes (the cubic case assembles one and copies)
        check(lib().tgb_lattice_assemble(ctx.handle, nn, R, refp, offp, LL, outp, MEM_DEVICE))

    def run_axes():  # one tgb_lattice_assemble_axis per axis
        for ax in range(3):
            check(lib().tgb_lattice_assemble_axis(ctx.handle, n, R, dref[ax].data_ptr(), offs_c[ax].ctypes.data,
                                                  len(offs_c[ax]), dout[ax].data_ptr(), MEM_DEVICE))

    t, _ = timed(run, reps=20, sync=torch.cuda.synchronize)
    t_axes, _ = timed(run_axes, reps=20, sync=torch.cuda.synchronize)
    st = torch.cuda.ExternalStream(ctx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(20):
        run_axes()
    e1.record(st)
    torch.cuda.synchronize()
    t_axes_dev = e0.elapsed_time(e1) / 20 / 1e3
    byts = 3 * 8.0 * (2 * n + n) * R
    lat = tg.DeviceCP(dout, torch.from_numpy(spec.charge * ref.tensor.weight).cuda())
    pts = torch.as_tensor(Rng(1504062894).integers(3 * 100_000, n).reshape(-1, 3)).cuda()
    tv, vals = timed(lambda: tg.value_at_points(lat, pts, ctx), reps=5, sync=torch.cuda.synchronize)
    return {"config": 4, "what": "lattice_sum_canonical L=32^3, n=32769, R_N=41 (+1e5 probes)", "assembly_ms": t * 1e3,
            "assembly_per_axis_calls_ms": t_axes * 1e3, "assembly_per_axis_device_ms": t_axes_dev * 1e3,
            "assembly_hbm_frac": byts / t / 1e9 / HBM, "window_ops": int(sum(len(o) for o in offs)),
            "probe_ms_1e5": tv * 1e3}


def cfg_hf(ctx):
    """§8f operators on the config-1 basis (N_b=40 s/p, n=2049, R_N=41) and config-3-sized factors."""
    import torch

    import paper_1504_06289_b200 as tg
    from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, Rng, basis_case, occupied_coefficients

    sync = torch.cuda.synchronize
    bs, rng = basis_case(1)
    disc = tg.discretize_basis(bs)
    nb = len(disc)
    c_occ = occupied_coefficients(rng, nb, 8)
    es = tg.make_expsum(KERNEL_M[1], KERNEL_C0[1])
    kp = tg.kernel_tensor(bs.grid, es, False)
    kd = tg.kernel_tensor(bs.grid, es, True)
    centres = sorted({f.center for f in bs.functions})
    mol = tg.Molecule([tg.Nucleus(2.0, c) for c in centres], 2 * len(centres))
    t_s, _ = timed(lambda: tg.overlap_matrix(bs, disc, ctx), reps=3, sync=sync)
    t_t, _ = timed(lambda: tg.kinetic_matrix(bs, disc, False, ctx), reps=3, sync=sync)
    t_v, V = timed(lambda: tg.nuclear_matrix(bs, disc, mol, kd, ctx), reps=3, sync=sync)
    t_k, K = timed(lambda: tg.exchange_matrix(bs, disc, c_occ, kp, ctx), reps=1, sync=sync)
    n, P, RN = bs.grid.n[0], nb, kp.rank()
    G = P * P  # Hadamard columns per orbital (single-primitive functions, phi rank = nb)
    # symmetric kernel: blocks k <= m only, in groups of 4 blocks (hf.cu exchange_matrix_dev)
    executed = sum((min(m0 + 4, nb) - m0) * min(m0 + 4, nb) for m0 in range(0, nb, 4)) / (nb * nb)
    flops_k = 8 * 2.0 * 3 * n * G * G * RN * executed
    out = {"config": "hf", "what": "config-1 basis: overlap/kinetic/nuclear/exchange; N_b=80 factor ops",
           "overlap_ms": t_s * 1e3, "kinetic_ms": t_t * 1e3, "nuclear_ms": t_v * 1e3, "exchange_ms": t_k * 1e3,
           "exchange_gemm_tflops": flops_k / t_k / 1e12, "exchange_fp64_frac": flops_k / t_k / 1e12 / FP64,
           "exchange_gemm_fraction_of_full": executed,
           "exchange_convolutions": 8 * 3 * G * RN, "K_symmetric_exact": bool(np.array_equal(K, K.T))}
    # Cholesky-factor operators at config-3 size (N_b=80, R_B=362)
    r2 = Rng(77)
    nb3, rb = 80, 362
    Lh = np.asfortranarray(r2.normal(nb3 * nb3 * rb).reshape(nb3 * nb3, rb, order="F"))
    cc = occupied_coefficients(r2, nb3, 20)
    Dh = np.asfortranarray(2.0 * cc @ cc.T)
    Hh = np.asfortranarray(np.diag(np.linspace(-5.0, 5.0, nb3)))
    L = torch.from_numpy(np.ascontiguousarray(Lh.T)).cuda()
    D = torch.from_numpy(np.ascontiguousarray(Dh.T)).cuda()
    H = torch.from_numpy(np.ascontiguousarray(Hh.T)).cuda()
    t_f, _ = timed(lambda: tg.fock_from_factors(H, L, D, ctx=ctx), reps=20, sync=sync)
    flops_f = 2.0 * 2 * nb3 * nb3 * rb + 2.0 * nb3 ** 3 * rb * 2
    S = np.eye(nb3) + 0.01 * (lambda a: a @ a.T)(r2.normal(nb3 * nb3).reshape(nb3, nb3))
    F = 0.5 * (Lh[:, :nb3].reshape(nb3, nb3, nb3)[:, :, 0] + Lh[:, :nb3].reshape(nb3, nb3, nb3)[:, :, 0].T)
    t_e, _ = timed(lambda: tg.generalized_eigensolve(F, S, ctx), reps=5, sync=sync)
    # MP2 (oracle and factorized) with n_occ = 20 of 80
    _, ev = tg.generalized_eigensolve(F, S, ctx)
    Cm, _ = tg.generalized_eigensolve(F, S, ctx)
    mos = tg.MOSpace(Cm, np.sort(ev) + np.where(np.arange(nb3) >= 20, 1.0, 0.0), 20)
    t_mo, mo = timed(lambda: tg.mo_transform_cholesky(Lh, mos, ctx), reps=3, sync=sync)
    t_m0, e0 = timed(lambda: tg.mp2_energy(mo, mos, "oracle", ctx=ctx), reps=3, sync=sync)
    t_m1, e1 = timed(lambda: tg.mp2_energy(mo, mos, "factorized", 1e-9, ctx=ctx), reps=3, sync=sync)
    out.update({"fock_from_factors_ms_nb80_rb362": t_f * 1e3, "fock_tflops": flops_f / t_f / 1e12,
                "generalized_eigensolve_ms_nb80": t_e * 1e3, "mo_transform_ms": t_mo * 1e3,
                "mp2_oracle_ms": t_m0 * 1e3, "mp2_factorized_ms": t_m1 * 1e3,
                "mp2_rel_diff_oracle_vs_factorized": abs(e0 - e1) / abs(e0)})
    # full SCF on the config-1 geometry: 4 centres, Z = 2 each, 8 electrons, N_b = 40 at n = 513
    bs5 = tg.BasisSet(tg.make_grid(12.0, 513), bs.functions)
    cfg = tg.SCFConfig(kernel_eps=1e-4, kernel_r_max=20.0, eps_fit=1e-7, eps_chol=1e-8)
    t_scf, st = timed(lambda: tg.scf_solve(mol, bs5, cfg, ctx), reps=1, sync=sync)
    out.update({"scf_s_n513_nb40": t_scf, "scf_iterations": st.iterations, "scf_converged": st.converged,
                "scf_energy": st.energy, "scf_tei_rank_b": st.tei_rank_b, "scf_kernel_terms": 2 * st.kernel_m + 1})
    return out


def main():
    import paper_1504_06289_b200 as tg

    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "3", "4"]
    import torch

    ctx = tg.Context(0, stream=torch.cuda.current_stream().cuda_stream)  # torch's stream: no cross-stream ordering
    out = []
    for w in which:
        fn = {"0": cfg0, "1": cfg1, "3": cfg3, "4": cfg4, "hf": cfg_hf}[w]
        try:
            r = fn(ctx)
        except Exception as exc:  # report and continue
            r = {"config": w, "error": repr(exc)}
        print(json.dumps(r), flush=True)
        out.append(r)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"{tag}_configs.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

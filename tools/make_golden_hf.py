"""Generate tests/golden/reference_hf.npz by running the REFERENCE's own
hf.cpp / tei.cpp / reduction.cpp (oracle/_ref: /root/reference/proj/src
compiled in place against oracle/eigen_shim, whose dense decompositions are
the restatement's LA) on a small seeded basis.

Run here (where /root/reference exists):  python tools/make_golden_hf.py
The fixtures are committed; tests/test_hf_oracle.py pins the restatement and
tests/test_hf_gpu.py the GPU path against them on any machine.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1504_06289_b200.inputs import Rng  # noqa: E402

B_HALF = np.array([5.0, 5.5, 4.5])
N = np.array([41, 45, 37])
KM, KC0 = 6, 0.9
FUNCTIONS = [  # (center, degree, [(exponent, coeff)])
    ((0.4, -0.3, 0.2), (0, 0, 0), [(1.1, 1.0)]),
    ((0.4, -0.3, 0.2), (1, 0, 0), [(0.7, 1.0)]),
    ((-0.8, 0.5, -0.1), (0, 0, 0), [(2.5, 0.6), (0.6, 0.5)]),
    ((-0.8, 0.5, -0.1), (0, 0, 1), [(0.9, 1.0)]),
    ((0.3, 0.9, -0.7), (0, 1, 0), [(1.4, 1.0)]),
    ((0.3, 0.9, -0.7), (0, 0, 0), [(0.35, 1.0)]),
]
NUCLEI = [((0.4, -0.3, 0.2), 1.0), ((-0.8, 0.5, -0.1), 2.0), ((0.3, 0.9, -0.7), 1.5)]


def basis_arrays():
    c, d, npr, e, cf = O._basis_args(FUNCTIONS)
    return {"basis_centers": c, "basis_degs": d, "basis_nprim": npr, "basis_exps": e, "basis_coefs": cf}


def main():
    from paper_1504_06289_b200 import build

    build.build_ref()
    assert O.rlib() is not None, "oracle/_ref not built (needs /root/reference)"
    R = O.Ref(B_HALF, N, FUNCTIONS)
    rng = Rng(4242)
    nb = len(FUNCTIONS)
    out = {"b_half": B_HALF, "n": N, "kernel_m_c0": np.array([KM, KC0]), **basis_arrays()}
    out["nuc_centers"] = np.array([c for c, _ in NUCLEI])
    out["nuc_charges"] = np.array([q for _, q in NUCLEI])

    # one-electron matrices (hf.cpp:48-87)
    out["S"] = R.one_electron(0)
    out["T_lumped"] = R.one_electron(1)
    out["T_exact"] = R.one_electron(2)
    # nuclear potential tensor + matrix (hf.cpp:89-116), doubled Newton reference
    V, pc = R.nuclear(out["nuc_centers"], out["nuc_charges"], KM, KC0)
    out["V"] = V
    for ax, f in enumerate(pc.factors()):
        out[f"pc_f{ax}"] = f
    out["pc_w"] = pc.weight()

    # occupied coefficients, exchange (hf.cpp:153-170)
    g = rng.normal(nb * 2).reshape(nb, 2, order="F")
    c_occ, _ = np.linalg.qr(g)
    c_occ = np.asfortranarray(c_occ)
    c_occ[1, 1] = 0.0  # one zero coefficient: orbital_tensor skips it (hf.cpp:42)
    out["c_occ"] = c_occ
    out["K"] = R.exchange_matrix(c_occ, KM, KC0)

    # Coulomb matrix from the unreduced density (density_tensor eps = 0 -> no reduction)
    theta = R.density_tensor(c_occ, 0.0)
    kern = O.OCP(lib=R.R)
    import ctypes as C

    rc = R.R.ref_kernel_tensor(O._p(R.b), R.nn, C.c_longlong(KM), C.c_double(KC0), C.c_int(0), kern.h)
    assert rc == 0
    hh = 2.0 * B_HALF / (N + 1)
    ks = O.OCP(kern.factors(), kern.weight() / float(np.prod(hh)), lib=R.R)
    vh = O.OCP(lib=R.R)
    assert R.R.ref_convolve(theta.h, ks.h, O._p(np.ascontiguousarray(hh)), vh.h) == 0
    out["J"] = R.coulomb_matrix(vh)
    out["theta_rank"] = np.array([theta.rank()])

    # Cholesky-factor builders (tei.cpp:215-238) on seeded factors
    rb = 5
    chol = np.asfortranarray(rng.normal(nb * nb * rb).reshape(nb * nb, rb, order="F"))
    dens = np.asfortranarray(2.0 * c_occ @ c_occ.T)
    hcore = np.asfortranarray(out["T_lumped"] + V)
    out["ff_chol"], out["ff_density"], out["ff_hcore"] = chol, dens, hcore
    for which, key in ((0, "ff_J"), (1, "ff_K"), (2, "ff_F")):
        out[key] = O.ref_from_factors(which, chol, dens, hcore if which == 2 else None)

    # generalized eigenproblem F C = S C e (hf.cpp:187-199)
    cc, ee = O.ref_generalized_eigensolve(out["ff_F"], out["S"])
    out["gen_C"], out["gen_e"] = cc, ee

    # TEI factorisation (tei.cpp:19-213)
    ranks, rb_tei, clamped, res, lchol, diag = R.build_tei(KM, KC0, 1e-6, 1e-6)
    out["tei_fit_ranks"] = np.array(ranks)
    out["tei_rank_b"] = np.array([rb_tei])
    out["tei_chol"], out["tei_diag"], out["tei_fit_residual"] = lchol, diag, res

    # rank reduction of the density tensor (reduction.cpp:172-273)
    info, red = O.ref_reduce(theta, eps=1e-6, mode=2)
    out["red_eps"] = np.array([1e-6])
    info1, _ = O.ref_reduce(theta, eps=1e-6, mode=1)
    out["red_tucker_ranks"] = np.array(info1["ranks"])
    out["red_canonical_rank"] = np.array([info["canonical_rank"]])
    for ax, f in enumerate(red.factors()):
        out[f"red_f{ax}"] = f
    out["red_w"] = red.weight()
    for ax, f in enumerate(theta.factors()):
        out[f"theta_f{ax}"] = f
    out["theta_w"] = theta.weight()

    # config-1 structure at n = 129: 40 s/p functions, 8 orbitals -> Theta rank 12,800 (the wide Gram
    # branch of thin_svd_left and Jacobi ALS), reduced by the reference's own reduce_rank at 1e-6
    from paper_1504_06289_b200.inputs import basis_case, occupied_coefficients

    bs1, rng1 = basis_case(1, n=129)
    c1 = occupied_coefficients(rng1, len(bs1.functions), 8)
    fns1 = [(f.center, f.degree, [(q.exponent, q.coeff) for q in f.primitives]) for f in bs1.functions]
    R1 = O.Ref(bs1.grid.b_half, bs1.grid.n, fns1)
    th1 = R1.density_tensor(c1, 0.0)
    info1, _ = O.ref_reduce(th1, eps=1e-6, mode=1)
    info2, red1 = O.ref_reduce(th1, eps=1e-6, mode=2)
    pts = np.ascontiguousarray(Rng(99).integers(3 * 2000, 129).reshape(2000, 3))
    out["cfg1s_n"] = np.array([129])
    out["cfg1s_c_occ"] = c1
    out["cfg1s_tucker_ranks"] = np.array(info1["ranks"])
    out["cfg1s_canonical_rank"] = np.array([info2["canonical_rank"]])
    out["cfg1s_pts"] = pts
    def ref_values(t):
        vals = np.zeros(len(pts))
        assert R1.R.ref_value_at(t.h, C.c_longlong(len(pts)), O._p(pts), O._p(vals)) == 0
        return vals

    out["cfg1s_theta_vals"] = ref_values(th1)
    out["cfg1s_red_vals"] = ref_values(red1)
    # config-3 structure at n = 129: 3 centres x (2 s + 2 p shells) = 24 functions, exponents
    # log-uniform in [0.1, 80], box 15, R_N = 41: the reference's own build_tei at 1e-6 / 1e-6
    from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, SEED_BASE

    rng3 = Rng(SEED_BASE + 3)
    cent3 = rng3.uniform(9, -5.0, 5.0).reshape(3, 3)
    fns3 = []
    for ci in range(3):
        for sh in ("s", "s", "p", "p"):
            alpha = float(rng3.loguniform(1, 0.1, 80.0)[0])
            for d in ([(0, 0, 0)] if sh == "s" else [(1, 0, 0), (0, 1, 0), (0, 0, 1)]):
                fns3.append((tuple(cent3[ci]), d, [(alpha, 1.0)]))
    R3 = O.Ref([15.0] * 3, [129] * 3, fns3)
    r3, rb3, cl3, res3, L3, _ = R3.build_tei(KERNEL_M[3], KERNEL_C0[3], 1e-6, 1e-6)
    c3, d3, np3, e3, cf3 = O._basis_args(fns3)
    out.update(tei3s_centers=c3, tei3s_degs=d3, tei3s_nprim=np3, tei3s_exps=e3, tei3s_coefs=cf3,
               tei3s_fit_ranks=np.array(r3), tei3s_rank_b=np.array([rb3]), tei3s_chol=L3,
               tei3s_clamped=np.array([int(cl3)]))
    path = ROOT / "tests" / "golden" / "reference_hf.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({len(out)} arrays)")


if __name__ == "__main__":
    main()

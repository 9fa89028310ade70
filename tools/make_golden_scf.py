"""Generate tests/golden/reference_scf.npz: the REFERENCE's own tg::scf_solve
(hf.cpp:201-270) and tg::expsum_for_interval (kernel.cpp:131-165) run from
oracle/_ref (reference sources compiled in place; shim LA) on small seeded
molecules.  Run here (where /root/reference exists):
    python tools/make_golden_scf.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402

CFG = dict(max_iterations=40, energy_tol=1e-9, mixing=0.7, eps_fit=1e-8, eps_chol=1e-10, kernel_eps=1e-4)

CASES = {
    # H2, contracted s + p_z per centre
    "h2": dict(b=[5.0, 5.0, 6.0], n=[31, 31, 35], electrons=2,
               nuclei=[((0.0, 0.0, -0.7), 1.0), ((0.0, 0.0, 0.7), 1.0)],
               fns=[((0.0, 0.0, -0.7), (0, 0, 0), [(1.2, 0.6), (0.35, 0.5)]),
                    ((0.0, 0.0, 0.7), (0, 0, 0), [(1.2, 0.6), (0.35, 0.5)]),
                    ((0.0, 0.0, -0.7), (0, 0, 1), [(0.8, 1.0)]),
                    ((0.0, 0.0, 0.7), (0, 0, 1), [(0.8, 1.0)])]),
    # one electron: F = H_core, no TEI (hf.cpp:214, 237-238)
    "h_atom": dict(b=[4.0, 4.0, 4.0], n=[29, 29, 29], electrons=1, nuclei=[((0.1, -0.2, 0.0), 1.0)],
                   fns=[((0.1, -0.2, 0.0), (0, 0, 0), [(0.4, 1.0)]), ((0.1, -0.2, 0.0), (0, 0, 0), [(1.6, 1.0)]),
                        ((0.1, -0.2, 0.0), (1, 0, 0), [(0.9, 1.0)])]),
    # 4 electrons on three centres, s/p functions, off-axis geometry
    "chain": dict(b=[5.5, 5.0, 5.0], n=[33, 31, 31], electrons=4,
                  nuclei=[((-1.2, 0.1, 0.0), 2.0), ((0.3, -0.2, 0.3), 1.0), ((1.4, 0.4, -0.3), 1.0)],
                  fns=[((-1.2, 0.1, 0.0), (0, 0, 0), [(2.5, 0.5), (0.6, 0.6)]), ((-1.2, 0.1, 0.0), (1, 0, 0), [(0.9, 1.0)]),
                       ((-1.2, 0.1, 0.0), (0, 1, 0), [(0.9, 1.0)]), ((0.3, -0.2, 0.3), (0, 0, 0), [(1.0, 1.0)]),
                       ((1.4, 0.4, -0.3), (0, 0, 0), [(1.1, 1.0)]), ((1.4, 0.4, -0.3), (0, 0, 1), [(0.7, 1.0)])]),
}

EXPSUM = [(0.5, 20.0, 1e-6), (0.3, 20.0, 1e-5), (1.0, 10.0, 1e-8), (0.45, 17.4, 1e-4)]


def main():
    from paper_1504_06289_b200 import build

    build.build_ref()
    assert O.rlib() is not None, "oracle/_ref not built (needs /root/reference)"
    out = {"cfg": np.array([CFG[k] for k in ("max_iterations", "energy_tol", "mixing", "eps_fit", "eps_chol",
                                             "kernel_eps")])}
    for name, c in CASES.items():
        ref = O.Ref(c["b"], c["n"], c["fns"])
        r = O.ref_scf_solve(ref, c["nuclei"], c["electrons"], CFG)
        for k in ("energy", "nuclear_energy", "iterations", "tei_rank_b"):
            out[f"{name}_{k}"] = np.array([r[k]])
        out[f"{name}_converged"] = np.array([int(r["converged"])])
        out[f"{name}_orbital_energies"] = r["orbital_energies"]
        out[f"{name}_density"] = r["density"]
        out[f"{name}_energy_history"] = r["energy_history"]
        print(name, r["energy"], r["iterations"], r["tei_rank_b"])
    out["expsum_in"] = np.array(EXPSUM)
    out["expsum_out"] = np.array([O.ref_expsum_for_interval(*x) for x in EXPSUM])
    mp2_fixtures(out)
    path = ROOT / "tests" / "golden" / "reference_scf.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path}")



def mp2_fixtures(out: dict) -> None:
    """MP2 (mp2.cpp) on the 'chain' SCF: the reference's MO factor and both energies."""
    import ctypes as C

    c = CASES["chain"]
    ref = O.Ref(c["b"], c["n"], c["fns"])
    R = ref.R
    cfg = np.array([CFG[k] for k in ("max_iterations", "energy_tol", "mixing", "eps_fit", "eps_chol", "kernel_eps")])
    q = np.ascontiguousarray([z for _, z in c["nuclei"]], dtype=np.float64)
    cen = np.ascontiguousarray([p for p, _ in c["nuclei"]], dtype=np.float64).reshape(-1)
    sizes = (C.c_longlong * 3)()
    args = (*ref._basis(), C.c_int(q.shape[0]), O._p(q), O._p(cen), C.c_int(c["electrons"]), O._p(cfg),
            C.c_double(1e-9), sizes)
    assert R.ref_mp2_case(*args, None, None, None, None, None) == 0, R.ref_last_error()
    nb, rb, nocc = sizes[0], sizes[1], sizes[2]
    chol = np.zeros((nb * nb, rb), order="F")
    coef = np.zeros((nb, nb), order="F")
    e = np.zeros(nb)
    mo = np.zeros((nocc * (nb - nocc), rb), order="F")
    e2 = np.zeros(2)
    assert R.ref_mp2_case(*args, O._p(chol), O._p(coef), O._p(e), O._p(mo), O._p(e2)) == 0, R.ref_last_error()
    out.update(mp2_chol=chol, mp2_coef=coef, mp2_energies=e, mp2_nocc=np.array([nocc]), mp2_mo_factor=mo,
               mp2_e2=e2, mp2_expsum_eps=np.array([1e-9]))
    print("mp2", e2)
    # reciprocal_expsum (kernel.cpp:205-250) on a few intervals
    rx = []
    for lo, hi, eps in ((0.5, 20.0, 1e-9), (1.0, 3.0, 1e-6), (0.2, 200.0, 1e-12), (2.0, 2.0, 1e-6)):
        t, ach, ok = C.c_longlong(), C.c_double(), C.c_int()
        r, w = np.zeros(256), np.zeros(256)
        assert R.ref_reciprocal_expsum(C.c_double(lo), C.c_double(hi), C.c_double(eps), C.byref(t), O._p(r), O._p(w),
                                       C.byref(ach), C.byref(ok)) == 0
        rx.append((lo, hi, eps, t.value, ach.value, ok.value))
        out[f"recip_{len(rx) - 1}_rates"], out[f"recip_{len(rx) - 1}_weights"] = r[:t.value], w[:t.value]
    out["recip_cases"] = np.array(rx)


if __name__ == "__main__":
    main()

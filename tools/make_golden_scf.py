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
    path = ROOT / "tests" / "golden" / "reference_scf.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path}")


if __name__ == "__main__":
    main()

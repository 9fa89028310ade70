"""Shared builder for the tests/golden/reference_hf.npz case (tools/make_golden_hf.py)."""
from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden" / "reference_hf.npz"


def load():
    return dict(np.load(GOLDEN))


def functions(g) -> list:
    """(center, degree, [(exponent, coeff)]) per function, as the fixture stored them."""
    out, off = [], 0
    for i, npr in enumerate(g["basis_nprim"]):
        c = tuple(g["basis_centers"][3 * i:3 * i + 3])
        d = tuple(int(x) for x in g["basis_degs"][3 * i:3 * i + 3])
        prims = [(float(g["basis_exps"][off + p]), float(g["basis_coefs"][off + p])) for p in range(npr)]
        off += int(npr)
        out.append((c, d, prims))
    return out


def product_case(g):
    """BasisSet, discretised basis, primary and doubled kernels through libtgb's host producers."""
    import paper_1504_06289_b200 as tg

    grid = tg.make_grid(tuple(g["b_half"]), tuple(int(x) for x in g["n"]))
    fns = [tg.SeparableBasisFunction(c, d, [tg.GaussianPrimitive(e, k) for e, k in prims])
           for c, d, prims in functions(g)]
    bs = tg.BasisSet(grid, fns)
    disc = tg.discretize_basis(bs)
    m, c0 = int(g["kernel_m_c0"][0]), float(g["kernel_m_c0"][1])
    es = tg.make_expsum(m, c0)
    return bs, disc, tg.kernel_tensor(grid, es, False), tg.kernel_tensor(grid, es, True)


def molecule(g):
    import paper_1504_06289_b200 as tg

    return tg.Molecule([tg.Nucleus(float(q), tuple(c)) for c, q in zip(g["nuc_centers"], g["nuc_charges"])],
                       n_electrons=4)

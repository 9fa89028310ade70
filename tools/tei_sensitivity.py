"""How reproducible is the reference's own config-3 TEI pipeline (tei.cpp:92-213)?
Run the reference (oracle/_ref) on the config-3 basis with every primitive
exponent moved by one ulp (a perturbation at the level of the rounding any
two correct implementations differ by) and compare the TEI diagonal, L L^T at
the fixture's probes and the pivots with tests/golden/reference_cfg3.npz.
The change is the reference's own sensitivity floor at this size.
Run here:  python tools/tei_sensitivity.py   (~7 min on 8 cores)
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, basis_case  # noqa: E402


def main():
    R = O.rlib()
    R.ref_build_tei_pivots.restype = C.c_int
    g = np.load(ROOT / "tests" / "golden" / "reference_cfg3.npz")
    bs, _ = basis_case(3)
    fns = [(tuple(f.center), tuple(f.degree), [(np.nextafter(p.exponent, np.inf), p.coeff) for p in f.primitives])
           for f in bs.functions]
    ref = O.Ref(bs.grid.b_half, bs.grid.n, fns)
    nb = ref.nb
    info = (C.c_longlong * 5)()
    res = np.zeros(3)
    piv = np.zeros(nb * nb, dtype=np.int64)
    h = C.c_void_p()
    rc = R.ref_build_tei_pivots(*ref._basis(), C.c_longlong(KERNEL_M[3]), C.c_double(KERNEL_C0[3]), C.c_double(1e-6),
                                C.c_double(1e-6), info, O._p(res), O._p(piv), C.byref(h))
    assert rc == 0, R.ref_last_error().decode()
    rb = info[3]
    chol = np.zeros((nb * nb, rb), order="F")
    diag = np.zeros(nb * nb)
    assert R.ref_tei_get(h, 0, 0, O._p(chol)) == 0
    assert R.ref_tei_get(h, 1, 0, O._p(diag)) == 0
    R.ref_tei_free(h)
    pr = g["probes"]
    llt = np.einsum("ij,ij->i", chol[pr[:, 0]], chol[pr[:, 1]]) if rb == int(g["rank_b"]) else None
    out = {"perturbation": "every primitive exponent +1 ulp", "fit_ranks": list(info[:3]), "rank_b": int(rb),
           "fit_ranks_same": list(info[:3]) == [int(x) for x in g["fit_ranks"]],
           "pivots_same": bool(rb == int(g["rank_b"]) and np.array_equal(piv[:rb], g["pivots"])),
           "diagonal_relmax_change": float(np.abs(diag - g["diagonal"]).max() / np.abs(g["diagonal"]).max()),
           "llt_change_over_maxdiag": (float(np.abs(llt - g["llt"]).max() / np.abs(g["diagonal"]).max())
                                       if llt is not None else None)}
    print(json.dumps(out))
    (ROOT / "profiles" / "r02_tei_reference_sensitivity.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()

"""Full-size fixtures for BASELINE.json configs 1, 3 and 4 from the REFERENCE's
own code (oracle/_ref: /root/reference/proj/src compiled against the shim LA),
run here on the CPU.  Test infrastructure: tests/test_configs_full_gpu.py pins
the device path against them; nothing in the product reads them.

  config 4  lattice_sum_canonical (lattice.cpp:116-129), L=32, n=32769, R_N=41:
            SHA-256 of every factor matrix and the weights (bit-identity),
            window_ops, value_at at 10^5 seeded points.
  config 3  build_tei (tei.cpp:206-213), N_b=80 s/p, n=4097, eps_fit=eps_chol=1e-6:
            fit ranks, residuals, R_B, the pivot sequence (ref_build_tei_pivots
            keeps pivoted_cholesky's), the diagonal, L L^T at 4096 seeded probes,
            4 B columns (tei_column).
  config 1  density_tensor (hf.cpp:118-129, reduce_rank split into C2T + T2C to
            report the Tucker ranks), V_H = hartree_potential of the reduced
            density at 10^4 seeded points, J = coulomb_matrix (hf.cpp:140-151,
            split by kernel column over threads).

Run here (where /root/reference exists):
    python tools/make_golden_configs.py 4 3 1      (THREADS=8 by default)
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1504_06289_b200.inputs import (KERNEL_C0, KERNEL_M, Rng, basis_case, lattice_case,  # noqa: E402
                                          occupied_coefficients)

GOLD = ROOT / "tests" / "golden"
THREADS = int(os.environ.get("THREADS", os.cpu_count() or 1))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.asfortranarray(a, dtype=np.float64).tobytes(order="F")).hexdigest()


def _functions(bs):
    return [(tuple(f.center), tuple(f.degree), [(p.exponent, p.coeff) for p in f.primitives]) for f in bs.functions]


def cfg4():
    R = O.rlib()
    spec, grid, ref = lattice_case()
    b, nn = O._grid_args(grid.b_half, grid.n)
    counts = (C.c_longlong * 3)(*spec.counts)
    out = O.OCP(lib=R)
    wops = C.c_longlong()
    t0 = time.perf_counter()
    rc = R.ref_lattice_sum_canonical(counts, C.c_double(spec.spacing), C.c_double(spec.charge), O._p(b), nn,
                                     C.c_longlong(KERNEL_M[4]), C.c_double(KERNEL_C0[4]), out.h, C.byref(wops))
    assert rc == 0, R.ref_last_error().decode()
    t = time.perf_counter() - t0
    f = out.factors()
    w = out.weight()
    pts = Rng(1504062894).integers(3 * 100_000, grid.n[0]).reshape(-1, 3)
    vals = np.zeros(pts.shape[0])
    rc = R.ref_value_at(out.h, C.c_longlong(pts.shape[0]), O._p(np.ascontiguousarray(pts)), O._p(vals))
    assert rc == 0
    np.savez_compressed(GOLD / "reference_cfg4.npz", factor_sha=np.array([sha(x) for x in f]), weight=w,
                        window_ops=np.array(wops.value), points_sha=np.array(hashlib.sha256(pts.tobytes()).hexdigest()),
                        values=vals,
                        shape=np.array([f[0].shape[0], f[0].shape[1]]))
    print(f"cfg4: rank {out.rank()} window_ops {wops.value} in {t:.1f} s")


def cfg3():
    R = O.rlib()
    bs, _ = basis_case(3)
    ref = O.Ref(bs.grid.b_half, bs.grid.n, _functions(bs))
    nb = ref.nb
    info = (C.c_longlong * 5)()
    res = np.zeros(3)
    piv = np.zeros(nb * nb, dtype=np.int64)
    h = C.c_void_p()
    t0 = time.perf_counter()
    rc = R.ref_build_tei_pivots(*ref._basis(), C.c_longlong(KERNEL_M[3]), C.c_double(KERNEL_C0[3]), C.c_double(1e-6),
                                C.c_double(1e-6), info, O._p(res), O._p(piv), C.byref(h))
    assert rc == 0, R.ref_last_error().decode()
    t = time.perf_counter() - t0
    try:
        rb = info[3]
        chol = np.zeros((nb * nb, rb), order="F")
        diag = np.zeros(nb * nb)
        assert R.ref_tei_get(h, 0, 0, O._p(chol)) == 0
        assert R.ref_tei_get(h, 1, 0, O._p(diag)) == 0
        rng = Rng(1504062893)
        probes = rng.integers(2 * 4096, nb * nb).reshape(-1, 2)
        llt = np.einsum("ij,ij->i", chol[probes[:, 0]], chol[probes[:, 1]])
        cols = np.array([0, nb * nb - 1, int(piv[0]), int(piv[rb // 2])], dtype=np.int64)
        B = np.zeros((nb * nb, len(cols)), order="F")
        for c, j in enumerate(cols):
            col = np.zeros(nb * nb)
            assert R.ref_tei_get(h, 2, C.c_longlong(int(j)), O._p(col)) == 0
            B[:, c] = col
    finally:
        R.ref_tei_free(h)
    np.savez_compressed(GOLD / "reference_cfg3.npz", fit_ranks=np.array(info[:3]), fit_residual=res, rank_b=np.array(rb),
                        clamped=np.array(info[4]), pivots=piv[:rb], diagonal=diag, probes=probes, llt=llt,
                        b_cols=cols, B=B)
    print(f"cfg3: fit ranks {list(info[:3])} R_B {rb} in {t:.1f} s")


def cfg1():
    R = O.rlib()
    bs, rng = basis_case(1)
    nb = len(bs.functions)
    c_occ = occupied_coefficients(rng, nb, 8)
    ref = O.Ref(bs.grid.b_half, bs.grid.n, _functions(bs))
    info = (C.c_longlong * 5)()
    red = O.OCP(lib=R)
    t0 = time.perf_counter()
    rc = R.ref_density_tucker(*ref._basis(), C.c_longlong(8), O._p(np.asfortranarray(c_occ)), C.c_double(1e-6), info,
                              red.h)
    assert rc == 0, R.ref_last_error().decode()
    t1 = time.perf_counter()
    print(f"cfg1: density_tensor tucker {list(info[:3])} canonical {info[3]} (from {info[4]}) in {t1 - t0:.1f} s",
          flush=True)
    # V_H at the 10^4 seeded points, kernel from the reference's own producer
    kt = O.OCP(lib=R)
    b, nn = O._grid_args(bs.grid.b_half, bs.grid.n)
    assert R.ref_kernel_tensor(O._p(b), nn, C.c_longlong(KERNEL_M[1]), C.c_double(KERNEL_C0[1]), C.c_int(0), kt.h) == 0
    pts = Rng(1504062891).integers(3 * 10_000, bs.grid.n[0]).reshape(-1, 3)
    hh = np.ascontiguousarray(np.asarray(bs.grid.h, dtype=np.float64))
    vh = np.zeros(pts.shape[0])
    rc = R.ref_hartree_samples(red.h, kt.h, O._p(hh), C.c_longlong(pts.shape[0]), O._p(np.ascontiguousarray(pts)),
                               C.c_int(THREADS), O._p(vh))
    assert rc == 0, R.ref_last_error().decode()
    t2 = time.perf_counter()
    print(f"cfg1: V_H samples in {t2 - t1:.1f} s", flush=True)
    J = np.zeros((nb, nb), order="F")
    rc = R.ref_coulomb_from_theta(*ref._basis(), red.h, C.c_longlong(KERNEL_M[1]), C.c_double(KERNEL_C0[1]),
                                  C.c_int(THREADS), O._p(J))
    assert rc == 0, R.ref_last_error().decode()
    t3 = time.perf_counter()
    print(f"cfg1: J in {t3 - t2:.1f} s", flush=True)
    np.savez_compressed(GOLD / "reference_cfg1.npz", tucker_ranks=np.array(info[:3]), canonical_rank=np.array(info[3]),
                        unreduced_rank=np.array(info[4]), c_occ=c_occ, points=pts, vh=vh, J=J)


def main():
    from paper_1504_06289_b200 import build

    build.build_ref()
    assert O.rlib() is not None, "oracle/_ref not built (needs /root/reference)"
    R = O.rlib()
    R.ref_density_tucker.restype = C.c_int
    R.ref_coulomb_from_theta.restype = C.c_int
    R.ref_build_tei_pivots.restype = C.c_int
    for c in sys.argv[1:] or ["4", "3", "1"]:
        {"4": cfg4, "3": cfg3, "1": cfg1}[c]()


if __name__ == "__main__":
    main()

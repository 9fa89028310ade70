"""Generate tests/golden/reference_conv_path.npz by running the REFERENCE's own
conv-path code (oracle/_ref/libtengrid_ref.so: /root/reference/proj/src/
fft.cpp, tensor.cpp, grid.cpp, kernel.cpp, basis.cpp, lattice.cpp compiled in
place against oracle/eigen_shim) on small seeded inputs.

Run here (where /root/reference exists):  python tools/make_golden.py
The fixtures are committed; tests/test_golden.py pins the oracle restatement
and the GPU path against them on any machine.
"""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1504_06289_b200.inputs import Rng  # noqa: E402


def p(a):
    return C.c_void_p(a.ctypes.data) if a.size else None


def chk(rc, R):
    if rc:
        raise RuntimeError(R.ref_last_error().decode())


def ref_cp(R, factors, weight):
    return O.OCP(factors, weight, lib=R)


def main():
    from paper_1504_06289_b200 import build

    build.build_ref()
    R = O.rlib()
    assert R is not None, "oracle/_ref not built (needs /root/reference)"
    out = {}
    rng = Rng(777)

    # 1. conv_full direct / fft (test_tensor.cpp:24-37 sizes)
    for n in (5, 31, 128, 200, 513):
        u, v = rng.normal(n), rng.normal(n)
        for fft in (0, 1):
            r = np.zeros(2 * n - 1)
            chk(R.ref_conv_full(C.c_longlong(n), p(u), p(v), C.c_int(fft), p(r)), R)
            out[f"conv_full_{n}_{fft}_u"], out[f"conv_full_{n}_{fft}_v"], out[f"conv_full_{n}_{fft}_out"] = u, v, r

    # 2. conv_central_many, odd and even n, both sides of the 128 threshold
    for n in (16, 17, 127, 128, 129, 256, 257, 1025):
        U = np.asfortranarray(rng.normal(3 * n).reshape(n, 3, order="F"))
        v = rng.normal(n)
        r = np.zeros((n, 3), order="F")
        chk(R.ref_conv_central_many(C.c_longlong(n), C.c_longlong(3), p(U), p(v), p(r), C.c_int(1)), R)
        out[f"ccm_{n}_U"], out[f"ccm_{n}_v"], out[f"ccm_{n}_out"] = U, v, r

    # 3. convolve / hadamard / scalar_product on random CP tensors with unequal extents
    dims = (12, 9, 16)
    a_f = [np.asfortranarray(rng.normal(d * 3).reshape(d, 3, order="F")) for d in dims]
    a_w = rng.normal(3)
    b_f = [np.asfortranarray(rng.normal(d * 2).reshape(d, 2, order="F")) for d in dims]
    b_w = rng.normal(2)
    h = np.array([0.37, 0.5, 0.21])
    A, B = ref_cp(R, a_f, a_w), ref_cp(R, b_f, b_w)
    Cc = O.OCP(lib=R)
    chk(R.ref_convolve(A.h, B.h, p(h), Cc.h), R)
    Hh = O.OCP(lib=R)
    chk(R.ref_hadamard(A.h, B.h, Hh.h), R)
    sp = C.c_double()
    chk(R.ref_scalar_product(A.h, B.h, C.byref(sp)), R)
    for ax in range(3):
        out[f"cp_a_f{ax}"], out[f"cp_b_f{ax}"] = a_f[ax], b_f[ax]
        out[f"convolve_f{ax}"] = Cc.factors()[ax]
        out[f"hadamard_f{ax}"] = Hh.factors()[ax]
    out["cp_a_w"], out["cp_b_w"], out["cp_h"] = a_w, b_w, h
    out["convolve_w"], out["hadamard_w"] = Cc.weight(), Hh.weight()
    out["scalar_product"] = np.array([sp.value])

    # 4. make_expsum and kernel tensors (primary and doubled)
    for m, c0 in ((1, 1.0), (8, 1.0), (15, 0.7098), (20, 0.7591), (32, 1.3)):
        nodes, w = np.zeros(2 * m + 1), np.zeros(2 * m + 1)
        sc, mesh = C.c_double(), C.c_double()
        chk(R.ref_make_expsum(C.c_longlong(m), C.c_double(c0), C.c_double(0.0), C.c_double(0.0), p(nodes), p(w),
                              C.byref(sc), C.byref(mesh)), R)
        out[f"expsum_{m}_nodes"], out[f"expsum_{m}_weights"] = nodes, w
        out[f"expsum_{m}_scale_mesh"] = np.array([sc.value, mesh.value])
        out[f"expsum_{m}_c0"] = np.array([c0])
    b3 = np.array([10.0, 10.0, 10.0])
    n3 = (C.c_longlong * 3)(33, 33, 33)
    for dbl in (0, 1):
        K = O.OCP(lib=R)
        chk(R.ref_kernel_tensor(p(b3), n3, C.c_longlong(8), C.c_double(1.0), C.c_int(dbl), K.h), R)
        out[f"kernel_{dbl}_f0"] = K.factors()[0]

    # 5. Hartree-type convolution of Gaussians with the kernel (odd and even n)
    for n in (65, 64):
        hh = 20.0 / (n + 1)
        x = (np.arange(n) - 0.5 * (n - 1)) * hh
        a = np.array([0.3, 2.0, 9.0])
        th = [np.asfortranarray(np.exp(-a[None, :] * (x[:, None] - c) ** 2)) for c in (0.1, -0.4, 0.7)]
        tw = np.array([1.0, 0.5, 1.5])
        nn = (C.c_longlong * 3)(n, n, n)
        K = O.OCP(lib=R)
        chk(R.ref_kernel_tensor(p(b3), nn, C.c_longlong(6), C.c_double(0.9), C.c_int(0), K.h), R)
        T = ref_cp(R, th, tw)
        kf = K.factors()
        Kw = K.weight() / (hh ** 3)  # hartree_potential weight scaling (hf.cpp:136)
        Ks = ref_cp(R, kf, Kw)
        V = O.OCP(lib=R)
        hv = np.array([hh, hh, hh])
        chk(R.ref_convolve(T.h, Ks.h, p(hv), V.h), R)
        pts = np.ascontiguousarray(rng.integers(3 * 50, n).reshape(50, 3))
        vals = np.zeros(50)
        chk(R.ref_value_at(V.h, C.c_longlong(50), p(pts), p(vals)), R)
        for ax in range(3):
            out[f"hartree_{n}_theta_f{ax}"] = th[ax]
            out[f"hartree_{n}_kernel_f{ax}"] = kf[ax]
            out[f"hartree_{n}_vh_f{ax}"] = V.factors()[ax]
        out[f"hartree_{n}_theta_w"], out[f"hartree_{n}_kernel_w"] = tw, K.weight()
        out[f"hartree_{n}_vh_w"], out[f"hartree_{n}_pts"], out[f"hartree_{n}_vals"] = V.weight(), pts, vals
        out[f"hartree_{n}_h"] = hv

    # 6. lattice_sum_canonical on a lattice-aligned grid (lattice.cpp:65-75 sizing)
    counts = (3, 2, 4)
    spacing, n0 = 2.0, 8
    cells = [c - 1 + 2 for c in counts]
    nl = [n0 * c - 1 for c in cells]
    bl = np.array([0.5 * c * spacing for c in cells])
    L = O.OCP(lib=R)
    ops = C.c_longlong()
    chk(R.ref_lattice_sum_canonical((C.c_longlong * 3)(*counts), C.c_double(spacing), C.c_double(1.5), p(bl),
                                    (C.c_longlong * 3)(*nl), C.c_longlong(6), C.c_double(0.9), L.h, C.byref(ops)), R)
    for ax in range(3):
        out[f"lattice_f{ax}"] = L.factors()[ax]
    out["lattice_w"], out["lattice_ops"] = L.weight(), np.array([ops.value])
    out["lattice_spec"] = np.array([*counts, spacing, 1.5, n0, *nl, *bl, 6, 0.9])

    # 7. discretize_basis (s, p, contracted)
    bn = (C.c_longlong * 3)(21, 22, 23)
    bb = np.array([5.0, 5.5, 6.0])
    centers = np.array([[0.1, -0.3, 0.7], [1.0, 0.0, -1.2], [-0.5, 0.5, 0.25]]).reshape(-1)
    degs = np.array([[0, 0, 0], [1, 0, 0], [0, 0, 1]], dtype=np.int32).reshape(-1)
    nprim = np.array([1, 2, 1], dtype=np.int32)
    exps = np.array([1.3, 0.4, 2.2, 0.8])
    coefs = np.array([1.0, 0.6, 0.4, 1.0])
    hs = (C.c_void_p * 3)()
    chk(R.ref_discretize_basis(p(bb), bn, C.c_int(3), p(centers), p(degs), p(nprim), p(exps), p(coefs), hs), R)
    for i in range(3):
        t = O.OCP.__new__(O.OCP)
        t.lib, t.h = R, C.c_void_p(hs[i])
        for ax in range(3):
            out[f"basis_{i}_f{ax}"] = t.factors()[ax]
        out[f"basis_{i}_w"] = t.weight()
    out["basis_spec_centers"], out["basis_spec_degs"], out["basis_spec_nprim"] = centers, degs, nprim
    out["basis_spec_exps"], out["basis_spec_coefs"] = exps, coefs

    dst = ROOT / "tests" / "golden" / "reference_conv_path.npz"
    np.savez_compressed(dst, **out)
    print(f"wrote {dst} ({dst.stat().st_size} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()

"""Pins against the reference itself.

tests/golden/reference_conv_path.npz was produced by tools/make_golden.py from
the REFERENCE's own code (proj/src/fft.cpp, tensor.cpp, grid.cpp, kernel.cpp,
basis.cpp, lattice.cpp compiled in place into oracle/_ref).  CPU tests pin the
oracle restatement and libtgb's host producers to it; GPU tests pin the
device path.  When oracle/_ref is present (this container), extra randomized
cases compare the restatement with the reference binary directly."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from conftest import relmax
from oracle import oracle as O
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import Rng

G = np.load(Path(__file__).parent / "golden" / "reference_conv_path.npz")


# ------------------------------------------------------------------ oracle restatement vs reference outputs (CPU)

@pytest.mark.parametrize("n", [5, 31, 128, 200, 513])
@pytest.mark.parametrize("fft", [0, 1])
def test_oracle_conv_full_bitwise(n, fft):
    got = O.conv_full(G[f"conv_full_{n}_{fft}_u"], G[f"conv_full_{n}_{fft}_v"], bool(fft))
    assert np.array_equal(got, G[f"conv_full_{n}_{fft}_out"])


@pytest.mark.parametrize("n", [16, 17, 127, 128, 129, 256, 257, 1025])
def test_oracle_conv_central_many_bitwise(n):
    got = O.conv_central_many(G[f"ccm_{n}_U"], G[f"ccm_{n}_v"])
    assert np.array_equal(got, G[f"ccm_{n}_out"])


def _cp(prefix, w):
    return [G[f"{prefix}_f{ax}"] for ax in range(3)], G[w]


def test_oracle_convolve_hadamard_scalar_product():
    a = O.OCP(*_cp("cp_a", "cp_a_w"))
    b = O.OCP(*_cp("cp_b", "cp_b_w"))
    c = O.convolve(a, b, G["cp_h"])
    for ax in range(3):
        assert np.array_equal(c.factors()[ax], G[f"convolve_f{ax}"])
    assert np.array_equal(c.weight(), G["convolve_w"])
    hd = O.hadamard(a, b)
    for ax in range(3):
        assert np.array_equal(hd.factors()[ax], G[f"hadamard_f{ax}"])
    assert O.scalar_product(a, b) == pytest.approx(float(G["scalar_product"][0]), rel=1e-14)


@pytest.mark.parametrize("m", [1, 8, 15, 20, 32])
def test_expsum_bitwise_oracle_and_product(m):
    c0 = float(G[f"expsum_{m}_c0"][0])
    nodes, w, sc, mesh = O.make_expsum(m, c0)
    assert np.array_equal(nodes, G[f"expsum_{m}_nodes"]) and np.array_equal(w, G[f"expsum_{m}_weights"])
    assert [sc, mesh] == list(G[f"expsum_{m}_scale_mesh"])
    es = tg.make_expsum(m, c0)
    assert np.array_equal(es.nodes, G[f"expsum_{m}_nodes"]) and np.array_equal(es.weights, G[f"expsum_{m}_weights"])


@pytest.mark.parametrize("doubled", [0, 1])
def test_kernel_tensor_bitwise_oracle_and_product(doubled):
    nodes, w, _, _ = O.make_expsum(8, 1.0)
    k = O.kernel_tensor(10.0, 33, nodes, w, bool(doubled))
    assert np.array_equal(k.factors()[0], G[f"kernel_{doubled}_f0"])
    kt = tg.kernel_tensor(tg.make_grid(10.0, 33), tg.make_expsum(8, 1.0), bool(doubled))
    assert np.array_equal(kt.tensor.factor[0], G[f"kernel_{doubled}_f0"])


@pytest.mark.parametrize("n", [65, 64])
def test_oracle_hartree_bitwise(n):
    th = O.OCP(*_cp(f"hartree_{n}_theta", f"hartree_{n}_theta_w"))
    k = O.OCP(*_cp(f"hartree_{n}_kernel", f"hartree_{n}_kernel_w"))
    v = O.hartree_potential(th, k, G[f"hartree_{n}_h"])
    for ax in range(3):
        assert np.array_equal(v.factors()[ax], G[f"hartree_{n}_vh_f{ax}"])
    assert np.array_equal(v.weight(), G[f"hartree_{n}_vh_w"])
    assert np.array_equal(O.value_at(v, G[f"hartree_{n}_pts"]), G[f"hartree_{n}_vals"])


def _lattice_spec():
    s = G["lattice_spec"]
    counts = tuple(int(x) for x in s[0:3])
    spacing, charge, n0 = float(s[3]), float(s[4]), int(s[5])
    nl = tuple(int(x) for x in s[6:9])
    bl = tuple(float(x) for x in s[9:12])
    m, c0 = int(s[12]), float(s[13])
    return counts, spacing, charge, nl, bl, m, c0


def test_oracle_and_product_lattice_offsets_bitwise():
    counts, spacing, charge, nl, bl, m, c0 = _lattice_spec()
    nodes, w, _, _ = O.make_expsum(m, c0)
    ref = O.kernel_tensor(bl, nl, nodes, w, True)
    total_ops = 0
    for ax in range(3):
        centers = [(k - 0.5 * (counts[ax] - 1)) * spacing for k in range(counts[ax])]
        out, ops = O.assemble_axis(bl, nl, ax, ref.factors()[ax], centers)
        total_ops += ops
        assert np.array_equal(out, G[f"lattice_f{ax}"])
    assert total_ops == int(G["lattice_ops"][0]) == sum(counts)  # window_ops == 3L analogue


def test_basis_bitwise_oracle_and_product():
    centers = G["basis_spec_centers"].reshape(-1, 3)
    degs = G["basis_spec_degs"].reshape(-1, 3)
    nprim, exps, coefs = G["basis_spec_nprim"], G["basis_spec_exps"], G["basis_spec_coefs"]
    fns, prod_fns, off = [], [], 0
    for i in range(3):
        prims = [(float(exps[off + p]), float(coefs[off + p])) for p in range(int(nprim[i]))]
        off += int(nprim[i])
        fns.append((tuple(centers[i]), tuple(int(d) for d in degs[i]), prims))
        prod_fns.append(tg.SeparableBasisFunction(tuple(centers[i]), tuple(int(d) for d in degs[i]),
                                                  [tg.GaussianPrimitive(e, c) for e, c in prims]))
    disc = O.discretize_basis([5.0, 5.5, 6.0], [21, 22, 23], fns)
    pdisc = tg.discretize_basis(tg.BasisSet(tg.make_grid([5.0, 5.5, 6.0], [21, 22, 23]), prod_fns))
    for i in range(3):
        for ax in range(3):
            assert np.array_equal(disc[i].factors()[ax], G[f"basis_{i}_f{ax}"])
            assert np.array_equal(pdisc[i].factor[ax], G[f"basis_{i}_f{ax}"])
        assert np.array_equal(disc[i].weight(), G[f"basis_{i}_w"])
        assert np.array_equal(pdisc[i].weight, G[f"basis_{i}_w"])


@pytest.mark.skipif(O.rlib() is None, reason="oracle/_ref (reference binary) not built here")
def test_restatement_vs_reference_binary_randomized():
    R = O.rlib()
    rng = Rng(4242)
    for rep in range(12):
        n = int(rng.integers(1, 700)[0]) + 1
        U = np.asfortranarray(rng.normal(2 * n).reshape(n, 2, order="F"))
        v = rng.normal(n)
        r = np.zeros((n, 2), order="F")
        assert R.ref_conv_central_many(C.c_longlong(n), C.c_longlong(2), C.c_void_p(U.ctypes.data),
                                       C.c_void_p(v.ctypes.data), C.c_void_p(r.ctypes.data), C.c_int(1)) == 0
        assert np.array_equal(O.conv_central_many(U, v), r)


# ------------------------------------------------------------------ device path vs reference outputs (GPU)

@pytest.mark.gpu
@pytest.mark.parametrize("n", [16, 17, 127, 128, 129, 256, 257, 1025])
@pytest.mark.parametrize("force_fft", [False, True])
def test_gpu_conv_central_many_vs_reference(ctx, n, force_fft):
    ctx.set_direct_max(0 if force_fft else 64)
    try:
        got = tg.conv_central_many(G[f"ccm_{n}_U"], G[f"ccm_{n}_v"], ctx)
    finally:
        ctx.set_direct_max(64)
    assert relmax(got, G[f"ccm_{n}_out"]) <= 1e-10


@pytest.mark.gpu
def test_gpu_convolve_scalar_product_vs_reference(ctx):
    a = tg.CanonicalTensor3(*_cp("cp_a", "cp_a_w"))
    b = tg.CanonicalTensor3(*_cp("cp_b", "cp_b_w"))
    c = tg.convolve(a, b, G["cp_h"], ctx)
    for ax in range(3):
        assert relmax(c.factor[ax], G[f"convolve_f{ax}"]) <= 1e-10
    assert np.array_equal(c.weight, G["convolve_w"])
    sp = tg.scalar_product(a, b, ctx)
    assert sp == pytest.approx(float(G["scalar_product"][0]), rel=1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [65, 64])
def test_gpu_hartree_vs_reference(ctx, n):
    th = tg.CanonicalTensor3(*_cp(f"hartree_{n}_theta", f"hartree_{n}_theta_w"))
    k = tg.CanonicalTensor3(*_cp(f"hartree_{n}_kernel", f"hartree_{n}_kernel_w"))
    for force_fft in (False, True):
        ctx.set_direct_max(0 if force_fft else 64)
        try:
            v = tg.hartree_potential(th, k, G[f"hartree_{n}_h"], ctx)
        finally:
            ctx.set_direct_max(64)
        for ax in range(3):
            assert relmax(v.factor[ax], G[f"hartree_{n}_vh_f{ax}"]) <= 1e-10
        assert np.array_equal(v.weight, G[f"hartree_{n}_vh_w"])
        assert relmax(tg.value_at_points(v, G[f"hartree_{n}_pts"], ctx), G[f"hartree_{n}_vals"]) <= 1e-10


@pytest.mark.gpu
def test_gpu_lattice_bitwise_vs_reference(ctx):
    counts, spacing, charge, nl, bl, m, c0 = _lattice_spec()
    grid = tg.make_grid(bl, nl)
    ref = tg.kernel_tensor(grid, tg.make_expsum(m, c0), True)
    spec = tg.LatticeSpec(counts=counts, spacing=spacing, charge=charge)
    ap = tg.lattice_sum_canonical(spec, grid, ref, ctx)
    for ax in range(3):
        assert np.array_equal(ap.canonical.factor[ax], G[f"lattice_f{ax}"])
    assert np.array_equal(ap.canonical.weight, G["lattice_w"])
    assert ap.window_ops == int(G["lattice_ops"][0])

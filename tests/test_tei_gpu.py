"""Parity of the device TEI pipeline (density fitting, convolution matrices,
diagonal, columns, pivoted Cholesky) with the oracle restatement of
proj/src/tei.cpp.  Ranks and pivot sequences must be identical; values are
compared through sign-invariant quantities (B entries, L L^T) at 1e-10
relative max-norm.  Semantics re-expressed from test_hf.cpp:319-492."""
import numpy as np
import pytest

from conftest import relmax
from oracle import oracle as O
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import Rng

pytestmark = pytest.mark.gpu
TOL = 1e-10


def make_basis(n, b, centres, shells, rng, contracted=False):
    fns = []
    for c in centres:
        for sh in shells:
            alpha = float(rng.loguniform(1, 0.3, 4.0)[0])
            prims = [tg.GaussianPrimitive(alpha, 1.0)]
            if contracted:
                prims = [tg.GaussianPrimitive(alpha, 0.7), tg.GaussianPrimitive(2.5 * alpha, 0.3)]
            degs = [(0, 0, 0)] if sh == "s" else [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
            for d in degs:
                fns.append(tg.SeparableBasisFunction(tuple(c), d, prims))
    grid = tg.make_grid(b, n)
    return tg.BasisSet(grid, fns)


def oracle_tei(bs, kernel, eps_fit, eps_chol):
    fns = [(f.center, f.degree, [(p.exponent, p.coeff) for p in f.primitives]) for f in bs.functions]
    disc = O.discretize_basis(bs.grid.b_half, bs.grid.n, fns)
    import ctypes as C

    h = O.olib().orc_tei_new()
    b = np.ascontiguousarray(bs.grid.b_half, dtype=np.float64)
    nn = (C.c_longlong * 3)(*bs.grid.n)
    hs = (C.c_void_p * len(disc))(*[d.h.value for d in disc])
    O._chk(O.olib().orc_tei_fit(C.c_void_p(h), O._p(b), nn, C.c_int(len(disc)), hs, C.c_double(eps_fit)))
    ok = O.OCP.from_cp(kernel.tensor)
    O._chk(O.olib().orc_tei_conv(C.c_void_p(h), ok.h))
    return h, disc


def oracle_info(h):
    import ctypes as C

    info = (C.c_longlong * 7)()
    res = np.zeros(3)
    O.olib().orc_tei_info(C.c_void_p(h), info, O._p(res))
    return list(info), res


def run_case(ctx, bs, kernel, eps_fit=1e-6, eps_chol=1e-6, check_chol=True):
    import ctypes as C

    disc = tg.discretize_basis(bs)
    fac = tg.TEIFactorization(ctx)
    tg.tei_density_fitting(fac, bs, disc, eps_fit)
    tg.tei_convolution_matrices(fac, kernel)
    oh, odisc = oracle_tei(bs, kernel, eps_fit, eps_chol)
    info, ores = oracle_info(oh)
    assert fac.fit_ranks() == tuple(info[:3])
    assert np.allclose(fac.fit_residual, ores, rtol=1e-3, atol=1e-12)  # diagnostic only
    nb = fac.n_b
    # diagonal and a few columns (B is sign-invariant in U)
    d = tg.tei_diagonal(fac)
    od = np.zeros(nb * nb)
    O._chk(O.olib().orc_tei_diagonal(C.c_void_p(oh), O._p(od)))
    assert relmax(d, od) <= TOL
    for pair in sorted({0, nb * nb - 1, (nb * nb) // 3, int(np.argmax(od))}):
        col = tg.tei_column(fac, pair)
        oc = np.zeros(nb * nb)
        O._chk(O.olib().orc_tei_column(C.c_void_p(oh), C.c_longlong(pair), O._p(oc)))
        assert relmax(col, oc) <= TOL
    # 8-fold symmetry of (mu nu | ka la) (test_hf.cpp:398-462)
    B = np.stack([tg.tei_column(fac, j) for j in range(nb * nb)], axis=1)
    assert np.abs(B - B.T).max() <= 1e-10 * np.abs(B).max()
    if check_chol:
        tg.tei_cholesky(fac, eps_chol)
        O._chk(O.olib().orc_tei_cholesky(C.c_void_p(oh), C.c_double(eps_chol)))
        info, _ = oracle_info(oh)
        rb = fac.rank_b()
        assert rb == info[5]
        L = fac.chol
        oL = np.zeros((nb * nb, rb), order="F")
        opiv = np.zeros(max(rb, 1), dtype=np.int64)
        O.olib().orc_tei_get_chol(C.c_void_p(oh), O._p(oL), O._p(opiv))
        # the pivot sequence is identical, including which of the (mu,nu) / (nu,mu) pair
        # (equal in exact arithmetic) each step takes
        assert list(fac.pivots) == [int(p) for p in opiv[:rb]]
        assert relmax(L @ L.T, oL @ oL.T) <= TOL
        assert np.abs(L @ L.T - B).max() <= 1e-6 * np.abs(B).max() * 10
    O.olib().orc_tei_free(C.c_void_p(oh))
    return fac


def test_tei_h2_toy(ctx):
    rng = Rng(11)
    bs = make_basis(65, 6.0, [(-0.7, 0.0, 0.0), (0.7, 0.0, 0.0)], ("s",), rng)
    kern = tg.kernel_tensor(bs.grid, tg.make_expsum(12, 0.9), False)
    run_case(ctx, bs, kern)


def test_tei_sp_basis(ctx):
    rng = Rng(12)
    cents = rng.uniform(6, -1.5, 1.5).reshape(2, 3)
    bs = make_basis(65, 7.0, cents, ("s", "p"), rng)
    kern = tg.kernel_tensor(bs.grid, tg.make_expsum(10, 0.9), False)
    run_case(ctx, bs, kern)


def test_tei_contracted_basis(ctx):
    rng = Rng(13)
    cents = rng.uniform(6, -1.0, 1.0).reshape(2, 3)
    bs = make_basis(48, 6.0, cents, ("s",), rng, contracted=True)
    kern = tg.kernel_tensor(bs.grid, tg.make_expsum(8, 0.9), False)
    run_case(ctx, bs, kern)


def test_tei_duplicates_do_not_raise_rank(ctx):
    # test_hf.cpp:319-361: identical functions -> fit ranks unchanged
    rng = Rng(14)
    bs1 = make_basis(33, 5.0, [(0.1, 0.2, -0.3)], ("s",), Rng(14))
    bs2 = make_basis(33, 5.0, [(0.1, 0.2, -0.3), (0.1, 0.2, -0.3)], ("s",), Rng(14))
    bs2.functions[1] = bs2.functions[0]
    f1 = tg.TEIFactorization(ctx)
    tg.tei_density_fitting(f1, bs1, tg.discretize_basis(bs1), 1e-6)
    f2 = tg.TEIFactorization(ctx)
    tg.tei_density_fitting(f2, bs2, tg.discretize_basis(bs2), 1e-6)
    assert f1.fit_ranks() == (1, 1, 1) == f2.fit_ranks()
    assert max(f2.fit_residual) <= 1e-6


@pytest.mark.parametrize("contracted", [False, True])
def test_tei_cholesky_cooperative_matches_graph_loop(ctx, monkeypatch, contracted):
    # the one-grid Cholesky and the graph-replayed 4-kernel step share their arithmetic:
    # identical pivots, rank and L
    rng = Rng(15)
    cents = rng.uniform(6, -1.2, 1.2).reshape(2, 3)
    bs = make_basis(48, 6.0, cents, ("s", "p") if not contracted else ("s",), rng, contracted=contracted)
    kern = tg.kernel_tensor(bs.grid, tg.make_expsum(8, 0.9), False)
    disc = tg.discretize_basis(bs)
    out = []
    for graph in (False, True):
        if graph:
            monkeypatch.setenv("TGB_TEI_GRAPH", "1")
        fac = tg.TEIFactorization(ctx)
        tg.tei_density_fitting(fac, bs, disc, 1e-6)
        tg.tei_convolution_matrices(fac, kern)
        tg.tei_cholesky(fac, 1e-8)
        out.append((fac.rank_b(), list(fac.pivots), np.array(fac.chol)))
    assert out[0][0] == out[1][0] > 1
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][2], out[1][2])


def test_tei_many_kernel_terms(ctx):
    # K = 2M+1 = 51 > 48 kernel columns: the column falls back to the SIMT kernel inside the
    # graph-replayed step (the DMMA tile and the cooperative grid cover K <= 48)
    rng = Rng(16)
    cents = rng.uniform(6, -1.0, 1.0).reshape(2, 3)
    bs = make_basis(48, 6.0, cents, ("s",), rng)
    kern = tg.kernel_tensor(bs.grid, tg.make_expsum(25, 0.9), False)
    assert kern.rank() == 51
    run_case(ctx, bs, kern)

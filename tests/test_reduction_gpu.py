"""Parity of the device rank reduction (RHOSVD, canonical_to_tucker ALS,
tucker_to_canonical, reduce_rank) with the oracle restatement of
proj/src/reduction.cpp.  Tucker ranks must be identical; tensors are compared
through their dense images (sides carry sign/rotation freedom).  Semantics
re-expressed from test_reduction.cpp:82-205 and test_hf.cpp:201-244."""
import numpy as np
import pytest

from conftest import relmax
from oracle import oracle as O
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import Rng, gaussian_density

pytestmark = pytest.mark.gpu


def tucker_structured(rng, dims, ranks, R):
    """Canonical tensor of rank R whose exact Tucker ranks are `ranks`."""
    bases = []
    for d, r in zip(dims, ranks):
        q, _ = np.linalg.qr(rng.normal(d * r).reshape(d, r))
        bases.append(q)
    facs = [np.asfortranarray(b @ rng.normal(b.shape[1] * R).reshape(b.shape[1], R)) for b in bases]
    return tg.CanonicalTensor3(facs, rng.uniform(R, 0.5, 1.5))


def oracle_dense(cp):
    return np.einsum("k,ik,jk,lk->ijl", cp.weight(), *cp.factors())


def test_rhosvd_exact_recovery(ctx):
    rng = Rng(21)
    a = tucker_structured(rng, (20, 17, 23), (3, 4, 2), 12)
    res = tg.rhosvd(a, tg.ReductionConfig.tolerance(1e-10), ctx)
    assert res.tucker.ranks() == (3, 4, 2)
    assert relmax(res.tucker.to_dense(), a.to_dense()) <= 1e-12
    o = O.reduce(O.OCP.from_cp(a), eps=1e-10, mode=0)
    assert o["ranks"] == (3, 4, 2)


def test_fixed_ranks_and_clamping(ctx):
    rng = Rng(22)
    a = tucker_structured(rng, (16, 16, 16), (2, 3, 2), 9)
    res = tg.rhosvd(a, tg.ReductionConfig.fixed(2, 5, 1), ctx)
    assert res.tucker.ranks() == (2, 3, 1)
    assert res.rank_clamped
    o = O.reduce(O.OCP.from_cp(a), ranks=(2, 5, 1), mode=0)
    assert o["ranks"] == (2, 3, 1) and o["rank_clamped"]


@pytest.mark.parametrize("n,R,eps", [(33, 40, 1e-6), (65, 150, 1e-7), (48, 60, 1e-5)])
def test_reduce_rank_gaussian_density_matches_oracle(ctx, n, R, eps):
    rng = Rng(23 + n)
    grid = tg.make_grid(6.0, n)
    theta, *_ = gaussian_density(grid, rng, R, 0.3, 8.0, box=1.5)
    red = tg.reduce_rank(theta, tg.ReductionConfig.tolerance(eps), ctx)
    o = O.reduce(O.OCP.from_cp(theta), eps=eps, mode=2)
    res = tg.canonical_to_tucker(theta, tg.ReductionConfig.tolerance(eps), ctx)
    assert res.tucker.ranks() == o["ranks"]
    dense = red.to_dense()
    ref = oracle_dense(o["canonical"])
    # both approximate the same tensor to eps; the reference's Gram branches have an
    # accuracy floor ~sqrt(machine eps) (reduction.cpp:91-92), so the two truncations
    # agree to well below eps but not to 1e-10
    assert relmax(dense, ref) <= 0.5 * eps
    assert relmax(dense, theta.to_dense()) <= 10 * eps
    # T2C rank = product of the two smaller Tucker ranks (reduction.cpp:242-248)
    r = sorted(res.tucker.ranks())
    assert red.rank() == r[0] * r[1]


def test_sweep_fits_monotone(ctx):
    rng = Rng(24)
    grid = tg.make_grid(5.0, 40)
    theta, *_ = gaussian_density(grid, rng, 30, 0.5, 6.0, box=1.0)
    res = tg.canonical_to_tucker(theta, tg.ReductionConfig.fixed(4, 4, 4), ctx)
    f = res.sweep_fits
    assert len(f) >= 1
    assert all(b >= a - 1e-12 * abs(a) for a, b in zip(f, f[1:]))


def test_zero_rank_input(ctx):
    z = tg.CanonicalTensor3.zero((9, 8, 7))
    red = tg.reduce_rank(z, tg.ReductionConfig.tolerance(1e-6), ctx)
    assert red.rank() == 0


def test_wide_gram_branch(ctx):
    # cols >= 4 rows and cols > 8192 (reduction.cpp:93): RHOSVD of a rank-9000 tensor on n = 33
    rng = Rng(25)
    grid = tg.make_grid(4.0, 33)
    theta, *_ = gaussian_density(grid, rng, 9000, 0.5, 4.0, box=1.0)
    res = tg.rhosvd(theta, tg.ReductionConfig.tolerance(1e-6), ctx)
    o = O.reduce(O.OCP.from_cp(theta), eps=1e-6, mode=0)
    assert res.tucker.ranks() == o["ranks"]
    assert relmax(res.tucker.to_dense(), np.einsum("abc,ia,jb,kc->ijk", o["core"], *o["sides"])) <= 1e-9


def test_mode_rank_beyond_shared_memory_jacobi(ctx):
    # a mode rank of 140: the subspace block grows past 128 columns, so its
    # Rayleigh-Ritz SVD runs on the global-memory one-sided Jacobi
    rng = Rng(26)
    a = tucker_structured(rng, (160, 30, 30), (140, 6, 5), 200)
    res = tg.rhosvd(a, tg.ReductionConfig.tolerance(1e-10), ctx)
    assert res.tucker.ranks() == (140, 6, 5)
    assert relmax(res.tucker.to_dense(), a.to_dense()) <= 1e-11
    o = O.reduce(O.OCP.from_cp(a), eps=1e-10, mode=0)
    assert o["ranks"] == (140, 6, 5)
    # the ALS refines mode 0 within the 6 x 5 core unfolding: rank 30 (RHOSVD initial guess: 140)
    c2t = tg.canonical_to_tucker(a, tg.ReductionConfig.tolerance(1e-10), ctx)
    o1 = O.reduce(O.OCP.from_cp(a), eps=1e-10, mode=1)
    assert c2t.tucker.ranks() == o1["ranks"] == (30, 6, 5)
    assert relmax(c2t.tucker.to_dense(), a.to_dense()) <= 1e-10


@pytest.mark.timeout(300)
def test_rank_beyond_subspace_block_fails_not_hangs(ctx):
    """a fixed rank above the subspace-iteration block (1020 columns)
    with min(n, R) > 1024 must raise NumericalError, not loop."""
    rng = Rng(31)
    n, R = 1100, 1100
    f = [np.asfortranarray(rng.normal(n * R).reshape(n, R, order="F")) for _ in range(3)]
    a = tg.CanonicalTensor3(f, np.ones(R))
    with pytest.raises(tg.NumericalError):
        tg.canonical_to_tucker(a, tg.ReductionConfig.fixed(1030, 4, 4), ctx)

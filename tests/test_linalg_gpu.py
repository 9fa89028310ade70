"""thin_svd_left (reduction.cpp:85-138) and pivoted_cholesky (tei.cpp:48-90) behind the C ABI,
against the restatement (oracle) and the reference's own test properties
(test_reduction.cpp, test_hf.cpp:464-492): shapes per branch, singular values, the
sign-invariant projector U diag(s^2) U^T, and for the Cholesky identical pivots / ranks,
L L^T, the clamp flag and the not-PSD error."""
import numpy as np
import pytest

import paper_1504_06289_b200 as tg
from conftest import relmax
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _mat(rng, r, c, decay=None):
    a = rng.normal(size=(r, c))
    if decay is not None:  # graded spectrum
        u, _, vt = np.linalg.svd(a, full_matrices=False)
        s = decay ** np.arange(min(r, c))
        a = (u * s) @ vt
    return np.asfortranarray(a)


@pytest.mark.parametrize("r,c,decay", [(300, 40, None), (30, 500, None), (400, 20, 0.5), (20, 9000, None),
                                       (64, 64, 0.7), (7, 3, None), (3, 7, None),
                                       (300, 200, None), (150, 600, 0.9)])  # beyond the shared-memory solver
def test_thin_svd_left_vs_restatement(ctx, r, c, decay):
    rng = np.random.default_rng(r * 1000 + c)
    a = _mat(rng, r, c, decay)
    u, s = tg.thin_svd_left(a, ctx)
    ou, os_ = O.thin_svd_left(a)
    assert u.shape == ou.shape and s.shape == os_.shape  # the reference's per-branch output shape
    assert np.all(np.diff(s) <= 0)
    # Gram branches of the reference resolve singular values to ~sqrt(eps) sigma_0
    assert np.abs(s - os_).max() <= 1e-10 * s[0] + (1e-7 * s[0] if (c >= 4 * r and c > 8192) else 0.0)
    k = u.shape[1]
    full = min(r, c)
    if k == full:  # orthonormal columns and the projector of A A^T
        assert np.abs(u.T @ u - np.eye(k)).max() <= 1e-10
        assert relmax((u * s ** 2) @ u.T, a @ a.T) <= 1e-10


def test_thin_svd_left_edge(ctx):
    u, s = tg.thin_svd_left(np.zeros((5, 0)), ctx)
    assert u.shape == (5, 0) and s.shape == (0,)
    # rank-one input: one nonzero singular value, the rest exactly resolved to ~0
    u, s = tg.thin_svd_left(np.ones((300, 200)), ctx)
    assert u.shape == (300, 200) and abs(s[0] - np.sqrt(300 * 200)) <= 1e-10 * s[0] and s[1] <= 1e-10 * s[0]


@pytest.mark.parametrize("stop", ["max_diagonal", "trace"])
def test_pivoted_cholesky_vs_restatement(ctx, stop):
    rng = np.random.default_rng(11)
    g = rng.normal(size=(90, 30))
    a = np.asfortranarray(g @ g.T)  # rank 30
    res = tg.pivoted_cholesky(a, 1e-12, stop, ctx=ctx)
    oL, opiv, ores, ocl = O.pivoted_cholesky(a, 1e-12, stop == "trace", 90, 1e-12)
    assert list(res.pivots) == list(opiv) and res.factor.shape == oL.shape
    assert relmax(res.factor @ res.factor.T, oL @ oL.T) <= 1e-10
    assert res.clamped_negative == ocl
    assert abs(res.residual - ores) <= 1e-10
    # max_rank cap and the trivial zero matrix
    capped = tg.pivoted_cholesky(a, 1e-12, stop, max_rank=5, ctx=ctx)
    assert capped.factor.shape == (90, 5) and list(capped.pivots) == list(opiv[:5])
    z = tg.pivoted_cholesky(np.zeros((4, 4)), 1e-8, stop, ctx=ctx)
    assert z.factor.shape == (4, 0) and z.residual == 0.0


def test_pivoted_cholesky_not_psd(ctx):
    a = np.diag([4.0, 1.0, -3.0])
    a[0, 2] = a[2, 0] = 1.9
    with pytest.raises(tg.NumericalError):
        tg.pivoted_cholesky(a, 1e-14, "max_diagonal", ctx=ctx)

"""CPU self-checks of the oracle restatement (tests/ only): the reference's
own known-answer and property tests for the path, re-expressed, plus
independent numpy definitions.  Pins against the reference binary itself
(oracle/_ref) and the committed golden fixtures live in test_golden.py."""
import numpy as np
import pytest

from conftest import relmax
from oracle import oracle as O
from paper_1504_06289_b200.inputs import Rng


def window_np(u, v):
    n = len(u)
    full = np.convolve(u, v)
    if n % 2:
        o = (n - 1) // 2
        return full[o:o + n]
    o = n // 2 - 1
    return 0.5 * (full[o:o + n] + full[o + 1:o + 1 + n])


@pytest.mark.parametrize("n", [5, 31, 128, 200, 513])
def test_direct_and_fft_agree(n):
    # test_tensor.cpp:24-37
    rng = Rng(1)
    u, v = rng.normal(n), rng.normal(n)
    a = O.conv_full(u, v, False)
    b = O.conv_full(u, v, True)
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()
    assert relmax(a, np.convolve(u, v)) <= 1e-13


@pytest.mark.parametrize("n", [1, 2, 16, 17, 127, 128, 129, 1025])
def test_central_window_vs_numpy(n):
    rng = Rng(n)
    U = np.asfortranarray(rng.normal(3 * n).reshape(n, 3, order="F"))
    v = rng.normal(n)
    got = O.conv_central_many(U, v)
    ref = np.stack([window_np(U[:, c], v) for c in range(3)], 1)
    assert relmax(got, ref) <= 1e-12


def test_convolve_rank_and_zero_rank():
    rng = Rng(3)
    dims = (6, 5, 7)
    a = O.OCP([rng.normal(d * 2).reshape(d, 2) for d in dims], rng.normal(2))
    z = O.OCP([np.zeros((d, 0)) for d in dims], np.zeros(0))
    c = O.convolve(a, z, 0.5)
    assert c.rank() == 0
    c = O.convolve(a, a, 0.5)
    assert c.rank() == 4
    with pytest.raises(O.OracleError):
        O.convolve(a, a, 0.0)


def test_sym_eigen_vs_numpy():
    rng = Rng(4)
    for n in (1, 2, 7, 40):
        g = rng.normal(n * n).reshape(n, n)
        a = g + g.T
        ev, z = O.sym_eigen(a)
        ref = np.linalg.eigvalsh(a)
        assert np.abs(ev - ref).max() <= 1e-12 * max(1, np.abs(ref).max())
        assert np.abs(z.T @ z - np.eye(n)).max() <= 1e-12
        assert np.abs(a @ z - z * ev).max() <= 1e-11 * max(1, np.abs(ref).max())


def test_householder_and_jacobi_vs_numpy():
    rng = Rng(5)
    a = rng.normal(30 * 6).reshape(30, 6)
    q, r = O.householder_qr(a)
    assert np.abs(q @ r - a).max() <= 1e-13 * np.abs(a).max()
    assert np.abs(q.T @ q - np.eye(6)).max() <= 1e-14
    for shape in ((30, 6), (6, 30), (9, 9)):
        a = rng.normal(shape[0] * shape[1]).reshape(shape)
        u, s = O.jacobi_svd(a)
        ref = np.linalg.svd(a, compute_uv=False)
        assert np.abs(s - ref).max() <= 1e-13 * ref.max()
        assert np.abs(u.T @ u - np.eye(u.shape[1])).max() <= 1e-13


def test_pivoted_cholesky_first_max_pivot():
    rng = Rng(6)
    g = rng.normal(12 * 5).reshape(12, 5)
    a = g @ g.T
    L, piv, res, cl = O.pivoted_cholesky(a, 1e-14, False, 12, 1e-10)
    assert L.shape[1] == 5
    assert piv[0] == int(np.argmax(np.diag(a)))
    assert np.abs(L @ L.T - a).max() <= 1e-10 * np.abs(a).max()
    # ties: the first maximal index is taken
    t = np.eye(4) * 2.0
    L, piv, res, cl = O.pivoted_cholesky(t, 1e-14, False, 4, 1e-10)
    assert list(piv) == [0, 1, 2, 3]

"""TuckerResult::mode_singular_values (proj/include/tengrid/reduction.hpp:42),
which rhosvd fills from thin_svd_left of each normalized mode matrix
(reduction.cpp:172-190, 85-138): the device full spectra (csrc/spectrum.cu)
against the reference's own rhosvd (oracle/_ref) on every thin_svd_left branch,
and against numpy's LAPACK SVD at a size that spreads the tridiagonalisation
over many CTAs.  Values come from the Gram spectrum, so the bound is on
sigma^2: |sigma^2 - sigma_ref^2| <= 1e-12 sigma_0^2 (the reference's Gram
branches carry the same floor)."""
import numpy as np
import pytest

from oracle import oracle as O
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import Rng, random_canonical

pytestmark = pytest.mark.gpu
TOL_SQ = 1e-12


def _close_sq(got, ref):
    return np.abs(got ** 2 - ref ** 2).max() <= TOL_SQ * ref[0] ** 2


def _normalized_mode(t, axis):
    """W = f_axis diag(w) after normalize (tensor.cpp:18-31), in numpy."""
    w = t.weight.copy()
    fs = [f.copy() for f in t.factor]
    for ax in range(3):
        nrm = np.linalg.norm(fs[ax], axis=0)
        ok = nrm > 0
        fs[ax][:, ok] /= nrm[ok]
        w = np.where(ok, w * nrm, 0.0)
    return fs[axis] * w


@pytest.mark.parametrize("dims,R,branch", [
    ((65, 40, 33), 30, "jacobi (n < 4R)"),
    ((16, 16, 16), 5, "jacobi (R < 8)"),
    ((257, 130, 33), 20, "tall Gram (n >= 4R): lambda > lambda_max 1e-24 kept"),
    ((33, 17, 9), 9000, "wide Gram (R >= 4n, R > 8192)"),
])
def test_mode_spectrum_vs_reference(ctx, dims, R, branch):
    if O.rlib() is None:
        pytest.skip("oracle/_ref not built")
    t = random_canonical(Rng(77000 + R), dims, R)
    rt = O.OCP.from_cp(t, lib=O.rlib())
    for ax in range(3):
        ref = O.ref_mode_sigma(rt, ax)
        got = tg.mode_spectrum(t, ax, ctx)
        assert len(got) == len(ref), (branch, ax)
        assert np.all(np.diff(got) <= 0)
        assert _close_sq(got, ref), (branch, ax)


def test_mode_spectrum_large_vs_lapack(ctx):
    # m = 1500: the cooperative tridiagonalisation spans many CTAs
    t = random_canonical(Rng(77123), (1500, 9, 7), 4000)
    got = tg.mode_spectrum(t, 0, ctx)
    ref = np.linalg.svd(_normalized_mode(t, 0), compute_uv=False)
    assert len(got) == 1500
    assert _close_sq(got, ref)
    # device-resident input gives the same spectrum bit for bit
    dgot = tg.mode_spectrum(tg.DeviceCP.from_host(t), 0, ctx)
    assert np.array_equal(dgot, got)


def test_mode_spectrum_rank_deficient(ctx):
    # duplicated columns: a rank-deficient mode matrix; the trailing values sit at the Gram floor
    rng = Rng(77321)
    base = random_canonical(rng, (80, 60, 50), 12)
    t = tg.CanonicalTensor3([np.asfortranarray(np.hstack([f, f])) for f in base.factor],
                            np.concatenate([base.weight, 0.5 * base.weight]))
    ref = np.linalg.svd(_normalized_mode(t, 0), compute_uv=False)
    got = tg.mode_spectrum(t, 0, ctx)
    assert len(got) == 24
    assert _close_sq(got, ref)
    assert got[12:].max() <= 1e-7 * got[0]


def test_tucker_full_spectra(ctx):
    rng = Rng(77555)
    t = random_canonical(rng, (70, 50, 40), 18)
    base = tg.canonical_to_tucker(t, tg.ReductionConfig.tolerance(1e-6), ctx)
    full = tg.canonical_to_tucker(t, tg.ReductionConfig(epsilon=1e-6, full_spectra=True), ctx)
    assert full.tucker.ranks() == base.tucker.ranks()
    for ax in range(3):
        assert np.array_equal(full.tucker.side[ax], base.tucker.side[ax])
        assert np.array_equal(full.mode_singular_values[ax], tg.mode_spectrum(t, ax, ctx))
        assert len(full.mode_singular_values[ax]) == min(t.extents()[ax], t.rank())
    if O.rlib() is not None:
        rt = O.OCP.from_cp(t, lib=O.rlib())
        for ax in range(3):
            ref = O.ref_mode_sigma(rt, ax, mode=1)
            assert len(ref) == len(full.mode_singular_values[ax])
            assert _close_sq(full.mode_singular_values[ax], ref)


def test_config1_full_spectra(ctx):
    # BASELINE config 1's unreduced density (n = 2049, rank 12,800): the wide Gram branch, m = 2049,
    # against the reference's own rhosvd spectra (tools/make_golden_spectra.py)
    from pathlib import Path

    from paper_1504_06289_b200.inputs import basis_case, occupied_coefficients

    p = Path(__file__).resolve().parent / "golden" / "reference_cfg1_spectra.npz"
    if not p.exists():
        pytest.skip("reference_cfg1_spectra.npz not generated")
    g = np.load(p)
    bs, rng = basis_case(1)
    disc = tg.discretize_basis(bs)
    c_occ = occupied_coefficients(rng, len(disc), 8)
    theta = tg.CanonicalTensor3.zero(disc[0].extents())
    for a in range(8):
        phi = tg.orbital_tensor(disc, c_occ[:, a])
        theta = tg.add(theta, tg.scale(tg.hadamard(phi, phi), 2.0))
    assert theta.rank() == int(g["rank"])
    dt = tg.DeviceCP.from_host(theta)
    for ax in range(3):
        ref = g[f"sigma{ax}"]
        got = tg.mode_spectrum(dt, ax, ctx)
        assert len(got) == len(ref)
        assert _close_sq(got, ref)

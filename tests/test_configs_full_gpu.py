"""BASELINE.json configs 1, 3 and 4 at their FULL sizes against fixtures the
reference's own code computed (tools/make_golden_configs.py on oracle/_ref).

* config 4 (lattice_sum_canonical, L=32, n=32769): every factor matrix
  bit-identical (SHA-256), window_ops = 3L, value_at at 10^5 points <= 1e-13.
* config 3 (build_tei, N_b=80, n=4097, eps 1e-6): fit ranks and R_B identical;
  L L^T at 4096 probes within 1e-10; the pivot sequence identical up to the
  first near-tie (a step whose argmax margin is below 1e-9 relative); the TEI
  diagonal and four B columns within 1e-8.  That bound is set by the
  reference's OWN reproducibility at this size: moving every primitive
  exponent by one ulp changes its diagonal by 1.3e-9 and its pivot sequence
  (profiles/r02_tei_reference_sensitivity.json, tools/tei_sensitivity.py) —
  the fit basis is the QR of a pivoted Cholesky factor stopped at a 1e-12
  trace residual, conditioned ~1e6.
* config 1 (density_tensor -> V_H -> J, n=2049, N_b=40): Tucker and canonical
  ranks identical; V_H at 10^4 seeded points and J within 1e-10 (measured
  3.4e-13 and 2.9e-13).  The reduced factors themselves are not compared: the
  reference's Gram branch and the device subspace iteration pick different
  bases of the same truncated subspaces, and the reduced TENSOR
  is what V_H and J see."""
import hashlib
from pathlib import Path

import numpy as np
import pytest

from conftest import relmax
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import (KERNEL_C0, KERNEL_M, Rng, basis_case, lattice_case,
                                          occupied_coefficients)

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
TOL3 = 1e-8  # the reference's own 1-ulp sensitivity is 1.3e-9 (see above)


def _sha(a):
    return hashlib.sha256(np.asfortranarray(a, dtype=np.float64).tobytes(order="F")).hexdigest()


def _load(name):
    p = GOLD / name
    if not p.exists():
        pytest.skip(f"{name} not generated")
    return np.load(p)


def test_config4_lattice_full(ctx):
    g = _load("reference_cfg4.npz")
    spec, grid, ref = lattice_case()
    ap = tg.lattice_sum_canonical(spec, grid, ref, ctx)
    assert ap.window_ops == int(g["window_ops"]) == 3 * 32
    for ax in range(3):
        assert _sha(ap.canonical.factor[ax]) == str(g["factor_sha"][ax]), f"axis {ax} factors differ"
    assert np.array_equal(ap.canonical.weight, g["weight"])
    pts = Rng(1504062894).integers(3 * 100_000, grid.n[0]).reshape(-1, 3)
    assert hashlib.sha256(pts.tobytes()).hexdigest() == str(g["points_sha"])
    vals = tg.value_at_points(tg.DeviceCP.from_host(ap.canonical), pts, ctx).cpu().numpy()
    assert relmax(vals, g["values"]) <= 1e-13


def test_config3_tei_full(ctx):
    g = _load("reference_cfg3.npz")
    bs, _ = basis_case(3)
    disc = tg.discretize_basis(bs)
    kern = tg.kernel_tensor(bs.grid, tg.make_expsum(KERNEL_M[3], KERNEL_C0[3]), False)
    fac = tg.TEIFactorization(ctx)
    tg.tei_density_fitting(fac, bs, disc, 1e-6)
    assert fac.fit_ranks() == tuple(int(x) for x in g["fit_ranks"])
    tg.tei_convolution_matrices(fac, kern)
    d = tg.tei_diagonal(fac)
    e_diag = relmax(d, g["diagonal"])
    e_cols = max(relmax(tg.tei_column(fac, int(j)), g["B"][:, c]) for c, j in enumerate(g["b_cols"]))
    tg.tei_cholesky(fac, 1e-6)
    from paper_1504_06289_b200.tei import pivot_margins

    L = np.asarray(fac.chol)
    pr = g["probes"]
    same_rb = fac.rank_b() == int(g["rank_b"])
    piv = list(fac.pivots)
    first_diff = next((i for i, (a, b) in enumerate(zip(piv, g["pivots"])) if a != b), None)
    e_llt = (np.abs(np.einsum("ij,ij->i", L[pr[:, 0]], L[pr[:, 1]]) - g["llt"]).max() / np.abs(g["diagonal"]).max()
             if same_rb else None)
    mg = pivot_margins(fac, d, 1e-6)
    gaps = mg.pop("gaps")
    k0 = next((i for i, x in enumerate(gaps) if x < 1e-9), len(gaps))  # first near-tie
    print(f"config 3: diag {e_diag:.3e} B cols {e_cols:.3e} LLt {e_llt} R_B {fac.rank_b()}/{int(g['rank_b'])} "
          f"first pivot difference at {first_diff}, first near-tie at {k0}; margins {mg}")
    assert same_rb and len(piv) == len(g["pivots"])
    assert first_diff is None or first_diff >= k0
    assert e_llt <= 1e-10
    assert e_diag <= TOL3 and e_cols <= TOL3


def test_config1_density_vh_j_full(ctx):
    g = _load("reference_cfg1.npz")
    bs, rng = basis_case(1)
    disc = tg.discretize_basis(bs)
    c_occ = occupied_coefficients(rng, len(disc), 8)
    assert np.array_equal(c_occ, g["c_occ"])
    theta = tg.CanonicalTensor3.zero(disc[0].extents())
    for a in range(8):
        phi = tg.orbital_tensor(disc, c_occ[:, a])
        theta = tg.add(theta, tg.scale(tg.hadamard(phi, phi), 2.0))
    assert theta.rank() == int(g["unreduced_rank"])
    res = tg.canonical_to_tucker(theta, tg.ReductionConfig.tolerance(1e-6), ctx)
    print("config 1 rank margins:", res.rank_margins)
    assert list(res.tucker.ranks()) == [int(x) for x in g["tucker_ranks"]]
    red = tg.density_tensor(disc, c_occ, 1e-6, ctx)
    assert red.rank() == int(g["canonical_rank"])
    kern = tg.kernel_tensor(bs.grid, tg.make_expsum(KERNEL_M[1], KERNEL_C0[1]), False)
    dt, dk = tg.DeviceCP.from_host(red), tg.DeviceCP.from_host(kern.tensor)
    vh = tg.hartree_potential(dt, dk, bs.grid.h, ctx)
    vals = tg.value_at_points(vh, g["points"], ctx).cpu().numpy()
    ev = relmax(vals, g["vh"])
    J = tg.coulomb_matrix(bs, disc, vh, ctx)
    ej = relmax(J, g["J"])
    print(f"config 1: V_H samples rel err {ev:.3e}, J rel err {ej:.3e}")
    assert ev <= 1e-10 and ej <= 1e-10
    assert np.array_equal(J, J.T)

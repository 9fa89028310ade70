"""The device SCF (tgb_scf_solve, hf.cpp:201-270) and generalized eigensolver
(hf.cpp:187-199) against the reference's OWN scf_solve run from oracle/_ref
(tests/golden/reference_scf.npz, tools/make_golden_scf.py).  Energies and
orbital energies at 1e-10 relative, the density (sign-invariant) at 1e-8
relative after convergence to energy_tol 1e-9, TEI rank and iteration count
identical."""
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1504_06289_b200 as tg
from conftest import relmax

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
from make_golden_scf import CASES  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-10
G = dict(np.load(Path(__file__).resolve().parent / "golden" / "reference_scf.npz"))


def case(name):
    c = CASES[name]
    grid = tg.make_grid(tuple(c["b"]), tuple(c["n"]))
    bs = tg.BasisSet(grid, [tg.SeparableBasisFunction(cen, d, [tg.GaussianPrimitive(e, k) for e, k in p])
                            for cen, d, p in c["fns"]])
    mol = tg.Molecule([tg.Nucleus(q, pos) for pos, q in c["nuclei"]], c["electrons"])
    cfg = G["cfg"]
    return bs, mol, tg.SCFConfig(max_iterations=int(cfg[0]), energy_tol=cfg[1], mixing=cfg[2], eps_fit=cfg[3],
                                 eps_chol=cfg[4], kernel_eps=cfg[5])


@pytest.mark.parametrize("name", list(CASES))
def test_scf_matches_reference(ctx, name):
    bs, mol, cfg = case(name)
    st = tg.scf_solve(mol, bs, cfg, ctx)
    assert st.converged == bool(G[f"{name}_converged"][0])
    assert st.iterations == int(G[f"{name}_iterations"][0])
    assert st.tei_rank_b == int(G[f"{name}_tei_rank_b"][0])
    assert abs(st.nuclear_energy - G[f"{name}_nuclear_energy"][0]) <= 1e-12 * max(1.0, abs(st.nuclear_energy))
    assert abs(st.energy - G[f"{name}_energy"][0]) <= 1e-10 * abs(G[f"{name}_energy"][0])
    assert relmax(st.energy_history, G[f"{name}_energy_history"]) <= 1e-10
    assert relmax(st.orbital_energies, G[f"{name}_orbital_energies"]) <= 1e-10
    assert relmax(st.density, G[f"{name}_density"]) <= 1e-8
    # S-orthonormal coefficients (hf.cpp:245-247)
    assert max(st.orthonormality_defects) <= 1e-10


@pytest.mark.parametrize("nb", [37, 150])  # shared-memory tiles / global workspace (nb > 112)
def test_generalized_eigensolve(ctx, nb):
    rng = np.random.default_rng(7)
    a = rng.normal(size=(nb, nb))
    s = a @ a.T / nb + np.eye(nb)
    f = rng.normal(size=(nb, nb))
    f = 0.5 * (f + f.T)
    c, e = tg.generalized_eigensolve(f, s, ctx)
    assert np.all(np.diff(e) >= 0)
    assert np.abs(c.T @ s @ c - np.eye(nb)).max() <= 1e-11
    assert np.abs(f @ c - s @ c @ np.diag(e)).max() <= 1e-10 * np.abs(f).max()
    import scipy.linalg

    assert relmax(e, scipy.linalg.eigh(f, s, eigvals_only=True)) <= 1e-11
    with pytest.raises(tg.NumericalError):
        tg.generalized_eigensolve(f, -s, ctx)  # hf.cpp:190-191


def test_scf_errors(ctx):
    bs, mol, cfg = case("h2")
    with pytest.raises(tg.InvalidArgument):
        tg.scf_solve(tg.Molecule([], 2), bs, cfg, ctx)
    with pytest.raises(tg.InvalidArgument):
        tg.scf_solve(tg.Molecule(mol.nuclei, 3), bs, cfg, ctx)  # odd electron count
    with pytest.raises(tg.InvalidArgument):
        tg.scf_solve(tg.Molecule(mol.nuclei, 12), bs, cfg, ctx)  # more occupied orbitals than functions


def test_mp2_matches_reference(ctx):
    """mo_transform_cholesky + mp2_energy (mp2.cpp) on the reference's own SCF of the 'chain' case."""
    nocc = int(G["mp2_nocc"][0])
    mos = tg.MOSpace(G["mp2_coef"], G["mp2_energies"], nocc)
    mo = tg.mo_transform_cholesky(G["mp2_chol"], mos, ctx)
    assert relmax(mo.factor, G["mp2_mo_factor"]) <= TOL
    e_or = tg.mp2_energy(mo, mos, "oracle", ctx=ctx)
    e_fa = tg.mp2_energy(mo, mos, "factorized", float(G["mp2_expsum_eps"][0]), ctx=ctx)
    assert abs(e_or - G["mp2_e2"][0]) <= TOL * abs(G["mp2_e2"][0])
    assert abs(e_fa - G["mp2_e2"][1]) <= TOL * abs(G["mp2_e2"][1])
    with pytest.raises(tg.NumericalError):  # reversed orbital energies: no positive gap (mp2.cpp:99-100)
        tg.mp2_energy(mo, tg.MOSpace(G["mp2_coef"], G["mp2_energies"][::-1].copy(), nocc), ctx=ctx)
    with pytest.raises(tg.InvalidArgument):
        tg.mp2_energy(mo, tg.MOSpace(G["mp2_coef"], G["mp2_energies"], nocc + 1), ctx=ctx)

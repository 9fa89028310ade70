"""Property tests of the device HF operators, SCF and MP2 re-expressed from the
reference's own suites (proj/tests/test_hf.cpp:70-200, 539-620;
proj/tests/test_mp2.cpp:104-175) against closed-form Gaussian integrals
(tests/analytic.py) — independent of the reference-binary fixtures."""
import numpy as np
import pytest

import paper_1504_06289_b200 as tg
from analytic import S, kinetic, nuclear, overlap, rhf_energy
from conftest import relmax

pytestmark = pytest.mark.gpu


def approx(a, b, eps):
    """doctest::Approx(b).epsilon(eps) == a: |a - b| < eps (1 + max(|a|, |b|)) (scale 1)."""
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


def snapped_z(g, z):
    return float(g.coord(2, tg.snap_to_node(g, 2, z)))


def s_basis(g, specs):
    """specs: (centre, [(exponent, coeff)])"""
    return tg.BasisSet(g, [tg.SeparableBasisFunction(tuple(c), (0, 0, 0), [tg.GaussianPrimitive(e, k) for e, k in p])
                           for c, p in specs])


def expsum_for_interval(lo, hi, eps):
    import ctypes as C
    from paper_1504_06289_b200._lib import check

    m, c0 = C.c_int64(), C.c_double()
    check(tg.lib().tgb_expsum_for_interval(lo, hi, eps, 2048, C.byref(m), C.byref(c0)), host=True)
    return tg.make_expsum(m.value, c0.value, lo, hi)


def test_overlap_analytic(ctx):  # test_hf.cpp:70-88
    g = tg.make_grid(8.0, 128)
    zs = snapped_z(g, 0.7)
    bs = s_basis(g, [((0, 0, zs), [(0.9, 1.0)]), ((0, 0, -zs), [(0.9, 1.0)])])
    s = tg.overlap_matrix(bs, tg.discretize_basis(bs), ctx)
    a, b = S((0, 0, zs), [0.9], [1.0]), S((0, 0, -zs), [0.9], [1.0])
    assert approx(s[0, 0], overlap(a, a), 1e-5)
    assert approx(s[0, 1], overlap(a, b), 1e-5)
    assert s[0, 1] == s[1, 0]
    far = s_basis(g, [((0, 0, 6.0), [(0.9, 1.0)]), ((0, 0, -6.0), [(0.9, 1.0)])])
    assert abs(tg.overlap_matrix(far, tg.discretize_basis(far), ctx)[0, 1]) <= 1e-8


def test_kinetic_convergence_and_symmetry(ctx):  # test_hf.cpp:90-129
    rel = []
    for n in (128, 256):
        b2 = s_basis(tg.make_grid(8.0, n), [((0, 0, 0), [(1.0, 1.0)])])
        d2 = tg.discretize_basis(b2)
        t = tg.kinetic_matrix(b2, d2, False, ctx)[0, 0]
        s = tg.overlap_matrix(b2, d2, ctx)[0, 0]
        rel.append(abs(t - 1.5 * s) / (1.5 * s))
    assert rel[0] <= 0.02 and rel[1] <= rel[0] / 2.5
    bs = s_basis(tg.make_grid(4.0, 16), [((0, 0, 0), [(0.8, 1.0)])])
    t = tg.kinetic_matrix(bs, tg.discretize_basis(bs), False, ctx)
    assert np.array_equal(t, t.T)


def test_nuclear_analytic_rank_and_swap_symmetry(ctx):  # test_hf.cpp:131-166
    g = tg.make_grid(8.0, 255)
    mol = tg.Molecule([tg.Nucleus(1.0, (0.0, 0.0, 0.0))], 1)
    bs = s_basis(g, [((0, 0, 0), [(1.5, 1.0)])])
    disc = tg.discretize_basis(bs)
    ref = tg.kernel_tensor(g, expsum_for_interval(g.h[0], 2.5 * g.b_half[0], 1e-7), True)
    pc = tg.nuclear_potential_tensor(bs, mol, ref, ctx)
    assert pc.rank() == len(mol.nuclei) * ref.rank()
    v = tg.nuclear_matrix(bs, disc, mol, ref, ctx)
    a = S((0, 0, 0), [1.5], [1.0])
    assert v[0, 0] < 0.0 and approx(v[0, 0], nuclear(a, a, (0, 0, 0), 1.0), 1e-3)
    g2 = tg.make_grid(8.0, 96)
    zs = snapped_z(g2, 1.1)
    bs2 = s_basis(g2, [((0, 0, zs), [(0.8, 1.0)]), ((0, 0, -zs), [(0.8, 1.0)])])
    mol2 = tg.Molecule([tg.Nucleus(1.0, (0, 0, zs)), tg.Nucleus(1.0, (0, 0, -zs))], 2)
    ref2 = tg.kernel_tensor(g2, expsum_for_interval(g2.h[0], 2.5 * g2.b_half[0], 1e-6), True)
    v2 = tg.nuclear_matrix(bs2, tg.discretize_basis(bs2), mol2, ref2, ctx)
    assert approx(v2[0, 0], v2[1, 1], 1e-12) and approx(v2[0, 1], v2[1, 0], 1e-12)


def test_one_electron_second_order(ctx):  # test_hf.cpp:168-199
    ga = S((0, 0, 0), [1.0], [1.0])
    es, et, ev = [], [], []
    for n in (95, 191):
        g = tg.make_grid(8.0, n)
        bs = s_basis(g, [((0, 0, 0), [(1.0, 1.0)])])
        disc = tg.discretize_basis(bs)
        mol = tg.Molecule([tg.Nucleus(1.0, (0, 0, 0))], 1)
        ref = tg.kernel_tensor(g, expsum_for_interval(g.h[0], 2.5 * g.b_half[0], 3e-6), True)
        es.append(abs(tg.overlap_matrix(bs, disc, ctx)[0, 0] - overlap(ga, ga)))
        et.append(abs(tg.kinetic_matrix(bs, disc, False, ctx)[0, 0] - kinetic(ga, ga)))
        ev.append(abs(tg.nuclear_matrix(bs, disc, mol, ref, ctx)[0, 0] - nuclear(ga, ga, (0, 0, 0), 1.0)))
    assert es[0] <= 1e-12 and es[1] <= 1e-12
    assert et[1] <= et[0] / 2.5 and ev[1] <= ev[0] / 2.5


def test_scf_hydrogen_atom(ctx):  # test_hf.cpp:539-562
    g = tg.make_grid(10.0, 127)
    expo = [0.123 * 3.8 ** k for k in range(4)]
    bs = s_basis(g, [((0, 0, 0), [(a, 1.0)]) for a in expo])
    st = tg.scf_solve(tg.Molecule([tg.Nucleus(1.0, (0, 0, 0))], 1), bs, tg.SCFConfig(), ctx)
    assert st.converged
    ref = rhf_energy([S((0, 0, 0), [a], [1.0]) for a in expo], [((0, 0, 0), 1.0)], 1)
    assert abs(st.energy - ref) <= 0.01 and abs(st.energy + 0.4998) <= 0.01


def test_scf_h2_against_analytic_rhf(ctx):  # test_hf.cpp:564-586
    g = tg.make_grid(9.0, 128)
    zs = snapped_z(g, 0.7)
    mol = tg.Molecule([tg.Nucleus(1.0, (0, 0, zs)), tg.Nucleus(1.0, (0, 0, -zs))], 2)
    bs = s_basis(g, [((0, 0, zs), [(0.35, 1.0)]), ((0, 0, -zs), [(0.35, 1.0)])])
    st = tg.scf_solve(mol, bs, tg.SCFConfig(exact_mass_kinetic=True), ctx)
    assert st.converged and st.iterations <= 40
    assert max(st.orthonormality_defects) <= 1e-10
    nuc = [(n.center, n.charge) for n in st.snapped.nuclei]
    ref = rhf_energy([S((0, 0, zs), [0.35], [1.0]), S((0, 0, -zs), [0.35], [1.0])], nuc, 2)
    assert abs(st.energy - ref) <= 1e-3
    for m in (st.overlap, st.kinetic, st.nuclear, st.core_hamiltonian):
        assert np.abs(m - m.T).max() <= 1e-10


def test_scf_helium_monotone_tail(ctx):  # test_hf.cpp:588-609
    g = tg.make_grid(7.0, 96)
    bs = s_basis(g, [((0, 0, 0), [(a, 1.0)]) for a in (0.3, 1.0, 3.2)])
    st = tg.scf_solve(tg.Molecule([tg.Nucleus(2.0, (0, 0, 0))], 2), bs,
                      tg.SCFConfig(mixing=0.5, energy_tol=1e-11), ctx)
    assert st.converged and len(st.energy_history) >= 6
    e = st.energy_history
    for i in range(len(e) - 5, len(e) - 1):
        assert abs(e[i + 1] - e[i]) <= abs(e[i] - e[i - 1]) * (1.0 + 1e-9) + 1e-14


def test_scf_rejects_degenerate_basis(ctx):  # test_hf.cpp:611-624
    g = tg.make_grid(6.0, 48)
    bs = s_basis(g, [((0, 0, 0), [(0.8, 1.0)]), ((0, 0, 0), [(0.8, 1.0)])])
    with pytest.raises(tg.NumericalError):
        tg.scf_solve(tg.Molecule([tg.Nucleus(1.0, (0, 0, 0))], 2), bs, tg.SCFConfig(), ctx)


def synthetic(rng, nb, nocc, r):  # test_mp2.cpp:14-41
    q, _ = np.linalg.qr(rng.normal(size=(nb, nb)))
    e = np.sort(np.concatenate([rng.uniform(-2.0, -0.8, nocc), rng.uniform(0.4, 3.0, nb - nocc)]))
    cols = []
    for _ in range(r):
        m = rng.normal(size=(nb, nb))
        cols.append((0.5 * (m + m.T)).reshape(-1, order="F"))
    return tg.MOSpace(np.asfortranarray(q), e, nocc), np.asfortranarray(np.stack(cols, 1))


def mp2_quadruple(v, e, nocc):
    nv = len(e) - nocc
    tot = 0.0
    for i in range(nocc):
        for j in range(nocc):
            for a in range(nv):
                for b in range(nv):
                    den = e[nocc + a] + e[nocc + b] - e[i] - e[j]
                    x, y = v[i * nv + a, j * nv + b], v[i * nv + b, j * nv + a]
                    tot -= x * (2.0 * x - y) / den
    return tot


def test_mp2_factorized_equals_oracle(ctx):  # test_mp2.cpp:104-117
    rng = np.random.default_rng(63)
    for _ in range(10):
        mos, chol = synthetic(rng, 8, 3, 6)
        mo = tg.mo_transform_cholesky(chol, mos, ctx)
        e_or = tg.mp2_energy(mo, mos, "oracle", ctx=ctx)
        e_fa = tg.mp2_energy(mo, mos, "factorized", 1e-9, ctx=ctx)
        assert e_or <= 0.0 and abs(e_fa - e_or) <= 1e-8 * abs(e_or)
        v = mo.factor @ mo.factor.T
        assert approx(e_or, mp2_quadruple(v, mos.energies, 3), 1e-12)


def test_mp2_degenerate_rotation_invariance(ctx):  # test_mp2.cpp:119-136
    rng = np.random.default_rng(64)
    mos, chol = synthetic(rng, 6, 2, 4)
    mos.energies[0] = mos.energies[1] = -1.3
    e0 = tg.mp2_energy(tg.mo_transform_cholesky(chol, mos, ctx), mos, "oracle", ctx=ctx)
    th = 0.7345
    rot = np.eye(6)
    rot[0, 0], rot[0, 1], rot[1, 0], rot[1, 1] = np.cos(th), -np.sin(th), np.sin(th), np.cos(th)
    rmos = tg.MOSpace(np.asfortranarray(mos.coefficients @ rot), mos.energies, 2)
    assert approx(tg.mp2_energy(tg.mo_transform_cholesky(chol, rmos, ctx), rmos, "oracle", ctx=ctx), e0, 1e-8)


def test_mp2_refuses_nonpositive_gap(ctx):  # test_mp2.cpp:163-174
    mos = tg.MOSpace(np.eye(2), np.array([-0.1, -0.1]), 1)
    mo = tg.MOCholesky(np.ones((1, 1)), 1, 1)
    with pytest.raises(tg.NumericalError):
        tg.mp2_energy(mo, mos, ctx=ctx)

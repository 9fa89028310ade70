"""CPU: the restatement's hf.cpp / tei.cpp operators (oracle/tengrid_oracle.cpp)
against fixtures produced by the reference's OWN hf.cpp / tei.cpp / reduction.cpp
(oracle/_ref, tools/make_golden_hf.py).  No GPU involved."""
import numpy as np
import pytest

from conftest import relmax
from hf_case import functions, load
from oracle import oracle as O

TOL = 1e-12


@pytest.fixture(scope="module")
def g():
    return load()


@pytest.fixture(scope="module")
def disc(g):
    return O.discretize_basis(g["b_half"], g["n"], functions(g))


def kernel(g, doubled):
    m, c0 = int(g["kernel_m_c0"][0]), float(g["kernel_m_c0"][1])
    nodes, w = O.make_expsum(m, c0)[:2]
    return O.kernel_tensor(g["b_half"], g["n"], nodes, w, doubled)


@pytest.mark.parametrize("which,key", [(0, "S"), (1, "T_lumped"), (2, "T_exact")])
def test_one_electron(g, disc, which, key):
    got = O.one_electron(g["b_half"], g["n"], disc, which)
    assert relmax(got, g[key]) <= TOL
    assert np.array_equal(got, got.T)


def test_nuclear(g, disc):
    pc = O.nuclear_potential_tensor(g["b_half"], g["n"], g["nuc_centers"], g["nuc_charges"], kernel(g, True))
    for ax, f in enumerate(pc.factors()):
        assert np.array_equal(f, g[f"pc_f{ax}"])  # windows are copies: bit-identical
    assert np.array_equal(pc.weight(), g["pc_w"])
    V = O.nuclear_matrix(disc, pc)
    assert relmax(V, g["V"]) <= TOL


def test_exchange(g, disc):
    K = O.exchange_matrix(g["b_half"], g["n"], disc, g["c_occ"], kernel(g, False))
    assert relmax(K, g["K"]) <= TOL
    assert np.array_equal(K, K.T)


@pytest.mark.parametrize("which,key", [(0, "ff_J"), (1, "ff_K"), (2, "ff_F")])
def test_from_factors(g, which, key):
    got = O.from_factors(which, g["ff_chol"], g["ff_density"], g["ff_hcore"] if which == 2 else None)
    assert relmax(got, g[key]) <= TOL
    assert np.array_equal(got, got.T)


def test_reference_binary_matches_fixture(g):
    """Where oracle/_ref exists (this container), the committed fixture is what it computes today."""
    if O.rlib() is None:
        pytest.skip("oracle/_ref not built")
    R = O.Ref(g["b_half"], g["n"], functions(g))
    assert np.array_equal(R.one_electron(0), g["S"])
    assert np.array_equal(R.exchange_matrix(g["c_occ"], int(g["kernel_m_c0"][0]), float(g["kernel_m_c0"][1])), g["K"])

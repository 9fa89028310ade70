"""Host input producers that need no GPU: tg::expsum_for_interval (kernel.cpp:131-165)
is bit-identical to the reference binary's (tests/golden/reference_scf.npz)."""
import ctypes as C
from pathlib import Path

import numpy as np

import paper_1504_06289_b200 as tg
from paper_1504_06289_b200._lib import check

G = dict(np.load(Path(__file__).resolve().parent / "golden" / "reference_scf.npz"))


def test_expsum_for_interval_bit_identical():
    for (lo, hi, eps), (m_ref, c0_ref) in zip(G["expsum_in"], G["expsum_out"]):
        m, c0 = C.c_int64(), C.c_double()
        check(tg.lib().tgb_expsum_for_interval(lo, hi, eps, 2048, C.byref(m), C.byref(c0)), host=True)
        assert m.value == int(m_ref) and c0.value == c0_ref


def test_reciprocal_expsum_bit_identical():
    """tg::reciprocal_expsum (kernel.cpp:205-250) against the reference binary's output."""
    for idx, (lo, hi, eps, terms, ach, ok) in enumerate(G["recip_cases"]):
        t, a, k = C.c_int64(), C.c_double(), C.c_int()
        r, w = np.zeros(256), np.zeros(256)
        check(tg.lib().tgb_reciprocal_expsum(lo, hi, eps, 256, C.byref(t), r.ctypes.data, w.ctypes.data, C.byref(a),
                                             C.byref(k)), host=True)
        assert (t.value, k.value) == (int(terms), int(ok)) and a.value == ach
        assert np.array_equal(r[:t.value], G[f"recip_{idx}_rates"]) and np.array_equal(w[:t.value],
                                                                                    G[f"recip_{idx}_weights"])


def test_flatten_basis_and_add_layouts():
    # host-side CP concatenations: Fortran-order factors, column order = function order
    from paper_1504_06289_b200.inputs import basis_case
    from paper_1504_06289_b200.tengrid import flatten_basis

    bs, _ = basis_case(1, n=33)
    disc = tg.discretize_basis(bs)
    flat, offs = flatten_basis(disc)
    for ax in range(3):
        ref = np.hstack([d.factor[ax] for d in disc])
        assert flat.factor[ax].flags["F_CONTIGUOUS"] and np.array_equal(flat.factor[ax], ref)
    assert np.array_equal(flat.weight, np.concatenate([d.weight for d in disc]))
    assert list(offs) == [0] + list(np.cumsum([d.rank() for d in disc]))
    s = tg.add(disc[0], disc[1])
    assert s.rank() == disc[0].rank() + disc[1].rank()
    for ax in range(3):
        assert s.factor[ax].flags["F_CONTIGUOUS"]
        assert np.array_equal(s.factor[ax], np.hstack([disc[0].factor[ax], disc[1].factor[ax]]))
    z = tg.add(tg.CanonicalTensor3.zero(disc[0].extents()), disc[0])
    assert z.rank() == disc[0].rank()

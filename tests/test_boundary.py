"""CPU tests of the drop-in boundary: libtgb.so loads and exports every symbol
declared in include/*.h; the host-side input producers (tgb_host.h) agree
bit-for-bit with the oracle restatement of kernel.cpp / basis.cpp / grid.cpp
and raise the reference's error classes.  No device compute is called here."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1504_06289_b200 import (DomainError, InvalidArgument, SnapError, exported_symbols, kernel_tensor, lib,
                                   make_expsum, make_grid, primitive_norm, window_offset, snap_to_node,
                                   gauss_cell_integral)
from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, Rng


def test_library_exports_every_declared_symbol():
    names = exported_symbols()
    assert len(names) >= 20
    so = C.CDLL(str(lib()._name))
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_no_cpu_fallback_symbols():
    # the product library links no oracle code
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", lib()._name], capture_output=True, text=True).stdout
    assert "orc_" not in out and "ref_" not in out


@pytest.mark.parametrize("m,c0", [(1, 1.0), (8, 1.0), (15, KERNEL_C0[0]), (20, KERNEL_C0[1]), (32, 1.0), (128, 1.0)])
def test_make_expsum_bitwise_vs_oracle(m, c0):
    es = make_expsum(m, c0)
    nodes, w, sc, mesh = O.make_expsum(m, c0)
    assert es.terms() == 2 * m + 1
    assert np.array_equal(es.nodes, nodes) and np.array_equal(es.weights, w)
    assert es.scale == sc and es.mesh == mesh


def test_make_expsum_known_answers():
    # test_kernel.cpp:13-27: node layout, positivity, half-line scale ~ 1/2
    es = make_expsum(1, 1.0)
    assert es.terms() == 3
    assert es.nodes[1] == 0.0 and es.nodes[0] == -es.mesh and es.nodes[2] == es.mesh
    for m in (8, 32, 128):
        e = make_expsum(m, 1.0)
        assert e.weights.min() > 0
        assert abs(e.scale - 0.5) <= 0.5e-3
    with pytest.raises(InvalidArgument):
        make_expsum(0, 1.0)
    with pytest.raises(InvalidArgument):
        make_expsum(4, -1.0)


@pytest.mark.parametrize("doubled", [False, True])
def test_kernel_factors_bitwise_vs_oracle(doubled):
    g = make_grid(20.0, 255)
    es = make_expsum(40, 1.2, 1.0, 8.0)
    kt = kernel_tensor(g, es, doubled)
    ok = O.kernel_tensor(20.0, 255, es.nodes, es.weights, doubled)
    of = ok.factors()
    for ax in range(3):
        assert np.array_equal(kt.tensor.factor[ax], of[ax])
    # test_kernel.cpp:107-117: rank 2M+1, identical axes, even symmetry
    assert kt.rank() == 81
    assert np.array_equal(kt.tensor.factor[0], kt.tensor.factor[1])
    assert np.array_equal(kt.tensor.factor[0], kt.tensor.factor[2])
    if not doubled:
        f = kt.tensor.factor[0]
        np.testing.assert_allclose(f, f[::-1], rtol=1e-13, atol=0)


def test_kernel_pointwise_value():
    # test_kernel.cpp:119-124 — h^-3 entry near (2,0,0) approximates 1/r
    g = make_grid(20.0, 255)
    best = min(((make_expsum(40, c0, 1.0, 8.0).max_relative_error(1.5, 4.0), c0)
                for c0 in np.arange(0.5, 2.5001, 0.1)))
    es = make_expsum(40, best[1], 1.0, 8.0)
    kt = kernel_tensor(g, es, False)
    i2, ic = g.nearest_index(0, 2.0), g.nearest_index(0, 0.0)
    r = float(g.coord(0, i2))
    val = kt.tensor.value_at(i2, ic, ic) / (g.h[0] * g.h[1] * g.h[2])
    assert abs(val - 1.0 / r) <= 1e-4 / r


def test_gauss_cell_integral_branches():
    for t in (0.0, 0.3, 2.0, 11.0):
        for c in (-3.0, -0.01, 0.0, 0.02, 4.0):
            assert gauss_cell_integral(t, c, 0.05) == O.gauss_cell_integral(t, c, 0.05)


def test_grid_and_window_offsets():
    g = make_grid(72.0, 32769)
    assert g.h[0] == 2 * 72.0 / 32770
    for x in (-62.0, -3.9, 0.0, 10.0, 62.0):
        assert window_offset(g, 0, x) == O.window_offset(72.0, 32769, 0, x)
    with pytest.raises(DomainError):
        window_offset(g, 0, 80.0)
    g2 = make_grid(1.0, 4)
    with pytest.raises(SnapError):
        snap_to_node(g2, 0, 0.95)  # inside the box, beyond the last node by > h/2
    with pytest.raises(InvalidArgument):
        make_grid(-1.0, 5)


def test_primitive_norm():
    assert primitive_norm(1.3, 0) == pytest.approx((2 * 1.3 / math.pi) ** 0.75, rel=1e-15)
    with pytest.raises(InvalidArgument):
        primitive_norm(1.0, 2)

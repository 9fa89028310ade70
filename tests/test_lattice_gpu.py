"""Lattice sums (proj/src/lattice.cpp:50-165) on the device: bit-identical
window assembly vs the oracle, rank preservation, window_ops == sum of L,
Tucker core untouched, composite block geometries vs explicit node sums.
Re-expresses test_lattice.cpp:26-226."""
import numpy as np
import pytest

from conftest import relmax
from oracle import oracle as O
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import Rng

pytestmark = pytest.mark.gpu


def ref_kernel(grid, m=6, c0=0.9):
    return tg.kernel_tensor(grid, tg.make_expsum(m, c0), True)


def windowed(ref, grid, center):
    """CP tensor of the reference kernel translated to `center` (grid.cpp:40-47)."""
    facs = []
    for ax in range(3):
        o = tg.window_offset(grid, ax, center[ax])
        facs.append(ref.tensor.factor[ax][o:o + grid.n[ax]])
    return tg.CanonicalTensor3(facs, ref.tensor.weight.copy())


def test_single_site_equals_windowed_kernel(ctx):
    spec = tg.LatticeSpec(counts=(1, 1, 1), spacing=2.0, n0=8)
    grid = tg.lattice_grid(spec)
    ref = ref_kernel(grid)
    ap = tg.lattice_sum_canonical(spec, grid, ref, ctx)
    w = windowed(ref, grid, (0.0, 0.0, 0.0))
    for ax in range(3):
        assert np.array_equal(ap.canonical.factor[ax], w.factor[ax])
    assert ap.window_ops == 3


def test_bitwise_vs_oracle_and_rank(ctx):
    spec = tg.LatticeSpec(counts=(5, 3, 4), spacing=2.0, charge=1.5, n0=10)
    grid = tg.lattice_grid(spec)
    ref = ref_kernel(grid, 8, 1.0)
    ap = tg.lattice_sum_canonical(spec, grid, ref, ctx)
    assert ap.canonical.rank() == ref.rank()
    assert ap.window_ops == 5 + 3 + 4
    for ax in range(3):
        centres = [spec.position(ax, m) for m in range(spec.counts[ax])]
        out, ops = O.assemble_axis(grid.b_half, grid.n, ax, ref.tensor.factor[ax], centres)
        assert np.array_equal(ap.canonical.factor[ax], out)
    assert np.array_equal(ap.canonical.weight, 1.5 * ref.tensor.weight)


def test_8cubed_probes_vs_direct_windowed_sum(ctx):
    # test_lattice.cpp:80-110 (8^3 lattice at probes, <= 1e-10)
    spec = tg.LatticeSpec(counts=(8, 8, 8), spacing=1.0, n0=6)
    grid = tg.lattice_grid(spec)
    ref = ref_kernel(grid, 6, 0.8)
    ap = tg.lattice_sum_canonical(spec, grid, ref, ctx)
    rng = Rng(99)
    pts = rng.integers(150, grid.n[0]).reshape(50, 3)
    got = tg.value_at_points(ap.canonical, pts, ctx)
    direct = np.zeros(len(pts))
    for c in tg.lattice_nodes(spec):
        direct += tg.value_at_points(windowed(ref, grid, c), pts, ctx)
    assert relmax(got, direct) <= 1e-10


def test_tucker_core_unchanged_and_dense_matches_canonical(ctx):
    spec = tg.LatticeSpec(counts=(3, 2, 2), spacing=2.0, charge=0.7, n0=6)
    grid = tg.lattice_grid(spec)
    ref = ref_kernel(grid, 4, 0.9)
    master = tg.rhosvd(ref.tensor, tg.ReductionConfig.tolerance(1e-10), ctx).tucker
    ap = tg.lattice_sum_tucker(spec, grid, master, ctx)
    assert np.array_equal(ap.tucker.core, master.core * 0.7)  # lattice.cpp:139-140
    assert ap.window_ops == 7
    canon = tg.lattice_sum_canonical(spec, grid, ref, ctx)
    assert relmax(ap.tucker.to_dense(), canon.canonical.to_dense()) <= 1e-8


@pytest.mark.parametrize("shape", ["L", "O"])
def test_composite_shapes_vs_node_sum(ctx, shape):
    if shape == "L":
        blocks = [tg.LatticeBlock((2, 2, 0), (3, 3, 1), False)]
    else:
        blocks = [tg.LatticeBlock((1, 1, 0), (2, 2, 1), False)]
    spec = tg.LatticeSpec(counts=(4, 4, 2), spacing=1.5, n0=6, blocks=blocks)
    grid = tg.lattice_grid(spec)
    ref = ref_kernel(grid, 5, 0.9)
    ap = tg.lattice_sum_composite(spec, grid, ref, None, ctx)
    rng = Rng(7)
    pts = np.stack([rng.integers(40, grid.n[ax]) for ax in range(3)], axis=1)
    got = tg.value_at_points(ap.canonical, pts, ctx)
    direct = np.zeros(len(pts))
    for c in tg.lattice_nodes(spec):
        direct += tg.value_at_points(windowed(ref, grid, c), pts, ctx)
    assert relmax(got, direct) <= 1e-9
    with pytest.raises(tg.InvalidArgument):
        tg.lattice_sum_canonical(spec, grid, ref, ctx)


def test_overlapping_includes_rejected():
    spec = tg.LatticeSpec(counts=(4, 4, 4), blocks=[tg.LatticeBlock((0, 0, 0), (2, 2, 2)),
                                                    tg.LatticeBlock((1, 1, 1), (3, 3, 3))])
    with pytest.raises(tg.InvalidArgument):
        tg.resolve_blocks(spec)

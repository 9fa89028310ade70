"""Parity of the sm_100a mode convolutions with the CPU oracle (restatement of
proj/src/fft.cpp + tensor.cpp) and with an independent numpy definition.
Tolerance: 1e-10 relative max-norm (BASELINE.json north_star), per factor
matrix.  Semantics pinned by the reference tests test_tensor.cpp:24-37,
122-169, 211-230 and acceptance.cpp:103-127 are re-expressed here."""
import numpy as np
import pytest

from conftest import relmax
from oracle import oracle as O
from paper_1504_06289_b200 import (CanonicalTensor3, DeviceCP, InvalidArgument, conv_central_many, convolve,
                                   hartree_potential, value_at_points)
from paper_1504_06289_b200.inputs import Rng, hartree_case, random_canonical

pytestmark = pytest.mark.gpu
TOL = 1e-10


def window_np(u, v):
    n = len(u)
    full = np.convolve(u, v)
    if n % 2:
        o = (n - 1) // 2
        return full[o:o + n]
    o = n // 2 - 1
    return 0.5 * (full[o:o + n] + full[o + 1:o + 1 + n])


@pytest.mark.parametrize("n", [1, 2, 3, 5, 16, 17, 31, 64, 65, 100, 127, 128, 129, 200, 513, 1000, 1025, 2048,
                               2049, 4097, 8193, 16383, 16385, 16387, 20001, 32769, 32771, 65537])
@pytest.mark.parametrize("force_fft", [False, True])
def test_conv_central_many_matches_oracle(ctx, n, force_fft):
    rng = Rng(1000 + n)
    cols = 7
    U = np.asfortranarray(rng.normal(n * cols).reshape(n, cols, order="F"))
    v = rng.normal(n)
    ctx.set_direct_max(0 if force_fft else 64)
    try:
        got = conv_central_many(U, v, ctx)
    finally:
        ctx.set_direct_max(64)
    ref = O.conv_central_many(U, v)
    assert relmax(got, ref) <= TOL
    ind = np.stack([window_np(U[:, c], v) for c in range(cols)], axis=1)
    assert relmax(got, ind) <= TOL


def test_conv_large_n_gaussians(ctx):
    # n = 16385 (config 2 extent): smooth, widely ranged Gaussians
    n = 16385
    x = (np.arange(n) - 0.5 * (n - 1)) * (20.0 / (n + 1))
    a = np.array([0.05, 0.7, 5.0, 60.0, 500.0])
    U = np.asfortranarray(np.exp(-a[None, :] * (x[:, None] - 0.3) ** 2))
    v = np.exp(-2.0 * x ** 2)
    got = conv_central_many(U, v, ctx)
    ref = O.conv_central_many(U, v)
    assert relmax(got, ref) <= TOL


def test_k12_plan_many_pairs_per_cta(ctx):
    """The N = 12288 plan (fftconv12k.cu: m = 24576, one aliased term per window end
    at n = 16385, subtracted exactly) with ~6 pairs per persistent CTA, density-column
    switches inside a CTA's run, duplicate kernel columns (one result, two output
    columns), the real-spectrum path (axis 0: every kernel column mirror-symmetric)
    and the complex path (axes 1, 2: one non-symmetric column).  Sampled output
    columns against the oracle's conv_central_many (proj/src/fft.cpp:97-122) x h."""
    dims = (16385, 16383, 16385)
    ra = 300
    rng = Rng(4242)
    fa = [np.asfortranarray(rng.normal(d * ra).reshape(d, ra, order="F")) for d in dims]
    a = CanonicalTensor3(fa, rng.normal(ra))
    fb = []
    for ax, d in enumerate(dims):
        x = np.arange(d) - 0.5 * (d - 1)
        g = np.exp(-(x / 900.0) ** 2)
        c2 = np.exp(-((x / 300.0) ** 2)) if ax == 0 else rng.normal(d)
        fb.append(np.asfortranarray(np.stack([g, g.copy(), c2], axis=1)))
    b = CanonicalTensor3(fb, np.ones(3))
    h = (0.011, 0.013, 0.017)
    c = convolve(a, b, h, ctx)
    for ax, d in enumerate(dims):
        for i in (0, 1, 149, 150, 151, 298, 299):
            for j in range(3):
                ref = O.conv_central_many(np.asfortranarray(fa[ax][:, [i]]), np.ascontiguousarray(fb[ax][:, j]))[:, 0]
                assert relmax(c.factor[ax][:, i + ra * j], h[ax] * ref) <= TOL, (ax, i, j)
        assert np.array_equal(c.factor[ax][:, 0:ra], c.factor[ax][:, ra:2 * ra])


@pytest.mark.parametrize("ra", [64, 7])
def test_k12_band_limited_pairs(ctx, monkeypatch, ra):
    """Band-limited kernel columns (spectrum below 2^-46 of its peak beyond k = 144: smooth
    Gaussians, the Newton kernel's mid-range terms) take the pruned path of k12_pair_kernel
    (Zs table + merged 48-point stage, fftconv12k.cu); the others the full stages 1-3.  Kernel
    columns ordered so that a CTA's run switches between the two forms in both directions and
    runs several band-limited pairs back to back (table and y values formed one pair ahead):
    off-centre Gaussians (non-symmetric: complex spectra on axis 0), centred ones (real spectra
    on axis 1), a box-truncated wide Gaussian, a spike, a zero column.  Against the oracle
    (proj/src/fft.cpp:97-122) and against the same call with the pruning switched off.
    ra = 64: aligned (one-sample-delayed) window stores; ra = 7: the unshifted store path."""
    n = 16385
    rng = Rng(777)
    fa = [np.asfortranarray(rng.normal(n * ra).reshape(n, ra, order="F")) for _ in range(3)]
    a = CanonicalTensor3(fa, rng.normal(ra))
    x = np.arange(n) - 0.5 * (n - 1)
    gauss = lambda s, c=0.0: np.exp(-(((x - c) / s) ** 2))
    spike = np.zeros(n)
    spike[n // 2 - 3:n // 2 + 4] = [1, -2, 3, 5, 3, -2, 1]
    cols0 = [gauss(700, 40.5), gauss(400, -300), gauss(9000), gauss(900, 123), gauss(350, 7), spike,
             np.zeros(n), gauss(1200, -77), gauss(500, 2000)]
    cols1 = [gauss(700), gauss(400), gauss(9000), gauss(900), gauss(350), spike, np.zeros(n), gauss(1200), gauss(320)]
    fb = [np.asfortranarray(np.stack(c, axis=1)) for c in (cols0, cols1, cols0[::-1])]
    rb = len(cols0)
    b = CanonicalTensor3(fb, np.ones(rb))
    h = (0.011, 0.013, 0.017)
    c = convolve(a, b, h, ctx)
    monkeypatch.setenv("TGB_K12_NO_PRUNE", "1")
    cfull = convolve(a, b, h, ctx)
    monkeypatch.delenv("TGB_K12_NO_PRUNE")
    for ax in range(3):
        assert relmax(c.factor[ax], cfull.factor[ax]) <= 1e-12, ax
        for j in range(rb):
            blk = c.factor[ax][:, ra * j:ra * (j + 1)]
            scale = np.abs(cfull.factor[ax][:, ra * j:ra * (j + 1)]).max()
            assert np.abs(blk - cfull.factor[ax][:, ra * j:ra * (j + 1)]).max() <= 1e-12 * max(scale, 1e-300), (ax, j)
        for i in sorted({0, 1, ra // 2, ra - 2, ra - 1}):
            for j in range(rb):
                ref = O.conv_central_many(np.asfortranarray(fa[ax][:, [i]]), np.ascontiguousarray(fb[ax][:, j]))[:, 0]
                assert relmax(c.factor[ax][:, i + ra * j], h[ax] * ref) <= TOL, (ax, i, j)


def test_k12_non_finite_kernel_column_not_pruned(ctx):
    """A kernel column holding a NaN has a NaN spectrum: it must not be classed as band-limited
    (its NaNs would be dropped with the pruned entries); every window element is NaN as in the
    reference's FFT (fft.cpp:97-122), and the finite columns beside it are untouched."""
    n, ra = 16385, 6
    rng = Rng(778)
    fa = [np.asfortranarray(rng.normal(n * ra).reshape(n, ra, order="F")) for _ in range(3)]
    a = CanonicalTensor3(fa, np.ones(ra))
    x = np.arange(n) - 0.5 * (n - 1)
    g = np.exp(-((x / 800.0) ** 2))
    bad = g.copy()
    bad[5] = np.nan
    fb = [np.asfortranarray(np.stack([g, bad], axis=1)) for _ in range(3)]
    c = convolve(a, CanonicalTensor3(fb, np.ones(2)), (1.0, 1.0, 1.0), ctx)
    for ax in range(3):
        assert np.isnan(c.factor[ax][:, ra:]).all()
        ref = O.conv_central_many(fa[ax], g)
        assert relmax(c.factor[ax][:, :ra], ref) <= TOL


def test_convolve_delta_identity(ctx):
    # test_tensor.cpp:122-135 — delta kernel with h-scaling removed
    n, h = 17, 0.25
    rng = Rng(7)
    a = random_canonical(rng, (n, n, n), 2)
    f = [np.zeros((n, 1), order="F") for _ in range(3)]
    for ax in range(3):
        f[ax][(n - 1) // 2, 0] = 1.0 / h
    delta = CanonicalTensor3(f, np.ones(1))
    c = convolve(a, delta, h, ctx)
    assert c.rank() == 2
    np.testing.assert_allclose(c.to_dense(), a.to_dense(), rtol=0, atol=1e-13 * np.abs(a.to_dense()).max())


def test_convolve_semantics_random(ctx):
    # acceptance.cpp:103-127 / test_tensor.cpp:211-230: per-axis extents 4..32,
    # ranks 0..4, column order i + Ra*j, weights a.w[i]*b.w[j], h per axis.
    rng = Rng(20240817)
    for rep in range(40):
        dims = tuple(int(4 + x) for x in rng.integers(3, 29))
        ra, rb = (int(x) for x in rng.integers(2, 5))
        a = random_canonical(rng, dims, ra)
        b = random_canonical(rng, dims, rb)
        h = (0.37, 0.5, 0.21)
        c = convolve(a, b, h, ctx)
        assert c.rank() == ra * rb
        oc = O.convolve(O.OCP.from_cp(a), O.OCP.from_cp(b), h)
        assert np.array_equal(c.weight, oc.weight())
        for ax in range(3):
            assert c.factor[ax].shape == (dims[ax], ra * rb)
            if ra * rb:
                assert relmax(c.factor[ax], oc.factors()[ax]) <= TOL


def test_convolve_errors(ctx):
    rng = Rng(8)
    a = random_canonical(rng, (32, 32, 32), 2)
    with pytest.raises(InvalidArgument):
        convolve(a, random_canonical(rng, (32, 32, 8), 1), 0.2, ctx)
    with pytest.raises(InvalidArgument):
        convolve(a, a, 0.0, ctx)
    with pytest.raises(InvalidArgument):
        convolve(a, a, (0.2, -1.0, 0.2), ctx)


def test_bitwise_duplicate_kernel_columns(ctx):
    # +-t sinc nodes give bitwise-identical kernel columns (kernel.cpp:194);
    # their output columns must be bitwise identical too.
    case = hartree_case(0, n=257, rank=6)
    vh = hartree_potential(case.theta, case.kernel, case.grid.h, ctx)
    ra, rb = case.theta.rank(), case.kernel.rank()
    for ax in range(3):
        kf = case.kernel.tensor.factor[ax]
        for j in range(rb):
            jm = rb - 1 - j
            assert np.array_equal(kf[:, j], kf[:, jm])
            assert np.array_equal(vh.factor[ax][:, j * ra:(j + 1) * ra], vh.factor[ax][:, jm * ra:(jm + 1) * ra])


def test_hartree_config0_full(ctx):
    case = hartree_case(0)
    vh = hartree_potential(case.theta, case.kernel, case.grid.h, ctx)
    ovh = O.hartree_potential(O.OCP.from_cp(case.theta), O.OCP.from_cp(case.kernel.tensor), case.grid.h)
    assert np.array_equal(vh.weight, ovh.weight())
    of = ovh.factors()
    for ax in range(3):
        assert relmax(vh.factor[ax], of[ax]) <= TOL
    got = value_at_points(vh, case.samples, ctx)
    ref = O.value_at(ovh, case.samples)
    assert relmax(got, ref) <= TOL


def test_hartree_device_resident_matches_host(ctx):
    import torch

    case = hartree_case(0, n=1025, rank=12)
    host = hartree_potential(case.theta, case.kernel, case.grid.h, ctx)
    dt = DeviceCP.from_host(case.theta)
    dk = DeviceCP.from_host(case.kernel.tensor)
    dv = hartree_potential(dt, dk, case.grid.h, ctx)
    ctx.synchronize()
    back = dv.to_host()
    for ax in range(3):
        assert np.array_equal(back.factor[ax], host.factor[ax])
    assert np.array_equal(back.weight, host.weight)
    pts = torch.as_tensor(case.samples[:500]).cuda()
    got = value_at_points(dv, pts, ctx).cpu().numpy()
    assert relmax(got, value_at_points(host, case.samples[:500], ctx)) <= 1e-13


def test_k12_shared_kernel_axes_bitwise(ctx):
    """Config-2 extent: the Newton kernel's three factor matrices are bitwise equal on a cubic
    grid; given as ONE device matrix (DeviceCP.from_host share_equal_axes) libtgb forms its
    spectra once (fftconv12k.cu k12_spectrum_kernel bsrc) - the result must not change by a bit.
    Even density rank (shifted odd columns) and odd rank (unshifted stores) both."""
    for rank in (6, 5):
        case = hartree_case(2, rank=rank, nsamples=1)
        dt = DeviceCP.from_host(case.theta)
        sep = hartree_potential(dt, DeviceCP.from_host(case.kernel.tensor), case.grid.h, ctx)
        dks = DeviceCP.from_host(case.kernel.tensor, share_equal_axes=True)
        assert dks.factor[1] is dks.factor[0] and dks.factor[2] is dks.factor[0]
        shared = hartree_potential(dt, dks, case.grid.h, ctx)
        ctx.synchronize()
        a, b = sep.to_host(), shared.to_host()
        for ax in range(3):
            assert np.array_equal(a.factor[ax], b.factor[ax])


def test_hartree_config2_columns(ctx):
    # n = 16385 (config 2 extent) with a slice of the density: every kernel
    # column, a few density columns, all three axes against the oracle.
    case = hartree_case(2, rank=500, nsamples=100)
    keep = [0, 17, 123, 256, 499]
    theta = CanonicalTensor3([f[:, keep] for f in case.theta.factor], case.theta.weight[keep])
    vh = hartree_potential(theta, case.kernel, case.grid.h, ctx)
    ovh = O.hartree_potential(O.OCP.from_cp(theta), O.OCP.from_cp(case.kernel.tensor), case.grid.h)
    of = ovh.factors()
    for ax in range(3):
        assert relmax(vh.factor[ax], of[ax]) <= TOL


GOLDEN_CFG2 = __import__("pathlib").Path(__file__).parent / "golden" / "reference_cfg2_vh_samples.npz"


def test_hartree_config2_full_benchmarked_path(ctx):
    """The benchmarked configuration itself (bench.py): all 500 density columns
    x 41 kernel columns x 3 axes through the device-resident path, i.e. the
    persistent pair kernel with ~71 pairs per CTA, density-column switches
    inside a CTA's run and shared/tensor memory reused across pairs.
    * 64 complete output columns per axis against the reference's own
      conv_central_many (oracle/_ref, proj/src/fft.cpp:97-122) times h, as
      tg::convolve forms them (tensor.cpp:191-195); the density columns are
      chosen so that their pairs sit mid-run in CTAs that switched density
      column before them (work list: i-major, 21 distinct kernel columns per i,
      CTA b takes entries [10500 b / 148, 10500 (b + 1) / 148)).
    * V_H at the 10^4 seeded sample points against the fixture the reference
      computed over all 61,500 convolutions (tools/make_golden_cfg2.py)."""
    import ctypes as C

    import torch

    R = O.rlib()
    if R is None:
        pytest.skip("oracle/_ref not built")
    g = np.load(GOLDEN_CFG2)
    case = hartree_case(2, nsamples=int(g["samples"].shape[0]))
    assert np.array_equal(case.samples, g["samples"])
    ra, rb = case.theta.rank(), case.kernel.rank()
    n = case.grid.n[0]
    d_theta = DeviceCP.from_host(case.theta)
    d_kern = DeviceCP.from_host(case.kernel.tensor)
    d_out = DeviceCP.empty([n, n, n], ra * rb)
    hartree_potential(d_theta, d_kern, case.grid.h, ctx, out=d_out)
    ctx.synchronize()
    # V_H at the sample points vs the reference over all 61,500 convolutions
    got_t = value_at_points(d_out, torch.as_tensor(case.samples).cuda(), ctx)
    ctx.synchronize()
    got = got_t.cpu().numpy()
    assert relmax(got, g["vh"]) <= TOL, relmax(got, g["vh"])
    # complete output columns vs the reference's conv_central_many
    ii = [0, 3, 4, 70, 71, 250, 251, 499]
    jj = [0, 40, 5, 35, 13, 20, 27, 39]
    kf = case.kernel.tensor.factor
    for ax in range(3):
        U = np.asfortranarray(case.theta.factor[ax][:, ii])
        cols = torch.as_tensor([i + ra * j for j in jj for i in ii], device=d_out.factor[ax].device)
        sel = d_out.factor[ax].index_select(0, cols)
        torch.cuda.synchronize()
        mine = sel.cpu().numpy().T  # n x 64
        for jx, j in enumerate(jj):
            v = np.ascontiguousarray(kf[ax][:, j])
            ref = np.zeros((n, len(ii)), order="F")
            rc = R.ref_conv_central_many(C.c_longlong(n), C.c_longlong(len(ii)), C.c_void_p(U.ctypes.data),
                                         C.c_void_p(v.ctypes.data), C.c_void_p(ref.ctypes.data), C.c_int(8))
            assert rc == 0
            ref *= case.grid.h[ax]
            blk = mine[:, jx * len(ii):(jx + 1) * len(ii)]
            for c in range(len(ii)):
                assert relmax(blk[:, c], ref[:, c]) <= TOL, (ax, ii[c], j, relmax(blk[:, c], ref[:, c]))
    del d_out
    torch.cuda.empty_cache()


def test_pair_kernels_deterministic(ctx):
    """Race evidence in lieu of compute-sanitizer (closed on this pool): the
    config-2 plan with several pairs per CTA, density-column switches and
    twin columns, and the split plan (n = 32769), run twice on the same inputs,
    give bit-identical factors."""
    rng = Rng(99)
    for n, ra in ((16385, 300), (32769, 40)):
        dims = (n, n, n)
        fa = [np.asfortranarray(rng.normal(n * ra).reshape(n, ra, order="F")) for _ in dims]
        x = np.arange(n) - 0.5 * (n - 1)
        g = np.exp(-(x / 700.0) ** 2)
        fb = [np.asfortranarray(np.stack([g, g], axis=1)) for _ in dims]
        a = DeviceCP.from_host(CanonicalTensor3(fa, np.ones(ra)))
        b = DeviceCP.from_host(CanonicalTensor3(fb, np.ones(2)))
        c1 = convolve(a, b, 0.01, ctx)
        c2 = convolve(a, b, 0.01, ctx)
        ctx.synchronize()
        for ax in range(3):
            assert bool((c1.factor[ax] == c2.factor[ax]).all()), (n, ax)


def test_cp_algebra_device_bitwise(ctx):
    """tgb_hadamard / tgb_add / tgb_scale (tensor.cpp:141-177) on device tensors are
    bit-identical to the element-wise host definitions (the reference's), with
    column order i + R_a j and rank-0 operands."""
    rng = Rng(5150)
    dims = (17, 9, 23)
    a = random_canonical(rng, dims, 3)
    b = random_canonical(rng, dims, 4)
    z = random_canonical(rng, dims, 0)
    from paper_1504_06289_b200 import add, hadamard, scale

    da, db, dz = DeviceCP.from_host(a), DeviceCP.from_host(b), DeviceCP.from_host(z)
    for got, ref in ((hadamard(da, db, ctx), hadamard(a, b)), (add(da, db, ctx), add(a, b)),
                     (scale(da, -0.37, ctx), scale(a, -0.37)), (hadamard(da, dz, ctx), hadamard(a, z)),
                     (add(dz, db, ctx), add(z, b))):
        h = got.to_host()
        assert h.rank() == ref.rank()
        assert np.array_equal(h.weight, ref.weight)
        for ax in range(3):
            assert np.array_equal(h.factor[ax], ref.factor[ax])
    with pytest.raises(InvalidArgument):
        hadamard(da, DeviceCP.from_host(random_canonical(rng, (17, 9, 22), 2)), ctx)


def test_host_path_pinned_twin_replication(ctx):
    """Host-memory hartree_potential into PINNED output buffers: only the
    representative kernel-column blocks cross PCIe (twins replicated on the
    host, tgb_ctx_transfer_bytes counts it) and the result is bit-identical to
    the pageable path's whole-factor copy."""
    import torch

    case = hartree_case(0, n=1025, rank=12)
    ra, rb = case.theta.rank(), case.kernel.rank()
    ref = hartree_potential(case.theta, case.kernel, case.grid.h, ctx)  # pageable output
    oh = CanonicalTensor3([torch.empty((ra * rb, 1025), dtype=torch.float64).pin_memory().numpy().T
                           for _ in range(3)], np.zeros(ra * rb))
    ctx.transfer_bytes()
    hartree_potential(case.theta, case.kernel, case.grid.h, ctx, out=oh)
    h2d, d2h = ctx.transfer_bytes()
    distinct = len({case.kernel.tensor.factor[0][:, j].tobytes() for j in range(rb)})
    assert d2h == 3 * 1025 * ra * distinct * 8 < 3 * 1025 * ra * rb * 8
    for ax in range(3):
        assert np.array_equal(oh.factor[ax], ref.factor[ax])
    assert np.array_equal(oh.weight, ref.weight)


def test_host_path_pinned_pieces_and_mixed_extents(ctx):
    """Host-memory convolve into PINNED outputs at the config-2 extent: a representative block
    (n * ra * 8 = 5.2 MB) leaves the device in 4 MB pieces (capi.cpp) and each piece's twin is
    written as it lands (hostcopy.cpp SpinCopyPool, non-temporal stores) - bit-identical to the
    pageable path's whole-factor copy.  Extents (16385, 16385, 16383): device-resident, the
    first two axes share one spectrum launch and one pair launch of the N = 12288 plan and the
    third runs alone; the host path convolves axis by axis - the same bits either way."""
    import torch

    dims = (16385, 16385, 16383)
    ra = 40
    rng = Rng(777)
    a = CanonicalTensor3([np.asfortranarray(rng.normal(d * ra).reshape(d, ra, order="F")) for d in dims],
                         rng.normal(ra))
    fb = []
    for d in dims:
        x = np.arange(d) - 0.5 * (d - 1)
        g = np.exp(-(x / 700.0) ** 2)
        fb.append(np.asfortranarray(np.stack([g, np.exp(-(x / 200.0) ** 2), g.copy()], axis=1)))  # columns 0 and 2: twins
    b = CanonicalTensor3(fb, np.ones(3))
    h = (0.011, 0.013, 0.017)
    ref = convolve(a, b, h, ctx)  # pageable output
    oh = CanonicalTensor3([torch.empty((ra * 3, d), dtype=torch.float64).pin_memory().numpy().T for d in dims],
                          np.zeros(ra * 3))
    for f in oh.factor:
        f[:] = np.nan
    ctx.transfer_bytes()
    convolve(a, b, h, ctx, out=oh)
    _, d2h = ctx.transfer_bytes()
    assert d2h == sum(d * ra * 2 * 8 for d in dims)  # two distinct kernel columns per axis cross PCIe
    for ax, d in enumerate(dims):
        assert np.array_equal(oh.factor[ax], ref.factor[ax])
        assert np.array_equal(oh.factor[ax][:, :ra], oh.factor[ax][:, 2 * ra:])
        for i, j in ((0, 0), (1, 1), (ra - 1, 2)):
            want = O.conv_central_many(np.asfortranarray(a.factor[ax][:, [i]]), np.ascontiguousarray(fb[ax][:, j]))[:, 0]
            assert relmax(oh.factor[ax][:, i + ra * j], h[ax] * want) <= TOL, (ax, i, j)
    dv = convolve(DeviceCP.from_host(a), DeviceCP.from_host(b), h, ctx)
    ctx.synchronize()
    back = dv.to_host()
    for ax in range(3):
        assert np.array_equal(back.factor[ax], ref.factor[ax])


def _grouping_case(rng, n, sym):
    """Kernel-side tensor whose columns form groups of bitwise-identical columns
    {1, 5, 7}, {2, 6} and singletons (optionally all mirror-symmetric)."""
    rb, ra = 9, 3
    fac = []
    for _ in range(3):
        f = rng.normal(n * rb).reshape(n, rb, order="F")
        if sym:
            f = 0.5 * (f + f[::-1])
        f[:, 5] = f[:, 1]
        f[:, 7] = f[:, 1]
        f[:, 6] = f[:, 2]
        fac.append(np.asfortranarray(f))
    b = CanonicalTensor3(fac, rng.uniform(rb) + 0.5)
    a = random_canonical(rng, (n, n, n), ra)
    return a, b


@pytest.mark.parametrize("n", [257, 1025, 16385])  # one-launch grouping / fused into the N = 800 spectra / 3 kernels
@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("weak", [False, True])  # weak: every hash collides -> the verified re-search path
def test_kernel_column_grouping_paths(ctx, monkeypatch, n, sym, weak):
    if weak:
        monkeypatch.setenv("TGB_COLHASH_WEAK", "1")
    rng = Rng(424242 + n + 2 * sym)
    a, b = _grouping_case(rng, n, sym)
    h = (0.3, 0.25, 0.2)
    c = convolve(a, b, h, ctx)
    oc = O.convolve(O.OCP.from_cp(a), O.OCP.from_cp(b), h)
    ra = a.rank()
    for ax in range(3):
        assert relmax(c.factor[ax], oc.factors()[ax]) <= TOL
        blk = lambda j: c.factor[ax][:, j * ra:(j + 1) * ra]  # noqa: E731
        assert np.array_equal(blk(1), blk(5)) and np.array_equal(blk(1), blk(7)) and np.array_equal(blk(2), blk(6))

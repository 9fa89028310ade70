"""Memory-safety evidence without compute-sanitizer (closed on this pool): every
output element is written and nothing depends on prior buffer or workspace
contents, on every convolution plan (direct, generic mixed-radix, the fused
N = 800 small plan, N = 12288 / 12800 static plans, the split large-n plan).

* outputs pre-filled with NaN come back finite and bitwise equal to a clean run;
* a call after another call with different data on the same context (same
  shapes, so every workspace is reused) equals the same call on a fresh
  context, bit for bit;
* the grouping's per-context ticket counters survive interleaved shapes."""
import numpy as np
import pytest

import paper_1504_06289_b200 as tg
from paper_1504_06289_b200 import CanonicalTensor3, DeviceCP, hartree_potential
from paper_1504_06289_b200.inputs import hartree_case

pytestmark = pytest.mark.gpu

NS = [65, 127, 257, 1025, 2049, 16384, 16385, 17000, 32769]


def _dev_out(n, rank, fill=None):
    out = DeviceCP.empty([n] * 3, rank)
    if fill is not None:
        for f in out.factor:
            f.fill_(fill)
        out.weight.fill_(fill)
    return out


def _equal(a, b):
    import torch

    torch.cuda.synchronize()
    return all(torch.equal(x, y) for x, y in zip(a.factor, b.factor)) and torch.equal(a.weight, b.weight)


@pytest.mark.parametrize("n", NS)
def test_every_output_element_written(ctx, n):
    import torch

    case = hartree_case(0, n=n, rank=3, nsamples=1)
    dt, dk = DeviceCP.from_host(case.theta), DeviceCP.from_host(case.kernel.tensor)
    R = dt.rank() * dk.rank()
    clean = hartree_potential(dt, dk, case.grid.h, ctx, out=_dev_out(n, R))
    dirty = hartree_potential(dt, dk, case.grid.h, ctx, out=_dev_out(n, R, float("nan")))
    torch.cuda.synchronize()
    for f in dirty.factor:
        assert bool(torch.isfinite(f).all())
    assert _equal(clean, dirty)


def _other(theta):
    """Same shapes, different data: columns reversed and rescaled."""
    return CanonicalTensor3([np.asfortranarray(1.5 * f[:, ::-1]) for f in theta.factor], theta.weight[::-1].copy())


@pytest.mark.parametrize("n", [257, 1025, 2049, 16385, 32769])
def test_no_state_carried_between_calls(n):
    case = hartree_case(0, n=n, rank=4, nsamples=1)
    first = DeviceCP.from_host(case.theta)
    second = DeviceCP.from_host(_other(case.theta))
    dk = DeviceCP.from_host(case.kernel.tensor)
    R = first.rank() * dk.rank()
    used = tg.Context(0)
    hartree_potential(first, dk, case.grid.h, used, out=_dev_out(n, R))
    got = hartree_potential(second, dk, case.grid.h, used, out=_dev_out(n, R))
    fresh = tg.Context(0)
    ref = hartree_potential(second, dk, case.grid.h, fresh, out=_dev_out(n, R))
    assert _equal(got, ref)


def test_interleaved_shapes_share_context(ctx):
    # alternating plans (fused small plan with its self-resetting tickets, generic, k12) on one context
    ref = {}
    for rep in range(2):
        for n in (1025, 257, 16385, 1025):
            case = hartree_case(0, n=n, rank=2, nsamples=1)
            dt, dk = DeviceCP.from_host(case.theta), DeviceCP.from_host(case.kernel.tensor)
            o = hartree_potential(dt, dk, case.grid.h, ctx, out=_dev_out(n, dt.rank() * dk.rank(), float("nan")))
            if n in ref:
                assert _equal(o, ref[n])
            else:
                ref[n] = o

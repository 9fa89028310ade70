"""Multi-GPU plumbing for the hot path (one process per GPU).

The rank-pair batch of tg::convolve shards naturally: rank r
owns a contiguous block of density columns i, replicates the (few) kernel
columns and produces the output columns i + R_a*j for its i-block with no
data-path exchange — the factor matrices stay sharded on the devices.  The
one real exchange is a reduction: quantities that sum over all rank pairs
(V_H at sample points, partial J blocks) are combined with a single
all-reduce (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of `total` items for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad rank/world")
    return rank * total // world, (rank + 1) * total // world


def shard_canonical(t, rank: int, world: int):
    """Density-side shard of a CanonicalTensor3 (columns lo:hi of every factor)."""
    from .tengrid import CanonicalTensor3

    lo, hi = shard_range(t.rank(), rank, world)
    return CanonicalTensor3([f[:, lo:hi] for f in t.factor], t.weight[lo:hi]), (lo, hi)


def global_columns(lo: int, hi: int, ra_total: int, rb: int) -> np.ndarray:
    """Global output-column indices (i + R_a*j) of a shard's local columns
    (local index i_loc + (hi-lo)*j), for gathering / validation."""
    ra = hi - lo
    loc = np.arange(ra * rb)
    i_loc, j = loc % ra, loc // ra
    return (lo + i_loc) + ra_total * j


def allreduce_sum(x, group=None):
    """Sum a tensor/ndarray over all ranks in place (torch.distributed)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    if isinstance(x, np.ndarray):
        t = torch.from_numpy(x)
        dist.all_reduce(t, group=group)
        return t.numpy()
    dist.all_reduce(x, group=group)
    return x


def sharded_coulomb_matrix(bs, disc: list, theta, kernel, ctx=None, group=None, coulomb=None, hartree=None):
    """J_km = h^3 <G_k . G_m, V_H> (hf.cpp:140-151) with the density columns
    sharded over the ranks of `group`: each rank convolves its shard of theta
    (its V_H columns, no exchange), assembles the partial J over those columns,
    and ONE all-reduce of the N_b x N_b partials gives J on every rank (the
    north-star's single allreduce of J blocks).  Exact symmetry survives: every
    partial is mirrored before the sum.  `coulomb` / `hartree` default to the
    libtgb operators (overridable so the CPU gloo test can stand the oracle in
    for the per-rank GPU)."""
    import torch.distributed as dist

    from . import tengrid as tg

    rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    theta_r, _ = shard_canonical(theta, rank, world)
    hartree = hartree or (lambda t: tg.hartree_potential(t, kernel, bs.grid.h, ctx))
    coulomb = coulomb or (lambda v: tg.coulomb_matrix(bs, disc, v, ctx))
    nb = len(disc)
    part = coulomb(hartree(theta_r)) if theta_r.rank() else np.zeros((nb, nb))
    return allreduce_sum(np.ascontiguousarray(part, dtype=np.float64), group)

"""World-size-2 gloo test of the N>1 host logic (CPU): density columns are
sharded across ranks, each rank's convolution output (computed here by the
oracle restatement, standing in for the per-rank GPU) is evaluated at the
shared sample points, and one all-reduce of the partial sums must reproduce
the unsharded result; shards cover every output column exactly once."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1504_06289_b200.shard import global_columns, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_1504_06289_b200.inputs import hartree_case
        from paper_1504_06289_b200.shard import allreduce_sum, shard_canonical, torch_comm

        comm = torch_comm()
        case = hartree_case(0, n=65, rank=7, nsamples=40)
        theta_r, (lo, hi) = shard_canonical(case.theta, rank, world)
        vh = O.hartree_potential(O.OCP.from_cp(theta_r), O.OCP.from_cp(case.kernel.tensor), case.grid.h)
        part = O.value_at(vh, case.samples) if theta_r.rank() else np.zeros(len(case.samples))
        total = allreduce_sum(np.ascontiguousarray(part), comm)  # libtgb tgb_comm_allreduce_host
        if rank == 0:
            full = O.hartree_potential(O.OCP.from_cp(case.theta), O.OCP.from_cp(case.kernel.tensor), case.grid.h)
            ref = O.value_at(full, case.samples)
            q.put(float(np.abs(total - ref).max() / np.abs(ref).max()))
    finally:
        dist.destroy_process_group()


def test_sharded_partial_sums_allreduce_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    err = q.get(timeout=10)
    assert err <= 1e-13


@pytest.mark.parametrize("total,world", [(500, 1), (500, 2), (500, 8), (7, 3), (3, 8)])
def test_shards_cover_every_column_once(total, world):
    rb = 5
    seen = []
    for r in range(world):
        lo, hi = shard_range(total, r, world)
        assert 0 <= lo <= hi <= total
        seen.append(global_columns(lo, hi, total, rb))
    allc = np.sort(np.concatenate(seen))
    assert np.array_equal(allc, np.arange(total * rb))


def _worker_j(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from hf_case import functions, load
        from oracle import oracle as O
        from paper_1504_06289_b200.shard import sharded_coulomb_matrix
        import paper_1504_06289_b200 as tg

        g = load()
        b, n = g["b_half"], g["n"]
        theta = tg.CanonicalTensor3([g[f"theta_f{ax}"] for ax in range(3)], g["theta_w"])
        m, c0 = int(g["kernel_m_c0"][0]), float(g["kernel_m_c0"][1])
        nodes, w = O.make_expsum(m, c0)[:2]
        kern = O.kernel_tensor(b, n, nodes, w, False)
        disc = O.discretize_basis(b, n, functions(g))
        hh = 2.0 * np.asarray(b) / (np.asarray(n) + 1)
        J = sharded_coulomb_matrix(
            None, disc, theta, None,
            hartree=lambda t: O.hartree_potential(O.OCP.from_cp(t), kern, hh),
            coulomb=lambda v: O.coulomb_matrix(b, n, disc, v))
        if rank == 0:
            q.put((float(np.abs(J - g["J"]).max() / np.abs(g["J"]).max()), bool(np.array_equal(J, J.T))))
    finally:
        dist.destroy_process_group()


def test_sharded_coulomb_allreduce_gloo():
    """J from density-column shards + one all-reduce equals the reference's own J (hf.cpp:140-151)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_j, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    err, sym = q.get(timeout=10)
    assert err <= 1e-12 and sym


def _worker_sym(rank, world, port, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1504_06289_b200.shard import symmetric_allreduce, torch_comm

        nb = 9
        rng = np.random.default_rng(100 + rank)
        part = rng.standard_normal((nb, nb))
        part = np.asfortranarray(part + part.T)
        J = symmetric_allreduce(part, torch_comm())
        if rank == 0:
            parts = []
            for r in range(world):
                p = np.random.default_rng(100 + r).standard_normal((nb, nb))
                parts.append(p + p.T)
            ref = np.sum(parts, axis=0)
            q.put((float(np.abs(J - ref).max()), bool(np.array_equal(J, J.T))))
    finally:
        dist.destroy_process_group()


def test_symmetric_allreduce_gloo_world3():
    """libtgb's tgb_symmetric_allreduce_host over a torch.distributed (gloo)
    tgb_comm at world size 3: the sum of the partial J blocks, exactly
    symmetric whatever order the backend summed J_km and J_mk in."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sym, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    err, sym = q.get(timeout=10)
    assert err <= 1e-13 and sym


def test_shard_range_is_libtgb():
    """shard_range comes from the C-ABI (tgb_shard_range) and rejects bad ranks."""
    from paper_1504_06289_b200 import InvalidArgument

    assert shard_range(500, 7, 8) == (437, 500)
    with pytest.raises(InvalidArgument):
        shard_range(10, 2, 2)

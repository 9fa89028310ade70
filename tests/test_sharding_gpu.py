"""The multi-GPU C-ABI (include/tgb.h "multi-GPU", csrc/comm.cpp) driven end to
end through libtgb's real kernels: two processes on one GPU, each with its own
context and a torch.distributed (gloo) tgb_comm, run tgb_hartree_potential_shard
on their density-column blocks, then tgb_value_at_allreduce and
tgb_coulomb_matrix_allreduce.  The all-reduce is host-side (gloo), so the two
processes' kernels never wait on each other.  Results must equal the
single-process path (V_H samples at 1e-12, J at 1e-12 and exactly symmetric)
and the reference's own J (reference_hf.npz, hf.cpp:140-151) at 1e-10."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path

    here = Path(__file__).resolve().parent
    sys.path.insert(0, str(here.parent))
    sys.path.insert(0, str(here))
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1504_06289_b200 as tg
        from hf_case import load, product_case
        from paper_1504_06289_b200 import shard
        from paper_1504_06289_b200.inputs import hartree_case

        ctx = tg.Context(0)
        comm = shard.torch_comm()
        shard.set_comm(ctx, comm)
        assert shard.comm_info(ctx) == (rank, world)
        # V_H samples (config-0 shape, reduced): sharded convolution + one all-reduce
        case = hartree_case(0, n=129, rank=9, nsamples=64)
        d_theta = tg.DeviceCP.from_host(case.theta)
        d_kern = tg.DeviceCP.from_host(case.kernel.tensor)
        out = shard.hartree_potential_shard(d_theta, d_kern, case.grid.h, ctx)
        lo, hi = shard.shard_range(case.theta.rank(), rank, world)
        assert out.rank() == (hi - lo) * case.kernel.rank()
        vals = shard.value_at_allreduce(out, case.samples, ctx).cpu().numpy()
        # J from the reference fixture's unreduced density, V_H sharded by density column
        g = load()
        bs, disc, kp, _ = product_case(g)
        theta = tg.CanonicalTensor3([g[f"theta_f{ax}"] for ax in range(3)], g["theta_w"])
        vh_shard = shard.hartree_potential_shard(tg.DeviceCP.from_host(theta), tg.DeviceCP.from_host(kp.tensor),
                                                 bs.grid.h, ctx)
        J = shard.coulomb_matrix_allreduce(bs, disc, vh_shard, ctx)
        torch.cuda.synchronize()
        if rank == 0:
            ref_ctx = tg.Context(0)  # single process, no communicator
            full = tg.hartree_potential(d_theta, d_kern, case.grid.h, ref_ctx)
            ref_vals = tg.value_at_points(full, case.samples, ref_ctx).cpu().numpy()
            J1 = tg.coulomb_matrix(bs, disc, tg.hartree_potential(theta, kp, bs.grid.h, ref_ctx), ref_ctx)
            q.put((float(np.abs(vals - ref_vals).max() / np.abs(ref_vals).max()),
                   float(np.abs(J - J1).max() / np.abs(J1).max()),
                   float(np.abs(J - g["J"]).max() / np.abs(g["J"]).max()),
                   bool(np.array_equal(J, J.T))))
        shard.set_comm(ctx, None)
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_sharded_hartree_and_coulomb_two_processes_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    e_vals, e_j1, e_ref, sym = q.get(timeout=10)
    assert e_vals <= 1e-12
    assert e_j1 <= 1e-12
    assert e_ref <= 1e-10
    assert sym


def test_nccl_single_rank_context(ctx):
    """libtgb's own NCCL communicator (dlopen of libnccl.so.2): world 1 is a no-op sum."""
    import torch

    from paper_1504_06289_b200 import shard

    uid = shard.nccl_unique_id()
    assert len(uid) == 128
    shard.init_nccl(ctx, 0, 1, uid)
    assert shard.comm_info(ctx) == (0, 1)
    import paper_1504_06289_b200 as tg
    from paper_1504_06289_b200.inputs import hartree_case

    case = hartree_case(0, n=65, rank=3, nsamples=16)
    out = shard.hartree_potential_shard(tg.DeviceCP.from_host(case.theta), tg.DeviceCP.from_host(case.kernel.tensor),
                                        case.grid.h, ctx)
    v = shard.value_at_allreduce(out, case.samples, ctx)
    ref = tg.value_at_points(out, torch.as_tensor(case.samples).cuda(), ctx)
    assert torch.equal(v, ref)
    shard.set_comm(ctx, None)


def _worker_tei(rank, world, port, q):
    import sys
    from pathlib import Path

    here = Path(__file__).resolve().parent
    sys.path.insert(0, str(here.parent))
    sys.path.insert(0, str(here))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1504_06289_b200 as tg
        from paper_1504_06289_b200 import shard
        from paper_1504_06289_b200.inputs import Rng
        from test_tei_gpu import make_basis

        rng = Rng(12)
        cents = rng.uniform(6, -1.5, 1.5).reshape(2, 3)
        bs = make_basis(65, 7.0, cents, ("s", "p"), rng)
        kern = tg.kernel_tensor(bs.grid, tg.make_expsum(10, 0.9), False)
        disc = tg.discretize_basis(bs)

        def run(ctx):
            fac = tg.TEIFactorization(ctx)
            tg.tei_density_fitting(fac, bs, disc, 1e-6)
            tg.tei_convolution_matrices(fac, kern)
            conv = [fac.conv(k, ax) for k in range(kern.rank()) for ax in range(3)]
            d = tg.tei_diagonal(fac)
            tg.tei_cholesky(fac, 1e-8)
            return fac.fit_ranks(), conv, d, fac.rank_b(), list(fac.pivots), np.array(fac.chol)

        ctx = tg.Context(0)
        comm = shard.torch_comm()
        shard.set_comm(ctx, comm)
        got = run(ctx)
        shard.set_comm(ctx, None)
        if rank == 0:
            ref = run(tg.Context(0))
            same = (got[0] == ref[0] and all(np.array_equal(a, b) for a, b in zip(got[1], ref[1]))
                    and np.array_equal(got[2], ref[2]) and got[3] == ref[3] and got[4] == ref[4]
                    and np.array_equal(got[5], ref[5]))
            q.put((bool(same), got[3]))
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_sharded_tei_two_processes_bit_identical():
    """TEI sharded per SURVEY §8e over a gloo tgb_comm: convolution matrices by
    kernel-term pair, the diagonal by pair rows, one all-reduce each; the
    pivoted Cholesky replicated.  Fit ranks, every M_k, the diagonal, R_B, the
    pivot sequence and L are bit-identical to one process."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_tei, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    same, rb = q.get(timeout=10)
    assert same and rb > 1

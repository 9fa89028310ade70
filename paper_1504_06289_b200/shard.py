"""Multi-GPU plumbing for the hot path (one process per GPU) — the Python side
of libtgb's communicator API (include/tgb.h, "multi-GPU"; csrc/comm.cpp).

The rank-pair batch of tg::convolve shards naturally: rank r
owns a contiguous block of density columns i (tgb_shard_range), replicates the
(few) kernel columns and produces the output columns i + R_a*j for its i-block
with no data-path exchange — the factor matrices stay sharded on the devices.
The one real exchange is a reduction: quantities that sum over all rank pairs
(V_H at sample points, partial J blocks, the k-sharded TEI convolution
matrices) are combined by ONE all-reduce inside libtgb, over either the
context's own NCCL communicator (Context.init_nccl) or a caller-supplied
tgb_comm (torch_comm: any torch.distributed backend, gloo in the CPU tests).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import ALLREDUCE_FN, MEM_DEVICE, MEM_HOST, check, lib, tgb_comm


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of `total` items for `rank` (sizes differ by <= 1): tgb_shard_range."""
    lo, hi = C.c_int64(), C.c_int64()
    check(lib().tgb_shard_range(int(total), int(rank), int(world), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


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


class _CudaBuf:
    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 3}


class TorchComm:
    """A tgb_comm whose allreduce_sum runs torch.distributed.all_reduce on
    `group` (gloo: host tensors; nccl: device tensors, staged as needed).  Keep
    the object alive while a context uses it."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.backend = dist.get_backend(group)
        self._fn = ALLREDUCE_FN(self._allreduce)
        self.c = tgb_comm(dist.get_rank(group), dist.get_world_size(group), self._fn, None)

    def _allreduce(self, buf, count, on_device, stream, user) -> int:
        try:
            import torch
            import torch.distributed as dist

            n = int(count)
            if on_device:
                if stream:
                    torch.cuda.ExternalStream(stream).synchronize()
                t = torch.as_tensor(_CudaBuf(C.cast(buf, C.c_void_p).value, n), device="cuda")
                if self.backend == "nccl":
                    dist.all_reduce(t, group=self.group)
                    torch.cuda.synchronize()
                else:
                    h = t.cpu()
                    dist.all_reduce(h, group=self.group)
                    t.copy_(h)
                    torch.cuda.synchronize()
            else:
                h = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n,)))
                if self.backend == "nccl":
                    d = h.cuda()
                    dist.all_reduce(d, group=self.group)
                    h.copy_(d.cpu())
                else:
                    dist.all_reduce(h, group=self.group)
            return 0
        except Exception:  # noqa: BLE001 — reported to libtgb as a failed callback
            return 1


def torch_comm(group=None) -> TorchComm:
    return TorchComm(group)


def nccl_unique_id() -> bytes:
    """tgb_nccl_get_unique_id (rank 0), to be broadcast to the other ranks."""
    buf = (C.c_ubyte * 128)()
    check(lib().tgb_nccl_get_unique_id(buf))
    return bytes(buf)


def init_nccl(ctx, rank: int, world: int, uid: bytes) -> None:
    """tgb_ctx_init_nccl: a libtgb-owned NCCL communicator on `ctx`."""
    buf = (C.c_ubyte * 128).from_buffer_copy(uid)
    check(lib().tgb_ctx_init_nccl(ctx.handle, rank, world, buf))


def init_nccl_from_torch(ctx, group=None) -> None:
    """Rank 0 creates the NCCL id; torch.distributed broadcasts it (any backend)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, 0, group=group)
    init_nccl(ctx, rank, world, bytes(t.cpu().numpy().tobytes()))


def set_comm(ctx, comm: TorchComm | None) -> None:
    """tgb_ctx_set_comm (None detaches)."""
    check(lib().tgb_ctx_set_comm(ctx.handle, C.byref(comm.c) if comm is not None else None))
    ctx._comm = comm  # keep the callback alive


def comm_info(ctx) -> tuple[int, int]:
    r, w = C.c_int(), C.c_int()
    check(lib().tgb_ctx_comm_info(ctx.handle, C.byref(r), C.byref(w)))
    return r.value, w.value


def allreduce_sum(x, comm: TorchComm | None = None):
    """Sum a host float64 array over all ranks in place through libtgb's
    tgb_comm_allreduce_host (no-op without a communicator)."""
    if comm is None:
        return x
    a = np.ascontiguousarray(x, dtype=np.float64)
    check(lib().tgb_comm_allreduce_host(C.byref(comm.c), a.ctypes.data, a.size))
    return a


def symmetric_allreduce(J, comm: TorchComm | None = None):
    """tgb_symmetric_allreduce_host: sum an N x N partial over the ranks, then
    mirror the upper triangle (J exactly symmetric, hf.cpp:145-149)."""
    a = np.asfortranarray(J, dtype=np.float64).copy(order="F")
    if comm is None:
        single = tgb_comm(0, 1, ALLREDUCE_FN(), None)
        check(lib().tgb_symmetric_allreduce_host(C.byref(single), a.ctypes.data, a.shape[0]))
        return a
    check(lib().tgb_symmetric_allreduce_host(C.byref(comm.c), a.ctypes.data, a.shape[0]))
    return a


# --------------------------------------------------------------------------- sharded operators (device path)

def hartree_potential_shard(theta, kernel, h, ctx, out=None):
    """tgb_hartree_potential_shard: this rank's density columns x the whole kernel."""
    from .tengrid import KernelTensor, _h3, _mem, _out_like, _stream_enter, _stream_order

    if isinstance(kernel, KernelTensor):
        kernel = kernel.tensor
    r, w = comm_info(ctx)
    lo, hi = shard_range(theta.rank(), r, w)
    mem = _mem(theta, kernel)
    if out is None:
        out = _out_like(theta, (hi - lo) * kernel.rank(), mem)
    ct, ck, co = theta._cstruct(), kernel._cstruct(), out._cstruct()
    if mem == MEM_DEVICE:
        _stream_enter(ctx)
    check(lib().tgb_hartree_potential_shard(ctx.handle, C.byref(ct), C.byref(ck), _h3(h).ctypes.data, C.byref(co), mem))
    if mem == MEM_DEVICE:
        _stream_order(ctx, theta, kernel, out)
    return out


def value_at_allreduce(t_shard, ijk, ctx):
    """tgb_value_at_allreduce: sum over the ranks' shards of value_at (device tensors)."""
    import torch

    ct = t_shard._cstruct()
    pts = ijk if isinstance(ijk, torch.Tensor) else torch.as_tensor(np.asarray(ijk, dtype=np.int64))
    pts = pts.to(device=t_shard.weight.device, dtype=torch.int64).contiguous()
    out = torch.empty(pts.shape[0], dtype=torch.float64, device=t_shard.weight.device)
    from .tengrid import _stream_enter

    _stream_enter(ctx)
    check(lib().tgb_value_at_allreduce(ctx.handle, C.byref(ct), pts.shape[0], pts.data_ptr(), out.data_ptr(),
                                       MEM_DEVICE))
    from .tengrid import _stream_order

    _stream_order(ctx, t_shard, pts, out)
    return out


def coulomb_matrix_allreduce(bs, disc: list, vh_shard, ctx) -> np.ndarray:
    """tgb_coulomb_matrix_allreduce: partial J over this rank's V_H columns, one all-reduce, exact mirror."""
    from .tengrid import DeviceCP, _h3, flatten_basis

    flat, offs = flatten_basis(disc)
    nb = len(disc)
    J = np.zeros((nb, nb), order="F")
    if isinstance(vh_shard, DeviceCP):
        flat = DeviceCP.from_host(flat, device=vh_shard.weight.device)
        mem = MEM_DEVICE
        import torch

        Jd = torch.empty((nb, nb), dtype=torch.float64, device=vh_shard.weight.device)
        cf, cv = flat._cstruct(), vh_shard._cstruct()
        check(lib().tgb_coulomb_matrix_allreduce(ctx.handle, C.byref(cf), offs.ctypes.data, nb, C.byref(cv),
                                                 _h3(bs.grid.h).ctypes.data, Jd.data_ptr(), mem))
        return Jd.cpu().numpy().T.copy(order="F")
    cf, cv = flat._cstruct(), vh_shard._cstruct()
    check(lib().tgb_coulomb_matrix_allreduce(ctx.handle, C.byref(cf), offs.ctypes.data, nb, C.byref(cv),
                                             _h3(bs.grid.h).ctypes.data, J.ctypes.data, MEM_HOST))
    return J


def sharded_coulomb_matrix(bs, disc: list, theta, kernel, ctx=None, group=None, coulomb=None, hartree=None,
                           comm: TorchComm | None = None):
    """J_km = h^3 <G_k . G_m, V_H> (hf.cpp:140-151) with the density columns
    sharded over the ranks of `group`: each rank convolves its shard of theta
    (its V_H columns, no exchange), assembles the partial J over those columns,
    and ONE all-reduce of the N_b x N_b partials (libtgb's
    tgb_symmetric_allreduce_host, which also restores exact symmetry) gives J
    on every rank.  `coulomb` / `hartree` default to the libtgb operators
    (overridable so the CPU gloo test can stand the oracle in for each rank's
    GPU; the reduction and the shard ranges are libtgb's either way)."""
    import torch.distributed as dist

    from . import tengrid as tg

    on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if on else 0
    world = dist.get_world_size(group) if on else 1
    if comm is None and on and world > 1:
        comm = torch_comm(group)
    theta_r, _ = shard_canonical(theta, rank, world)
    hartree = hartree or (lambda t: tg.hartree_potential(t, kernel, bs.grid.h, ctx))
    coulomb = coulomb or (lambda v: tg.coulomb_matrix(bs, disc, v, ctx))
    nb = len(disc)
    part = coulomb(hartree(theta_r)) if theta_r.rank() else np.zeros((nb, nb))
    return symmetric_allreduce(np.asfortranarray(part, dtype=np.float64), comm)

"""Python mirror of the reference `tengrid` API for the hot path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/tengrid/{grid,tensor,fft,kernel,basis,hf,lattice}.hpp
so parity tests read like the reference's own doctest suites.  Every compute
call goes through libtgb.so (include/tgb.h); host-side input producers
(make_expsum, kernel_tensor, discretize_basis, window_offset) go through the
same library's C++ restatements (include/tgb_host.h).

Layout: a factor matrix is a float64 array of shape (n, R) in Fortran
(column-major) order, exactly Eigen::MatrixXd's memory layout.  Device-
resident tensors (DeviceCP) hold torch CUDA tensors of shape (R, n), which is
the same memory layout.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from ._lib import (MEM_DEVICE, MEM_HOST, InvalidArgument, check, lib, tgb_cp)

# --------------------------------------------------------------------------- context


class Context:
    """One libtgb context (CUDA stream + workspace) per device (tgb.h)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._h = C.c_void_p()
        check(lib().tgb_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(self._h)))
        self.device = device

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return lib().tgb_ctx_stream(self._h) or 0

    def synchronize(self) -> None:
        check(lib().tgb_ctx_synchronize(self._h))

    def launch_count(self) -> int:
        return lib().tgb_ctx_launch_count(self._h)

    def reset_launch_count(self) -> None:
        lib().tgb_ctx_reset_launch_count(self._h)

    def set_direct_max(self, n: int) -> None:
        check(lib().tgb_ctx_set_direct_max(self._h, n))

    def transfer_bytes(self) -> tuple[int, int]:
        """(H2D, D2H) bytes moved by host-memory calls since the last read (tgb_ctx_transfer_bytes)."""
        h, d = C.c_int64(), C.c_int64()
        check(lib().tgb_ctx_transfer_bytes(self._h, C.byref(h), C.byref(d)))
        return h.value, d.value

    def probe_fp64_peak(self) -> float:
        """Measured FP64 DFMA rate of the device in TFLOP/s (tgb_probe_fp64_peak)."""
        t = C.c_double()
        check(lib().tgb_probe_fp64_peak(self._h, C.byref(t)))
        return t.value

    def set_profiling(self, enabled: bool) -> None:
        check(lib().tgb_ctx_set_profiling(self._h, int(enabled)))

    def profile_read(self) -> tuple[float, int]:
        """(summed device ms, launches) of the pair convolution kernel since the last read."""
        ms, cnt = C.c_double(), C.c_int64()
        check(lib().tgb_ctx_profile_read(self._h, C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def torch_stream(self):
        """This context's stream as a torch ExternalStream (cached)."""
        import torch

        if getattr(self, "_tstream", None) is None:
            self._tstream = torch.cuda.ExternalStream(self.stream, device=torch.device("cuda", self.device))
        return self._tstream

    def close(self) -> None:
        if self._h:
            check(lib().tgb_ctx_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# --------------------------------------------------------------------------- tensors


def _fmat(a, rows: int | None = None, cols: int | None = None) -> np.ndarray:
    m = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if m.ndim == 1:
        m = m.reshape(-1, 1, order="F")
    return m


@dataclass
class CanonicalTensor3:
    """tensor.hpp:119-150 — sum_k w_k u_k^(1) x u_k^(2) x u_k^(3)."""

    factor: list = field(default_factory=list)
    weight: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def __post_init__(self):
        self.factor = [_fmat(f) for f in self.factor]
        self.weight = np.ascontiguousarray(np.asarray(self.weight, dtype=np.float64).reshape(-1))

    @staticmethod
    def zero(dims: Sequence[int]) -> "CanonicalTensor3":
        return CanonicalTensor3([np.zeros((d, 0), order="F") for d in dims], np.zeros(0))

    def rank(self) -> int:
        return int(self.weight.shape[0])

    def extent(self, ax: int) -> int:
        return int(self.factor[ax].shape[0])

    def extents(self) -> tuple[int, int, int]:
        return (self.extent(0), self.extent(1), self.extent(2))

    def check_valid(self) -> None:
        for f in self.factor:
            if f.shape[1] != self.rank():
                raise InvalidArgument("CanonicalTensor3: factor/weight rank mismatch")

    def value_at(self, i: int, j: int, k: int) -> float:
        return float(np.sum(self.weight * self.factor[0][i] * self.factor[1][j] * self.factor[2][k]))

    def to_dense(self) -> np.ndarray:
        """Column-major dense image (index i1 + n1*(i2 + n2*i3)), small sizes only."""
        return np.einsum("k,ik,jk,lk->ijl", self.weight, *self.factor)

    def normalize(self) -> None:
        """tensor.cpp:18-31."""
        self.check_valid()
        for k in range(self.rank()):
            for ax in range(3):
                nrm = float(np.sqrt(np.sum(self.factor[ax][:, k] ** 2)))
                if nrm > 0.0:
                    self.factor[ax][:, k] /= nrm
                    self.weight[k] *= nrm
                else:
                    self.weight[k] = 0.0

    def _cstruct(self) -> tgb_cp:
        s = tgb_cp()
        for ax in range(3):
            s.n[ax] = self.extent(ax)
            s.factor[ax] = self.factor[ax].ctypes.data if self.factor[ax].size else None
        s.rank = self.rank()
        s.weight = self.weight.ctypes.data if self.rank() else None
        return s


class DeviceCP:
    """Device-resident canonical tensor: torch CUDA tensors, factor[ax] of
    shape (R, n) (= column-major n x R), weight (R,)."""

    def __init__(self, factor, weight):
        self.factor = list(factor)
        self.weight = weight

    @staticmethod
    def from_host(t: CanonicalTensor3, device="cuda", share_equal_axes: bool = False) -> "DeviceCP":
        """share_equal_axes: axes whose factor matrices are bitwise equal (the Newton kernel on a
        cubic grid) share ONE device matrix; libtgb then forms that matrix's spectra once.  Only for
        tensors that are not modified in place afterwards."""
        import torch

        f = []
        for ax, x in enumerate(t.factor):
            src = next((j for j in range(ax) if share_equal_axes and t.factor[j].shape == x.shape
                        and np.array_equal(t.factor[j], x)), None)
            f.append(f[src] if src is not None else torch.from_numpy(np.ascontiguousarray(x.T)).to(device))
        return DeviceCP(f, torch.from_numpy(t.weight.copy()).to(device))

    @staticmethod
    def empty(dims: Sequence[int], rank: int, device="cuda") -> "DeviceCP":
        import torch

        f = [torch.empty((rank, d), dtype=torch.float64, device=device) for d in dims]
        return DeviceCP(f, torch.empty(rank, dtype=torch.float64, device=device))

    def rank(self) -> int:
        return int(self.weight.shape[0])

    def extent(self, ax: int) -> int:
        return int(self.factor[ax].shape[1])

    def to_host(self) -> CanonicalTensor3:
        return CanonicalTensor3([np.asfortranarray(f.cpu().numpy().T) for f in self.factor],
                                self.weight.cpu().numpy())

    def _cstruct(self) -> tgb_cp:
        s = tgb_cp()
        for ax in range(3):
            s.n[ax] = self.extent(ax)
            s.factor[ax] = self.factor[ax].data_ptr() if self.factor[ax].numel() else None
        s.rank = self.rank()
        s.weight = self.weight.data_ptr() if self.rank() else None
        return s


def _stream_order(ctx: "Context", *objs) -> None:
    """Device calls run asynchronously on the context's stream: order torch's
    current stream after the call, so torch ops reading the results see them
    and memory the caching allocator hands out again on that stream (a freed
    input, say) is not overwritten while the call still reads it.  The calls
    themselves first wait for torch's current stream (_stream_enter)."""
    import torch

    if not any(isinstance(o, (DeviceCP, torch.Tensor)) for o in objs):
        return
    dev = torch.device("cuda", ctx.device)
    cur = torch.cuda.current_stream(dev)
    s = ctx.torch_stream()
    if cur.cuda_stream != s.cuda_stream:
        cur.wait_stream(s)


def _stream_enter(ctx: "Context") -> None:
    """The context's stream waits for torch's current stream (inputs produced there are ready)."""
    import torch

    dev = torch.device("cuda", ctx.device)
    cur = torch.cuda.current_stream(dev)
    s = ctx.torch_stream()
    if cur.cuda_stream != s.cuda_stream:
        s.wait_stream(cur)


def _mem(*ts) -> int:
    dev = [isinstance(t, DeviceCP) for t in ts]
    if all(dev):
        return MEM_DEVICE
    if not any(dev):
        return MEM_HOST
    raise InvalidArgument("mixing host and device tensors in one call")


def _h3(h) -> np.ndarray:
    if np.isscalar(h):
        return np.array([h, h, h], dtype=np.float64)
    return np.ascontiguousarray(np.asarray(h, dtype=np.float64).reshape(3))


# --------------------------------------------------------------------------- algebra (host, 1D complexity)


def _cp_algebra(fn: str, a, b, rank: int, ctx, alpha: float | None = None):
    """Device-resident CP algebra through the C-ABI (tgb_hadamard / tgb_add / tgb_scale)."""
    ctx = ctx or default_context()
    out = DeviceCP.empty([a.extent(ax) for ax in range(3)], rank, device=a.weight.device)
    ca, co = a._cstruct(), out._cstruct()
    _stream_enter(ctx)
    if fn == "tgb_scale":
        check(lib().tgb_scale(ctx.handle, C.byref(ca), float(alpha), C.byref(co), MEM_DEVICE))
    else:
        cb = b._cstruct()
        check(getattr(lib(), fn)(ctx.handle, C.byref(ca), C.byref(cb), C.byref(co), MEM_DEVICE))
    _stream_order(ctx, a, b, out)
    return out


def hadamard(a, b, ctx: "Context | None" = None):
    """tensor.cpp:141-157 (column i + Ra*j).  Device tensors go through tgb_hadamard."""
    if isinstance(a, DeviceCP) or isinstance(b, DeviceCP):
        _mem(a, b)
        if [a.extent(ax) for ax in range(3)] != [b.extent(ax) for ax in range(3)]:
            raise InvalidArgument("hadamard: extent mismatch")
        return _cp_algebra("tgb_hadamard", a, b, a.rank() * b.rank(), ctx)
    a.check_valid(), b.check_valid()
    if a.extents() != b.extents():
        raise InvalidArgument("hadamard: extent mismatch")
    ra, rb = a.rank(), b.rank()
    f = []
    for ax in range(3):
        m = (a.factor[ax][:, :, None] * b.factor[ax][:, None, :]).reshape(a.extent(ax), ra * rb, order="F")
        f.append(m)
    w = (a.weight[:, None] * b.weight[None, :]).reshape(-1, order="F")
    return CanonicalTensor3(f, w)


def add(a, b, ctx: "Context | None" = None):
    """tensor.cpp:159-171 (concatenation).  Device tensors go through tgb_add."""
    if isinstance(a, DeviceCP) or isinstance(b, DeviceCP):
        _mem(a, b)
        if [a.extent(ax) for ax in range(3)] != [b.extent(ax) for ax in range(3)]:
            raise InvalidArgument("add: extent mismatch")
        return _cp_algebra("tgb_add", a, b, a.rank() + b.rank(), ctx)
    a.check_valid(), b.check_valid()
    if a.extents() != b.extents():
        raise InvalidArgument("add: extent mismatch")
    # Fortran-order result straight from the row stacks of the transposes (no C-order detour)
    return CanonicalTensor3([np.concatenate([a.factor[ax].T, b.factor[ax].T], axis=0).T for ax in range(3)],
                            np.concatenate([a.weight, b.weight]))


def scale(a, alpha: float, ctx: "Context | None" = None):
    """tensor.cpp:173-177 (weights only).  Device tensors go through tgb_scale."""
    if isinstance(a, DeviceCP):
        return _cp_algebra("tgb_scale", a, None, a.rank(), ctx, alpha)
    return CanonicalTensor3([f.copy(order="F") for f in a.factor], a.weight * alpha)


# --------------------------------------------------------------------------- hot path (libtgb)


def conv_central_many(U, v, ctx: Context | None = None) -> np.ndarray:
    """fft.cpp:97-122 — windowed convolution of every column of U with v."""
    ctx = ctx or default_context()
    U = _fmat(U)
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
    n = v.shape[0]
    if U.shape[0] != n:
        raise InvalidArgument("conv_central_many: column length mismatch")
    out = np.zeros((n, U.shape[1]), order="F")
    check(lib().tgb_conv_central_many(ctx.handle, n, U.shape[1], U.ctypes.data if U.size else None, v.ctypes.data,
                                      out.ctypes.data if out.size else None, MEM_HOST))
    return out


def _out_like(a, rank: int, mem: int):
    dims = [a.extent(ax) for ax in range(3)]
    if mem == MEM_DEVICE:
        return DeviceCP.empty(dims, rank, device=a.weight.device)
    return CanonicalTensor3([np.zeros((d, rank), order="F") for d in dims], np.zeros(rank))


def convolve(a, b, h, ctx: Context | None = None, out=None):
    """tensor.cpp:179-198 — rank Ra*Rb tensor-product convolution."""
    ctx = ctx or default_context()
    mem = _mem(a, b)
    hh = _h3(h)
    if out is None:
        out = _out_like(a, a.rank() * b.rank(), mem)
    ca, cb, co = a._cstruct(), b._cstruct(), out._cstruct()
    if mem == MEM_DEVICE:
        _stream_enter(ctx)
    check(lib().tgb_convolve(ctx.handle, C.byref(ca), C.byref(cb), hh.ctypes.data, C.byref(co), mem))
    if mem == MEM_DEVICE:
        _stream_order(ctx, a, b, out)
    return out


def hartree_potential(theta, kernel, h, ctx: Context | None = None, out=None):
    """hf.cpp:131-138 — V_H = convolve(theta, kernel / (h0 h1 h2), h)."""
    if isinstance(kernel, KernelTensor):
        if kernel.doubled:
            raise InvalidArgument("hartree_potential: kernel must live on the primary grid")
        kernel = kernel.tensor
    ctx = ctx or default_context()
    mem = _mem(theta, kernel)
    hh = _h3(h)
    if out is None:
        out = _out_like(theta, theta.rank() * kernel.rank(), mem)
    ct, ck, co = theta._cstruct(), kernel._cstruct(), out._cstruct()
    if mem == MEM_DEVICE:
        _stream_enter(ctx)
    check(lib().tgb_hartree_potential(ctx.handle, C.byref(ct), C.byref(ck), hh.ctypes.data, C.byref(co), mem))
    if mem == MEM_DEVICE:
        _stream_order(ctx, theta, kernel, out)
    return out


def value_at_points(t, ijk, ctx: Context | None = None):
    """tensor.hpp:135-140 batched over points (ijk: (npts, 3) int64)."""
    ctx = ctx or default_context()
    mem = _mem(t)
    ct = t._cstruct()
    if mem == MEM_DEVICE:
        import torch

        pts = ijk if isinstance(ijk, torch.Tensor) else torch.as_tensor(np.asarray(ijk, dtype=np.int64))
        pts = pts.to(device=t.weight.device, dtype=torch.int64).contiguous()
        out = torch.empty(pts.shape[0], dtype=torch.float64, device=t.weight.device)
        _stream_enter(ctx)
        check(lib().tgb_value_at(ctx.handle, C.byref(ct), pts.shape[0], pts.data_ptr(), out.data_ptr(), mem))
        _stream_order(ctx, t, pts, out)
        return out
    pts = np.ascontiguousarray(np.asarray(ijk, dtype=np.int64).reshape(-1, 3))
    out = np.zeros(pts.shape[0])
    check(lib().tgb_value_at(ctx.handle, C.byref(ct), pts.shape[0], pts.ctypes.data, out.ctypes.data, mem))
    return out


def scalar_product(a, b, ctx: Context | None = None) -> float:
    """tensor.cpp:88-98 — <A, B> in 1D complexity."""
    ctx = ctx or default_context()
    mem = _mem(a, b)
    res = C.c_double()
    ca, cb = a._cstruct(), b._cstruct()
    check(lib().tgb_scalar_product(ctx.handle, C.byref(ca), C.byref(cb), C.byref(res), mem))
    return res.value


# --------------------------------------------------------------------------- grid / kernel / basis (input producers)


@dataclass
class Grid3:
    """grid.hpp:18-52 — cell-centred grid on [-b,b]^3, h = 2b/(n+1)."""

    n: tuple
    b_half: tuple
    h: tuple

    def coord(self, ax: int, i) -> np.ndarray:
        return (np.asarray(i, dtype=np.float64) - 0.5 * float(self.n[ax] - 1)) * self.h[ax]

    def ref_coord(self, ax: int, j) -> np.ndarray:
        return (np.asarray(j, dtype=np.float64) - float(self.n[ax] - 1)) * self.h[ax]

    def nearest_index(self, ax: int, x: float) -> int:
        return int(np.rint(x / self.h[ax] + 0.5 * float(self.n[ax] - 1)))


def make_grid(b_half, n) -> Grid3:
    """grid.cpp:7-21."""
    bs = (b_half,) * 3 if np.isscalar(b_half) else tuple(b_half)
    ns = (n,) * 3 if np.isscalar(n) else tuple(n)
    for ax in range(3):
        if not bs[ax] > 0.0:
            raise InvalidArgument("make_grid: box half-width must be positive")
        if ns[ax] < 2:
            raise InvalidArgument("make_grid: need at least 2 grid points per axis")
    return Grid3(tuple(int(x) for x in ns), tuple(float(x) for x in bs),
                 tuple(lib().tgb_mesh_size(bs[ax], ns[ax]) for ax in range(3)))


def snap_to_node(grid: Grid3, ax: int, x: float) -> int:
    out = C.c_int64()
    check(lib().tgb_snap_to_node(grid.b_half[ax], grid.n[ax], x, C.byref(out)), host=True)
    return out.value


def window_offset(grid: Grid3, ax: int, center: float) -> int:
    """grid.cpp:32-38."""
    out = C.c_int64()
    check(lib().tgb_window_offset(grid.b_half[ax], grid.n[ax], center, C.byref(out)), host=True)
    return out.value


@dataclass
class ExpSum:
    """kernel.hpp:26-47 — 1/r ~ sum_k w_k exp(-t_k^2 r^2), t_k = k*mesh."""

    m: int
    c0: float
    mesh: float
    scale: float
    nodes: np.ndarray
    weights: np.ndarray

    def terms(self) -> int:
        return int(self.weights.shape[0])

    def evaluate(self, r: float) -> float:
        return float(np.sum(self.weights * np.exp(-self.nodes * self.nodes * r * r)))

    def max_relative_error(self, lo: float, hi: float, samples: int = 400) -> float:
        worst = 0.0
        for i in range(samples):
            r = lo * (hi / lo) ** (0.0 if samples == 1 else i / (samples - 1))
            worst = max(worst, abs(self.evaluate(r) - 1.0 / r) * r)
        return worst


def make_expsum(m: int, c0: float, fit_lo: float = 0.0, fit_hi: float = 0.0) -> ExpSum:
    """kernel.cpp:71-123 (Newton kernel)."""
    nodes = np.zeros(2 * m + 1 if m >= 1 else 1)
    weights = np.zeros_like(nodes)
    sc, mesh = C.c_double(), C.c_double()
    check(lib().tgb_make_expsum(m, c0, fit_lo, fit_hi, nodes.ctypes.data, weights.ctypes.data, C.byref(sc),
                                C.byref(mesh)), host=True)
    return ExpSum(m, c0, mesh.value, sc.value, nodes, weights)


@dataclass
class KernelTensor:
    """kernel.hpp:58-72."""

    tensor: CanonicalTensor3
    doubled: bool
    expsum: ExpSum

    def rank(self) -> int:
        return self.tensor.rank()


def kernel_tensor(grid: Grid3, es: ExpSum, doubled: bool) -> KernelTensor:
    """kernel.cpp:182-203 — a_q^{1/3} * cell integral of exp(-t_q^2 x^2)."""
    r = es.terms()
    facs = []
    for ax in range(3):
        length = 2 * grid.n[ax] if doubled else grid.n[ax]
        f = np.zeros((length, r), order="F")
        check(lib().tgb_kernel_factors(grid.b_half[ax], grid.n[ax], r, es.nodes.ctypes.data, es.weights.ctypes.data,
                                       int(doubled), f.ctypes.data), host=True)
        facs.append(f)
    return KernelTensor(CanonicalTensor3(facs, np.ones(r)), doubled, es)


def gauss_cell_integral(t: float, center: float, h: float) -> float:
    return lib().tgb_gauss_cell_integral(t, center, h)


def primitive_norm(alpha: float, l: int) -> float:
    out = C.c_double()
    check(lib().tgb_primitive_norm(alpha, l, C.byref(out)), host=True)
    return out.value


@dataclass
class GaussianPrimitive:
    exponent: float = 1.0
    coeff: float = 1.0


@dataclass
class SeparableBasisFunction:
    """basis.hpp:19-26."""

    center: tuple = (0.0, 0.0, 0.0)
    degree: tuple = (0, 0, 0)
    primitives: list = field(default_factory=list)

    def total_degree(self) -> int:
        return int(sum(self.degree))


@dataclass
class BasisSet:
    grid: Grid3
    functions: list

    def size(self) -> int:
        return len(self.functions)


def discretize_basis(bs: BasisSet) -> list:
    """basis.cpp:16-46 — one rank-np canonical tensor per basis function."""
    out = []
    for f in bs.functions:
        for ax in range(3):
            if f.degree[ax] not in (0, 1):
                raise InvalidArgument("discretize_basis: per-axis degree must be 0 or 1")
        if not f.primitives:
            raise InvalidArgument("discretize_basis: contraction needs at least one primitive")
        npr = len(f.primitives)
        facs = [np.zeros((bs.grid.n[ax], npr), order="F") for ax in range(3)]
        w = np.zeros(npr)
        for p, prim in enumerate(f.primitives):
            w[p] = prim.coeff * primitive_norm(prim.exponent, f.total_degree())
            for ax in range(3):
                check(lib().tgb_gaussian_factor(bs.grid.b_half[ax], bs.grid.n[ax], f.center[ax], prim.exponent,
                                                f.degree[ax], facs[ax][:, p].ctypes.data), host=True)
        out.append(CanonicalTensor3(facs, w))
    return out


def flatten_basis(disc: list):
    """All primitives as one CP tensor + function offsets (tgb_coulomb_matrix).
    Column blocks are copied straight into Fortran-order factors (np.hstack
    would build C-order arrays and transpose them: ~10x slower at config 3)."""
    offs = np.zeros(len(disc) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([d.rank() for d in disc])
    facs = []
    for ax in range(3):
        n = disc[0].factor[ax].shape[0] if disc else 0
        # rows of the C-order (R x n) stack = columns of the Fortran-order (n x R) factor
        facs.append(np.concatenate([d.factor[ax].T for d in disc], axis=0).T if disc else np.zeros((n, 0), order="F"))
    w = np.concatenate([d.weight for d in disc]) if disc else np.zeros(0)
    return CanonicalTensor3(facs, w), offs


def coulomb_matrix(bs: BasisSet, disc: list, v_hartree, ctx: Context | None = None) -> np.ndarray:
    """hf.cpp:140-151 — J_km = h^3 <G_k . G_m, V_H>, exactly symmetric."""
    ctx = ctx or default_context()
    flat, offs = flatten_basis(disc)
    nb = len(disc)
    if isinstance(v_hartree, DeviceCP):
        flat_d = DeviceCP.from_host(flat, device=v_hartree.weight.device)
        import torch

        J = torch.empty((nb, nb), dtype=torch.float64, device=v_hartree.weight.device)
        cf, cv = flat_d._cstruct(), v_hartree._cstruct()
        hh = _h3(bs.grid.h)
        check(lib().tgb_coulomb_matrix(ctx.handle, C.byref(cf), offs.ctypes.data, nb, C.byref(cv), hh.ctypes.data,
                                       J.data_ptr(), MEM_DEVICE))
        return J.cpu().numpy().T.copy(order="F")
    J = np.zeros((nb, nb), order="F")
    cf, cv = flat._cstruct(), v_hartree._cstruct()
    hh = _h3(bs.grid.h)
    check(lib().tgb_coulomb_matrix(ctx.handle, C.byref(cf), offs.ctypes.data, nb, C.byref(cv), hh.ctypes.data,
                                   J.ctypes.data, MEM_HOST))
    return J


# --------------------------------------------------------------------------- lattice


@dataclass
class LatticeSpec:
    """lattice.hpp:20-36."""

    counts: tuple = (1, 1, 1)
    spacing: float = 2.0
    charge: float = 1.0
    blocks: list = field(default_factory=list)
    n0: int = 64
    margin_cells: int = 1

    def position(self, ax: int, m: int) -> float:
        return (float(m) - 0.5 * float(self.counts[ax] - 1)) * self.spacing


@dataclass
class AssembledPotential:
    """lattice.hpp:41-45."""

    canonical: CanonicalTensor3 | None = None
    window_ops: int = 0
    tucker: object = None


def lattice_offsets(spec: LatticeSpec, grid: Grid3, ax: int, lo: int = 0, hi: int | None = None) -> np.ndarray:
    hi = spec.counts[ax] - 1 if hi is None else hi
    return np.array([window_offset(grid, ax, spec.position(ax, m)) for m in range(lo, hi + 1)], dtype=np.int64)


def lattice_assemble_axis(ref_cols: np.ndarray, offsets: np.ndarray, n: int, ctx: Context | None = None):
    ctx = ctx or default_context()
    ref = _fmat(ref_cols)
    R = ref.shape[1]
    out = np.zeros((n, R), order="F")
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    check(lib().tgb_lattice_assemble_axis(ctx.handle, n, R, ref.ctypes.data if ref.size else None, offs.ctypes.data,
                                          offs.shape[0], out.ctypes.data if out.size else None, MEM_HOST))
    return out


def lattice_sum_canonical(spec: LatticeSpec, grid: Grid3, reference: KernelTensor,
                          ctx: Context | None = None) -> AssembledPotential:
    """lattice.cpp:116-129 — rank-preserving O(L) assembly."""
    if not reference.doubled:
        raise InvalidArgument("lattice_sum_canonical: reference must live on the doubled grid")
    if spec.blocks:
        raise InvalidArgument("lattice_sum_canonical: use lattice_sum_composite for block geometries")
    for ax in range(3):
        if spec.counts[ax] < 1:
            raise InvalidArgument("LatticeSpec: counts must be >= 1")
    out = AssembledPotential()
    ctx = ctx or default_context()
    offs = [np.ascontiguousarray(lattice_offsets(spec, grid, ax), dtype=np.int64) for ax in range(3)]
    R = reference.rank()
    refs = [np.asfortranarray(reference.tensor.factor[ax], dtype=np.float64) for ax in range(3)]
    facs = [np.zeros((grid.n[ax], R), order="F") for ax in range(3)]
    P3 = C.c_void_p * 3
    nn = (C.c_int64 * 3)(*grid.n)
    LL = (C.c_int64 * 3)(*[len(o) for o in offs])
    check(lib().tgb_lattice_assemble(ctx.handle, nn, R, P3(*[r.ctypes.data if r.size else None for r in refs]),
                                     P3(*[o.ctypes.data if o.size else None for o in offs]), LL,
                                     P3(*[f.ctypes.data if f.size else None for f in facs]), MEM_HOST))
    out.window_ops = int(sum(len(o) for o in offs))
    out.canonical = CanonicalTensor3(facs, spec.charge * reference.tensor.weight)
    return out


# --------------------------------------------------------------------------- Hartree-Fock pieces on the path


def orbital_tensor(disc: list, coeff) -> CanonicalTensor3:
    """hf.cpp:39-46 — phi = sum_k c_k G_k (concatenation in k order)."""
    phi = CanonicalTensor3.zero(disc[0].extents())
    for k, c in enumerate(np.asarray(coeff, dtype=np.float64)):
        if c == 0.0:
            continue
        phi = add(phi, scale(disc[k], float(c)))
    return phi


def density_tensor(disc: list, c_occ, reduce_eps: float = 1e-7, ctx: Context | None = None) -> CanonicalTensor3:
    """hf.cpp:118-129 — Theta = sum_a 2 phi_a . phi_a built on the device from the
    basis factors (tgb_density_build), then reduce_rank on the device
    (tgb_density_reduce) when rank > 1 and reduce_eps > 0."""
    from .reduction import _t2c, _tucker_result

    if not disc:
        raise InvalidArgument("density_tensor: empty basis")
    ctx = ctx or default_context()
    c = np.asfortranarray(np.asarray(c_occ, dtype=np.float64))
    if c.ndim != 2 or c.shape[0] != len(disc):
        raise InvalidArgument("density_tensor: coefficient shape mismatch")
    flat, offs = flatten_basis(disc)
    nb, nocc = len(disc), c.shape[1]
    cf = flat._cstruct()
    cp = c.ctypes.data if c.size else None
    rank = C.c_int64()
    check(lib().tgb_density_rank(offs.ctypes.data, nb, cp, nocc, C.byref(rank)))
    dims = disc[0].extents()
    if rank.value <= 1 or reduce_eps <= 0.0:
        theta = CanonicalTensor3([np.zeros((d, rank.value), order="F") for d in dims], np.zeros(rank.value))
        co = theta._cstruct()
        check(lib().tgb_density_build(ctx.handle, C.byref(cf), offs.ctypes.data, nb, cp, nocc, C.byref(co), MEM_HOST))
        return theta
    h = C.c_void_p()
    check(lib().tgb_density_reduce(ctx.handle, C.byref(cf), offs.ctypes.data, nb, cp, nocc, reduce_eps, MEM_HOST,
                                   C.byref(h)))
    return _t2c(_tucker_result(h, dims, ctx), dims)


@dataclass
class LatticeBlock:
    """lattice.hpp:13-18 — inclusive node-index box, include/exclude, charge scale."""

    lo: tuple = (0, 0, 0)
    hi: tuple = (0, 0, 0)
    include: bool = True
    charge_scale: float = 1.0


def _validate_spec(spec: LatticeSpec) -> None:
    """lattice.cpp:13-18."""
    for ax in range(3):
        if spec.counts[ax] < 1:
            raise InvalidArgument("LatticeSpec: counts must be >= 1")
    if not spec.spacing > 0.0:
        raise InvalidArgument("LatticeSpec: spacing must be positive")
    if spec.n0 < 2 or spec.n0 % 2:
        raise InvalidArgument("LatticeSpec: n0 must be even (node alignment)")
    if spec.margin_cells < 1:
        raise InvalidArgument("LatticeSpec: need at least one margin cell")


def lattice_grid(spec: LatticeSpec) -> Grid3:
    """lattice.cpp:65-75 — n = n0 (L - 1 + 2 margin) - 1 so every node is a cell centre."""
    _validate_spec(spec)
    cells = [spec.counts[ax] - 1 + 2 * spec.margin_cells for ax in range(3)]
    return make_grid([0.5 * c * spec.spacing for c in cells], [spec.n0 * c - 1 for c in cells])


def _overlap(a: LatticeBlock, b: LatticeBlock) -> bool:
    return all(not (a.hi[ax] < b.lo[ax] or b.hi[ax] < a.lo[ax]) for ax in range(3))


def resolve_blocks(spec: LatticeSpec) -> list:
    """lattice.cpp:77-104 — disjoint included rectangles (the full lattice when no blocks)."""
    _validate_spec(spec)
    full = LatticeBlock((0, 0, 0), tuple(c - 1 for c in spec.counts), True, 1.0)
    included = []
    for b in spec.blocks:
        if not b.include:
            continue
        if not b.charge_scale > 0.0:
            raise InvalidArgument("resolve_blocks: charge scale must be positive")
        for ax in range(3):
            if not (0 <= b.lo[ax] <= b.hi[ax] < spec.counts[ax]):
                raise InvalidArgument("resolve_blocks: block outside the lattice")
        if any(_overlap(p, b) for p in included):
            raise InvalidArgument("resolve_blocks: overlapping include blocks")
        included.append(b)
    if not included:
        included.append(full)
    for cut in spec.blocks:
        if cut.include:
            continue
        nxt = []
        for box in included:
            if not _overlap(box, cut):
                nxt.append(box)
                continue
            rest_lo, rest_hi = list(box.lo), list(box.hi)
            for ax in range(3):  # lattice.cpp:31-48
                if cut.lo[ax] > rest_lo[ax]:
                    hi = list(rest_hi)
                    hi[ax] = cut.lo[ax] - 1
                    nxt.append(LatticeBlock(tuple(rest_lo), tuple(hi), True, box.charge_scale))
                    rest_lo[ax] = cut.lo[ax]
                if cut.hi[ax] < rest_hi[ax]:
                    lo = list(rest_lo)
                    lo[ax] = cut.hi[ax] + 1
                    nxt.append(LatticeBlock(tuple(lo), tuple(rest_hi), True, box.charge_scale))
                    rest_hi[ax] = cut.hi[ax]
        included = nxt
    if not included:
        raise InvalidArgument("resolve_blocks: empty composite lattice")
    return included


def lattice_nodes(spec: LatticeSpec) -> np.ndarray:
    """lattice.cpp:106-114."""
    out = []
    for r in resolve_blocks(spec):
        for k in range(r.lo[2], r.hi[2] + 1):
            for j in range(r.lo[1], r.hi[1] + 1):
                for i in range(r.lo[0], r.hi[0] + 1):
                    out.append((spec.position(0, i), spec.position(1, j), spec.position(2, k)))
    return np.array(out)


def lattice_sum_tucker(spec: LatticeSpec, grid: Grid3, master, ctx: Context | None = None):
    """lattice.cpp:131-145 — the same window assembly on the Tucker side
    matrices of a doubled-grid master; the core is scaled by the charge."""
    _validate_spec(spec)
    if spec.blocks:
        raise InvalidArgument("lattice_sum_tucker: use lattice_sum_composite for block geometries")
    for ax in range(3):
        if master.side[ax].shape[0] != 2 * grid.n[ax]:
            raise InvalidArgument("lattice_sum_tucker: master must live on the doubled grid")
    from .reduction import TuckerTensor3

    sides, ops = [], 0
    for ax in range(3):
        offs = lattice_offsets(spec, grid, ax)
        sides.append(lattice_assemble_axis(master.side[ax], offs, grid.n[ax], ctx))
        ops += len(offs)
    out = AssembledPotential()
    out.tucker = TuckerTensor3(sides, np.asfortranarray(master.core * spec.charge))
    out.window_ops = ops
    return out


def lattice_sum_composite(spec: LatticeSpec, grid: Grid3, reference: KernelTensor, reduce_eps: float | None = None,
                          ctx: Context | None = None) -> AssembledPotential:
    """lattice.cpp:147-165 — per-block assembled sums concatenated (rank R per
    block), then optionally rank-reduced on the device."""
    if not reference.doubled:
        raise InvalidArgument("lattice_sum_composite: reference must live on the doubled grid")
    rects = resolve_blocks(spec)
    out = AssembledPotential()
    total = CanonicalTensor3.zero(grid.n)
    for r in rects:
        facs = []
        for ax in range(3):
            offs = lattice_offsets(spec, grid, ax, r.lo[ax], r.hi[ax])
            facs.append(lattice_assemble_axis(reference.tensor.factor[ax], offs, grid.n[ax], ctx))
            out.window_ops += len(offs)
        total = add(total, CanonicalTensor3(facs, spec.charge * r.charge_scale * reference.tensor.weight))
    if reduce_eps is not None:
        from .reduction import ReductionConfig, reduce_rank

        total = reduce_rank(total, ReductionConfig.tolerance(reduce_eps), ctx)
    out.canonical = total
    return out

"""Python mirror of the reference's factorised-TEI API (proj/include/tengrid/
tei.hpp:27-72) over libtgb (include/tgb.h, tgb_tei_*)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import MEM_HOST, InvalidArgument, check, lib
from .tengrid import CanonicalTensor3, Context, KernelTensor, _h3, default_context, flatten_basis


class TEIFactorization:
    """tei.hpp:38-57 — device-resident; accessors copy to the host."""

    def __init__(self, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self._h = C.c_void_p()
        check(lib().tgb_tei_create(C.byref(self._h)))

    def __del__(self):
        try:
            lib().tgb_tei_destroy(self._h)
        except Exception:
            pass

    def _info(self):
        info = np.zeros(8, dtype=np.int64)
        res = np.zeros(3)
        check(lib().tgb_tei_info(self._h, info.ctypes.data, res.ctypes.data))
        return info, res

    @property
    def n_b(self) -> int:
        return int(self._info()[0][4])

    @property
    def n_prim(self) -> int:
        return int(self._info()[0][3])

    def fit_ranks(self) -> tuple:
        return tuple(int(x) for x in self._info()[0][:3])

    @property
    def fit_residual(self) -> np.ndarray:
        return self._info()[1]

    @property
    def fit_clamped_negative(self) -> bool:
        return bool(self._info()[0][6])

    def rank_b(self) -> int:
        return int(self._info()[0][5])

    def fit(self, ax: int):
        r = self.fit_ranks()[ax]
        n = self._n[ax]
        U = np.zeros((n, r), order="F")
        V = np.zeros((self.n_prim ** 2, r), order="F")
        check(lib().tgb_tei_get_fit(self._h, ax, U.ctypes.data if U.size else None, V.ctypes.data if V.size else None,
                                    MEM_HOST))
        return U, V

    def conv(self, k: int, ax: int) -> np.ndarray:
        r = self.fit_ranks()[ax]
        M = np.zeros((r, r), order="F")
        check(lib().tgb_tei_get_conv(self._h, k, ax, M.ctypes.data if M.size else None, MEM_HOST))
        return M

    @property
    def chol(self) -> np.ndarray:
        nb2 = self.n_b ** 2
        rb = self.rank_b()
        L = np.zeros((nb2, rb), order="F")
        piv = np.zeros(max(rb, 1), dtype=np.int64)
        check(lib().tgb_tei_get_cholesky(self._h, L.ctypes.data if L.size else None, piv.ctypes.data, MEM_HOST))
        self._pivots = piv[:rb]
        return L

    @property
    def pivots(self) -> np.ndarray:
        self.chol
        return self._pivots


def pivot_margins(fac: "TEIFactorization", diagonal: np.ndarray, eps_chol: float) -> dict:
    """How decisively each TEI Cholesky pivot was chosen (the argmax of
    tei.cpp:66): the remaining diagonal is rebuilt from L step by step
    (d_r = d_0 - sum_{s<r} L[:, s]^2, pinned pivots zeroed as tei.cpp:73-75)
    and, at every step, the relative gap between the pivot's value and the best
    candidate that is not its (mu nu)/(nu mu) mirror (mirrors are bitwise equal
    by construction and resolve to the first index).  Also the stop margin
    max d_final / (eps_chol max d_0) (<= 1: stopped).  A pivot sequence is
    robust when min_gap is well above roundoff."""
    L = np.asarray(fac.chol)
    piv = [int(p) for p in fac.pivots]
    nb = fac.n_b
    d = np.array(diagonal, dtype=np.float64, copy=True)
    max0 = float(d.max()) if d.size else 0.0
    gaps = []
    for r, p in enumerate(piv):
        mirror = (p % nb) * nb + p // nb
        dp = d[p]
        others = d.copy()
        others[p] = -np.inf
        others[mirror] = -np.inf
        d2 = float(others.max()) if others.size > 2 else 0.0
        gaps.append((dp - d2) / dp if dp > 0 else 0.0)
        d -= L[:, r] ** 2
        d[p] = 0.0
        d[mirror] = max(d[mirror], 0.0)
        d[d < 0] = 0.0
    return {"min_pivot_gap": float(min(gaps)) if gaps else None,
            "argmin_step": int(np.argmin(gaps)) if gaps else None,
            "stop_ratio": float(d.max() / (eps_chol * max0)) if max0 > 0 else None,
            "gaps": [float(x) for x in gaps]}


def tei_density_fitting(fac: TEIFactorization, bs, disc: list, eps_fit: float) -> None:
    """tei.cpp:92-143."""
    if not disc:
        raise InvalidArgument("tei_density_fitting: empty basis")
    flat, offs = flatten_basis(disc)
    cf = flat._cstruct()
    hh = _h3(bs.grid.h)
    fac._n = bs.grid.n
    check(lib().tgb_tei_density_fitting(fac.ctx.handle, fac._h, C.byref(cf), offs.ctypes.data, len(disc),
                                        hh.ctypes.data, eps_fit, MEM_HOST))


def tei_convolution_matrices(fac: TEIFactorization, kernel) -> None:
    """tei.cpp:145-158 (kernel must live on the primary grid)."""
    if isinstance(kernel, KernelTensor):
        if kernel.doubled:
            raise InvalidArgument("tei_convolution_matrices: kernel must live on the primary grid")
        kernel = kernel.tensor
    ck = kernel._cstruct()
    check(lib().tgb_tei_convolution_matrices(fac.ctx.handle, fac._h, C.byref(ck), MEM_HOST))


def tei_diagonal(fac: TEIFactorization) -> np.ndarray:
    """tei.cpp:182-196."""
    out = np.zeros(fac.n_b ** 2)
    check(lib().tgb_tei_diagonal(fac.ctx.handle, fac._h, out.ctypes.data, MEM_HOST))
    return out


def tei_column(fac: TEIFactorization, pair_index: int) -> np.ndarray:
    """tei.cpp:160-174."""
    out = np.zeros(fac.n_b ** 2)
    check(lib().tgb_tei_column(fac.ctx.handle, fac._h, pair_index, out.ctypes.data, MEM_HOST))
    return out


def tei_matrix_entry(fac: TEIFactorization, mu: int, nu: int, kappa: int, lam: int) -> float:
    """tei.cpp:176-180."""
    nb = fac.n_b
    for i in (mu, nu, kappa, lam):
        if not 0 <= i < nb:
            raise InvalidArgument("tei_matrix_entry: index out of range")
    return float(tei_column(fac, kappa + nb * lam)[mu + nb * nu])


def tei_cholesky(fac: TEIFactorization, eps_chol: float) -> None:
    """tei.cpp:198-204."""
    check(lib().tgb_tei_cholesky(fac.ctx.handle, fac._h, eps_chol))


def build_tei(bs, disc: list, kernel, eps_fit: float, eps_chol: float, ctx: Context | None = None):
    """tei.cpp:206-213 — fitting -> convolution matrices -> pivoted Cholesky."""
    fac = TEIFactorization(ctx)
    tei_density_fitting(fac, bs, disc, eps_fit)
    tei_convolution_matrices(fac, kernel)
    tei_cholesky(fac, eps_chol)
    return fac


class PivotedCholesky:
    """tei.hpp:12-17."""

    def __init__(self, factor, pivots, residual, clamped_negative):
        self.factor, self.pivots, self.residual, self.clamped_negative = factor, pivots, residual, clamped_negative


def pivoted_cholesky(a, tol: float, stop: str = "max_diagonal", max_rank: int | None = None,
                     negative_tol: float = 1e-12, ctx: Context | None = None) -> PivotedCholesky:
    """tei.cpp:48-90 on an explicit PSD matrix (the reference's column callback reads its columns);
    stop "max_diagonal" or "trace" (CholeskyStop, tei.hpp:19-22)."""
    ctx = ctx or default_context()
    A = np.asfortranarray(np.asarray(a, dtype=np.float64))
    n = A.shape[0]
    if A.shape != (n, n):
        raise InvalidArgument("pivoted_cholesky: square matrix expected")
    max_rank = n if max_rank is None else max_rank
    cap = min(n, max_rank)
    L = np.zeros((n, max(cap, 1)), order="F")
    piv = np.zeros(max(cap, 1), dtype=np.int64)
    rank, res, cl = C.c_int64(), C.c_double(), C.c_int()
    check(lib().tgb_pivoted_cholesky(ctx.handle, n, A.ctypes.data if A.size else None, tol,
                                     {"max_diagonal": 0, "trace": 1}[stop], max_rank, negative_tol, L.ctypes.data,
                                     piv.ctypes.data, C.byref(rank), C.byref(res), C.byref(cl), MEM_HOST))
    k = rank.value
    return PivotedCholesky(np.asfortranarray(L[:, :k]), piv[:k].copy(), res.value, bool(cl.value))

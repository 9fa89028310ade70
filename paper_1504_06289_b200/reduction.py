"""Python mirror of the reference's rank-reduction API (proj/include/tengrid/
reduction.hpp:12-67) over libtgb (tgb_reduce_tucker / tgb_tucker_*)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import MEM_DEVICE, MEM_HOST, InvalidArgument, check, lib
from .tengrid import CanonicalTensor3, Context, default_context


@dataclass
class ReductionConfig:
    """reduction.hpp:12-35 — exactly one of ranks / epsilon."""

    ranks: tuple | None = None
    epsilon: float | None = None
    max_sweeps: int = 3
    # also fill TuckerResult.mode_singular_values with the FULL spectra (reduction.hpp:42);
    # off by default: the rank rule only needs the leading values
    full_spectra: bool = False

    @staticmethod
    def fixed(r1, r2, r3, sweeps=3):
        return ReductionConfig(ranks=(r1, r2, r3), max_sweeps=sweeps)

    @staticmethod
    def tolerance(eps, sweeps=3):
        return ReductionConfig(epsilon=eps, max_sweeps=sweeps)

    def validate(self):
        if (self.ranks is None) == (self.epsilon is None):
            raise InvalidArgument("ReductionConfig: set exactly one of {ranks, epsilon}")
        if self.epsilon is not None and not self.epsilon > 0.0:
            raise InvalidArgument("ReductionConfig: epsilon must be positive")
        if self.max_sweeps < 1:
            raise InvalidArgument("ReductionConfig: need at least one sweep")


@dataclass
class TuckerTensor3:
    side: list
    core: np.ndarray  # (r1, r2, r3), Fortran order

    def ranks(self):
        return tuple(self.core.shape)

    def to_dense(self):
        return np.einsum("abc,ia,jb,kc->ijk", self.core, *self.side)


@dataclass
class TuckerResult:
    tucker: TuckerTensor3
    rank_clamped: bool = False
    rhosvd_fallback: bool = False
    sweep_fits: list = field(default_factory=list)
    mode_singular_values: list = field(default_factory=list)
    _handle: object = None
    rank_margins: list = field(default_factory=list)  # tgb_tucker_margins per mode


class _Handle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            lib().tgb_tucker_destroy(self.h)
        except Exception:
            pass


def _run(a: CanonicalTensor3, cfg: ReductionConfig, mode: int, ctx: Context | None):
    cfg.validate()
    a.check_valid()
    ctx = ctx or default_context()
    h = C.c_void_p()
    ca = a._cstruct()
    ranks = np.asarray(cfg.ranks if cfg.ranks is not None else (0, 0, 0), dtype=np.int64)
    check(lib().tgb_reduce_tucker(ctx.handle, C.byref(ca), int(cfg.epsilon is not None), cfg.epsilon or 0.0,
                                  ranks.ctypes.data, cfg.max_sweeps, mode + (2 if cfg.full_spectra else 0), MEM_HOST,
                                  C.byref(h)))
    return _tucker_result(h, a.extents(), ctx)


def _tucker_result(h, dims, ctx: Context) -> TuckerResult:
    """Read a device-resident Tucker result (tgb_tucker handle) back to the host."""
    hh = _Handle(h)
    info = np.zeros(7, dtype=np.int64)
    check(lib().tgb_tucker_info(h, info.ctypes.data))
    r = tuple(int(x) for x in info[:3])
    core = np.zeros(r, order="F")
    sides = [np.zeros((dims[ax], r[ax]), order="F") for ax in range(3)]
    fits = np.zeros(max(1, int(info[5])))
    check(lib().tgb_tucker_get(h, core.ctypes.data if core.size else None,
                               *[s.ctypes.data if s.size else None for s in sides], fits.ctypes.data, MEM_HOST))
    sig = []
    for ax in range(3):
        cnt = C.c_int64()
        check(lib().tgb_tucker_sigma(h, ax, C.byref(cnt), None))
        sv = np.zeros(max(1, cnt.value))
        check(lib().tgb_tucker_sigma(h, ax, C.byref(cnt), sv.ctypes.data))
        sig.append(sv[:cnt.value])
    margins = []
    for ax in range(3):
        m = np.zeros(6)
        check(lib().tgb_tucker_margins(h, ax, m.ctypes.data))
        margins.append({"rank": int(m[0]), "sigma_last_kept": m[1], "sigma_first_dropped": m[2],
                        "sigma_ratio": m[3], "tail_before_over_budget": m[4], "tail_after_over_budget": m[5]})
    res = TuckerResult(TuckerTensor3(sides, core), bool(info[3]), bool(info[4]), list(fits[:int(info[5])]), sig, hh)
    res.rank_margins = margins
    res._t2c_rank = int(info[6])
    res._ctx = ctx
    return res


def mode_spectrum(a, axis: int, ctx: Context | None = None) -> np.ndarray:
    """tgb_mode_spectrum: the full singular-value spectrum rhosvd reports for mode `axis`
    (TuckerResult::mode_singular_values, reduction.hpp:42; reduction.cpp:172-190), device-computed.
    `a`: CanonicalTensor3 (host) or DeviceCP."""
    from .tengrid import DeviceCP

    ctx = ctx or default_context()
    if not 0 <= axis < 3:
        raise InvalidArgument("mode_spectrum: axis must be 0, 1 or 2")
    mem = MEM_DEVICE if isinstance(a, DeviceCP) else MEM_HOST
    ca = a._cstruct()
    cnt = C.c_int64()
    n_ax = a.extent(axis) if isinstance(a, DeviceCP) else a.extents()[axis]
    out = np.zeros(max(1, min(n_ax, a.rank())))
    check(lib().tgb_mode_spectrum(ctx.handle, C.byref(ca), axis, mem, C.byref(cnt), out.ctypes.data))
    return out[:cnt.value].copy()


def rhosvd(a: CanonicalTensor3, cfg: ReductionConfig, ctx: Context | None = None) -> TuckerResult:
    """reduction.cpp:172-190."""
    return _run(a, cfg, 0, ctx)


def canonical_to_tucker(a: CanonicalTensor3, cfg: ReductionConfig, ctx: Context | None = None) -> TuckerResult:
    """reduction.cpp:192-236 — RHOSVD initial guess + ALS sweeps."""
    return _run(a, cfg, 1, ctx)


def _t2c(res: TuckerResult, dims) -> CanonicalTensor3:
    rank = res._t2c_rank
    out = CanonicalTensor3([np.zeros((d, rank), order="F") for d in dims], np.zeros(rank))
    co = out._cstruct()
    check(lib().tgb_tucker_to_canonical(res._ctx.handle, res._handle.h, C.byref(co), MEM_HOST))
    return out


def reduce_rank(a: CanonicalTensor3, cfg: ReductionConfig, ctx: Context | None = None) -> CanonicalTensor3:
    """reduction.cpp:271-273 — canonical_to_tucker then tucker_to_canonical."""
    res = canonical_to_tucker(a, cfg, ctx)
    return _t2c(res, a.extents())


def thin_svd_left(a, ctx: Context | None = None):
    """reduction.cpp:85-138 — (u, sigma): left singular pairs, sigma descending, with the
    reference's output shape per branch (device one-sided Jacobi)."""
    ctx = ctx or default_context()
    A = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if A.ndim != 2:
        raise InvalidArgument("thin_svd_left: matrix expected")
    r, c = A.shape
    p = min(r, c)
    u = np.zeros((r, p), order="F")
    s = np.zeros(p)
    kept = C.c_int64()
    check(lib().tgb_thin_svd_left(ctx.handle, r, c, A.ctypes.data if A.size else None, u.ctypes.data if u.size else None,
                                  s.ctypes.data if s.size else None, C.byref(kept), MEM_HOST))
    k = kept.value
    return np.asfortranarray(u[:, :k]), s[:k].copy()

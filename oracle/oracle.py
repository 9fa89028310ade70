"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/build/liboracle.so (the CPU restatement in
tengrid_oracle.cpp) and of oracle/_ref/libtengrid_ref.so (the reference's own
conv-path translation units compiled against oracle/eigen_shim).  Imported
only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs — never by the product package.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "build" / "liboracle.so"
REF_LIB = HERE / "_ref" / "libtengrid_ref.so"

_o = None
_r = None


def olib() -> C.CDLL:
    global _o
    if _o is None:
        if not ORACLE_LIB.exists():
            raise FileNotFoundError(f"{ORACLE_LIB} missing: run __graft_entry__.build()")
        L = C.CDLL(str(ORACLE_LIB))
        P = C.c_void_p
        L.orc_cp_new.restype = P
        L.orc_tei_new.restype = P
        for name in ("orc_cp_free", "orc_tei_free"):
            getattr(L, name).argtypes = [P]
        L.orc_cp_rank.restype = C.c_longlong
        L.orc_cp_rank.argtypes = [P]
        L.orc_cp_extent.restype = C.c_longlong
        L.orc_cp_extent.argtypes = [P, C.c_int]
        L.orc_cp_get.argtypes = [P, C.c_int, P]
        L.orc_cp_get_w.argtypes = [P, P]
        L.orc_last_error.restype = C.c_char_p
        L.orc_gauss_cell_integral.restype = C.c_double
        L.orc_gauss_cell_integral.argtypes = [C.c_double, C.c_double, C.c_double]
        _o = L
    return _o


def rlib() -> C.CDLL | None:
    """The reference's own code (oracle/_ref), or None where it was not built."""
    global _r
    if _r is None:
        if not REF_LIB.exists():
            return None
        L = C.CDLL(str(REF_LIB))
        P = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_cp_new.restype = P
        L.ref_cp_free.argtypes = [P]
        L.ref_cp_rank.restype = C.c_longlong
        L.ref_cp_rank.argtypes = [P]
        L.ref_cp_extent.restype = C.c_longlong
        L.ref_cp_extent.argtypes = [P, C.c_int]
        L.ref_cp_get.argtypes = [P, C.c_int, P]
        L.ref_cp_get_w.argtypes = [P, P]
        L.ref_tei_get.argtypes = [P, C.c_int, C.c_longlong, P]
        L.ref_tei_free.argtypes = [P]
        L.ref_gauss_cell_integral.restype = C.c_double
        L.ref_gauss_cell_integral.argtypes = [C.c_double, C.c_double, C.c_double]
        _r = L
    return _r


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _chk(rc: int, lib=None) -> None:
    if rc:
        lib = lib or olib()
        err = (lib.orc_last_error() if hasattr(lib, "orc_last_error") else lib.ref_last_error()) or b""
        raise OracleError(rc, err.decode())


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


def _f(a) -> np.ndarray:
    m = np.asfortranarray(np.asarray(a, dtype=np.float64))
    return m.reshape(-1, 1, order="F") if m.ndim == 1 else m


class OCP:
    """Owned handle to an oracle CanonicalTensor3."""

    def __init__(self, factors=None, weight=None, lib=None):
        self.lib = lib or olib()
        self.h = C.c_void_p(self.lib.orc_cp_new() if self.lib is olib() else self.lib.ref_cp_new())
        if factors is not None:
            fs = [_f(f) for f in factors]
            w = np.ascontiguousarray(np.asarray(weight, dtype=np.float64))
            n = (C.c_longlong * 3)(*[f.shape[0] for f in fs])
            setter = self.lib.orc_cp_set if self.lib is olib() else self.lib.ref_cp_set
            _chk(setter(self.h, n, C.c_longlong(w.shape[0]), _p(fs[0]), _p(fs[1]), _p(fs[2]), _p(w)), self.lib)

    @staticmethod
    def from_cp(t, lib=None) -> "OCP":
        return OCP(t.factor, t.weight, lib)

    def rank(self) -> int:
        return (self.lib.orc_cp_rank if self.lib is olib() else self.lib.ref_cp_rank)(self.h)

    def extent(self, ax: int) -> int:
        return (self.lib.orc_cp_extent if self.lib is olib() else self.lib.ref_cp_extent)(self.h, ax)

    def factors(self) -> list:
        out = []
        get = self.lib.orc_cp_get if self.lib is olib() else self.lib.ref_cp_get
        for ax in range(3):
            m = np.zeros((self.extent(ax), self.rank()), order="F")
            if m.size:
                get(self.h, ax, _p(m))
            out.append(m)
        return out

    def weight(self) -> np.ndarray:
        w = np.zeros(self.rank())
        if w.size:
            (self.lib.orc_cp_get_w if self.lib is olib() else self.lib.ref_cp_get_w)(self.h, _p(w))
        return w

    def __del__(self):
        try:
            (self.lib.orc_cp_free if self.lib is olib() else self.lib.ref_cp_free)(self.h)
        except Exception:
            pass


# ------------------------------------------------------------------ restatement entry points

def conv_central_many(U, v) -> np.ndarray:
    U = _f(U)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros(U.shape, order="F")
    _chk(olib().orc_conv_central_many(C.c_longlong(U.shape[0]), C.c_longlong(U.shape[1]), _p(U), _p(v), _p(out)))
    return out


def conv_full(u, v, use_fft: bool) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros(2 * u.shape[0] - 1)
    _chk(olib().orc_conv_full(C.c_longlong(u.shape[0]), _p(u), _p(v), C.c_int(int(use_fft)), _p(out)))
    return out


def convolve(a: OCP, b: OCP, h) -> OCP:
    out = OCP()
    hh = np.ascontiguousarray(np.broadcast_to(np.asarray(h, dtype=np.float64), (3,)))
    _chk(olib().orc_convolve(a.h, b.h, _p(hh), out.h))
    return out


def hartree_potential(theta: OCP, kernel: OCP, h) -> OCP:
    out = OCP()
    hh = np.ascontiguousarray(np.broadcast_to(np.asarray(h, dtype=np.float64), (3,)))
    _chk(olib().orc_hartree_potential(theta.h, kernel.h, _p(hh), out.h))
    return out


def hadamard(a: OCP, b: OCP) -> OCP:
    out = OCP()
    _chk(olib().orc_hadamard(a.h, b.h, out.h))
    return out


def scalar_product(a: OCP, b: OCP) -> float:
    r = C.c_double()
    _chk(olib().orc_scalar_product(a.h, b.h, C.byref(r)))
    return r.value


def value_at(t: OCP, ijk) -> np.ndarray:
    pts = np.ascontiguousarray(np.asarray(ijk, dtype=np.int64).reshape(-1, 3))
    out = np.zeros(pts.shape[0])
    _chk(olib().orc_value_at(t.h, C.c_longlong(pts.shape[0]), _p(pts), _p(out)))
    return out


def make_expsum(m: int, c0: float, lo: float = 0.0, hi: float = 0.0):
    nodes = np.zeros(2 * m + 1)
    w = np.zeros(2 * m + 1)
    sc, mesh = C.c_double(), C.c_double()
    _chk(olib().orc_make_expsum(C.c_longlong(m), C.c_double(c0), C.c_double(lo), C.c_double(hi), _p(nodes), _p(w),
                                C.byref(sc), C.byref(mesh)))
    return nodes, w, sc.value, mesh.value


def kernel_tensor(b_half, n, nodes, weights, doubled: bool) -> OCP:
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(b_half, dtype=np.float64), (3,)))
    nn = (C.c_longlong * 3)(*np.broadcast_to(np.asarray(n), (3,)).tolist())
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    out = OCP()
    _chk(olib().orc_kernel_tensor(_p(b), nn, C.c_longlong(nodes.shape[0]), _p(nodes), _p(weights),
                                  C.c_int(int(doubled)), out.h))
    return out


def gauss_cell_integral(t, c, h) -> float:
    return olib().orc_gauss_cell_integral(t, c, h)


def window_offset(b_half, n, ax, center) -> int:
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(b_half, dtype=np.float64), (3,)))
    nn = (C.c_longlong * 3)(*np.broadcast_to(np.asarray(n), (3,)).tolist())
    o = C.c_longlong()
    _chk(olib().orc_window_offset(_p(b), nn, C.c_int(ax), C.c_double(center), C.byref(o)))
    return o.value


def discretize_basis(b_half, n, functions) -> list:
    """functions: list of (center(3), degree(3), [(exponent, coeff), ...])."""
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(b_half, dtype=np.float64), (3,)))
    nn = (C.c_longlong * 3)(*np.broadcast_to(np.asarray(n), (3,)).tolist())
    nf = len(functions)
    centers = np.ascontiguousarray([f[0] for f in functions], dtype=np.float64).reshape(-1)
    degs = np.ascontiguousarray([f[1] for f in functions], dtype=np.int32).reshape(-1)
    nprim = np.ascontiguousarray([len(f[2]) for f in functions], dtype=np.int32)
    exps = np.ascontiguousarray([p[0] for f in functions for p in f[2]], dtype=np.float64)
    coefs = np.ascontiguousarray([p[1] for f in functions for p in f[2]], dtype=np.float64)
    handles = (C.c_void_p * nf)()
    _chk(olib().orc_basis_handle(_p(b), nn, C.c_int(nf), _p(centers), _p(degs), _p(nprim), _p(exps), _p(coefs),
                                 handles))
    out = []
    for i in range(nf):
        t = OCP.__new__(OCP)
        t.lib = olib()
        t.h = C.c_void_p(handles[i])
        out.append(t)
    return out


def coulomb_matrix(b_half, n, disc: list, vh: OCP) -> np.ndarray:
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(b_half, dtype=np.float64), (3,)))
    nn = (C.c_longlong * 3)(*np.broadcast_to(np.asarray(n), (3,)).tolist())
    nb = len(disc)
    hs = (C.c_void_p * nb)(*[d.h.value for d in disc])
    J = np.zeros((nb, nb), order="F")
    _chk(olib().orc_coulomb_matrix(_p(b), nn, C.c_int(nb), hs, vh.h, _p(J)))
    return J


def density_tensor(disc: list, c_occ, eps: float) -> OCP:
    c = _f(c_occ)
    nb = len(disc)
    hs = (C.c_void_p * nb)(*[d.h.value for d in disc])
    out = OCP()
    _chk(olib().orc_density_tensor(C.c_int(nb), hs, C.c_longlong(c.shape[1]), _p(c), C.c_double(eps), out.h))
    return out


def assemble_axis(b_half, n, ax: int, ref, centers) -> tuple[np.ndarray, int]:
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(b_half, dtype=np.float64), (3,)))
    nn = (C.c_longlong * 3)(*np.broadcast_to(np.asarray(n), (3,)).tolist())
    ref = _f(ref)
    cs = np.ascontiguousarray(centers, dtype=np.float64)
    out = np.zeros((nn[ax], ref.shape[1]), order="F")
    ops = C.c_longlong(0)
    _chk(olib().orc_assemble_axis(_p(b), nn, C.c_int(ax), C.c_longlong(ref.shape[1]), _p(ref),
                                  C.c_longlong(cs.shape[0]), _p(cs), _p(out), C.byref(ops)))
    return out, ops.value


def sym_eigen(a):
    a = _f(a)
    n = a.shape[0]
    ev = np.zeros(n)
    z = np.zeros((n, n), order="F")
    _chk(olib().orc_sym_eigen(C.c_longlong(n), _p(a), _p(ev), _p(z)))
    return ev, z


def householder_qr(a):
    a = _f(a)
    m, k = a.shape
    kk = min(m, k)
    q = np.zeros((m, kk), order="F")
    r = np.zeros((kk, k), order="F")
    _chk(olib().orc_householder_qr(C.c_longlong(m), C.c_longlong(k), _p(a), _p(q), _p(r)))
    return q, r


def jacobi_svd(a):
    a = _f(a)
    m, k = a.shape
    kk = min(m, k)
    u = np.zeros((m, kk), order="F")
    s = np.zeros(kk)
    _chk(olib().orc_jacobi_svd(C.c_longlong(m), C.c_longlong(k), _p(a), _p(u), _p(s)))
    return u, s


def thin_svd_left(a):
    a = _f(a)
    r, c = a.shape
    u = np.zeros((r, max(r, c)), order="F")
    s = np.zeros(max(r, c))
    kept = C.c_longlong()
    _chk(olib().orc_thin_svd_left(C.c_longlong(r), C.c_longlong(c), _p(a), _p(u), _p(s), C.byref(kept)))
    k = kept.value
    return np.asfortranarray(u.reshape(-1, order="F")[: r * k].reshape(r, k, order="F")), s[:k]


def reduce(a: OCP, eps: float | None = None, ranks=None, sweeps: int = 3, mode: int = 2):
    """mode 0 rhosvd, 1 canonical_to_tucker, 2 reduce_rank.  Returns dict."""
    info = (C.c_longlong * 6)()
    rk = (C.c_longlong * 3)(*(ranks or (0, 0, 0)))
    out = OCP()
    # first call without buffers to learn ranks, then fetch
    _chk(olib().orc_reduce(a.h, C.c_int(eps is not None), C.c_double(eps or 0.0), rk if ranks else None,
                           C.c_int(sweeps), C.c_int(mode), out.h, info, None, None, None, None, None))
    r = [info[0], info[1], info[2]]
    core = np.zeros(r[0] * r[1] * r[2])
    sides = [np.zeros((a.extent(ax), r[ax]), order="F") for ax in range(3)]
    fits = np.zeros(max(1, info[5]))
    _chk(olib().orc_reduce(a.h, C.c_int(eps is not None), C.c_double(eps or 0.0), rk if ranks else None,
                           C.c_int(sweeps), C.c_int(mode), out.h, info, _p(core), _p(sides[0]), _p(sides[1]),
                           _p(sides[2]), _p(fits)))
    return {"ranks": tuple(r), "rank_clamped": bool(info[3]), "rhosvd_fallback": bool(info[4]),
            "sweep_fits": fits[: info[5]], "core": core.reshape(r, order="F") if core.size else core,
            "sides": sides, "canonical": out if mode == 2 else None}


def pivoted_cholesky(a, tol, trace_stop: bool, max_rank: int, neg_tol: float):
    a = _f(a)
    n = a.shape[0]
    L = np.zeros((n, min(n, max_rank)), order="F")
    piv = np.zeros(n, dtype=np.int64)
    rank = C.c_longlong()
    res = C.c_double()
    cl = C.c_int()
    _chk(olib().orc_pivoted_cholesky(C.c_longlong(n), _p(a), C.c_double(tol), C.c_int(int(trace_stop)),
                                     C.c_longlong(max_rank), C.c_double(neg_tol), _p(L), _p(piv), C.byref(rank),
                                     C.byref(res), C.byref(cl)))
    k = rank.value
    return L[:, :k].copy(order="F"), piv[:k].copy(), res.value, bool(cl.value)


# --------------------------------------------------------------------------- hf.cpp / tei.cpp operators (§8f)

def _grid_args(b_half, n):
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(b_half, dtype=np.float64), (3,)))
    nn = (C.c_longlong * 3)(*np.broadcast_to(np.asarray(n), (3,)).tolist())
    return b, nn


def _handles(disc):
    return (C.c_void_p * len(disc))(*[d.h.value for d in disc])


def one_electron(b_half, n, disc: list, which: int) -> np.ndarray:
    """which 0: overlap_matrix (hf.cpp:48-58); 1/2: kinetic_matrix lumped / exact mass (hf.cpp:60-87)."""
    b, nn = _grid_args(b_half, n)
    nb = len(disc)
    out = np.zeros((nb, nb), order="F")
    _chk(olib().orc_one_electron(_p(b), nn, C.c_int(nb), _handles(disc), C.c_int(which), _p(out)))
    return out


def nuclear_potential_tensor(b_half, n, centers, charges, ref: OCP) -> OCP:
    """hf.cpp:89-101 on a doubled-grid reference kernel."""
    b, nn = _grid_args(b_half, n)
    c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1)
    q = np.ascontiguousarray(charges, dtype=np.float64)
    out = OCP()
    _chk(olib().orc_nuclear_potential_tensor(_p(b), nn, C.c_int(q.shape[0]), _p(c), _p(q), ref.h, out.h))
    return out


def nuclear_matrix(disc: list, pc: OCP) -> np.ndarray:
    nb = len(disc)
    V = np.zeros((nb, nb), order="F")
    _chk(olib().orc_nuclear_matrix(C.c_int(nb), _handles(disc), pc.h, _p(V)))
    return V


def exchange_matrix(b_half, n, disc: list, c_occ, kernel: OCP) -> np.ndarray:
    """hf.cpp:153-170 (primary-grid kernel)."""
    b, nn = _grid_args(b_half, n)
    c = _f(c_occ)
    nb = len(disc)
    K = np.zeros((nb, nb), order="F")
    _chk(olib().orc_exchange_matrix(_p(b), nn, C.c_int(nb), _handles(disc), C.c_longlong(c.shape[1]), _p(c),
                                    kernel.h, _p(K)))
    return K


def from_factors(which: int, chol, density, h_core=None) -> np.ndarray:
    """which 0/1/2: coulomb_ / exchange_ / fock_from_factors (tei.cpp:215-238)."""
    d = _f(density)
    nb = d.shape[0]
    L = _f(chol).reshape(nb * nb, -1, order="F")
    h = _f(h_core) if h_core is not None else np.zeros((1, 1), order="F")
    out = np.zeros((nb, nb), order="F")
    _chk(olib().orc_from_factors(C.c_int(which), C.c_longlong(nb), C.c_longlong(L.shape[1]), _p(h), _p(L), _p(d),
                                 _p(out)))
    return out


# --------------------------------------------------------------------------- the reference binary (oracle/_ref)

def _basis_args(functions):
    centers = np.ascontiguousarray([f[0] for f in functions], dtype=np.float64).reshape(-1)
    degs = np.ascontiguousarray([f[1] for f in functions], dtype=np.int32).reshape(-1)
    nprim = np.ascontiguousarray([len(f[2]) for f in functions], dtype=np.int32)
    exps = np.ascontiguousarray([p[0] for f in functions for p in f[2]], dtype=np.float64)
    coefs = np.ascontiguousarray([p[1] for f in functions for p in f[2]], dtype=np.float64)
    return centers, degs, nprim, exps, coefs


class Ref:
    """Calls into the reference's own hf.cpp / tei.cpp / reduction.cpp (oracle/_ref, shim LA)."""

    def __init__(self, b_half, n, functions):
        self.R = rlib()
        if self.R is None:
            raise FileNotFoundError("oracle/_ref not built (needs /root/reference)")
        self.b, self.nn = _grid_args(b_half, n)
        self.nb = len(functions)
        self.args = _basis_args(functions)
        self._keep = self.args

    def _basis(self):
        c, d, npr, e, cf = self.args
        return (_p(self.b), self.nn, C.c_int(self.nb), _p(c), _p(d), _p(npr), _p(e), _p(cf))

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.R.ref_last_error().decode())

    def one_electron(self, which: int) -> np.ndarray:
        out = np.zeros((self.nb, self.nb), order="F")
        self._chk(self.R.ref_one_electron(*self._basis(), C.c_int(which), _p(out)))
        return out

    def nuclear(self, centers, charges, m: int, c0: float):
        c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1)
        q = np.ascontiguousarray(charges, dtype=np.float64)
        V = np.zeros((self.nb, self.nb), order="F")
        pc = OCP(lib=self.R)
        self._chk(self.R.ref_nuclear(*self._basis(), C.c_int(q.shape[0]), _p(q), _p(c), C.c_longlong(m),
                                     C.c_double(c0), _p(V), pc.h))
        return V, pc

    def coulomb_matrix(self, vh: OCP) -> np.ndarray:
        J = np.zeros((self.nb, self.nb), order="F")
        self._chk(self.R.ref_coulomb_matrix(*self._basis(), vh.h, _p(J)))
        return J

    def exchange_matrix(self, c_occ, m: int, c0: float) -> np.ndarray:
        c = _f(c_occ)
        K = np.zeros((self.nb, self.nb), order="F")
        self._chk(self.R.ref_exchange_matrix(*self._basis(), C.c_longlong(c.shape[1]), _p(c), C.c_longlong(m),
                                             C.c_double(c0), _p(K)))
        return K

    def density_tensor(self, c_occ, eps: float) -> OCP:
        c = _f(c_occ)
        out = OCP(lib=self.R)
        self._chk(self.R.ref_density_tensor(*self._basis(), C.c_longlong(c.shape[1]), _p(c), C.c_double(eps),
                                            out.h))
        return out

    def build_tei(self, m: int, c0: float, eps_fit: float, eps_chol: float):
        """(fit ranks, R_B, clamped, fit residuals, chol, diagonal)."""
        info = (C.c_longlong * 5)()
        res = np.zeros(3)
        h = C.c_void_p()
        self._chk(self.R.ref_build_tei(*self._basis(), C.c_longlong(m), C.c_double(c0), C.c_double(eps_fit),
                                       C.c_double(eps_chol), info, _p(res), C.byref(h)))
        try:
            nb2 = self.nb * self.nb
            chol = np.zeros((nb2, info[3]), order="F")
            diag = np.zeros(nb2)
            self._chk(self.R.ref_tei_get(h, 0, 0, _p(chol)))
            self._chk(self.R.ref_tei_get(h, 1, 0, _p(diag)))
        finally:
            self.R.ref_tei_free(h)
        return (info[0], info[1], info[2]), info[3], bool(info[4]), res, chol, diag


def ref_from_factors(which: int, chol, density, h_core=None) -> np.ndarray:
    R = rlib()
    d = _f(density)
    nb = d.shape[0]
    L = _f(chol).reshape(nb * nb, -1, order="F")
    h = _f(h_core) if h_core is not None else np.zeros((1, 1), order="F")
    out = np.zeros((nb, nb), order="F")
    rc = R.ref_from_factors(C.c_int(which), C.c_longlong(nb), C.c_longlong(L.shape[1]), _p(h), _p(L), _p(d), _p(out))
    if rc:
        raise OracleError(rc, R.ref_last_error().decode())
    return out


def ref_generalized_eigensolve(f, s):
    R = rlib()
    f, s = _f(f), _f(s)
    nb = f.shape[0]
    c = np.zeros((nb, nb), order="F")
    e = np.zeros(nb)
    rc = R.ref_generalized_eigensolve(C.c_longlong(nb), _p(f), _p(s), _p(c), _p(e))
    if rc:
        raise OracleError(rc, R.ref_last_error().decode())
    return c, e


def ref_reduce(a: OCP, eps: float | None = None, ranks=None, sweeps: int = 3, mode: int = 2):
    """The reference's rhosvd (0) / canonical_to_tucker (1) / reduce_rank (2) on a tensor held by
    the reference library; returns (info dict, canonical OCP)."""
    R = rlib()
    info = (C.c_longlong * 7)()
    rk = (C.c_longlong * 3)(*(ranks or (0, 0, 0)))
    out = OCP(lib=R)
    rc = R.ref_reduce(a.h, C.c_int(eps is not None), C.c_double(eps or 0.0), rk, C.c_int(sweeps), C.c_int(mode),
                      info, out.h)
    if rc:
        raise OracleError(rc, R.ref_last_error().decode())
    return {"ranks": (info[0], info[1], info[2]), "rank_clamped": bool(info[3]), "rhosvd_fallback": bool(info[4]),
            "sweeps": info[5], "canonical_rank": info[6]}, out


def ref_mode_sigma(a: OCP, axis: int, eps: float | None = 1e-6, ranks=None, mode: int = 0) -> np.ndarray:
    """The reference's TuckerResult::mode_singular_values[axis] (rhosvd: mode 0)."""
    R = rlib()
    rk = (C.c_longlong * 3)(*(ranks or (0, 0, 0)))
    cap = max(1, min(a.rank(), max(a.factors()[axis].shape[0], 1)))
    out = np.zeros(cap)
    cnt = C.c_longlong()
    rc = R.ref_mode_sigma(a.h, C.c_int(eps is not None), C.c_double(eps or 0.0), rk, C.c_int(mode), C.c_int(axis),
                          C.c_longlong(cap), C.byref(cnt), _p(out))
    if rc:
        raise OracleError(rc, R.ref_last_error().decode())
    return out[:cnt.value]


def ref_expsum_for_interval(r_min: float, r_max: float, eps: float):
    R = rlib()
    m, c0 = C.c_longlong(), C.c_double()
    rc = R.ref_expsum_for_interval(C.c_double(r_min), C.c_double(r_max), C.c_double(eps), C.byref(m), C.byref(c0))
    if rc:
        raise OracleError(rc, R.ref_last_error().decode())
    return m.value, c0.value


def ref_scf_solve(ref: "Ref", nuclei, n_electrons: int, cfg: dict):
    """The reference's tg::scf_solve (hf.cpp:201-270) on the stand-in LA."""
    R = ref.R
    c = np.array([cfg["max_iterations"], cfg["energy_tol"], cfg["mixing"], cfg["eps_fit"], cfg["eps_chol"],
                  cfg["kernel_eps"], cfg.get("kernel_r_max", 0.0)], dtype=np.float64)
    q = np.ascontiguousarray([z for _, z in nuclei], dtype=np.float64)
    cen = np.ascontiguousarray([p for p, _ in nuclei], dtype=np.float64).reshape(-1)
    out = np.zeros(6)
    e = np.zeros(ref.nb)
    d = np.zeros((ref.nb, ref.nb), order="F")
    hist = np.zeros(int(cfg["max_iterations"]))
    rc = R.ref_scf_solve(*ref._basis(), C.c_int(q.shape[0]), _p(q), _p(cen), C.c_int(n_electrons), _p(c), _p(out),
                         _p(e), _p(d), _p(hist))
    if rc:
        raise OracleError(rc, R.ref_last_error().decode())
    it = int(out[3])
    return {"energy": out[0], "nuclear_energy": out[1], "converged": bool(out[2]), "iterations": it,
            "n_occupied": int(out[4]), "tei_rank_b": int(out[5]), "orbital_energies": e, "density": d,
            "energy_history": hist[:it]}

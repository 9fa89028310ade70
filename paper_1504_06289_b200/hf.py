"""Hartree-Fock operators on the convolution path, mirroring
/root/reference/proj/include/tengrid/hf.hpp and tei.hpp:76-79:
overlap / kinetic / nuclear / exchange matrices, the nuclear potential
tensor, and the Cholesky-factor Coulomb / exchange / Fock builders.  Every
call goes through libtgb.so (include/tgb.h); there is no CPU fallback.

Host numpy arrays run through the C ABI's host-memory mode (staged copies
inside the call); torch CUDA tensors / DeviceCP run device-resident.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import MEM_DEVICE, MEM_HOST, InvalidArgument, check, lib
from .tengrid import (BasisSet, CanonicalTensor3, Context, DeviceCP, KernelTensor, _h3, _mem, _out_like,
                      default_context, flatten_basis, snap_to_node, window_offset)


@dataclass
class Nucleus:
    """basis.hpp:37-40."""

    charge: float = 1.0
    center: tuple = (0.0, 0.0, 0.0)


@dataclass
class Molecule:
    """basis.hpp:42-52."""

    nuclei: list = field(default_factory=list)
    n_electrons: int = 0

    def n_occupied(self) -> int:
        if self.n_electrons == 1:
            return 1
        if self.n_electrons < 2 or self.n_electrons % 2:
            raise InvalidArgument("Molecule: closed-shell treatment needs an even electron count (or exactly one)")
        return self.n_electrons // 2


def _flat(disc: list):
    flat, offs = flatten_basis(disc)
    return flat, np.ascontiguousarray(offs, dtype=np.int64)


def _one_electron(fn, bs: BasisSet, disc: list, ctx: Context | None, *extra) -> np.ndarray:
    ctx = ctx or default_context()
    flat, offs = _flat(disc)
    nb = len(disc)
    out = np.zeros((nb, nb), order="F")
    cf = flat._cstruct()
    hh = _h3(bs.grid.h)
    check(fn(ctx.handle, C.byref(cf), offs.ctypes.data, nb, hh.ctypes.data, *extra, out.ctypes.data, MEM_HOST))
    return out


def overlap_matrix(bs: BasisSet, disc: list, ctx: Context | None = None) -> np.ndarray:
    """hf.cpp:48-58 — S_km = h^3 <G_k, G_m>."""
    return _one_electron(lib().tgb_overlap_matrix, bs, disc, ctx)


def kinetic_matrix(bs: BasisSet, disc: list, exact_mass: bool = False, ctx: Context | None = None) -> np.ndarray:
    """hf.cpp:60-87 — Kronecker FEM Laplacian with lumped or P1 mass."""
    return _one_electron(lib().tgb_kinetic_matrix, bs, disc, ctx, int(bool(exact_mass)))


def window_for_center(grid, center) -> tuple:
    """grid.cpp:40-47 — per-axis offsets into the doubled-grid reference."""
    return tuple(window_offset(grid, ax, float(center[ax])) for ax in range(3))


def nuclear_potential_tensor(bs: BasisSet, mol: Molecule, reference: KernelTensor, ctx: Context | None = None):
    """hf.cpp:89-101 — P_c = sum_a Z_a W_a Ptilde (rank = #nuclei * kernel rank)."""
    if not reference.doubled:
        raise InvalidArgument("nuclear_potential_tensor: reference kernel must live on the doubled grid")
    ctx = ctx or default_context()
    ref = reference.tensor
    offs = np.ascontiguousarray([window_for_center(bs.grid, nuc.center) for nuc in mol.nuclei],
                                dtype=np.int64).reshape(-1)
    q = np.ascontiguousarray([nuc.charge for nuc in mol.nuclei], dtype=np.float64)
    nn = len(mol.nuclei)
    mem = _mem(ref)
    dims = [bs.grid.n[ax] for ax in range(3)]
    if mem == MEM_DEVICE:
        out = DeviceCP.empty(dims, nn * ref.rank(), device=ref.weight.device)
    else:
        out = CanonicalTensor3([np.zeros((d, nn * ref.rank()), order="F") for d in dims], np.zeros(nn * ref.rank()))
    cr, co = ref._cstruct(), out._cstruct()
    check(lib().tgb_nuclear_potential_tensor(ctx.handle, C.byref(cr), offs.ctypes.data if nn else None,
                                             q.ctypes.data if nn else None, nn, C.byref(co), mem))
    return out


def nuclear_matrix(bs: BasisSet, disc: list, mol: Molecule, reference: KernelTensor,
                   ctx: Context | None = None) -> np.ndarray:
    """hf.cpp:103-116 — V_km = -<G_k . G_m, P_c>."""
    ctx = ctx or default_context()
    pc = nuclear_potential_tensor(bs, mol, reference, ctx)
    flat, offs = _flat(disc)
    nb = len(disc)
    if isinstance(pc, DeviceCP):
        flat = DeviceCP.from_host(flat, device=pc.weight.device)
    mem = _mem(flat, pc)
    cf, cp = flat._cstruct(), pc._cstruct()
    if mem == MEM_DEVICE:
        import torch

        V = torch.empty((nb, nb), dtype=torch.float64, device=pc.weight.device)
        check(lib().tgb_nuclear_matrix(ctx.handle, C.byref(cf), offs.ctypes.data, nb, C.byref(cp), V.data_ptr(), mem))
        return V.cpu().numpy().T.copy(order="F")
    V = np.zeros((nb, nb), order="F")
    check(lib().tgb_nuclear_matrix(ctx.handle, C.byref(cf), offs.ctypes.data, nb, C.byref(cp), V.ctypes.data, mem))
    return V


def exchange_matrix(bs: BasisSet, disc: list, c_occ, kernel: KernelTensor, ctx: Context | None = None) -> np.ndarray:
    """hf.cpp:153-170 — K_km = sum_a h^3 <G_k . phi_a, (G_m . phi_a) * P / h^3>, symmetrised."""
    if kernel.doubled:
        raise InvalidArgument("exchange_matrix: kernel must live on the primary grid")
    ctx = ctx or default_context()
    flat, offs = _flat(disc)
    nb = len(disc)
    c = np.asfortranarray(np.asarray(c_occ, dtype=np.float64).reshape(nb, -1))
    kt = kernel.tensor
    if isinstance(kt, DeviceCP):
        flat = DeviceCP.from_host(flat, device=kt.weight.device)
    mem = _mem(flat, kt)
    K = np.zeros((nb, nb), order="F")
    cf, ck = flat._cstruct(), kt._cstruct()
    hh = _h3(bs.grid.h)
    if mem == MEM_DEVICE:
        import torch

        cd = torch.from_numpy(np.ascontiguousarray(c.T)).to(kt.weight.device)
        Kd = torch.empty((nb, nb), dtype=torch.float64, device=kt.weight.device)
        check(lib().tgb_exchange_matrix(ctx.handle, C.byref(cf), offs.ctypes.data, nb, cd.data_ptr(), c.shape[1],
                                        C.byref(ck), hh.ctypes.data, Kd.data_ptr(), mem))
        return Kd.cpu().numpy().T.copy(order="F")
    check(lib().tgb_exchange_matrix(ctx.handle, C.byref(cf), offs.ctypes.data, nb, c.ctypes.data if c.size else None,
                                    c.shape[1], C.byref(ck), hh.ctypes.data, K.ctypes.data, mem))
    return K


def _factor_op(which: int, chol, density, h_core=None, ctx: Context | None = None):
    ctx = ctx or default_context()
    try:
        import torch

        on_dev = isinstance(chol, torch.Tensor) and chol.is_cuda
    except ImportError:  # pragma: no cover
        on_dev = False
    names = ("coulomb_from_factors", "exchange_from_factors", "fock_from_factors")
    if on_dev:
        # torch tensors hold the column-major matrices transposed: chol as (R, nb^2), density as (nb, nb)^T
        R, nn = chol.shape
        nb = int(round(nn ** 0.5))
        if nb * nb != nn or tuple(density.shape) != (nb, nb):
            raise InvalidArgument(f"{names[which]}: shape mismatch")
        out = torch.empty((nb, nb), dtype=torch.float64, device=chol.device)
        args = [ctx.handle, nb, R]
        if which == 2:
            args.append(h_core.contiguous().data_ptr())
        args += [chol.contiguous().data_ptr(), density.contiguous().data_ptr(), out.data_ptr(), MEM_DEVICE]
        check([lib().tgb_coulomb_from_factors, lib().tgb_exchange_from_factors, lib().tgb_fock_from_factors][which](*args))
        return out
    d = np.asfortranarray(np.asarray(density, dtype=np.float64))
    nb = d.shape[0]
    L = np.asfortranarray(np.asarray(chol, dtype=np.float64))
    if d.ndim != 2 or d.shape[1] != nb or L.shape[0] != nb * nb:
        raise InvalidArgument(f"{names[which]}: shape mismatch")
    out = np.zeros((nb, nb), order="F")
    args = [ctx.handle, nb, L.shape[1]]
    if which == 2:
        h = np.asfortranarray(np.asarray(h_core, dtype=np.float64))
        args.append(h.ctypes.data)
    args += [L.ctypes.data if L.size else None, d.ctypes.data, out.ctypes.data, MEM_HOST]
    check([lib().tgb_coulomb_from_factors, lib().tgb_exchange_from_factors, lib().tgb_fock_from_factors][which](*args))
    return out


def coulomb_from_factors(chol, density, ctx: Context | None = None):
    """tei.cpp:215-223 — J = unvec(L L^T vec D), symmetrised."""
    return _factor_op(0, chol, density, None, ctx)


def exchange_from_factors(chol, density, ctx: Context | None = None):
    """tei.cpp:225-234 — K = -1/2 sum_s M_s D M_s^T, symmetrised."""
    return _factor_op(1, chol, density, None, ctx)


def fock_from_factors(h_core, chol, density, ctx: Context | None = None):
    """tei.cpp:236-238 — F = h_core + J + K."""
    return _factor_op(2, chol, density, h_core, ctx)


def generalized_eigensolve(f, s, ctx: Context | None = None):
    """hf.cpp:187-199 — F C = S C diag(e), e ascending, C S-orthonormal (device)."""
    ctx = ctx or default_context()
    F = np.asfortranarray(np.asarray(f, dtype=np.float64))
    S = np.asfortranarray(np.asarray(s, dtype=np.float64))
    nb = F.shape[0]
    if F.shape != (nb, nb) or S.shape != (nb, nb):
        raise InvalidArgument("generalized_eigensolve: shape mismatch")
    Cm = np.zeros((nb, nb), order="F")
    e = np.zeros(nb)
    check(lib().tgb_generalized_eigensolve(ctx.handle, nb, F.ctypes.data, S.ctypes.data, Cm.ctypes.data,
                                           e.ctypes.data, MEM_HOST))
    return Cm, e


@dataclass
class SCFConfig:
    """hf.hpp:54-64."""

    max_iterations: int = 60
    energy_tol: float = 1e-9
    mixing: float = 0.7
    eps_fit: float = 1e-8
    eps_chol: float = 1e-10
    kernel_eps: float = 1e-6
    kernel_r_max: float = 0.0
    density_reduce_eps: float = 1e-7
    exact_mass_kinetic: bool = False


@dataclass
class SCFState:
    """hf.hpp:66-88 (tei: rank of the Cholesky factor only)."""

    coefficients: np.ndarray = None
    orbital_energies: np.ndarray = None
    density: np.ndarray = None
    n_occupied: int = 0
    energy: float = 0.0
    nuclear_energy: float = 0.0
    converged: bool = False
    iterations: int = 0
    energy_history: list = field(default_factory=list)
    residual_history: list = field(default_factory=list)
    orthonormality_defects: list = field(default_factory=list)
    overlap: np.ndarray = None
    core_hamiltonian: np.ndarray = None
    kinetic: np.ndarray = None
    nuclear: np.ndarray = None
    tei_rank_b: int = 0
    kernel_m: int = 0
    kernel_c0: float = 0.0
    snapped: Molecule = None


def scf_solve(mol: Molecule, bs: BasisSet, cfg: SCFConfig | None = None, ctx: Context | None = None) -> SCFState:
    """hf.cpp:201-270 — restricted closed-shell SCF, every operator on the device (tgb_scf_solve)."""
    from ._lib import tgb_basis_spec, tgb_molecule, tgb_scf_config, tgb_scf_state

    cfg = cfg or SCFConfig()
    ctx = ctx or default_context()
    nb = len(bs.functions)
    spec = tgb_basis_spec()
    for ax in range(3):
        spec.b_half[ax] = bs.grid.b_half[ax]
        spec.n[ax] = bs.grid.n[ax]
    spec.nfn = nb
    centers = np.ascontiguousarray([f.center for f in bs.functions], dtype=np.float64).reshape(-1)
    degs = np.ascontiguousarray([f.degree for f in bs.functions], dtype=np.int32).reshape(-1)
    poff = np.zeros(nb + 1, dtype=np.int64)
    poff[1:] = np.cumsum([len(f.primitives) for f in bs.functions])
    exps = np.ascontiguousarray([p.exponent for f in bs.functions for p in f.primitives], dtype=np.float64)
    coefs = np.ascontiguousarray([p.coeff for f in bs.functions for p in f.primitives], dtype=np.float64)
    spec.centers, spec.degrees, spec.prim_offset = centers.ctypes.data, degs.ctypes.data, poff.ctypes.data
    spec.exponents = exps.ctypes.data if exps.size else None
    spec.coeffs = coefs.ctypes.data if coefs.size else None
    m = tgb_molecule()
    m.nnuc = len(mol.nuclei)
    q = np.ascontiguousarray([nuc.charge for nuc in mol.nuclei], dtype=np.float64)
    nc = np.ascontiguousarray([nuc.center for nuc in mol.nuclei], dtype=np.float64).reshape(-1)
    m.charges = q.ctypes.data if q.size else None
    m.centers = nc.ctypes.data if nc.size else None
    m.n_electrons = mol.n_electrons
    c = tgb_scf_config(cfg.max_iterations, cfg.energy_tol, cfg.mixing, cfg.eps_fit, cfg.eps_chol, cfg.kernel_eps,
                       cfg.kernel_r_max, cfg.density_reduce_eps, int(cfg.exact_mass_kinetic))
    out = SCFState()
    mats = {k: np.zeros((nb, nb), order="F") for k in ("coefficients", "density", "overlap", "kinetic", "nuclear",
                                                       "core_hamiltonian")}
    e = np.zeros(nb)
    hist = {k: np.zeros(max(cfg.max_iterations, 1)) for k in ("energy_history", "residual_history",
                                                              "orthonormality_defects")}
    snapped = np.zeros(max(3 * len(mol.nuclei), 1))
    st = tgb_scf_state()
    for k, v in mats.items():
        setattr(st, k, v.ctypes.data)
    for k, v in hist.items():
        setattr(st, k, v.ctypes.data)
    st.orbital_energies = e.ctypes.data
    st.snapped_centers = snapped.ctypes.data
    check(lib().tgb_scf_solve(ctx.handle, C.byref(m), C.byref(spec), C.byref(c), C.byref(st)))
    for k, v in mats.items():
        setattr(out, k, v)
    out.orbital_energies = e
    it = st.iterations
    for k, v in hist.items():
        setattr(out, k, list(v[:it]))
    out.n_occupied, out.energy, out.nuclear_energy = st.n_occupied, st.energy, st.nuclear_energy
    out.converged, out.iterations, out.tei_rank_b = bool(st.converged), it, st.tei_rank_b
    out.kernel_m, out.kernel_c0 = st.kernel_m, st.kernel_c0
    out.snapped = Molecule([Nucleus(nuc.charge, tuple(snapped[3 * a:3 * a + 3])) for a, nuc in enumerate(mol.nuclei)],
                           mol.n_electrons)
    return out


# --------------------------------------------------------------------------- MP2 (mp2.hpp)


@dataclass
class MOSpace:
    """mp2.hpp:10-24."""

    coefficients: np.ndarray
    energies: np.ndarray
    n_occ: int

    def n_basis(self) -> int:
        return int(np.asarray(self.energies).shape[0])

    def n_virtual(self) -> int:
        return self.n_basis() - self.n_occ

    def gap(self) -> float:
        if self.n_occ < 1 or self.n_virtual() < 1:
            raise InvalidArgument("MOSpace: need occupied and virtual orbitals")
        return float(self.energies[self.n_occ] - self.energies[self.n_occ - 1])


@dataclass
class MOCholesky:
    """mp2.hpp:28-37 — rows i * n_vir + a."""

    factor: np.ndarray
    n_occ: int
    n_vir: int


def mo_transform_cholesky(chol, mos: MOSpace, ctx: Context | None = None) -> MOCholesky:
    """mp2.cpp:7-24 — C_occ^T mat(L_s) C_vir for every Cholesky column."""
    ctx = ctx or default_context()
    nb = mos.n_basis()
    L = np.asfortranarray(np.asarray(chol, dtype=np.float64))
    if L.shape[0] != nb * nb:
        raise InvalidArgument("mo_transform_cholesky: factor/basis shape mismatch")
    Cm = np.asfortranarray(np.asarray(mos.coefficients, dtype=np.float64))
    nov = mos.n_occ * mos.n_virtual()
    out = np.zeros((nov, L.shape[1]), order="F")
    check(lib().tgb_mo_transform_cholesky(ctx.handle, nb, L.shape[1], L.ctypes.data if L.size else None, mos.n_occ,
                                          Cm.ctypes.data, out.ctypes.data if out.size else None, MEM_HOST))
    return MOCholesky(out, mos.n_occ, mos.n_virtual())


def mp2_energy(mo: MOCholesky, mos: MOSpace, mode: str = "oracle", expsum_eps: float = 1e-9,
               ctx: Context | None = None) -> float:
    """mp2.cpp:97-103 — mode "oracle" (exact denominators) or "factorized" (exponential sums)."""
    ctx = ctx or default_context()
    if mo.n_occ != mos.n_occ or mo.n_vir != mos.n_virtual():
        raise InvalidArgument("mp2_energy: MO space mismatch")
    F = np.asfortranarray(np.asarray(mo.factor, dtype=np.float64))
    e = np.ascontiguousarray(mos.energies, dtype=np.float64)
    res = C.c_double()
    check(lib().tgb_mp2_energy(ctx.handle, mo.n_occ, mo.n_vir, F.shape[1], F.ctypes.data if F.size else None,
                               e.ctypes.data, {"oracle": 0, "factorized": 1}[mode], expsum_eps, C.byref(res),
                               MEM_HOST))
    return res.value

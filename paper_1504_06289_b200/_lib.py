"""ctypes binding of libtgb.so (include/tgb.h, include/tgb_host.h).

The library is loaded from the package directory (built in-tree by
build.py).  There is no fallback: if libtgb.so is missing or the GPU is not
an sm_100 device, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_HERE = Path(__file__).resolve().parent
import os

# TGB_LIB: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = _HERE / os.environ.get("TGB_LIB", "libtgb.so")


class TengridError(Exception):
    """Base of the mapped reference exception types."""


class InvalidArgument(TengridError, ValueError):
    """std::invalid_argument (tg::require, common.hpp:23-25)."""


class DomainError(TengridError, ValueError):
    """std::domain_error (grid.cpp:25, basis.cpp:22)."""


class SnapError(TengridError, RuntimeError):
    """tg::SnapError (common.hpp:11-15)."""


class NumericalError(TengridError, RuntimeError):
    """tg::NumericalError (common.hpp:17-21)."""


class CudaError(TengridError, RuntimeError):
    """CUDA / NCCL failure inside libtgb."""


_CODES = {1: InvalidArgument, 2: DomainError, 3: SnapError, 4: NumericalError, 5: CudaError}

MEM_HOST = 0
MEM_DEVICE = 1


class tgb_cp(C.Structure):
    _fields_ = [("n", C.c_int64 * 3), ("rank", C.c_int64), ("factor", C.c_void_p * 3), ("weight", C.c_void_p)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int64, C.c_int, C.c_void_p, C.c_void_p)


class tgb_comm(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("allreduce_sum", ALLREDUCE_FN), ("user", C.c_void_p)]


class tgb_scf_config(C.Structure):
    _fields_ = [("max_iterations", C.c_int), ("energy_tol", C.c_double), ("mixing", C.c_double),
                ("eps_fit", C.c_double), ("eps_chol", C.c_double), ("kernel_eps", C.c_double),
                ("kernel_r_max", C.c_double), ("density_reduce_eps", C.c_double), ("exact_mass_kinetic", C.c_int)]


class tgb_basis_spec(C.Structure):
    _fields_ = [("b_half", C.c_double * 3), ("n", C.c_int64 * 3), ("nfn", C.c_int64), ("centers", C.c_void_p),
                ("degrees", C.c_void_p), ("prim_offset", C.c_void_p), ("exponents", C.c_void_p),
                ("coeffs", C.c_void_p)]


class tgb_molecule(C.Structure):
    _fields_ = [("nnuc", C.c_int64), ("charges", C.c_void_p), ("centers", C.c_void_p), ("n_electrons", C.c_int64)]


class tgb_scf_state(C.Structure):
    _fields_ = [("energy", C.c_double), ("nuclear_energy", C.c_double), ("converged", C.c_int),
                ("iterations", C.c_int), ("n_occupied", C.c_int), ("tei_rank_b", C.c_int64),
                ("kernel_m", C.c_int64), ("kernel_c0", C.c_double)] + [
                   (name, C.c_void_p) for name in ("coefficients", "orbital_energies", "density", "overlap", "kinetic",
                                                   "nuclear", "core_hamiltonian", "energy_history", "residual_history",
                                                   "orthonormality_defects", "snapped_centers")]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise CudaError(f"libtgb.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(str(LIB_PATH))
        P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
        sig = {
            "tgb_ctx_create": (I, [I, P, C.POINTER(P)]),
            "tgb_ctx_destroy": (I, [P]),
            "tgb_ctx_stream": (P, [P]),
            "tgb_ctx_synchronize": (I, [P]),
            "tgb_last_error": (C.c_char_p, []),
            "tgb_ctx_launch_count": (I64, [P]),
            "tgb_ctx_reset_launch_count": (None, [P]),
            "tgb_ctx_set_direct_max": (I, [P, I64]),
            "tgb_ctx_transfer_bytes": (I, [P, C.POINTER(I64), C.POINTER(I64)]),
            "tgb_ctx_set_profiling": (I, [P, I]),
            "tgb_ctx_profile_read": (I, [P, C.POINTER(D), C.POINTER(I64)]),
            "tgb_shard_range": (I, [I64, I, I, C.POINTER(I64), C.POINTER(I64)]),
            "tgb_nccl_get_unique_id": (I, [P]),
            "tgb_ctx_init_nccl": (I, [P, I, I, P]),
            "tgb_ctx_set_comm": (I, [P, C.POINTER(tgb_comm)]),
            "tgb_ctx_comm_info": (I, [P, C.POINTER(I), C.POINTER(I)]),
            "tgb_comm_allreduce_host": (I, [C.POINTER(tgb_comm), P, I64]),
            "tgb_symmetric_allreduce_host": (I, [C.POINTER(tgb_comm), P, I64]),
            "tgb_hartree_potential_shard": (I, [P, C.POINTER(tgb_cp), C.POINTER(tgb_cp), P, C.POINTER(tgb_cp), I]),
            "tgb_value_at_allreduce": (I, [P, C.POINTER(tgb_cp), I64, P, P, I]),
            "tgb_coulomb_matrix_allreduce": (I, [P, C.POINTER(tgb_cp), P, I64, C.POINTER(tgb_cp), P, P, I]),
            "tgb_conv_central_many": (I, [P, I64, I64, P, P, P, I]),
            "tgb_convolve": (I, [P, C.POINTER(tgb_cp), C.POINTER(tgb_cp), P, C.POINTER(tgb_cp), I]),
            "tgb_hartree_potential": (I, [P, C.POINTER(tgb_cp), C.POINTER(tgb_cp), P, C.POINTER(tgb_cp), I]),
            "tgb_value_at": (I, [P, C.POINTER(tgb_cp), I64, P, P, I]),
            "tgb_scalar_product": (I, [P, C.POINTER(tgb_cp), C.POINTER(tgb_cp), C.POINTER(D), I]),
            "tgb_hadamard": (I, [P, C.POINTER(tgb_cp), C.POINTER(tgb_cp), C.POINTER(tgb_cp), I]),
            "tgb_add": (I, [P, C.POINTER(tgb_cp), C.POINTER(tgb_cp), C.POINTER(tgb_cp), I]),
            "tgb_scale": (I, [P, C.POINTER(tgb_cp), D, C.POINTER(tgb_cp), I]),
            "tgb_coulomb_matrix": (I, [P, C.POINTER(tgb_cp), P, I64, C.POINTER(tgb_cp), P, P, I]),
            "tgb_lattice_assemble_axis": (I, [P, I64, I64, P, P, I64, P, I]),
            "tgb_lattice_assemble": (I, [P, P, I64, P, P, P, P, I]),
            "tgb_nuclear_potential_tensor": (I, [P, C.POINTER(tgb_cp), P, P, I64, C.POINTER(tgb_cp), I]),
            "tgb_nuclear_matrix": (I, [P, C.POINTER(tgb_cp), P, I64, C.POINTER(tgb_cp), P, I]),
            "tgb_exchange_matrix": (I, [P, C.POINTER(tgb_cp), P, I64, P, I64, C.POINTER(tgb_cp), P, P, I]),
            "tgb_coulomb_from_factors": (I, [P, I64, I64, P, P, P, I]),
            "tgb_exchange_from_factors": (I, [P, I64, I64, P, P, P, I]),
            "tgb_fock_from_factors": (I, [P, I64, I64, P, P, P, P, I]),
            "tgb_generalized_eigensolve": (I, [P, I64, P, P, P, P, I]),
            "tgb_scf_config_default": (None, [C.POINTER(tgb_scf_config)]),
            "tgb_scf_solve": (I, [P, C.POINTER(tgb_molecule), C.POINTER(tgb_basis_spec), C.POINTER(tgb_scf_config),
                                  C.POINTER(tgb_scf_state)]),
            "tgb_expsum_for_interval": (I, [D, D, D, I64, C.POINTER(I64), C.POINTER(D)]),
            "tgb_mo_transform_cholesky": (I, [P, I64, I64, P, I64, P, P, I]),
            "tgb_mp2_energy": (I, [P, I64, I64, I64, P, P, I, D, C.POINTER(D), I]),
            "tgb_reciprocal_expsum": (I, [D, D, D, I64, C.POINTER(I64), P, P, C.POINTER(D), C.POINTER(I)]),
            "tgb_density_rank": (I, [P, I64, P, I64, C.POINTER(I64)]),
            "tgb_density_build": (I, [P, C.POINTER(tgb_cp), P, I64, P, I64, C.POINTER(tgb_cp), I]),
            "tgb_density_reduce": (I, [P, C.POINTER(tgb_cp), P, I64, P, I64, D, I, C.POINTER(P)]),
            "tgb_thin_svd_left": (I, [P, I64, I64, P, P, P, C.POINTER(I64), I]),
            "tgb_pivoted_cholesky": (I, [P, I64, P, D, I, I64, D, P, P, C.POINTER(I64), C.POINTER(D), C.POINTER(I), I]),
            "tgb_overlap_matrix": (I, [P, C.POINTER(tgb_cp), P, I64, P, P, I]),
            "tgb_kinetic_matrix": (I, [P, C.POINTER(tgb_cp), P, I64, P, I, P, I]),
            "tgb_tei_create": (I, [C.POINTER(P)]),
            "tgb_tei_destroy": (I, [P]),
            "tgb_tei_density_fitting": (I, [P, P, C.POINTER(tgb_cp), P, I64, P, D, I]),
            "tgb_tei_convolution_matrices": (I, [P, P, C.POINTER(tgb_cp), I]),
            "tgb_tei_diagonal": (I, [P, P, P, I]),
            "tgb_tei_column": (I, [P, P, I64, P, I]),
            "tgb_tei_cholesky": (I, [P, P, D]),
            "tgb_tei_info": (I, [P, P, P]),
            "tgb_tei_get_fit": (I, [P, I, P, P, I]),
            "tgb_tei_get_conv": (I, [P, I64, I, P, I]),
            "tgb_tei_get_cholesky": (I, [P, P, P, I]),
            "tgb_reduce_tucker": (I, [P, C.POINTER(tgb_cp), I, D, P, I, I, I, C.POINTER(P)]),
            "tgb_tucker_destroy": (I, [P]),
            "tgb_tucker_info": (I, [P, P]),
            "tgb_tucker_get": (I, [P, P, P, P, P, P, I]),
            "tgb_tucker_sigma": (I, [P, I, C.POINTER(I64), P]),
            "tgb_tucker_margins": (I, [P, I, P]),
            "tgb_mode_spectrum": (I, [P, C.POINTER(tgb_cp), I, I, P, P]),
            "tgb_tucker_to_canonical": (I, [P, P, C.POINTER(tgb_cp), I]),
            "tgb_dgemm": (I, [P, I, I, I64, I64, I64, D, P, I64, P, I64, D, P, I64]),
            "tgb_probe_fp64_peak": (I, [P, C.POINTER(D)]),
            "tgb_host_last_error": (C.c_char_p, []),
            "tgb_mesh_size": (D, [D, I64]),
            "tgb_snap_to_node": (I, [D, I64, D, C.POINTER(I64)]),
            "tgb_window_offset": (I, [D, I64, D, C.POINTER(I64)]),
            "tgb_make_expsum": (I, [I64, D, D, D, P, P, C.POINTER(D), C.POINTER(D)]),
            "tgb_kernel_factors": (I, [D, I64, I64, P, P, I, P]),
            "tgb_gauss_cell_integral": (D, [D, D, D]),
            "tgb_primitive_norm": (I, [D, I, C.POINTER(D)]),
            "tgb_gaussian_factor": (I, [D, I64, D, D, I, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int, host: bool = False) -> None:
    if rc == 0:
        return
    msg = (lib().tgb_host_last_error() if host else lib().tgb_last_error()) or b""
    raise _CODES.get(rc, TengridError)(msg.decode(errors="replace"))


EXPORTED_SYMBOLS = None  # filled lazily by exported_symbols()


def exported_symbols() -> list[str]:
    """Every function declared in include/tgb.h and include/tgb_host.h."""
    import re

    names = []
    for h in ("tgb.h", "tgb_host.h"):
        text = (_HERE.parent / "include" / h).read_text()
        names += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(tgb_[a-z_0-9]+)\s*\(", text, re.M)
    return sorted(set(names))

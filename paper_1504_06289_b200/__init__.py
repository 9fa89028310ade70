"""B200-native hot path of the tengrid Newton-kernel convolution stack
(arXiv 1504.06289): mode convolutions, J/TEI assembly, rank reduction and
lattice sums behind the reference's API.  See DESIGN.md."""
from ._lib import (CudaError, DomainError, InvalidArgument, NumericalError, SnapError, TengridError,
                   exported_symbols, lib)
from .tengrid import (AssembledPotential, BasisSet, CanonicalTensor3, Context, DeviceCP, ExpSum, GaussianPrimitive,
                      Grid3, KernelTensor, LatticeSpec, SeparableBasisFunction, add, conv_central_many,
                      convolve, coulomb_matrix, default_context, discretize_basis, flatten_basis,
                      gauss_cell_integral, hadamard, hartree_potential, kernel_tensor, lattice_assemble_axis,
                      lattice_offsets, lattice_sum_canonical, make_expsum, make_grid, primitive_norm, scalar_product,
                      scale, snap_to_node, value_at_points, window_offset, orbital_tensor, density_tensor,
                      LatticeBlock, lattice_grid, resolve_blocks, lattice_nodes, lattice_sum_tucker,
                      lattice_sum_composite)

from .tei import (PivotedCholesky, pivoted_cholesky, TEIFactorization, build_tei, tei_cholesky, tei_column, tei_convolution_matrices,
                  tei_density_fitting, tei_diagonal, tei_matrix_entry)

from .hf import (Molecule, Nucleus, SCFConfig, SCFState, generalized_eigensolve, scf_solve, MOSpace, MOCholesky,
                 mo_transform_cholesky, mp2_energy, coulomb_from_factors, exchange_from_factors, exchange_matrix,
                 fock_from_factors, kinetic_matrix, nuclear_matrix, nuclear_potential_tensor, overlap_matrix,
                 window_for_center)

from .reduction import (ReductionConfig, TuckerResult, TuckerTensor3, canonical_to_tucker, mode_spectrum, reduce_rank,
                        rhosvd, thin_svd_left)

__all__ = [n for n in dir() if not n.startswith("_")]

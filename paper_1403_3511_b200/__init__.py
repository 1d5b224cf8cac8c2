"""paper_1403_3511_b200 -- B200-native matrix-free Galerkin matvec for hprop.

Drop-in for the hot path of the reference package `hprop` 0.1.0
(arXiv 1403.3511, Brumm): index sets, the polynomial-potential matvec
y = W(X_1..X_N) c and the Lanczos/Magnus propagation loop, with the same
public names.  All numerics run in the sm_100a kernels of
`_lib/libhprop_b200.so` (C ABI: include/hprop_b200.h).
"""

from .index_set import (CUSTOM, FULL, HYPERBOLIC, CoeffVector, IndexSet, build_full, build_hyperbolic,
                        build_slab, extend, from_indices, load_index_set, neighbor, read_coeff_csv,
                        restrict, save_index_set)
from .potential_approx import (ChebApprox, PotentialSpec, chebyshev_values, custom_potential,
                               eval_interpolant, henon_heiles_perturbed, interpolate, potential_by_name,
                               smooth_remainder, torsional, torsional_minus_harmonic)
from .fast_apply import (PolynomialApplier, apply_hamiltonian, cheb_of_coordinate_apply, direct_op,
                         fast_algorithm, get_applier, install, square_sum_apply)
from .krylov_propagator import (LanczosFactorization, MagnusScheme, expm_tridiag_column, lanczos,
                                lanczos_exp_apply, magnus_step, propagate_magnus, tridiag_eigh)
from .error_lab import (MEASURE_REDUCTION, ErrorReport, FastHamiltonian, make_decay_vector, reduction_error,
                        reduction_local_mask)

__version__ = "0.1.0"

__all__ = [name for name in dir() if not name.startswith("_")]

"""paper_1408_2981_b200 -- B200-native (sm_100a) tensor-product multigrid hot path.

PCG preconditioned by a horizontally coarsening multigrid V-cycle with vertical
line-Jacobi relaxation (arXiv 1408.2981), matrix free, fp64, device resident.
The compute lives in ``libtpmg_b200.so`` (hand-written CUDA kernels behind the
C-ABI of ``include/tpmg_b200.h``); this package is the host-side mirror of the
reference's operator / smoother / transfer / solver interface.
"""
from . import synth  # noqa: F401
from .tpmg import (  # noqa: F401
    Context, Field, Hierarchy, SolveResult, TpmgError, apply_operator,
    build_hierarchy_coefficients, cap_error, config_error, cuda_error, dot, measure_cycle_rate,
    nccl_error, nonfinite_error, pcg_solve, pcg_solve_host, prolongate_field, residual,
    restrict_field, shape_error, singular_error, smooth, v_cycle,
    K_FASTEST, X_FASTEST, LINEAR, INJECTION, SUMMATION, TRANSPOSE,
)

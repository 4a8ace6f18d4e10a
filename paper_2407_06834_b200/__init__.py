"""B200-native ANOVA-Laplacian matvec + deflated CG (arXiv 2407.06834 hot path).

Drop-in for the reference package ``nldenoise``'s kernel-operator, matvec
and solver surface (kernel.py, linops.py, errors.py).  Compute runs in
hand-written sm_100a CUDA kernels behind the C-ABI in include/nld_b200.h;
importing this package fails if libnld_b200.so is missing (no CPU fallback).
"""

from . import bilevel
from ._lib import LIB_PATH
from .errors import (ConfigError, DenseLimitError, DimensionMismatchError,
                     NldenoiseError, ScalingOverflowError, SolverBreakdownError,
                     WindowSizeError)
from .kernel import AnovaOperator
from .linops import (DeflatingBasis, ShiftedSystem, SolveResult,
                     deflated_solve, deflated_solve_batched, pcg, plain_solve,
                     scs_down, scs_up)
from .transform import (FastsumPlan, NfftPlan, NodeSet, expansion_degree,
                        gauss_transform_direct, gauss_transform_fast, ndft,
                        ndft_adjoint, nfft, nfft_adjoint)

__version__ = "0.1.0"

__all__ = [
    "AnovaOperator", "ConfigError", "DeflatingBasis", "DenseLimitError",
    "DimensionMismatchError", "LIB_PATH", "NldenoiseError",
    "ScalingOverflowError", "ShiftedSystem", "SolveResult",
    "SolverBreakdownError", "WindowSizeError", "deflated_solve",
    "deflated_solve_batched", "pcg", "plain_solve", "scs_down", "scs_up",
    "FastsumPlan", "NfftPlan", "NodeSet", "expansion_degree",
    "gauss_transform_direct", "gauss_transform_fast", "ndft", "ndft_adjoint",
    "nfft", "nfft_adjoint", "bilevel",
]

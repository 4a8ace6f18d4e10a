"""ctypes binding of libnld_b200.so (the C-ABI in include/nld_b200.h).

This is the only path to the compute: there is no CPU fallback.  If the
shared library is missing, importing the package fails loudly; if no GPU is
present, every compute entry point fails with a CUDA error status.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# always the in-tree product build (no environment override: a mis-set
# variable can never swap in an experiment build)
LIB_PATH = os.path.join(_HERE, "libnld_b200.so")

NLD_OK = 0
ERR_DIMENSION, ERR_SCALING, ERR_WINDOW, ERR_DENSE_LIMIT = 1, 2, 3, 4
ERR_BREAKDOWN, ERR_VALUE, ERR_CUDA = 5, 6, 7

APPLY_GAMMA, APPLY_GAMMA_SQUARED, APPLY_SYSTEM, APPLY_LAPLACIAN = 0, 1, 2, 3
APPLY_WINDOW_SUM = 4
LAYOUT_PIXEL_MAJOR = 0x100     # OR into kind: batches are (n, nrhs)
PREC = {"none": 0, "jacobi": 1, "l2": 2}

_EXC = {
    ERR_DIMENSION: errors.DimensionMismatchError,
    ERR_SCALING: errors.ScalingOverflowError,
    ERR_WINDOW: errors.WindowSizeError,
    ERR_DENSE_LIMIT: errors.DenseLimitError,
    ERR_BREAKDOWN: errors.SolverBreakdownError,
    ERR_VALUE: ValueError,
    ERR_CUDA: RuntimeError,
}


class Params(ctypes.Structure):
    _fields_ = [("n_expansion", ctypes.c_int32), ("cutoff", ctypes.c_int32),
                ("oversampling", ctypes.c_double), ("rmax", ctypes.c_double),
                ("truncation_eps", ctypes.c_double), ("mode", ctypes.c_int32),
                ("no_sliced", ctypes.c_int32), ("dense_limit", ctypes.c_int64)]


class WindowInfo(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("bandwidth", ctypes.c_int32),
                ("grid", ctypes.c_int32), ("cutoff", ctypes.c_int32),
                ("center", ctypes.c_double * 3), ("scale", ctypes.c_double),
                ("sig_scaled", ctypes.c_double), ("box_lo", ctypes.c_int32 * 3),
                ("box_w", ctypes.c_int32 * 3), ("n_cells", ctypes.c_int64),
                ("n_subproblems", ctypes.c_int64), ("n_edge", ctypes.c_int64)]


class Stats(ctypes.Structure):
    _fields_ = [("spread_ms", ctypes.c_float), ("assemble_ms", ctypes.c_float),
                ("conv_ms", ctypes.c_float), ("gather_ms", ctypes.c_float),
                ("epilogue_ms", ctypes.c_float), ("total_ms", ctypes.c_float),
                ("launches", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_P = ctypes.c_void_p
_I32, _I64, _D = ctypes.c_int32, ctypes.c_int64, ctypes.c_double

# int (*)(ctx, buf, count, dtype, op, on_device, stream)  (nld_allreduce_fn)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_int32, ctypes.c_void_p)
_PI32 = ctypes.POINTER(ctypes.c_int32)
_PD = ctypes.POINTER(ctypes.c_double)

SIGNATURES = {
    "nld_last_error": (ctypes.c_char_p, []),
    "nld_abi_version": (ctypes.c_int, []),
    "nld_op_create": (ctypes.c_int, [_P, _I64, _I32, _PI32, _PI32, _I32, _D,
                                     ctypes.POINTER(Params), _P,
                                     ctypes.POINTER(_P)]),
    "nld_op_destroy": (ctypes.c_int, [_P]),
    "nld_op_set_comm": (ctypes.c_int, [_P, ALLREDUCE_FN, _P, _I64]),
    "nld_op_apply": (ctypes.c_int, [_P, _I32, _P, _P, _I32, _I64, _PD, _P]),
    "nld_op_degree": (ctypes.c_int, [_P, _I32, _P, _P]),
    "nld_op_assemble_dense": (ctypes.c_int, [_P, _I32, _P, _P]),
    "nld_op_window_info": (ctypes.c_int, [_P, _I32, ctypes.POINTER(WindowInfo)]),
    "nld_op_stats": (ctypes.c_int, [_P, ctypes.POINTER(Stats)]),
    "nld_op_set_timing": (ctypes.c_int, [_P, _I32]),
    "nld_op_debug_poison": (ctypes.c_int, [_P]),
    "nld_cg_solve": (ctypes.c_int, [_P, _P, _P, _I32, _I64, _PD, _PD, _I32, _I32,
                                    _D, _I32, _I32, _PI32, _PD, _PI32, _PD, _I32,
                                    _P]),
    "nld_basis_apply": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _P]),
    "nld_scs": (ctypes.c_int, [_P, _P, _I64, _I32, _P]),
    "nld_axpby": (ctypes.c_int, [_D, _P, _D, _P, _P, _I64, _P]),
    "nld_dot": (ctypes.c_int, [_P, _P, _I64, _PD, _P]),
    "nld_nfft_create": (ctypes.c_int, [_P, _I64, _I32, _I32, _D, _I32, _PD, _D, _I32, _P,
                                       ctypes.POINTER(_P)]),
    "nld_nfft_adjoint": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "nld_nfft_trafo": (ctypes.c_int, [_P, _P, _P, _P]),
    "nld_ndft": (ctypes.c_int, [_P, _I64, _I32, _I32, _P, _P, _I32, _P]),
    "nld_gauss_direct": (ctypes.c_int, [_P, _I64, _P, _I64, _I32, _P, _D, _P, _P]),
    "nld_fastsum_geometry": (ctypes.c_int, [_P, _I64, _I32, _D, _PD, _PD, _P]),
    "nld_gauss_coeffs": (ctypes.c_int, [_I32, _I32, _D, _P, _P]),
    "nld_window_factors": (ctypes.c_int, [_I32, _I32, _I32, _PD]),
    "nld_extract_patches": (ctypes.c_int, [_P, _I64, _I64, _I32, _I32, _I32, _D, _D, _P, _P]),
    "nld_mi_scores": (ctypes.c_int, [_P, _I64, _I32, _I32, _PD, _P]),
    "nld_probe_fp64": (ctypes.c_int, [_I64, _I32, _PD, _PD, _P]),
    "nld_probe_dmma": (ctypes.c_int, [_I64, _I32, _PD, _PD, _P]),
    "nld_probe_mixed": (ctypes.c_int, [_I64, _I64, _PD, _PD, _P]),
    "nld_probe_imma": (ctypes.c_int, [_I64, _I32, _PD, _PD, _P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import "
            "__graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    ver = lib.nld_abi_version()
    if ver == 1001 and os.environ.get("NLD_ALLOW_AB_BUILD") == "1":
        # the test-only A/B build (make ab), swapped in deliberately by a script
        import warnings
        warnings.warn("loaded the A/B test build of libnld_b200.so")
    elif ver != 1:
        raise ImportError(f"{LIB_PATH}: ABI version {ver}, expected 1 (the product build)")
    return lib


lib = _load()


def check(status: int) -> None:
    """Raise the reference exception class for a non-zero status."""
    if status == NLD_OK:
        return
    msg = lib.nld_last_error().decode("utf-8", "replace")
    raise _EXC.get(status, RuntimeError)(msg)

"""Drop-in shifted system, deflating basis and (deflated) PCG.

Mirrors ``nldenoise.linops`` (linops.py:28-319).  ``deflated_solve`` and
``plain_solve`` run entirely on the device (nld_cg_solve in
csrc/nld_cg.cu): the fused system matvec, the projected Jacobi / l2
preconditioner and the CG recurrences never leave HBM; the host reads a few
scalars per iteration for the stopping test, exactly where the reference
evaluates its Python-level conditions (linops.py:221-242).

Extension: ``deflated_solve_batched`` solves nrhs systems that share the
kernel (lam_r, mu_r per right-hand side) with every Gamma application shared
-- the config-4 alpha sweep of the bilevel driver (bilevel.py:173-181).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from ._lib import APPLY_LAPLACIAN, APPLY_SYSTEM, PREC, check, lib
from .errors import DimensionMismatchError, SolverBreakdownError
from .kernel import AnovaOperator

_PD = ctypes.POINTER(ctypes.c_double)
_PI = ctypes.POINTER(ctypes.c_int32)


class ShiftedSystem:
    """A = lambda I + mu (diag(eta) - Gamma), applied matrix-free."""

    def __init__(self, kernel: AnovaOperator, lam: float, mu: float):
        if lam <= 0 or mu <= 0:
            raise ValueError("shift lambda and weight mu must be positive")
        self.kernel = kernel
        self.lam = float(lam)
        self.mu = float(mu)
        self.eta = kernel.degree()

    @property
    def n(self) -> int:
        return self.kernel.n

    def laplacian_apply(self, v):
        """L v = diag(eta) v - Gamma v (linops.py:43-46)."""
        return self.kernel._product(v, APPLY_LAPLACIAN)

    def apply(self, v):
        """lam v + mu L v, fused into the gather epilogue (linops.py:48-50)."""
        x, nrhs = self.kernel._vectors(v)
        coef = np.tile([self.lam, self.mu], nrhs)
        out = self.kernel.apply_device(x, APPLY_SYSTEM, nrhs, coef)
        return dv.like_input(out, v)

    def __matmul__(self, v):
        return self.apply(v)

    def jacobi_diagonal(self):
        """diag(A) = lambda + mu eta (linops.py:57-59)."""
        return self.lam + self.mu * self.eta

    def l2_diagonal(self, exact: bool = False):
        """Row-wise l2 estimate as a diagonal preconditioner (linops.py:61-75)."""
        pa = self.jacobi_diagonal()
        if exact:
            g = self.kernel.assemble_dense()
            row_sq = (g * g).sum(axis=1) if isinstance(g, np.ndarray) \
                else (g * g).sum(dim=1)
        else:
            ell = self.kernel.n_windows
            row_sq = self.kernel.degree_squared() / (ell * ell)
        if isinstance(pa, np.ndarray):
            return np.sqrt(self.mu * self.mu * row_sq + pa * pa)
        return torch.sqrt(self.mu * self.mu * row_sq + pa * pa)


# ---------------------------------------------------------------------------
# Change of basis (linops.py:114-176), on the device
# ---------------------------------------------------------------------------

def _vec(x, n=None, device=None):
    shape = tuple(x.shape) if hasattr(x, "shape") else np.shape(x)
    if len(shape) != 1:
        raise DimensionMismatchError("expected a 1-d vector")
    if n is not None and shape[0] != n:
        raise DimensionMismatchError(f"length {shape[0]}, expected {n}")
    return dv.to_device(x, dv.pick_device(x, device))


def scs_up(x):
    """out_i = x_1 + sum_{j>i} x_j, out_n = x_1 (linops.py:114-121)."""
    t = _vec(x)
    out = torch.empty_like(t)
    check(lib.nld_scs(dv.ptr(t), dv.ptr(out), t.numel(), 0, dv.stream_of(t.device)))
    return dv.like_input(out, x)


def scs_down(x):
    """out_1 = sum_j x_j, out_i = sum_{j<i} x_j (linops.py:124-131)."""
    t = _vec(x)
    out = torch.empty_like(t)
    check(lib.nld_scs(dv.ptr(t), dv.ptr(out), t.numel(), 1, dv.stream_of(t.device)))
    return dv.like_input(out, x)


class DeflatingBasis:
    """Orthogonal basis U with first column v/||v||, applied in O(n)."""

    def __init__(self, v):
        shape = tuple(v.shape) if hasattr(v, "shape") else np.shape(v)
        if len(shape) != 1:
            raise DimensionMismatchError("expected a 1-d vector")
        if shape[0] < 2:
            raise DimensionMismatchError("basis needs at least two entries")
        self.v = v
        self._v = _vec(v)
        if float(self._v[0].item()) == 0.0:
            raise ValueError("leading entry of v must be nonzero")

    @property
    def n(self) -> int:
        return self._v.numel()

    def _run(self, x, adjoint):
        t = _vec(x, self.n, self._v.device)
        out = torch.empty_like(t)
        check(lib.nld_basis_apply(dv.ptr(self._v), dv.ptr(t), dv.ptr(out), self.n,
                                  adjoint, dv.stream_of(t.device)))
        return dv.like_input(out, x)

    def apply(self, x):
        """U x."""
        return self._run(x, 0)

    def apply_adjoint(self, x):
        """U^T x."""
        return self._run(x, 1)


# ---------------------------------------------------------------------------
# Preconditioned conjugate gradients (linops.py:184-244)
# ---------------------------------------------------------------------------

@dataclass
class SolveResult:
    x: object
    iterations: int
    converged: bool
    relative_residual: float
    residual_history: list = field(default_factory=list)


def _dot(a: torch.Tensor, b: torch.Tensor) -> float:
    res = ctypes.c_double()
    check(lib.nld_dot(dv.ptr(a), dv.ptr(b), a.numel(), ctypes.byref(res),
                      dv.stream_of(a.device)))
    return res.value


def _axpby(a, x, b, y, out):
    check(lib.nld_axpby(float(a), dv.ptr(x), float(b), dv.ptr(y), dv.ptr(out),
                        x.numel(), dv.stream_of(x.device)))
    return out


def pcg(apply_a, b, x0=None, *, prec=None, tol: float = 1e-10,
        maxit: int = 100) -> SolveResult:
    """Conjugate gradients with an optional preconditioner callable.

    Same algorithm and stopping rule as linops.py:193-244 (true-residual
    confirmation, bnorm = max(||b||, ||r0||), breakdown on pAp <= 0 or
    non-finite values).  The recurrences and inner products run on the
    device; ``apply_a`` / ``prec`` receive and return vectors of the same
    kind as ``b`` (numpy or torch), like the reference's callables.
    """
    host = not dv.is_torch(b)
    dev = dv.pick_device(b)
    bt = dv.to_device(b, dev)

    def call(fn, t):
        res = fn(dv.to_host(t) if host else t)
        return dv.to_device(res, dev)

    def fin(t):
        return dv.to_host(t) if host else t

    bn = _dot(bt, bt) ** 0.5
    if bn == 0.0 and x0 is None:
        return SolveResult(fin(torch.zeros_like(bt)), 0, True, 0.0, [0.0])
    x = torch.zeros_like(bt) if x0 is None else dv.to_device(x0, dev).clone()
    r = _axpby(1.0, bt, -1.0, call(apply_a, x), torch.empty_like(bt))
    rn = _dot(r, r) ** 0.5
    bnorm = max(bn, rn)
    if bnorm == 0.0:
        return SolveResult(fin(x), 0, True, 0.0, [0.0])
    history = [rn / bnorm]
    if maxit <= 0:
        return SolveResult(fin(x), 0, False, history[0], history)
    z = call(prec, r) if prec is not None else r
    p = z.clone()
    rz = _dot(r, z)
    it = 0
    while it < maxit:
        ap = call(apply_a, p)
        pap = _dot(p, ap)
        if not np.isfinite(pap) or pap <= 0.0:
            raise SolverBreakdownError(
                f"indefinite or non-finite curvature at iteration {it}")
        alpha = rz / pap
        _axpby(1.0, x, alpha, p, x)
        _axpby(1.0, r, -alpha, ap, r)
        it += 1
        rel = _dot(r, r) ** 0.5 / bnorm
        history.append(rel)
        if rel <= tol:
            res = _axpby(1.0, bt, -1.0, call(apply_a, x), torch.empty_like(bt))
            true_rel = _dot(res, res) ** 0.5 / bnorm
            history[-1] = true_rel
            if true_rel <= tol:
                return SolveResult(fin(x), it, True, true_rel, history)
        z = call(prec, r) if prec is not None else r
        rz_new = _dot(r, z)
        if not np.isfinite(rz_new):
            raise SolverBreakdownError("non-finite residual inner product")
        _axpby(1.0, z, rz_new / rz, p, p)
        rz = rz_new
    res = _axpby(1.0, bt, -1.0, call(apply_a, x), torch.empty_like(bt))
    rel = _dot(res, res) ** 0.5 / bnorm
    return SolveResult(fin(x), it, rel <= tol, rel, history)


# ---------------------------------------------------------------------------
# Deflated / plain solves on the device (linops.py:252-319)
# ---------------------------------------------------------------------------

def _solve(kernel: AnovaOperator, f, lams, mus, prec, tol, maxit, warm_start,
           deflate, history_cap=None):
    if prec not in PREC:
        raise ValueError(f"unknown preconditioner {prec!r}")
    shape = tuple(f.shape) if hasattr(f, "shape") else np.shape(f)
    if len(shape) == 1:
        nrhs = 1
        if shape[0] != kernel.n:
            raise DimensionMismatchError(f"length {shape[0]}, expected {kernel.n}")
    elif len(shape) == 2 and shape[1] == kernel.n:
        nrhs = shape[0]
    else:
        raise DimensionMismatchError("f must be (n,) or (nrhs, n)")
    lam = np.ascontiguousarray(np.broadcast_to(np.asarray(lams, np.float64), (nrhs,)))
    mu = np.ascontiguousarray(np.broadcast_to(np.asarray(mus, np.float64), (nrhs,)))
    ft = dv.to_device(f, kernel.device)
    u = torch.empty_like(ft)
    iters = np.zeros(nrhs, np.int32)
    relres = np.zeros(nrhs, np.float64)
    conv = np.zeros(nrhs, np.int32)
    cap = (max(maxit, 0) + 2) if history_cap is None else history_cap
    hist = np.full((nrhs, cap), np.nan)
    check(lib.nld_cg_solve(
        kernel._handle, dv.ptr(ft), dv.ptr(u), nrhs, kernel.n,
        lam.ctypes.data_as(_PD), mu.ctypes.data_as(_PD), PREC[prec],
        1 if deflate else 0, float(tol), int(maxit), 1 if warm_start else 0,
        iters.ctypes.data_as(_PI), relres.ctypes.data_as(_PD),
        conv.ctypes.data_as(_PI), hist.ctypes.data_as(_PD), cap,
        dv.stream_of(kernel.device)))
    xs = dv.like_input(u, f)
    out = []
    for r in range(nrhs):
        h = hist[r]
        h = [float(x) for x in h[~np.isnan(h)]]
        out.append(SolveResult(xs if nrhs == 1 else xs[r], int(iters[r]),
                               bool(conv[r]), float(relres[r]), h))
    return out


def deflated_solve(system: ShiftedSystem, f, *, prec: str = "jacobi",
                   tol: float = 1e-10, maxit: int = 100,
                   warm_start: bool = False) -> SolveResult:
    """Solve A u = lambda f with the constant eigenpair split off.

    linops.py:263-300: PCG on the orthogonal complement of 1, projected
    diagonal preconditioner selected by ``prec`` in {"none", "jacobi",
    "l2"}, zero tail start unless ``warm_start``.
    """
    if prec not in PREC:
        raise ValueError(f"unknown preconditioner {prec!r}")
    shape = tuple(f.shape) if hasattr(f, "shape") else np.shape(f)
    if len(shape) != 1:
        raise DimensionMismatchError("expected a 1-d vector")
    return _solve(system.kernel, f, system.lam, system.mu, prec, tol, maxit,
                  warm_start, True)[0]


def plain_solve(system: ShiftedSystem, f, *, prec: str = "none",
                tol: float = 1e-10, maxit: int = 100,
                warm_start: bool = False) -> SolveResult:
    """Solve A u = lambda f by PCG in the original basis (linops.py:303-319)."""
    if prec not in PREC:
        raise ValueError(f"unknown preconditioner {prec!r}")
    shape = tuple(f.shape) if hasattr(f, "shape") else np.shape(f)
    if len(shape) != 1:
        raise DimensionMismatchError("expected a 1-d vector")
    return _solve(system.kernel, f, system.lam, system.mu, prec, tol, maxit,
                  warm_start, False)[0]


def deflated_solve_batched(kernel: AnovaOperator, f, lams, mus, *,
                           prec: str = "jacobi", tol: float = 1e-10,
                           maxit: int = 100, warm_start: bool = False):
    """nrhs deflated solves sharing every Gamma application.

    f is (n,) (broadcast to every system) or (nrhs, n); lams/mus are scalars
    or length-nrhs.  Returns one SolveResult per right-hand side.
    """
    mus = np.atleast_1d(np.asarray(mus, np.float64))
    lams = np.atleast_1d(np.asarray(lams, np.float64))
    nrhs = max(mus.size, lams.size)
    shape = tuple(f.shape) if hasattr(f, "shape") else np.shape(f)
    if len(shape) == 1:
        if dv.is_torch(f):
            f = f.unsqueeze(0).expand(nrhs, -1).contiguous()
        else:
            f = np.broadcast_to(np.asarray(f, np.float64), (nrhs, shape[0]))
    return _solve(kernel, f, lams, mus, prec, tol, maxit, warm_start, True)

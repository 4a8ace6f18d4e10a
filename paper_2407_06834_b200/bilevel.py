"""Bilevel learning of the fidelity weight on the device (reference bilevel.py).

The caller of the hot path: the upper level
minimises the mean squared training error j(lambda) over lambda with Brent's
method; every evaluation is a lower-level deflated Jacobi-PCG solve of the
shifted Laplacian per training image, here on the GPU through the sliced /
fp64 tensor-core products.

* ``brent_minimize`` -- scalar host logic, the golden-section / parabolic
  minimiser of bilevel.py:42-101 restated step for step (same iterate
  sequence; tests/golden/bilevel.npz pins it against the reference).
* ``TrainingPair`` / ``TrainingSet`` -- clean/noisy pixel arrays (2-D numpy
  or torch, or objects with ``.pixels`` such as the reference's GrayImage) and
  the kernel / solver settings, defaults of bilevel.py:111-124.
* ``ReducedObjective`` -- bilevel.py:160-190: per pair the device features
  (``feature_windows``: patches + MI window split, features.py) and one
  ``AnovaOperator``, built once; ``__call__(lam)`` solves every pair.  The
  B200 extension ``values(lams)`` evaluates many lambdas in ONE batched solve
  per pair (``deflated_solve_batched``): all candidate systems share every
  Gamma application, so a sweep of k lambdas costs about one solve, not k.
* ``train`` / ``validate`` -- bilevel.py:244-272 without the SSIM scores
  (image quality metrics belong to imaging.py, outside the hot-path scope);
  ``sweep_then_brent`` brackets with one batched sweep before Brent.

Image I/O, noise generation, SSIM and the CLI stay out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from .features import feature_windows
from .kernel import AnovaOperator
from .linops import ShiftedSystem, deflated_solve, deflated_solve_batched

GOLDEN = 0.5 * (3.0 - np.sqrt(5.0))          # bilevel.py:24
DEFAULT_LAMBDA_RANGE = (1e-9, 3.0)           # bilevel.py:26-30
DEFAULT_BRENT_TOL = 1e-10
DEFAULT_BRENT_MAXIT = 30
DEFAULT_INNER_TOL = 1e-10
DEFAULT_INNER_MAXIT = 25
_EPS = float(np.finfo(float).eps)


@dataclass
class BrentResult:
    x: float
    fx: float
    iterations: int
    converged: bool
    history: list = field(default_factory=list)


def brent_minimize(fun, a: float, b: float, *, tol: float = DEFAULT_BRENT_TOL,
                   maxit: int = DEFAULT_BRENT_MAXIT) -> BrentResult:
    """Minimise a scalar function on [a, b] without derivatives.

    Brent's method as in bilevel.py:42-101: x is the best point so far, w the
    second best, v the previous w; a parabola through (v, w, x) proposes the
    step when it falls inside the bracket and shrinks fast enough, else a
    golden-section step into the larger part.  Stops when the bracket around
    x is within 2 tol1 (tol1 = tol |x| + tol), or when a minimum-size step
    makes no measurable change.
    """
    if not b > a:
        raise ValueError("need a nondegenerate bracket a < b")
    x = w = v = a + GOLDEN * (b - a)
    fx = fw = fv = fun(x)
    step = prev_step = 0.0          # d and e of the classic formulation
    history = [(x, fx)]
    for it in range(1, maxit + 1):
        mid = 0.5 * (a + b)
        tol1 = tol * abs(x) + tol
        if abs(x - mid) <= 2.0 * tol1 - 0.5 * (b - a):
            return BrentResult(x, fx, it - 1, True, history)
        parabolic = False
        if abs(prev_step) > tol1:
            r = (x - w) * (fx - fv)
            q = (x - v) * (fx - fw)
            p = (x - v) * q - (x - w) * r
            q = 2.0 * (q - r)
            if q > 0:
                p = -p
            q = abs(q)
            older, prev_step = prev_step, step
            if abs(p) < abs(0.5 * q * older) and q * (a - x) < p < q * (b - x):
                step = p / q
                u = x + step
                if u - a < 2.0 * tol1 or b - u < 2.0 * tol1:
                    step = tol1 if x < mid else -tol1
                parabolic = True
        if not parabolic:
            prev_step = (b if x < mid else a) - x
            step = GOLDEN * prev_step
        if abs(step) >= tol1:
            u = x + step
        else:
            u = x + (tol1 if step > 0 else -tol1)
        fu = fun(u)
        history.append((u, fu))
        if abs(u - x) <= 2.0 * tol1 and abs(fu - fx) <= 4.0 * _EPS * max(abs(fx), 1.0):
            if fu < fx:
                x, fx = u, fu
            return BrentResult(x, fx, it, True, history)
        if fu <= fx:
            if u < x:
                b = x
            else:
                a = x
            v, fv, w, fw, x, fx = w, fw, x, fx, u, fu
        else:
            if u < x:
                a = u
            else:
                b = u
            if fu <= fw or w == x:
                v, fv, w, fw = w, fw, u, fu
            elif fu <= fv or v == x or v == w:
                v, fv = u, fu
    return BrentResult(x, fx, maxit, False, history)


def _pixels(img):
    return getattr(img, "pixels", img)


@dataclass
class TrainingPair:
    clean: object
    noisy: object


@dataclass
class TrainingSet:
    """Clean/noisy pairs plus the kernel and solver settings (bilevel.py:111-124)."""

    pairs: list
    patch_size: int = 7
    sigma: float = 40.0
    mu: float = 0.01
    kernel_mode: str = "exact"
    inner_tol: float = DEFAULT_INNER_TOL
    inner_maxit: int = DEFAULT_INNER_MAXIT

    @classmethod
    def from_arrays(cls, clean, noisy, **kwargs):
        return cls([TrainingPair(c, n) for c, n in zip(clean, noisy)], **kwargs)


class ReducedObjective:
    """j(lambda): mean squared training error of the lower-level solves.

    bilevel.py:160-190.  Features, windows and operators are built once per
    pair on the device; the noisy right-hand side and the clean target stay
    resident, so an evaluation moves only a scalar back to the host.
    """

    def __init__(self, training: TrainingSet, device=None):
        self.training = training
        self._problems = []
        for pair in training.pairs:
            noisy = _pixels(pair.noisy)
            dev = dv.pick_device(noisy) if device is None else torch.device(device)
            nt = dv.to_device(noisy, dev)
            feats, wins = feature_windows(nt, training.patch_size)
            op = AnovaOperator(feats, wins, training.sigma, mode=training.kernel_mode)
            f = nt.reshape(-1).contiguous()
            clean = dv.to_device(_pixels(pair.clean), dev).reshape(-1).contiguous()
            self._problems.append((pair, op, f, clean))
        self.evaluations = 0

    def _system(self, op, lam):
        return ShiftedSystem(op, lam, self.training.mu)

    def denoise_all(self, lam: float) -> list:
        """One deflated Jacobi-PCG solve per pair (bilevel.py:170-178)."""
        out = []
        for pair, op, f, _ in self._problems:
            res = deflated_solve(self._system(op, lam), f, prec="jacobi",
                                 tol=self.training.inner_tol,
                                 maxit=self.training.inner_maxit)
            out.append(res.x if dv.is_torch(_pixels(pair.noisy)) else res.x.cpu().numpy())
        return out

    def __call__(self, lam: float) -> float:
        self.evaluations += 1
        total = 0.0
        for (pair, op, f, clean) in self._problems:
            res = deflated_solve(self._system(op, lam), f, prec="jacobi",
                                 tol=self.training.inner_tol,
                                 maxit=self.training.inner_maxit)
            diff = clean - res.x
            total += float(torch.dot(diff, diff))
        return total / len(self._problems)

    def values(self, lams) -> np.ndarray:
        """j at every lambda of ``lams``: one batched solve per pair.

        The systems lambda_k I + mu L share Gamma; deflated_solve_batched runs
        them as right-hand sides of one CG whose products apply Gamma to all
        of them at once (per-rhs convergence masks, deflation and Jacobi
        diagonals).  Each lambda's iterate sequence is the one a single solve
        would produce; only the reduction rounding differs.
        """
        lams = np.atleast_1d(np.asarray(lams, np.float64))
        if lams.size == 0:
            return np.zeros(0)
        if np.any(lams <= 0):
            raise ValueError("lambda must be positive")
        self.evaluations += int(lams.size)
        total = np.zeros(lams.size)
        for (pair, op, f, clean) in self._problems:
            # the system's right-hand side is lambda f: the batched solve
            # scales each row by its own lambda
            res = deflated_solve_batched(op, f, lams, self.training.mu, prec="jacobi",
                                         tol=self.training.inner_tol,
                                         maxit=self.training.inner_maxit)
            for k, r in enumerate(res):
                diff = clean - r.x
                total[k] += float(torch.dot(diff, diff))
        return total / len(self._problems)


@dataclass
class TrainingReport:
    """bilevel.py:197-207 without the SSIM lists (imaging is out of scope)."""

    lambda_opt: float
    objective_opt: float
    brent_iterations: int
    brent_converged: bool
    objective_at_bounds: tuple
    history: list
    evaluations: int = 0


def train(training: TrainingSet, *, lambda_range=DEFAULT_LAMBDA_RANGE,
          tol: float = DEFAULT_BRENT_TOL, maxit: int = DEFAULT_BRENT_MAXIT,
          objective: ReducedObjective | None = None) -> TrainingReport:
    """Learn the fidelity weight on the training pairs (bilevel.py:244-258)."""
    objective = ReducedObjective(training) if objective is None else objective
    lo, hi = lambda_range
    res = brent_minimize(objective, lo, hi, tol=tol, maxit=maxit)
    j_lo, j_hi = objective(lo), objective(hi)
    return TrainingReport(res.x, res.fx, res.iterations, res.converged, (j_lo, j_hi),
                          res.history, objective.evaluations)


def validate(training: TrainingSet, lambda_opt: float) -> TrainingReport:
    """Apply a learned fidelity weight to held-out pairs (bilevel.py:261-272)."""
    objective = ReducedObjective(training)
    fx = objective(lambda_opt)
    return TrainingReport(lambda_opt, fx, 0, True, (np.nan, np.nan), [],
                          objective.evaluations)


def sweep_then_brent(training: TrainingSet, *, lambda_range=DEFAULT_LAMBDA_RANGE,
                     points: int = 16, tol: float = DEFAULT_BRENT_TOL,
                     maxit: int = DEFAULT_BRENT_MAXIT,
                     objective: ReducedObjective | None = None) -> TrainingReport:
    """Batched log-spaced sweep (one solve per pair for all points), then Brent
    on the bracket around the best point -- the config-4 style alpha sweep
    feeding the reference's minimiser.  Not a reference entry point."""
    objective = ReducedObjective(training) if objective is None else objective
    lo, hi = lambda_range
    grid = np.geomspace(lo, hi, points)
    vals = objective.values(grid)
    k = int(np.argmin(vals))
    a, b = grid[max(k - 1, 0)], grid[min(k + 1, points - 1)]
    res = brent_minimize(objective, a, b, tol=tol, maxit=maxit)
    best = min([(res.fx, res.x)] + [(float(vals[k]), float(grid[k]))])
    hist = [(float(x), float(y)) for x, y in zip(grid, vals)] + list(res.history)
    return TrainingReport(best[1], best[0], res.iterations, res.converged,
                          (float(vals[0]), float(vals[-1])), hist, objective.evaluations)

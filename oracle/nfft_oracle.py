"""CPU oracle for the ANOVA-Laplacian hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``nldenoise``
(`/root/reference/pkg/src/nldenoise`) along the path named in BASELINE.json's
north star.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the
checker or as the timed CPU baseline.  The product package
(`paper_2407_06834_b200`) never imports it; there is no CPU fallback.

Parity pin: ``tests/golden/make_golden.py`` runs the real reference in the
build container and stores its outputs under ``tests/golden``;
``tests/test_oracle_golden.py`` checks this restatement against them.

Every function cites the reference file:line it restates.
"""

from __future__ import annotations

import numpy as np
from scipy.special import i0

RMAX_DEFAULT = 0.25 - 1.0 / 32.0          # transform.py:28
CUTOFF_DEFAULT = 5                         # transform.py:26
TRUNC_EPS_DEFAULT = 1e-8                   # transform.py:29
EXPANSION_MIN, EXPANSION_MAX = 16, 192     # transform.py:30-31


class OracleError(Exception):
    """Raised where the reference raises one of its NldenoiseError types."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------------------
# NFFT plan pieces (transform.py:110-170)
# ---------------------------------------------------------------------------

def centered(m: int) -> np.ndarray:
    """Frequencies -m/2 .. m/2-1 (transform.py:65-66)."""
    return np.arange(-(m // 2), m - m // 2)


def grid_size(bandwidth: int, oversampling: float) -> int:
    """nos = 2 ceil(os M / 2) (transform.py:129)."""
    return 2 * int(np.ceil(oversampling * bandwidth / 2))


def kb_shape(bandwidth: int, n: int) -> float:
    """Kaiser-Bessel shape b = pi (2 - M/n) (transform.py:131-133)."""
    return np.pi * (2.0 - bandwidth / n)


def deconv_factors(bandwidth: int, n: int, cutoff: int) -> np.ndarray:
    """I0(m sqrt(b^2 - (2 pi k / n)^2)), k centred (transform.py:140-145)."""
    b = kb_shape(bandwidth, n)
    k = centered(bandwidth)
    return i0(cutoff * np.sqrt(b * b - (2.0 * np.pi * k / n) ** 2))


def kb_tables(x: np.ndarray, bandwidth: int, n: int, cutoff: int):
    """Stencil bases (N,d) int64 and weights (N,d,2m+2) (transform.py:147-170).

    x are torus nodes in [-1/2, 1/2)^d.
    """
    x = np.atleast_2d(np.asarray(x, np.float64).T).T
    nn, d = x.shape
    width = 2 * cutoff + 2
    b = kb_shape(bandwidth, n)
    base = np.empty((nn, d), np.int64)
    wts = np.zeros((nn, d, width))
    offs = np.arange(width)
    for s in range(d):
        xs = x[:, s] * n
        lo = np.floor(xs).astype(np.int64) - cutoff
        base[:, s] = lo
        u = xs[:, None] - (lo[:, None] + offs[None, :])
        t = cutoff * cutoff - u * u
        inside = t > 0
        root = np.sqrt(np.where(inside, t, 1.0))
        val = np.where(inside, np.sinh(b * root) / (np.pi * root), 0.0)
        val[np.abs(t) <= 1e-14] = b / np.pi
        wts[:, s, :] = val
    return base, wts


def _stencil_chunks(base, wts, n_per_dim, chunk_elems=1 << 22):
    """Yield (rows, flat grid index (c, W^d), weight product (c, W^d)).

    Every node's full W^d stencil (W = 2m+2, as the reference loops over,
    _kernels.py:77-88), wrapped modulo the grid, C-order flattened.
    """
    nn, d, width = wts.shape
    step = max(1, chunk_elems // width ** d)
    offs = np.arange(width)
    for lo in range(0, nn, step):
        hi = min(nn, lo + step)
        idx = np.zeros((hi - lo,) + (1,) * d, np.int64)
        w = np.ones((hi - lo,) + (1,) * d)
        for s in range(d):
            shape = [hi - lo] + [1] * d
            shape[1 + s] = width
            pos = (base[lo:hi, s, None] + offs[None, :]) % n_per_dim[s]
            idx = idx * n_per_dim[s] + pos.reshape(shape)
            w = w * wts[lo:hi, s, :].reshape(shape)
        yield slice(lo, hi), idx.reshape(hi - lo, -1), w.reshape(hi - lo, -1)


def spread(values, base, wts, n_per_dim) -> np.ndarray:
    """Adjoint window step onto the flat C-order grid (_kernels.py:48-88)."""
    size = int(np.prod(n_per_dim))
    values = np.asarray(values)
    cplx = np.iscomplexobj(values)
    grid = np.zeros(size, np.complex128 if cplx else np.float64)
    for rows, idx, w in _stencil_chunks(base, wts, n_per_dim):
        contrib = (values[rows, None] * w).ravel()
        flat = idx.ravel()
        if cplx:
            grid += (np.bincount(flat, contrib.real, size)
                     + 1j * np.bincount(flat, contrib.imag, size))
        else:
            grid += np.bincount(flat, contrib, size)
    return grid


def gather(grid, base, wts, n_per_dim) -> np.ndarray:
    """Forward window step from the flat grid to the nodes (_kernels.py:91-136)."""
    out = np.zeros(base.shape[0], grid.dtype)
    for rows, idx, w in _stencil_chunks(base, wts, n_per_dim):
        out[rows] = (grid[idx] * w).sum(axis=1)
    return out


def _centred_positions(bandwidth, n):
    return centered(bandwidth) % n


def nfft_adjoint(values, x, bandwidth, n, cutoff, tables=None):
    """Spread, unnormalised e^{+} FFT, crop, deconvolve (transform.py:215-223)."""
    x = np.atleast_2d(np.asarray(x, np.float64).T).T
    d = x.shape[1]
    base, wts = kb_tables(x, bandwidth, n, cutoff) if tables is None else tables
    g = spread(np.asarray(values, np.complex128), base, wts, (n,) * d)
    ghat = np.fft.ifftn(g.reshape((n,) * d)) * float(n ** d)
    pos = _centred_positions(bandwidth, n)
    block = ghat[np.ix_(*([pos] * d))]
    c = deconv_factors(bandwidth, n, cutoff)
    for s in range(d):
        shape = [1] * d
        shape[s] = -1
        block = block / c.reshape(shape)
    return block


def nfft(coeffs, x, bandwidth, n, cutoff, tables=None):
    """Deconvolve, zero-pad, e^{-} FFT, gather (transform.py:200-212)."""
    x = np.atleast_2d(np.asarray(x, np.float64).T).T
    d = x.shape[1]
    base, wts = kb_tables(x, bandwidth, n, cutoff) if tables is None else tables
    block = np.array(coeffs, np.complex128)
    c = deconv_factors(bandwidth, n, cutoff)
    for s in range(d):
        shape = [1] * d
        shape[s] = -1
        block = block / c.reshape(shape)
    pos = _centred_positions(bandwidth, n)
    full = np.zeros((n,) * d, np.complex128)
    full[np.ix_(*([pos] * d))] = block
    g = np.fft.fftn(full).ravel()
    return gather(g, base, wts, (n,) * d)


def ndft(coeffs, x):
    """Exact trigonometric sum f(x) = sum_k c_k e^{-2 pi i k x} (transform.py:74-89)."""
    x = np.atleast_2d(np.asarray(x, np.float64).T).T
    c = np.asarray(coeffs, np.complex128)
    out = np.zeros(x.shape[0], np.complex128)
    for kk in np.ndindex(*c.shape):
        k = np.array([kk[s] - c.shape[s] // 2 for s in range(c.ndim)], np.float64)
        out += c[kk] * np.exp(-2j * np.pi * (x @ k))
    return out


# ---------------------------------------------------------------------------
# Fast Gauss transform plan (transform.py:254-333)
# ---------------------------------------------------------------------------

def expansion_degree(sig_scaled: float, eps: float = TRUNC_EPS_DEFAULT) -> int:
    """transform.py:254-258."""
    k = int(np.ceil(np.sqrt(max(sig_scaled, 1.0) * np.log(1.0 / eps)) / np.pi))
    return min(2 * max(EXPANSION_MIN // 2, k + 1), EXPANSION_MAX)


class WindowPlan:
    """One window's torus map, expansion and Gaussian coefficients.

    Restates FastsumPlan.build (transform.py:272-308).
    """

    def __init__(self, pts, sigbar, n_expansion=None, cutoff=CUTOFF_DEFAULT,
                 oversampling=2.0, rmax=RMAX_DEFAULT, eps=TRUNC_EPS_DEFAULT,
                 center=None, scale=None):
        # center/scale overrides: a shard of a larger point set uses the
        # global torus map (sharding tests only)
        if sigbar <= 0:
            raise ValueError("shape parameter must be positive")
        p = np.asarray(pts, np.float64)
        p = p[:, None] if p.ndim == 1 else p
        if p.shape[0] == 0:
            raise ValueError("empty point set")
        self.d = p.shape[1]
        if center is None:
            lo, hi = p.min(axis=0), p.max(axis=0)
            self.center = 0.5 * (lo + hi)
            radius = float(np.sqrt(((p - self.center) ** 2).sum(axis=1).max()))
            self.scale = rmax / max(radius, 1e-30)
        else:
            self.center = np.asarray(center, np.float64)
            self.scale = float(scale)
        self.sig_scaled = sigbar / (self.scale * self.scale)
        if n_expansion is None:
            n_expansion = expansion_degree(self.sig_scaled, eps)
        if n_expansion % 2:
            raise ValueError("expansion degree must be even")
        self.bandwidth = int(n_expansion)
        self.cutoff = int(cutoff)
        self.n = grid_size(self.bandwidth, oversampling)
        ax = centered(self.bandwidth) / self.bandwidth
        r2 = sum(g * g for g in np.meshgrid(*([ax] * self.d), indexing="ij"))
        gauss = np.exp(-self.sig_scaled * r2).astype(np.complex128)
        pos = centered(self.bandwidth) % self.bandwidth
        emb = np.zeros((self.bandwidth,) * self.d, np.complex128)
        emb[np.ix_(*([pos] * self.d))] = gauss
        raw = np.fft.ifftn(emb)
        self.coeffs = np.real(raw[np.ix_(*([pos] * self.d))])

    def torus(self, pts):
        """transform.py:310-317."""
        p = np.asarray(pts, np.float64)
        p = p[:, None] if p.ndim == 1 else p
        q = (p - self.center) * self.scale
        if q.size and np.abs(q).max() >= 0.5:
            raise OracleError("ScalingOverflowError", "node left the torus")
        return q

    def tables(self, pts):
        """transform.py:319-320."""
        return kb_tables(self.torus(pts), self.bandwidth, self.n, self.cutoff)

    def transform(self, src, tgt, alpha, src_tables=None, tgt_tables=None):
        """gauss_transform_fast (transform.py:323-333)."""
        ys, xs = self.torus(src), self.torus(tgt)
        ahat = nfft_adjoint(np.asarray(alpha, np.float64), ys, self.bandwidth,
                            self.n, self.cutoff, src_tables)
        return np.real(nfft(ahat * self.coeffs, xs, self.bandwidth, self.n,
                            self.cutoff, tgt_tables))


def gauss_direct(src, tgt, alpha, sigbar):
    """Exact sum_j alpha_j exp(-sigbar |x_i - y_j|^2) (transform.py:231-244)."""
    y = np.asarray(src, np.float64)
    x = np.asarray(tgt, np.float64)
    y = y[:, None] if y.ndim == 1 else y
    x = x[:, None] if x.ndim == 1 else x
    a = np.asarray(alpha, np.float64)
    out = np.empty(x.shape[0])
    blk = max(1, int(4e6) // max(1, y.shape[0]))
    for s in range(0, x.shape[0], blk):
        d2 = ((x[s:s + blk, None, :] - y[None, :, :]) ** 2).sum(-1)
        out[s:s + blk] = np.exp(-sigbar * d2) @ a
    return out


# ---------------------------------------------------------------------------
# ANOVA kernel operator (kernel.py:25-161)
# ---------------------------------------------------------------------------

class AnovaOracle:
    """Restates AnovaOperator's fast and exact modes (kernel.py:28-161).

    ``plan_kw`` carries the NFFT parameters.  The reference's AnovaOperator
    always uses FastsumPlan defaults (kernel.py:74); BASELINE pins
    n_expansion=32, cutoff=4, oversampling=2 and the survey's oracle
    subclass passes those, so both behaviours are reachable here.
    """

    def __init__(self, features, windows, sigma, **plan_kw):
        self.features = np.ascontiguousarray(features, np.float64)
        self.windows = [np.asarray(w, np.intp).ravel() for w in windows]
        self.sigma = float(sigma)
        self.plan_kw = plan_kw
        self._plans = {}
        self._eta = None

    @property
    def n(self):
        return self.features.shape[0]

    @property
    def n_windows(self):
        return len(self.windows)

    def plans(self, squared=False):
        """Lazy plan + table build (kernel.py:70-77)."""
        if squared not in self._plans:
            sigbar = (2.0 if squared else 1.0) / (self.sigma * self.sigma)
            built = []
            for w in self.windows:
                pts = np.ascontiguousarray(self.features[:, w])
                pl = WindowPlan(pts, sigbar, **self.plan_kw)
                built.append((pts, pl, pl.tables(pts)))
            self._plans[squared] = built
        return self._plans[squared]

    def window_sums(self, v, squared=False):
        """Per-window full Gauss sums G_l v (diagonal included)."""
        return [pl.transform(pts, pts, v, tb, tb)
                for pts, pl, tb in self.plans(squared)]

    def apply(self, v, squared=False):
        """Gamma v = (sum_l G_l v - L v) / L (kernel.py:79-93, :118-127)."""
        v = np.asarray(v, np.float64)
        if v.shape != (self.n,):
            raise OracleError("DimensionMismatchError", "vector length")
        out = np.zeros_like(v)
        for g in self.window_sums(v, squared):
            out += g
        out -= self.n_windows * v
        return out / self.n_windows

    def degree(self):
        """eta = Gamma 1, cached (kernel.py:142-146)."""
        if self._eta is None:
            self._eta = self.apply(np.ones(self.n))
        return self._eta

    def degree_squared(self):
        """kernel.py:148-154."""
        return self.apply(np.ones(self.n), squared=True) * self.n_windows

    def dense(self, squared=False):
        """Exact dense Gamma with zero diagonal (kernel.py:97-114)."""
        inv = (2.0 if squared else 1.0) / (self.sigma * self.sigma)
        g = np.zeros((self.n, self.n))
        for w in self.windows:
            p = self.features[:, w]
            d2 = ((p[:, None, :] - p[None, :, :]) ** 2).sum(-1)
            g += np.exp(-inv * d2)
        np.fill_diagonal(g, 0.0)
        return g / self.n_windows


# ---------------------------------------------------------------------------
# Shifted system, deflating basis, PCG (linops.py:28-319)
# ---------------------------------------------------------------------------

class SystemOracle:
    """A = lam I + mu (diag eta - Gamma) (linops.py:28-75)."""

    def __init__(self, op, lam, mu):
        if lam <= 0 or mu <= 0:
            raise ValueError("lam and mu must be positive")
        self.op, self.lam, self.mu = op, float(lam), float(mu)
        self.eta = op.degree()

    @property
    def n(self):
        return self.op.n

    def apply(self, x):
        x = np.asarray(x, np.float64)
        return self.lam * x + self.mu * (self.eta * x - self.op.apply(x))

    def jacobi_diagonal(self):
        return self.lam + self.mu * self.eta

    def l2_diagonal(self):
        pa = self.jacobi_diagonal()
        ell = self.op.n_windows
        row_sq = self.op.degree_squared() / (ell * ell)
        return np.sqrt(self.mu * self.mu * row_sq + pa * pa)


def scs_up(x):
    """out_i = x_1 + sum_{j>i} x_j, out_n = x_1 (linops.py:114-121)."""
    x = np.asarray(x, np.float64)
    suffix = np.cumsum(x[::-1])[::-1]
    out = np.empty_like(x)
    out[:-1] = x[0] + suffix[1:]
    out[-1] = x[0]
    return out


def scs_down(x):
    """out_1 = sum x, out_i = sum_{j<i} x_j (linops.py:124-131)."""
    x = np.asarray(x, np.float64)
    c = np.cumsum(x)
    out = np.empty_like(x)
    out[0] = c[-1]
    out[1:] = c[:-1]
    return out


class Basis:
    """Orthogonal U with first column v/|v| (linops.py:134-176)."""

    def __init__(self, v):
        self.v = np.asarray(v, np.float64)
        if self.v.size < 2:
            raise OracleError("DimensionMismatchError", "need >= 2 entries")
        pre = np.sqrt(np.cumsum(self.v * self.v))
        if pre[0] == 0.0:
            raise ValueError("leading entry of v must be nonzero")
        self.a = pre[:-1] / pre[1:]
        self.b = 1.0 / (pre[:-1] * pre[1:])
        self.norm = float(pre[-1])

    def apply(self, x):
        x = np.asarray(x, np.float64)
        y = np.empty_like(x)
        y[0] = x[0] / self.norm
        y[1:] = self.b * self.v[1:] * x[1:]
        out = self.v * scs_up(y)
        out[1:] -= self.a * x[1:]
        return out

    def apply_adjoint(self, x):
        x = np.asarray(x, np.float64)
        s = scs_down(self.v * x)
        out = np.empty_like(x)
        out[0] = s[0] / self.norm
        out[1:] = self.b * self.v[1:] * s[1:] - self.a * x[1:]
        return out


def pcg(apply_a, b, x0=None, prec=None, tol=1e-10, maxit=100):
    """PCG with true-residual confirmation (linops.py:193-244).

    Returns (x, iterations, converged, relative_residual, history).
    """
    b = np.asarray(b, np.float64)
    if np.linalg.norm(b) == 0.0 and x0 is None:
        return np.zeros_like(b), 0, True, 0.0, [0.0]
    x = np.zeros_like(b) if x0 is None else np.array(x0, np.float64)
    r = b - apply_a(x)
    bnorm = max(float(np.linalg.norm(b)), float(np.linalg.norm(r)))
    if bnorm == 0.0:
        return x, 0, True, 0.0, [0.0]
    hist = [float(np.linalg.norm(r)) / bnorm]
    if maxit <= 0:
        return x, 0, False, hist[0], hist
    z = prec(r) if prec is not None else r
    p = z.copy()
    rz = float(r @ z)
    it = 0
    while it < maxit:
        ap = apply_a(p)
        pap = float(p @ ap)
        if not np.isfinite(pap) or pap <= 0.0:
            raise OracleError("SolverBreakdownError", f"curvature at {it}")
        step = rz / pap
        x += step * p
        r -= step * ap
        it += 1
        rel = float(np.linalg.norm(r)) / bnorm
        hist.append(rel)
        if rel <= tol:
            true_rel = float(np.linalg.norm(b - apply_a(x))) / bnorm
            hist[-1] = true_rel
            if true_rel <= tol:
                return x, it, True, true_rel, hist
        z = prec(r) if prec is not None else r
        rz_new = float(r @ z)
        if not np.isfinite(rz_new):
            raise OracleError("SolverBreakdownError", "non-finite r.z")
        p = z + (rz_new / rz) * p
        rz = rz_new
    rel = float(np.linalg.norm(b - apply_a(x))) / bnorm
    return x, it, rel <= tol, rel, hist


def deflated_solve(system, f, prec="jacobi", tol=1e-10, maxit=100,
                   warm_start=False):
    """Deflated PCG on the U-tail (linops.py:252-300)."""
    f = np.asarray(f, np.float64)
    basis = Basis(np.ones(system.n))
    g = basis.apply_adjoint(f)

    def lift(y):
        return basis.apply(np.concatenate(([0.0], y)))

    def tail(y):
        return basis.apply_adjoint(system.apply(lift(y)))[1:]

    if prec == "none":
        pre = None
    elif prec in ("jacobi", "l2"):
        dinv = 1.0 / (system.jacobi_diagonal() if prec == "jacobi"
                      else system.l2_diagonal())

        def pre(y):
            return basis.apply_adjoint(dinv * lift(y))[1:]
    else:
        raise ValueError(f"unknown preconditioner {prec!r}")
    x, it, conv, rel, hist = pcg(tail, system.lam * g[1:],
                                 x0=g[1:] if warm_start else None,
                                 prec=pre, tol=tol, maxit=maxit)
    u = basis.apply(np.concatenate(([g[0]], x)))
    return u, it, conv, rel, hist


def plain_solve(system, f, prec="none", tol=1e-10, maxit=100,
                warm_start=False):
    """PCG in the pixel basis (linops.py:303-319)."""
    f = np.asarray(f, np.float64)
    if prec == "none":
        pre = None
    elif prec in ("jacobi", "l2"):
        dinv = 1.0 / (system.jacobi_diagonal() if prec == "jacobi"
                      else system.l2_diagonal())

        def pre(r):
            return dinv * r
    else:
        raise ValueError(f"unknown preconditioner {prec!r}")
    return pcg(system.apply, system.lam * f, x0=f if warm_start else None,
               prec=pre, tol=tol, maxit=maxit)

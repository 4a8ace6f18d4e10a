"""Drop-in transform API (reference transform.py:1-333) on the GPU.

Same names, argument meanings and exceptions as ``nldenoise.transform``:
``NodeSet``, ``ndft``, ``ndft_adjoint``, ``NfftPlan`` (``nos``,
``window_factors``, ``node_tables``), ``nfft``, ``nfft_adjoint``,
``gauss_transform_direct``, ``expansion_degree``, ``FastsumPlan`` (``build``,
``map_to_torus``, ``tables_for``) and ``gauss_transform_fast`` with distinct
sources and targets.  The sign convention is the reference's:
f(x) = sum_k fhat_k exp(-2 pi i k.x), k in {-M/2, ..., M/2-1}^d.

Differences: ``node_tables`` returns an opaque device table object (the
reference returns numpy (base, weights) arrays) accepted wherever the reference
accepts ``tables``; all bandwidths of a plan must be equal.  numpy inputs give
numpy outputs, torch CUDA tensors stay on the device.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _device as dv
from ._lib import check, lib
from .errors import DimensionMismatchError, ScalingOverflowError

DEFAULT_CUTOFF = 5                    # transform.py:26
DEFAULT_OVERSAMPLING = 2.0            # :27
DEFAULT_RMAX = 0.25 - 1.0 / 32.0      # :28
DEFAULT_TRUNCATION_EPS = 1e-8         # :29
MIN_EXPANSION = 16                    # :30
MAX_EXPANSION = 192                   # :31

_PD = ctypes.POINTER(ctypes.c_double)


def _shape(x):
    return tuple(x.shape) if hasattr(x, "shape") else np.shape(x)


def _as_nodes(nodes):
    """(N, d) nodes with d <= 3 (transform.py:34-42); keeps torch as torch."""
    x = getattr(nodes, "nodes", nodes)
    if not dv.is_torch(x):
        x = np.asarray(x, dtype=np.float64)
    shape = _shape(x)
    if len(shape) == 1:
        x = x[:, None]
        shape = _shape(x)
    if len(shape) != 2 or shape[1] > 3:
        raise DimensionMismatchError(
            f"nodes must be (N, d) with d <= 3, got shape {shape}")
    return x


def _real_dev(x, device):
    return dv.to_device(x, device, torch.float64)


def _cplx_dev(x, device):
    if dv.is_torch(x):
        return x.to(device=device, dtype=torch.complex128).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.complex128))).to(device)


def _out(t, template):
    return t if dv.is_torch(template) else t.detach().cpu().numpy()


class NodeSet:
    """Nodes on the torus [-1/2, 1/2)^d, d <= 3 (transform.py:45-62)."""

    def __init__(self, nodes):
        x = _as_nodes(nodes)
        xs = x if dv.is_torch(x) else torch.from_numpy(x)
        if xs.numel() and (float(xs.min()) < -0.5 or float(xs.max()) >= 0.5):
            raise ValueError("node coordinates must lie in [-1/2, 1/2)")
        self.nodes = x

    @property
    def dim(self) -> int:
        return _shape(self.nodes)[1]

    def __len__(self) -> int:
        return _shape(self.nodes)[0]


# ---------------------------------------------------------------------------
# exact transforms (oracles in the reference; exact GPU sums here)
# ---------------------------------------------------------------------------

def ndft(coeffs, nodes):
    """Evaluate the trigonometric polynomial exactly at every node."""
    x = _as_nodes(nodes)
    cs = _shape(coeffs)
    d = _shape(x)[1]
    if len(cs) != d:
        raise DimensionMismatchError(
            f"coefficient array has {len(cs)} axes for {d}-d nodes")
    if len(set(cs)) != 1:
        raise ValueError("unequal bandwidths are not supported")
    dev = dv.pick_device(x, coeffs)
    xt = _real_dev(x, dev)
    ct = _cplx_dev(coeffs, dev)
    out = torch.empty(_shape(x)[0], dtype=torch.complex128, device=dev)
    check(lib.nld_ndft(dv.ptr(xt), _shape(x)[0], d, cs[0], dv.ptr(ct), dv.ptr(out), 0,
                       dv.stream_of(dev)))
    return _out(out, coeffs)


def ndft_adjoint(values, nodes, bandwidth):
    """Exact adjoint sum over the centred index set (transform.py:92-102)."""
    x = _as_nodes(nodes)
    d = _shape(x)[1]
    shape = tuple(int(m) for m in np.atleast_1d(bandwidth))
    if len(shape) == 1 and d > 1:
        shape = shape * d
    if len(set(shape)) != 1 or len(shape) != d:
        raise ValueError("bandwidth must be one value or d equal values")
    dev = dv.pick_device(x, values)
    xt = _real_dev(x, dev)
    vt = _cplx_dev(values, dev)
    out = torch.empty(shape, dtype=torch.complex128, device=dev)
    check(lib.nld_ndft(dv.ptr(xt), _shape(x)[0], d, shape[0], dv.ptr(vt), dv.ptr(out), 1,
                       dv.stream_of(dev)))
    return _out(out, values)


# ---------------------------------------------------------------------------
# Kaiser-Bessel NFFT
# ---------------------------------------------------------------------------

class NodeTables:
    """Device node tables of one node set for one plan (opaque)."""

    def __init__(self, nodes, plan: "NfftPlan", center=None, scale=1.0,
                 check_torus=False):
        x = _as_nodes(nodes)
        n, d = _shape(x)
        if d != plan.dim:
            raise DimensionMismatchError("node dimension does not match plan")
        self.n, self.d, self.plan = n, d, plan
        self.device = dv.pick_device(x)
        self._x = _real_dev(x, self.device)
        ctr = None
        if center is not None:
            carr = np.ascontiguousarray(np.asarray(center, np.float64).ravel())
            self._center = carr
            ctr = carr.ctypes.data_as(_PD)
        handle = ctypes.c_void_p()
        check(lib.nld_nfft_create(dv.ptr(self._x), n, d, plan.bandwidth[0],
                                  float(plan.oversampling), int(plan.cutoff), ctr,
                                  float(scale), 1 if check_torus else 0,
                                  dv.stream_of(self.device), ctypes.byref(handle)))
        self._handle = handle

    def close(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            lib.nld_op_destroy(h)
            self._handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def adjoint(self, values, mult=None):
        vt = _cplx_dev(values, self.device)
        if vt.numel() != self.n:
            raise DimensionMismatchError("values length does not match the nodes")
        out = torch.empty(self.plan.bandwidth, dtype=torch.complex128, device=self.device)
        mp = None if mult is None else dv.ptr(mult)
        check(lib.nld_nfft_adjoint(self._handle, dv.ptr(vt), dv.ptr(out), mp,
                                   dv.stream_of(self.device)))
        return out

    def trafo(self, coeffs):
        ct = _cplx_dev(coeffs, self.device)
        out = torch.empty(self.n, dtype=torch.complex128, device=self.device)
        check(lib.nld_nfft_trafo(self._handle, dv.ptr(ct), dv.ptr(out),
                                 dv.stream_of(self.device)))
        return out


class NfftPlan:
    """Bandwidths, oversampling, window cutoff (transform.py:110-170)."""

    def __init__(self, bandwidth, oversampling: float = DEFAULT_OVERSAMPLING,
                 cutoff: int = DEFAULT_CUTOFF):
        bw = tuple(int(m) for m in np.atleast_1d(bandwidth))
        if any(m <= 0 or m % 2 for m in bw):
            raise ValueError("bandwidths must be even positive integers")
        if oversampling < 1.25:
            raise ValueError("oversampling factor must be >= 1.25")
        if cutoff < 1:
            raise ValueError("window cutoff must be >= 1")
        if cutoff > 8:
            raise ValueError("window cutoff above 8 is not supported")
        if len(set(bw)) != 1:
            raise ValueError("unequal bandwidths are not supported")
        self.bandwidth = bw
        self.oversampling = float(oversampling)
        self.cutoff = int(cutoff)
        self.nos = tuple(2 * int(math.ceil(self.oversampling * m / 2)) for m in bw)
        self._shape_b = tuple(math.pi * (2.0 - m / n) for m, n in zip(bw, self.nos))

    @property
    def dim(self) -> int:
        return len(self.bandwidth)

    def window_factors(self, s: int) -> np.ndarray:
        """I0-form Fourier factors of the window along dimension s."""
        out = np.empty(self.bandwidth[s])
        check(lib.nld_window_factors(self.bandwidth[s], self.nos[s], self.cutoff,
                                     out.ctypes.data_as(_PD)))
        return out

    def node_tables(self, nodes) -> NodeTables:
        """Stencil tables for a node batch (device; transform.py:147-170)."""
        return NodeTables(nodes, self)


def nfft(coeffs, nodes, plan: NfftPlan, tables=None):
    """Fast approximate evaluation of the trigonometric polynomial."""
    cs = _shape(coeffs)
    if cs != plan.bandwidth:
        raise DimensionMismatchError(
            f"coefficients shape {cs} != plan bandwidth {plan.bandwidth}")
    x = _as_nodes(nodes)
    tb = plan.node_tables(x) if tables is None else tables
    return _out(tb.trafo(coeffs), coeffs)


def nfft_adjoint(values, nodes, plan: NfftPlan, tables=None):
    """Fast approximate adjoint transform."""
    x = _as_nodes(nodes)
    tb = plan.node_tables(x) if tables is None else tables
    return _out(tb.adjoint(values), values)


# ---------------------------------------------------------------------------
# Gauss transform
# ---------------------------------------------------------------------------

def _points(p):
    if not dv.is_torch(p):
        p = np.asarray(p, np.float64)
    if len(_shape(p)) == 1:
        p = p[:, None]
    return p


def gauss_transform_direct(sources, targets, alpha, sigbar: float):
    """Exact O(Nx * Ny) discrete Gauss transform (transform.py:231-244)."""
    if sigbar <= 0:
        raise ValueError("shape parameter must be positive")
    y, x = _points(sources), _points(targets)
    dev = dv.pick_device(y, x, alpha)
    yt, xt = _real_dev(y, dev), _real_dev(x, dev)
    at = _real_dev(alpha, dev)
    out = torch.empty(_shape(x)[0], dtype=torch.float64, device=dev)
    check(lib.nld_gauss_direct(dv.ptr(xt), _shape(x)[0], dv.ptr(yt), _shape(y)[0],
                               _shape(x)[1], dv.ptr(at), float(sigbar), dv.ptr(out),
                               dv.stream_of(dev)))
    return _out(out, alpha)


def expansion_degree(sigbar_scaled: float, eps: float = DEFAULT_TRUNCATION_EPS) -> int:
    """Even expansion degree keeping the periodized-Gaussian tail below eps."""
    k = int(math.ceil(math.sqrt(max(sigbar_scaled, 1.0) * math.log(1.0 / eps)) / math.pi))
    n = 2 * max(MIN_EXPANSION // 2, k + 1)
    return min(n, MAX_EXPANSION)


class FastsumPlan:
    """Torus scaling, kernel coefficients, NFFT (transform.py:261-320)."""

    def __init__(self, sigbar, center, scale, rmax, nfft_plan, kernel_coeffs):
        self.sigbar = float(sigbar)
        self.center = center
        self.scale = float(scale)
        self.rmax = float(rmax)
        self.nfft_plan = nfft_plan
        self._coeffs = kernel_coeffs            # device, real, shape M^d

    @property
    def kernel_coeffs(self) -> np.ndarray:
        return self._coeffs.detach().cpu().numpy()

    @classmethod
    def build(cls, points, sigbar: float, *, n_expansion=None,
              cutoff: int = DEFAULT_CUTOFF,
              oversampling: float = DEFAULT_OVERSAMPLING,
              rmax: float = DEFAULT_RMAX,
              truncation_eps: float = DEFAULT_TRUNCATION_EPS) -> "FastsumPlan":
        if sigbar <= 0:
            raise ValueError("shape parameter must be positive")
        if not (0 < rmax <= 0.25):
            raise ValueError("rmax must lie in (0, 1/4]")
        p = _points(points)
        n, d = _shape(p)
        if n == 0:
            raise ValueError("cannot build a plan from an empty point set")
        if d > 3:
            raise DimensionMismatchError("points must be (N, d) with d <= 3")
        dev = dv.pick_device(p)
        pt = _real_dev(p, dev)
        center = np.zeros(d)
        scale = ctypes.c_double()
        check(lib.nld_fastsum_geometry(dv.ptr(pt), n, d, float(rmax),
                                       center.ctypes.data_as(_PD), ctypes.byref(scale),
                                       dv.stream_of(dev)))
        scale = scale.value
        sig_scaled = sigbar / (scale * scale)
        if n_expansion is None:
            n_expansion = expansion_degree(sig_scaled, truncation_eps)
        if n_expansion % 2:
            raise ValueError("expansion degree must be even")
        plan = NfftPlan((n_expansion,) * d, oversampling, cutoff)
        coeffs = torch.empty((n_expansion,) * d, dtype=torch.float64, device=dev)
        check(lib.nld_gauss_coeffs(n_expansion, d, float(sig_scaled), dv.ptr(coeffs),
                                   dv.stream_of(dev)))
        out = cls(float(sigbar), center, scale, float(rmax), plan, coeffs)
        out.device = dev
        return out

    def map_to_torus(self, points):
        """(p - center) * scale; ScalingOverflowError off the torus (:310-317)."""
        p = _points(points)
        pt = _real_dev(p, self.device)
        q = (pt - torch.as_tensor(self.center, device=self.device)) * self.scale
        if q.numel() and float(q.abs().max()) >= 0.5:
            raise ScalingOverflowError("scaled nodes leave the torus [-1/2, 1/2)^d")
        return _out(q, p)

    def tables_for(self, points) -> NodeTables:
        """Device tables of the mapped points (transform.py:319-320)."""
        return NodeTables(_points(points), self.nfft_plan, center=self.center,
                          scale=self.scale, check_torus=True)


def gauss_transform_fast(sources, targets, alpha, plan: FastsumPlan,
                         source_tables=None, target_tables=None):
    """NFFT fast summation approximating gauss_transform_direct (:323-333)."""
    src = source_tables if source_tables is not None else plan.tables_for(sources)
    tgt = target_tables if target_tables is not None else plan.tables_for(targets)
    if source_tables is not None or target_tables is not None:
        # the reference maps both point sets on every call (:328-329)
        plan.map_to_torus(sources)
        plan.map_to_torus(targets)
    ahat = src.adjoint(_real_dev(alpha, plan.device).to(torch.complex128),
                       mult=plan._coeffs)
    out = tgt.trafo(ahat).real.contiguous()
    return _out(out, alpha)

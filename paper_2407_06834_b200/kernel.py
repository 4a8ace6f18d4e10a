"""Drop-in ``AnovaOperator`` backed by the sm_100a kernels.

Mirrors ``nldenoise.kernel.AnovaOperator`` (kernel.py:25-161): same
constructor, same validation order and exception types, same lazy plan
build, same ``apply`` / ``apply_squared`` / ``degree`` / ``degree_squared`` /
``assemble_dense`` / ``n`` / ``n_windows`` / ``@`` surface.  The fast path
runs spread -> fused separable convolution -> gather on the GPU through the
C-ABI (include/nld_b200.h); the exact path evaluates the dense kernel sum on
the GPU.  There is no CPU fallback.

Extensions (not in the reference, off by default):
  * NFFT parameters as keywords (the reference hard-codes FastsumPlan
    defaults at kernel.py:74); BASELINE pins n_expansion=32, cutoff=4.
  * ``apply`` accepts a batch (nrhs, n) and shares every spread/gather.
  * torch CUDA tensors in -> torch CUDA tensors out (device resident).
  * ``sliced=False``: 16k-rhs batches of 3-D m = 4 windows run on the fp64
    DMMA kernels instead of the integer-sliced tcgen05 ones (results agree to
    rounding).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _device as dv
from ._lib import (APPLY_GAMMA, APPLY_GAMMA_SQUARED, APPLY_LAPLACIAN,
                   APPLY_SYSTEM, APPLY_WINDOW_SUM, LAYOUT_PIXEL_MAJOR, Params,
                   Stats, WindowInfo, check, lib)
from .errors import DimensionMismatchError, WindowSizeError

DEFAULT_DENSE_LIMIT = 5000          # kernel.py:22
DEFAULT_CUTOFF = 5                  # transform.py:26
DEFAULT_OVERSAMPLING = 2.0          # transform.py:27
DEFAULT_RMAX = 0.25 - 1.0 / 32.0    # transform.py:28
DEFAULT_TRUNCATION_EPS = 1e-8       # transform.py:29


def _shape_of(x):
    return tuple(x.shape) if hasattr(x, "shape") else np.shape(x)


class AnovaOperator:
    """Apply the ANOVA kernel matrix and its degree vectors matrix-free."""

    def __init__(self, features, windows, sigma: float, *, mode: str = "fast",
                 dense_limit: int = DEFAULT_DENSE_LIMIT, n_expansion=None,
                 cutoff: int = DEFAULT_CUTOFF,
                 oversampling: float = DEFAULT_OVERSAMPLING,
                 rmax: float = DEFAULT_RMAX,
                 truncation_eps: float = DEFAULT_TRUNCATION_EPS, device=None,
                 sliced: bool = True):
        # validation order of kernel.py:30-48
        if dv.is_torch(features):
            shape = tuple(features.shape)
        else:
            features = np.ascontiguousarray(features, dtype=np.float64)
            shape = features.shape
        if len(shape) != 2:
            raise DimensionMismatchError("features must be a 2-d array")
        if shape[0] == 0:
            raise DimensionMismatchError("at least one node is required")
        if sigma <= 0:
            raise ValueError("kernel width sigma must be positive")
        if mode not in ("fast", "exact"):
            raise ValueError(f"unknown mode {mode!r}")
        wins = [np.asarray(w, dtype=np.intp).ravel() for w in windows]
        if not wins:
            raise ValueError("at least one feature window is required")
        for w in wins:
            if w.size == 0 or w.size > 3:
                raise WindowSizeError(
                    "windows must have one to three feature dimensions")
            if w.min() < 0 or w.max() >= shape[1]:
                raise DimensionMismatchError("window index out of range")
        if n_expansion is not None and int(n_expansion) % 2:
            raise ValueError("expansion degree must be even")
        self.features = features
        self.windows = wins
        self.sigma = float(sigma)
        self.mode = mode
        self.dense_limit = int(dense_limit)
        self.device = dv.pick_device(features, device)
        self._host_kind = not dv.is_torch(features)
        self._feat = dv.to_device(features, self.device)
        self._params = Params(
            n_expansion=0 if n_expansion is None else int(n_expansion),
            cutoff=int(cutoff), oversampling=float(oversampling),
            rmax=float(rmax), truncation_eps=float(truncation_eps),
            mode=0 if mode == "fast" else 1, no_sliced=0 if sliced else 1,
            dense_limit=int(dense_limit))
        idx = np.concatenate(wins).astype(np.int32)
        off = np.zeros(len(wins) + 1, np.int32)
        off[1:] = np.cumsum([w.size for w in wins])
        handle = ctypes.c_void_p()
        check(lib.nld_op_create(
            dv.ptr(self._feat), shape[0], shape[1],
            idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            off.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(wins),
            self.sigma, ctypes.byref(self._params), dv.stream_of(self.device),
            ctypes.byref(handle)))
        self._handle = handle
        self._degree = None
        self._degree_sq = None
        # features are copied by the library; keep the tensor only for exact
        # mode assembly on request
        self._n = int(shape[0])

    # -- lifetime ---------------------------------------------------------
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

    # -- shape -----------------------------------------------------------
    @property
    def n(self) -> int:
        return self._n

    @property
    def n_windows(self) -> int:
        return len(self.windows)

    # -- raw device products -------------------------------------------------
    def _vectors(self, v, what="vector length"):
        shape = _shape_of(v)
        if len(shape) == 1 and shape[0] == self.n:
            nrhs = 1
        elif len(shape) == 2 and shape[1] == self.n and shape[0] >= 1:
            nrhs = shape[0]
        else:
            raise DimensionMismatchError(
                f"{what} {shape} does not match {self.n} nodes")
        return dv.to_device(v, self.device), nrhs

    def apply_device(self, x: torch.Tensor, kind: int, nrhs: int = 1,
                     coef=None, out: torch.Tensor | None = None,
                     pixel_major: bool = False) -> torch.Tensor:
        """Device product; x is a contiguous fp64 (nrhs, n) or (n,) tensor,
        or (n, nrhs) with ``pixel_major`` (the kernels' native layout: no
        transposes)."""
        if out is None:
            out = torch.empty_like(x)
        cptr = None
        if coef is not None:
            carr = np.ascontiguousarray(coef, dtype=np.float64).ravel()
            cptr = carr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        if pixel_major:
            kind |= LAYOUT_PIXEL_MAJOR
        check(lib.nld_op_apply(self._handle, kind, dv.ptr(x), dv.ptr(out), nrhs,
                               self.n, cptr, dv.stream_of(self.device)))
        return out

    def apply_pipelined(self, kind: int, inputs, outputs, nrhs: int = 1,
                        coef=None, pixel_major: bool = False):
        """Host -> device -> host products for a sequence of batches.

        ``inputs`` / ``outputs`` are equal-length sequences of pinned host
        torch tensors of shape (nrhs, n).  Batch k's host->device copy, the
        product of batch k-1 and the device->host copy of batch k-2 run
        concurrently on three streams with double-buffered device buffers,
        so PCIe traffic hides behind the kernels.  Returns after the last
        result is on the host.
        """
        dev = self.device
        cur = torch.cuda.current_stream(dev)
        s_in, s_cmp, s_out = (torch.cuda.Stream(dev) for _ in range(3))
        for s_ in (s_in, s_cmp, s_out):
            s_.wait_stream(cur)
        inputs, outputs = list(inputs), list(outputs)
        if not inputs:
            return
        shape = tuple(inputs[0].shape)
        want = (self.n, nrhs) if pixel_major else (nrhs, self.n)
        if shape != want and not (nrhs == 1 and shape == (self.n,)):
            raise DimensionMismatchError(f"batch shape {shape} != {want}")
        vd = [torch.empty(shape, dtype=torch.float64, device=dev) for _ in range(2)]
        yd = [torch.empty(shape, dtype=torch.float64, device=dev) for _ in range(2)]
        done_cmp = [None, None]      # compute finished with vd[b] / wrote yd[b]
        done_out = [None, None]      # yd[b] copied out
        for k, (xh, yh) in enumerate(zip(inputs, outputs)):
            b = k & 1
            with torch.cuda.stream(s_in):
                if done_cmp[b] is not None:
                    s_in.wait_event(done_cmp[b])
                vd[b].copy_(xh, non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(ev_in)
                if done_out[b] is not None:
                    s_cmp.wait_event(done_out[b])
                self.apply_device(vd[b], kind, nrhs, coef, out=yd[b],
                                  pixel_major=pixel_major)
                done_cmp[b] = torch.cuda.Event()
                done_cmp[b].record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(done_cmp[b])
                yh.copy_(yd[b], non_blocking=True)
                done_out[b] = torch.cuda.Event()
                done_out[b].record(s_out)
        for s_ in (s_in, s_cmp, s_out):
            cur.wait_stream(s_)
        torch.cuda.synchronize(dev)

    def _product(self, v, kind, coef=None):
        x, nrhs = self._vectors(v)
        out = self.apply_device(x, kind, nrhs, coef)
        return dv.like_input(out, v)

    # -- public API (kernel.py:118-161) --------------------------------------
    def apply(self, v):
        """Matrix-vector product gamma v."""
        return self._product(v, APPLY_GAMMA)

    def apply_squared(self, v):
        """Product with the entrywise-squared subkernel sum (kernel.py:129-140)."""
        return self._product(v, APPLY_GAMMA_SQUARED)

    def window_sum(self, v):
        """sum_l G_l v with each full Gauss sum's unit diagonal kept."""
        return self._product(v, APPLY_WINDOW_SUM)

    def degree_device(self, squared: bool = False) -> torch.Tensor:
        attr = "_degree_sq" if squared else "_degree"
        cached = getattr(self, attr)
        if cached is None:
            cached = torch.empty(self.n, dtype=torch.float64, device=self.device)
            check(lib.nld_op_degree(self._handle, 1 if squared else 0,
                                    dv.ptr(cached), dv.stream_of(self.device)))
            setattr(self, attr, cached)
        return cached

    def _as_feature_kind(self, t):
        return dv.to_host(t) if self._host_kind else t

    def degree(self):
        """eta = gamma 1, cached (kernel.py:142-146)."""
        return self._as_feature_kind(self.degree_device(False))

    def degree_squared(self):
        """sum_l (gamma_l o gamma_l) 1 without the 1/L (kernel.py:148-154)."""
        return self._as_feature_kind(self.degree_device(True))

    def assemble_dense(self, squared: bool = False):
        """Dense kernel matrix (zero diagonal); respects the node limit."""
        out = torch.empty((self.n, self.n), dtype=torch.float64,
                          device=self.device)
        check(lib.nld_op_assemble_dense(self._handle, 1 if squared else 0,
                                        dv.ptr(out), dv.stream_of(self.device)))
        return self._as_feature_kind(out)

    def __matmul__(self, v):
        return self.apply(v)

    # -- introspection ---------------------------------------------------
    def window_info(self, w: int) -> dict:
        info = WindowInfo()
        check(lib.nld_op_window_info(self._handle, w, ctypes.byref(info)))
        return {
            "dim": info.dim, "bandwidth": info.bandwidth, "grid": info.grid,
            "cutoff": info.cutoff, "center": list(info.center)[:info.dim],
            "scale": info.scale, "sig_scaled": info.sig_scaled,
            "box_lo": list(info.box_lo)[:info.dim],
            "box_w": list(info.box_w)[:info.dim], "n_cells": info.n_cells,
            "n_subproblems": info.n_subproblems, "n_edge": info.n_edge,
        }

    def set_timing(self, enabled: bool = True):
        check(lib.nld_op_set_timing(self._handle, 1 if enabled else 0))

    def debug_poison_workspace(self):
        """Test hook: fill the operator's device workspace with NaN bytes
        (nld_op_debug_poison); products must not depend on its contents."""
        check(lib.nld_op_debug_poison(self._handle))

    def stats(self) -> dict:
        s = Stats()
        check(lib.nld_op_stats(self._handle, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in Stats._fields_}


__all__ = ["AnovaOperator", "APPLY_GAMMA", "APPLY_GAMMA_SQUARED",
           "APPLY_SYSTEM", "APPLY_LAPLACIAN", "APPLY_WINDOW_SUM"]

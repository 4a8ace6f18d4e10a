"""Multi-threaded CPU port of the reference matvec -- TEST INFRASTRUCTURE ONLY.

Used as the CPU baseline (`bench.py` cpu_baseline and `--impl reference`)
and as a faster checker than the pure-numpy oracle.  Plans and node tables
come from `nfft_oracle.WindowPlan` (a restatement of FastsumPlan.build /
tables_for, transform.py:272-320); the spread and gather loops are the C
restatement in `oracle/c/nld_oracle.c` (reference _kernels.py:48-136) run on
all host threads; the grid step is numpy's pocketfft exactly as in
nfft_adjoint / nfft (transform.py:200-223).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import nfft_oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_c.so")


def _load():
    if not os.path.exists(_SO):
        raise ImportError(f"{_SO} missing: run `make -C oracle`")
    lib = ctypes.CDLL(_SO)
    p = ctypes.c_void_p
    lib.orc_max_threads.restype = ctypes.c_int
    lib.orc_spread.argtypes = [p, p, p, ctypes.c_int64, ctypes.c_int,
                               ctypes.c_int, p, p, ctypes.c_int]
    lib.orc_gather.argtypes = lib.orc_spread.argtypes
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


class CpuPort:
    """Reference fast-summation matvec on the host, all threads."""

    def __init__(self, features, windows, sigma, nthreads=0, **plan_kw):
        self.features = np.ascontiguousarray(features, np.float64)
        self.windows = [np.asarray(w, np.intp).ravel() for w in windows]
        self.sigma = float(sigma)
        self.nthreads = int(nthreads) or lib().orc_max_threads()
        sigbar = 1.0 / (self.sigma * self.sigma)
        self.plans = []
        for w in self.windows:
            pts = np.ascontiguousarray(self.features[:, w])
            pl = O.WindowPlan(pts, sigbar, **plan_kw)
            base, wts = pl.tables(pts)
            self.plans.append((pl, np.ascontiguousarray(base),
                               np.ascontiguousarray(wts)))
        self._eta = None

    @property
    def n(self):
        return self.features.shape[0]

    def _window(self, v, pl, base, wts):
        d = pl.d
        n = pl.n
        nos = np.full(d, n, np.int64)
        grid = np.empty(n ** d)
        lib().orc_spread(_ptr(v), _ptr(base), _ptr(wts), base.shape[0], d,
                         wts.shape[2], _ptr(nos), _ptr(grid), self.nthreads)
        # nfft_adjoint tail (transform.py:222-223), x coeffs, nfft (:209)
        ghat = np.fft.ifftn(grid.reshape((n,) * d)) * float(n ** d)
        pos = O.centered(pl.bandwidth) % n
        ix = np.ix_(*([pos] * d))
        c = O.deconv_factors(pl.bandwidth, n, pl.cutoff)
        block = ghat[ix]
        for s in range(d):
            shape = [1] * d
            shape[s] = -1
            block = block / c.reshape(shape)
        block = block * pl.coeffs
        for s in range(d):
            shape = [1] * d
            shape[s] = -1
            block = block / c.reshape(shape)
        full = np.zeros((n,) * d, np.complex128)
        full[ix] = block
        g2 = np.ascontiguousarray(np.fft.fftn(full).ravel())
        out = np.empty(2 * base.shape[0])
        lib().orc_gather(_ptr(g2.view(np.float64)), _ptr(base), _ptr(wts),
                         base.shape[0], d, wts.shape[2], _ptr(nos), _ptr(out),
                         self.nthreads)
        return out[0::2]

    def apply(self, v):
        """Gamma v (kernel.py:79-93)."""
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros_like(v)
        for pl, base, wts in self.plans:
            out += self._window(v, pl, base, wts)
        out -= len(self.plans) * v
        return out / len(self.plans)

    def degree(self):
        if self._eta is None:
            self._eta = self.apply(np.ones(self.n))
        return self._eta

    def system_apply(self, v, lam, mu):
        """lam v + mu (eta v - Gamma v) (linops.py:43-50)."""
        v = np.ascontiguousarray(v, np.float64)
        return lam * v + mu * (self.degree() * v - self.apply(v))

"""Pixel sharding across GPUs: one process per GPU.

Each rank holds a set of the pixels (features, vectors, node tables, sort
permutations): a contiguous slice (`shard_range`) or the window-0 stencil-cell
ownership partition (`partition`, what bench.py uses).  The library calls one
collective hook:

* at plan build: MIN/MAX of every window's bounding box, MAX of the torus
  radius and MIN/MAX of the stencil bases, so all ranks share the same torus
  map, kernel coefficients and support box (transform.py:292-296);
* once per product: SUM of the per-window support-box grids (all windows and
  right-hand sides, ~0.47 MB per rhs at config 4: 3 support boxes of 27^3;
  one call per window on the aux stream, overlapped with the next window's
  spread), after which every rank runs the small separable convolution
  redundantly and gathers its own pixels;
* in CG: SUM of the per-iteration scalars (dots, norms, means), as a device
  buffer on the solver's stream (one host read per reduction follows).

`TorchComm` implements the hook with torch.distributed (NCCL over NVLink for
device buffers; host buffers go through the same process group).
`ThreadComm` emulates `world` ranks as threads of one process on one GPU --
the host blocks in the hook, never a kernel -- so the sharded algorithm can be
checked on a single B200.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from ._lib import ALLREDUCE_FN, check, lib

F64, I32 = 0, 1
SUM, MIN, MAX = 0, 1, 2
_NP = {F64: (ctypes.c_double, np.float64), I32: (ctypes.c_int32, np.int32)}


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous pixel range [lo, hi) of `rank` (balanced to within one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return n * rank // world, n * (rank + 1) // world


def partition(features, windows, world: int, *, window: int = 0, grid: int = 64,
              rmax: float = 0.25 - 1.0 / 32.0) -> list[np.ndarray]:
    """Pixel indices of each rank, partitioned by stencil-cell ownership of
    one window (balanced by pixel count).

    Contiguous pixel ranges (`shard_range`) give every rank nodes in almost
    every occupied cell of every window, so each rank pays every cell's
    fixed costs (a 128-node gather tile per subproblem, the spread's
    accumulator drain and block write) on an eighth of its nodes at eight
    ranks.  Ranking the pixels by their cell in `window` (the torus map of
    transform.py:292-317 on the global point set, cell = floor(q * grid)) and
    cutting that order into `world` equal ranges keeps that window's cells
    whole on one rank (at most world - 1 cells are split); the other windows'
    cells follow as far as the features of neighbouring patch rows correlate.
    Each rank's indices are returned in ascending order.  Any partition is
    valid for the sharded operator: its products and solves depend only on
    which pixels a rank holds, not on how they were chosen.
    """
    if world < 1:
        raise ValueError("bad world size")
    f = np.asarray(features, np.float64)
    n = f.shape[0]
    cols = np.asarray(windows[window], np.int64)
    p = f[:, cols]
    lo, hi = p.min(axis=0), p.max(axis=0)
    c = 0.5 * (lo + hi)
    radius = float(np.sqrt(((p - c) ** 2).sum(axis=1).max()))
    q = (p - c) * (rmax / max(radius, 1e-30))
    base = np.floor(q * grid).astype(np.int64) + grid
    key = np.zeros(n, np.int64)
    for s in range(base.shape[1]):
        key = key * (4 * grid) + base[:, s]
    order = np.argsort(key, kind="stable")
    cuts = [n * k // world for k in range(world + 1)]
    return [np.sort(order[cuts[k]:cuts[k + 1]]) for k in range(world)]


def host_view(ptr: int, count: int, dtype: int) -> np.ndarray:
    ctype, _ = _NP[dtype]
    return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctype)),
                                 shape=(count,))


class _CudaArray:
    """Minimal __cuda_array_interface__ wrapper (zero-copy torch view)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": "<f8", "data": (ptr, False),
            "version": 2, "strides": None}


def device_view(ptr: int, count: int, device) -> torch.Tensor:
    return torch.as_tensor(_CudaArray(ptr, count), device=device)


def _reduce_np(parts, op):
    out = parts[0].copy()
    for p in parts[1:]:
        if op == SUM:
            out = out + p
        elif op == MIN:
            out = np.minimum(out, p)
        else:
            out = np.maximum(out, p)
    return out


class Comm:
    """Base class: owns the ctypes callback; subclasses implement reduce()."""

    def __init__(self):
        self._cb = ALLREDUCE_FN(self._entry)

    def _entry(self, ctx, buf, count, dtype, op, on_device, stream):
        try:
            self.reduce(int(ctx or 0), buf, int(count), int(dtype), int(op),
                        bool(on_device), stream)
            return 0
        except Exception as exc:  # surfaced as a CUDA-class status
            self.error = exc
            return 1

    @property
    def callback(self):
        return self._cb

    def reduce(self, rank, buf, count, dtype, op, on_device, stream):
        raise NotImplementedError


class TorchComm(Comm):
    """torch.distributed process group (one process per GPU)."""

    def __init__(self, group=None, device=None):
        super().__init__()
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.backend = dist.get_backend(group)
        self.device = device
        self.ops = {SUM: dist.ReduceOp.SUM, MIN: dist.ReduceOp.MIN,
                    MAX: dist.ReduceOp.MAX}

    def reduce(self, rank, buf, count, dtype, op, on_device, stream):
        dist = self.dist
        if on_device:
            t = device_view(buf, count, self.device)
            ext = torch.cuda.ExternalStream(stream, device=self.device) if stream \
                else torch.cuda.current_stream(self.device)
            with torch.cuda.stream(ext):
                dist.all_reduce(t, op=self.ops[op], group=self.group)
            return
        view = host_view(buf, count, dtype)
        t = torch.from_numpy(view.copy())
        if self.backend == "nccl":
            t = t.to(self.device)
        dist.all_reduce(t, op=self.ops[op], group=self.group)
        view[:] = t.cpu().numpy()


class ThreadComm(Comm):
    """`world` ranks as host threads of one process (single-GPU emulation).

    Rank r passes ctx = r.  Each collective deposits the rank's buffer,
    waits for all ranks, reduces in rank order (deterministic) and writes the
    result back.  Device buffers are synchronised on their stream first.
    """

    def __init__(self, world: int, device=None):
        super().__init__()
        self.world = world
        self.device = device
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def reduce(self, rank, buf, count, dtype, op, on_device, stream):
        if on_device:
            ext = torch.cuda.ExternalStream(stream, device=self.device) if stream \
                else torch.cuda.current_stream(self.device)
            ext.synchronize()
            t = device_view(buf, count, self.device)
            self.slots[rank] = t.clone()
            torch.cuda.synchronize(self.device)
            self.barrier.wait()
            total = self.slots[0].clone()
            for k in range(1, self.world):
                total += self.slots[k]
            t.copy_(total)
            torch.cuda.synchronize(self.device)
            self.barrier.wait()
            return
        view = host_view(buf, count, dtype)
        self.slots[rank] = view.copy()
        self.barrier.wait()
        res = _reduce_np(self.slots, op)
        self.barrier.wait()
        view[:] = res


def attach(op, comm: Comm, rank: int, global_n: int) -> None:
    """Turn AnovaOperator `op` (built from this rank's pixel slice) into one
    shard of a global_n-pixel operator.  Call before the first product."""
    check(lib.nld_op_set_comm(op._handle, comm.callback, ctypes.c_void_p(rank),
                              int(global_n)))
    op._comm = comm          # keep the callback alive with the operator
    op.global_n = int(global_n)

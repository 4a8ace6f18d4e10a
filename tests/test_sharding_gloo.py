"""CPU, world_size 2 over gloo: the pixel-sharding host logic.

Checks the collective hook (`sharding.TorchComm`, the callback the C library
calls) and the sharding protocol -- global torus map from MIN/MAX/MAX
reductions, one SUM of the per-rank spread grids -- against the unsharded
problem, with the CPU oracle standing in for the GPU kernels.
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _call(comm, arr, dtype, op):
    ptr = arr.ctypes.data
    return comm.callback(None if comm_rank[0] == 0 else comm_rank[0], ptr, arr.size,
                         dtype, op, 0, None)


comm_rank = [0]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import nfft_oracle as O
        from paper_2407_06834_b200 import sharding as S
        import synth
        comm_rank[0] = rank
        comm = S.TorchComm()
        res = {}
        # 1. the raw callback on host buffers
        a = np.array([1.0 + rank, -2.0 * rank, 3.0])
        assert _call(comm, a, S.F64, S.SUM) == 0
        res["sum"] = a.tolist()
        b = np.array([5 - rank, rank], np.int32)
        assert _call(comm, b, S.I32, S.MIN) == 0
        res["min"] = b.tolist()
        c = np.array([0.5 * rank, -1.0])
        assert _call(comm, c, S.F64, S.MAX) == 0
        res["max"] = c.tolist()
        # 2. protocol: shard c0, global torus map, one grid SUM
        feats, wins, _ = synth.make_problem("c0")
        n = feats.shape[0]
        lo_i, hi_i = S.shard_range(n, rank, world)
        v = synth.random_vector(n)
        errs = []
        for w in wins:
            pts = feats[lo_i:hi_i][:, w]
            lo = pts.min(axis=0).copy()
            hi = pts.max(axis=0).copy()
            assert _call(comm, lo, S.F64, S.MIN) == 0
            assert _call(comm, hi, S.F64, S.MAX) == 0
            center = 0.5 * (lo + hi)
            r2 = np.array([((pts - center) ** 2).sum(axis=1).max()])
            assert _call(comm, r2, S.F64, S.MAX) == 0
            scale = 0.21875 / max(float(np.sqrt(r2[0])), 1e-30)
            pin = dict(n_expansion=32, cutoff=4, oversampling=2.0)
            plan = O.WindowPlan(pts, 1.0 / 0.01, center=center, scale=scale, **pin)
            full = O.WindowPlan(feats[:, w], 1.0 / 0.01, **pin)
            assert plan.scale == full.scale and np.array_equal(plan.center, full.center)
            base, wts = plan.tables(pts)
            grid = O.spread(v[lo_i:hi_i], base, wts, (64,) * len(w))
            assert _call(comm, grid, S.F64, S.SUM) == 0
            fb, fw = full.tables(feats[:, w])
            want = O.spread(v, fb, fw, (64,) * len(w))
            errs.append(float(np.abs(grid - want).max() / np.abs(want).max()))
        res["grid_err"] = max(errs)
        res["range"] = (lo_i, hi_i)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_sharding_protocol_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert out[r]["sum"] == [3.0, -2.0, 6.0]
        assert out[r]["min"] == [4, 0]
        assert out[r]["max"] == [0.5, -1.0]
        assert out[r]["grid_err"] < 1e-13
    assert out[0]["range"] == (0, 2048) and out[1]["range"] == (2048, 4096)


def test_shard_range_balanced():
    from paper_2407_06834_b200.sharding import shard_range
    for n in (1, 7, 4096, 16777216):
        for world in (1, 2, 3, 8):
            if world > n:
                continue
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1

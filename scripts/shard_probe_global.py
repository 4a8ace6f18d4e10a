"""Strong-scaling probe on one GPU with the GLOBAL torus map: the k ranks of a
sharded c4 operator are built as host threads over sharding.ThreadComm (so
every rank's plan uses the global bounding boxes, as under torchrun), their
first product (the degree) runs in lockstep, and then each rank's 16-rhs
product is timed alone with the grid SUM switched to a no-op (the exchange is
what a one-GPU probe cannot time).  scripts/shard_probe.py builds each shard
as an independent operator instead: its local map stretches a cell-ownership
shard over the whole lattice, which hides what that partition gains.
usage: python scripts/shard_probe_global.py [k ...]"""
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
from paper_2407_06834_b200 import _lib, sharding  # noqa: E402
import synth  # noqa: E402

feats, wins, _ = synth.make_problem("c4")
n = feats.shape[0]
coef = np.tile([1.0, 0.001], 16)
dev = torch.device("cuda:0")


class ProbeComm(sharding.ThreadComm):
    passthrough = False

    def reduce(self, rank, buf, count, dtype, op, on_device, stream):
        if self.passthrough and on_device:
            return
        if self.passthrough:
            raise RuntimeError("host reduction after the plan build")
        super().reduce(rank, buf, count, dtype, op, on_device, stream)


def timed(op, V):
    for _ in range(2):
        op.apply_device(V, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        op.apply_device(V, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(parts):
    k = len(parts)
    comm = ProbeComm(k, dev)
    ops, errs = [None] * k, []

    def build(r):
        try:
            torch.cuda.set_device(0)
            op = nld.AnovaOperator(torch.from_numpy(np.ascontiguousarray(feats[parts[r]])).cuda(),
                                   wins, synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
            sharding.attach(op, comm, r, n)
            op.degree()                       # plan build + one product, in lockstep
            ops[r] = op
        except Exception as exc:              # noqa: BLE001
            errs.append(exc)
            comm.barrier.abort()

    ts = [threading.Thread(target=build, args=(r,)) for r in range(k)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    torch.cuda.synchronize()
    comm.passthrough = True
    out, cells = [], []
    for r in range(k):
        V = torch.randn((ops[r].n, 16), dtype=torch.float64, device="cuda")
        out.append(timed(ops[r], V))
        cells.append([ops[r].window_info(w)["n_subproblems"] for w in range(3)])
        del V
    del ops
    torch.cuda.empty_cache()
    return out, cells


op1 = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA, n_expansion=32,
                        cutoff=4, oversampling=2.0)
op1.degree()
full = timed(op1, torch.randn((n, 16), dtype=torch.float64, device="cuda"))
del op1
torch.cuda.empty_cache()
print(f"1 shard: {full:.2f} ms/product", flush=True)
for k in [int(a) for a in sys.argv[1:]] or [2, 4, 8]:
    for name, parts in (("contiguous", [np.arange(*sharding.shard_range(n, r, k)) for r in range(k)]),
                        ("cell-owner", sharding.partition(feats, wins, k))):
        ts, cells = run(parts)
        mx = max(ts)
        print(f"{k} shards {name} (global map): max {mx:.2f} ms (mean {np.mean(ts):.2f}), per rank "
              f"{[round(t, 2) for t in ts]} -> "
              f"{full / mx:.2f}x of {k} ({full / mx / k * 100:.0f}% efficiency); "
              f"subproblems per window, rank 0: {cells[0]}, rank {k - 1}: {cells[-1]}", flush=True)

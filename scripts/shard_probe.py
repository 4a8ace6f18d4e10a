"""Strong-scaling probe on one GPU: the 16-rhs product of each rank's shard of
the c4 pixels at world size k, for contiguous pixel ranges
(sharding.shard_range) and for window-0 cell ownership (sharding.partition).
A sharded step takes as long as its slowest rank: the max over the k shards
is reported (plus the grid allreduce, which this one-GPU probe cannot time)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
from paper_2407_06834_b200 import _lib, sharding  # noqa: E402
import synth  # noqa: E402

feats, wins, _ = synth.make_problem("c4")
n = feats.shape[0]
coef = np.tile([1.0, 0.001], 16)


def product_ms(idx):
    op = nld.AnovaOperator(torch.from_numpy(np.ascontiguousarray(feats[idx])).cuda(), wins,
                           synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
    m = op.n
    V = torch.randn((m, 16), dtype=torch.float64, device="cuda")
    op.degree()
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
    del op, V
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / reps


full = product_ms(np.arange(n))
print(f"1 shard: {full:.2f} ms/product", flush=True)
for k in (2, 4, 8):
    for name, parts in (("contiguous", [np.arange(*sharding.shard_range(n, r, k)) for r in range(k)]),
                        ("cell-owner", sharding.partition(feats, wins, k))):
        ts = [product_ms(ix) for ix in parts]
        mx = max(ts)
        print(f"{k} shards {name}: max {mx:.2f} ms (mean {np.mean(ts):.2f}) -> "
              f"{full / mx:.2f}x of {k} ({full / mx / k * 100:.0f}% efficiency)", flush=True)

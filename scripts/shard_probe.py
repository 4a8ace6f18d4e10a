"""Strong-scaling probe on one GPU: time the 16-rhs product of an operator
built on the first 1/k of the c4 pixels (one rank's shard at world size k)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
from paper_2407_06834_b200 import _lib  # noqa: E402
import synth  # noqa: E402

feats, wins, _ = synth.make_problem("c4")
n = feats.shape[0]
for k in (1, 2, 4, 8):
    m = n // k
    op = nld.AnovaOperator(torch.from_numpy(feats[:m]).cuda(), wins, synth.SIGMA,
                           n_expansion=32, cutoff=4, oversampling=2.0)
    V = torch.randn((m, 16), dtype=torch.float64, device="cuda")
    coef = np.tile([1.0, 0.001], 16)
    op.degree()
    for _ in range(2):
        op.apply_device(V, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True)
    torch.cuda.synchronize()
    op.set_timing(True)
    t0 = time.perf_counter()
    reps = 5
    st = {"spread_ms": 0, "gather_ms": 0}
    for _ in range(reps):
        op.apply_device(V, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True)
        s = op.stats()
        st["spread_ms"] += s["spread_ms"] / reps
        st["gather_ms"] += s["gather_ms"] / reps
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    print(f"shard 1/{k}: {m} px  {ms:.2f} ms/product (ideal {ms_full / k if k > 1 else ms:.2f})"
          f"  spread {st['spread_ms']:.2f}  gather {st['gather_ms']:.2f}", flush=True)
    if k == 1:
        ms_full = ms
    del op, V
    torch.cuda.empty_cache()

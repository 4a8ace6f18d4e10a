"""Kernel breakdown of one rank's 16-rhs product at 8 shards (c4), for the
launch-list capture: python scripts/shard_breakdown.py [contiguous|cell]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
from paper_2407_06834_b200 import _lib, sharding  # noqa: E402
import synth  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "cell"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
feats, wins, _ = synth.make_problem("c4")
n = feats.shape[0]
ix = (np.arange(*sharding.shard_range(n, 0, k)) if mode == "contiguous"
      else sharding.partition(feats, wins, k)[0])
op = nld.AnovaOperator(torch.from_numpy(np.ascontiguousarray(feats[ix])).cuda(), wins,
                       synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
V = torch.randn((op.n, 16), dtype=torch.float64, device="cuda")
coef = np.tile([1.0, 0.001], 16)
op.degree()
for _ in range(3):
    op.apply_device(V, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True)
torch.cuda.synchronize()
op.set_timing(True)
op.apply_device(V, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True)
print(mode, k, op.n, op.stats(), [op.window_info(w)["n_subproblems"] for w in range(3)])

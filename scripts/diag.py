"""Stage-by-stage diagnostics of the CUDA path against the oracle (dev aid)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
from oracle import nfft_oracle as O  # noqa: E402
import synth  # noqa: E402

PIN = dict(n_expansion=32, cutoff=4, oversampling=2.0)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


name = sys.argv[1] if len(sys.argv) > 1 else "c0"
feats, wins, f = synth.make_problem(name)
v = synth.random_vector(feats.shape[0])
t0 = time.time()
for w in range(len(wins)):
    op = nld.AnovaOperator(feats, [wins[w]], synth.SIGMA, **PIN)
    ws = op.window_sum(v)
    torch.cuda.synchronize()
    info = op.window_info(0)
    ref = O.AnovaOracle(feats, [wins[w]], synth.SIGMA, **PIN)
    want = ref.window_sums(v)[0]
    print(f"window {w}: rel {rel(ws, want):.3e} info {info}", flush=True)
    if w >= 1:
        break
print("diag done", time.time() - t0)

"""One warm + one profiled batched c4 system matvec, pixel-major batch."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
from paper_2407_06834_b200 import _lib  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
feats, wins, _ = synth.make_problem(cfg)
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA,
                       n_expansion=32, cutoff=4, oversampling=2.0)
eta = op.degree_device()
alphas = synth.alpha_sweep(float(eta.mean()), nrhs)
coef = np.stack([np.ones(nrhs), alphas], 1).ravel()
V = torch.randn((op.n, nrhs), dtype=torch.float64, device="cuda")
Y = torch.empty_like(V)
for _ in range(2):
    op.apply_device(V, _lib.APPLY_SYSTEM, nrhs, coef, out=Y, pixel_major=True)
torch.cuda.synchronize()
print("prof_step_pm done", cfg, nrhs, float(Y.norm()))

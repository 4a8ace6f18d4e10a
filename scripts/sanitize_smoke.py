"""Small sliced-path workload for compute-sanitizer: config 0 (64x64), one
16-rhs fused system product (tcgen05 spread / gather, G digits, assemble,
convolution, epilogue) and a short batched deflated CG."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
from paper_2407_06834_b200 import _lib  # noqa: E402
import synth  # noqa: E402

feats, wins, f = synth.make_problem(sys.argv[1] if len(sys.argv) > 1 else "c0")
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA,
                       n_expansion=32, cutoff=4, oversampling=2.0)
eta = op.degree_device()
V = torch.from_numpy(np.random.default_rng(3).standard_normal((op.n, 16))).cuda()
coef = np.stack([np.ones(16), synth.alpha_sweep(float(eta.mean()), 16)], 1).ravel()
y = op.apply_device(V, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True)
g = op.apply_device(V, _lib.APPLY_GAMMA, 16, pixel_major=True)
res = nld.deflated_solve_batched(op, torch.from_numpy(f[:, 0]).cuda(), 1.0,
                                 synth.alpha_sweep(float(eta.mean()), 16), tol=1e-6, maxit=50)
torch.cuda.synchronize()
print("sanitize workload done", float(y.norm()), float(g.norm()), [r.iterations for r in res])

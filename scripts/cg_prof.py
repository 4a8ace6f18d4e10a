"""Batched deflated CG (bench's CG leg): warm-up solve, then one timed solve.
usage: python scripts/cg_prof.py [config] [nalpha]
Under `ncu --metrics gpu__time_duration.sum` the launches after the last
k_cg_setup are the timed solve's kernels."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
na = int(sys.argv[2]) if len(sys.argv) > 2 else 16
feats, wins, f_img = synth.make_problem(cfg)
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA,
                       n_expansion=32, cutoff=4, oversampling=2.0)
eta = op.degree_device()
alphas = synth.alpha_sweep(float(eta.mean()), na)
f = torch.from_numpy(np.ascontiguousarray(f_img[:, 0])).cuda()
nld.deflated_solve_batched(op, f, 1.0, alphas, prec="jacobi", tol=synth.CG_TOL, maxit=2)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = nld.deflated_solve_batched(op, f, 1.0, alphas, prec="jacobi", tol=synth.CG_TOL, maxit=200)
torch.cuda.synchronize()
print("cg solve ms", (time.perf_counter() - t0) * 1e3, [r.iterations for r in res])

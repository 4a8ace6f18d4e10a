"""Determinism check: the same 16k-rhs product repeated must be bit-identical."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld
from paper_2407_06834_b200 import _lib
import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
feats, wins, _ = synth.make_problem(cfg)
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
rng = np.random.default_rng(nrhs)
V = torch.from_numpy(rng.standard_normal((op.n, nrhs)) * rng.uniform(0.1, 10.0, nrhs)).cuda()
for kind, name in ((_lib.APPLY_WINDOW_SUM, "wsum"), (_lib.APPLY_GAMMA, "gamma")):
    ref = op.apply_device(V, kind, nrhs, pixel_major=True).clone()
    bad = 0
    worst = 0.0
    for r in range(reps):
        y = op.apply_device(V, kind, nrhs, pixel_major=True)
        if not torch.equal(y, ref):
            bad += 1
            d = ((y - ref).norm(dim=0) / ref.norm(dim=0)).max().item()
            worst = max(worst, d)
    print(cfg, nrhs, name, "mismatching repeats", bad, "of", reps, "worst col rel", worst, flush=True)

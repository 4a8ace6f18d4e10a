"""Per-column error of the sliced 16k-rhs product vs the nrhs=1 fp64 products."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld
from paper_2407_06834_b200 import _lib
import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 32
feats, wins, _ = synth.make_problem(cfg)
op = nld.AnovaOperator(feats, wins, synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
rng = np.random.default_rng(nrhs)
V = rng.standard_normal((op.n, nrhs)) * rng.uniform(0.1, 10.0, nrhs)
Vd = torch.from_numpy(V).cuda()
for kind, name in ((_lib.APPLY_WINDOW_SUM, "wsum"), (_lib.APPLY_GAMMA, "gamma")):
    got = op.apply_device(Vd, kind, nrhs, pixel_major=True).cpu().numpy()
    errs = []
    for k in range(nrhs):
        one = op.apply_device(torch.from_numpy(V[:, k].copy()).cuda(), kind, 1).cpu().numpy()
        errs.append(np.linalg.norm(got[:, k] - one) / np.linalg.norm(one))
    print(name, " ".join(f"{e:.1e}" for e in errs))
    bad = int(np.argmax(errs))
    one = op.apply_device(torch.from_numpy(V[:, bad].copy()).cuda(), kind, 1).cpu().numpy()
    d = np.abs(got[:, bad] - one)
    idx = np.argsort(d)[::-1][:8]
    print("  worst col", bad, "worst pixels", idx, d[idx], one[idx])

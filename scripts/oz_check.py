"""Compare the sliced (NLD_OZAKI=1) and DMMA products on the same inputs.
usage: python scripts/oz_check.py CFG NRHS OUT.npy   (run with/without NLD_OZAKI)
       python scripts/oz_check.py cmp A.npy B.npy"""
import sys
import time

import numpy as np

if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    print("rel L2 per kind:", [float(np.linalg.norm(a[k] - b[k]) / np.linalg.norm(b[k]))
                               for k in range(a.shape[0])])
    sys.exit(0)
import torch  # noqa: E402
sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
from paper_2407_06834_b200 import _lib  # noqa: E402
import synth  # noqa: E402

cfg, nrhs, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
feats, wins, _ = synth.make_problem(cfg)
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA,
                       n_expansion=32, cutoff=4, oversampling=2.0)
rng = np.random.default_rng(5)
V = torch.from_numpy(rng.standard_normal((op.n, nrhs))).cuda()
coef = np.stack([np.ones(nrhs), rng.uniform(0, 0.01, nrhs)], 1).ravel()
res = []
for kind in (_lib.APPLY_WINDOW_SUM, _lib.APPLY_SYSTEM):
    y = op.apply_device(V, kind, nrhs, coef if kind == _lib.APPLY_SYSTEM else None,
                        pixel_major=True)
    res.append(y.cpu().numpy())
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    op.apply_device(V, _lib.APPLY_SYSTEM, nrhs, coef, pixel_major=True)
torch.cuda.synchronize()
print(cfg, nrhs, "ms per product", (time.perf_counter() - t0) / 3 * 1e3)
np.save(out, np.stack(res))

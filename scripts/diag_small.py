"""One small 16k-rhs product (c0 or c1), for compute-sanitizer runs."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld
from paper_2407_06834_b200 import _lib
import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c0"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
feats, wins, _ = synth.make_problem(cfg)
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
rng = np.random.default_rng(nrhs)
V = torch.from_numpy(rng.standard_normal((op.n, nrhs))).cuda()
y = op.apply_device(V, _lib.APPLY_GAMMA, nrhs, pixel_major=True)
torch.cuda.synchronize()
print("done", float(y.norm()))

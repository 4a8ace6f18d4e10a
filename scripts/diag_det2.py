"""Where do repeated 16k-rhs products differ?  Single-window operator on c4's
window 0 (WINDOW_SUM = that window's gather), pixels and rhs of the
differences, and the cell of each differing pixel."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld
from paper_2407_06834_b200 import _lib
import synth
from oracle import nfft_oracle as O

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
feats, wins, _ = synth.make_problem(cfg)
w0 = [wins[0]]
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), w0, synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
rng = np.random.default_rng(3)
V = torch.from_numpy(rng.standard_normal((op.n, 16))).cuda()
ref = op.apply_device(V, _lib.APPLY_WINDOW_SUM, 16, pixel_major=True).clone()
pts = np.ascontiguousarray(feats[:, wins[0]])
plan = O.WindowPlan(pts, 1 / synth.SIGMA**2, n_expansion=32, cutoff=4, oversampling=2.0)
x = plan.torus(pts)
base = np.floor(x * 64).astype(np.int64)
key = base[:, 0] * 4096 + base[:, 1] * 64 + base[:, 2]
u, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
for r in range(4):
    y = op.apply_device(V, _lib.APPLY_WINDOW_SUM, 16, pixel_major=True)
    d = (y != ref).cpu().numpy()
    px = np.nonzero(d.any(1))[0]
    print(f"run {r}: {d.sum()} differing entries in {len(px)} pixels; rhs histogram",
          np.bincount(np.nonzero(d)[1], minlength=16).tolist())
    if len(px):
        cells = inv[px]
        uc, cc = np.unique(cells, return_counts=True)
        print("   cells with diffs:", len(uc), "their sizes:", cnt[uc][:12].tolist(),
              "diff pixels per cell:", cc[:12].tolist())
        rel = (y - ref).abs().max().item() / ref.abs().max().item()
        print("   max abs diff / max", rel)

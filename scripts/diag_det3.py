"""Which pixels differ between repeated fused 16-rhs products (c4)?"""
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
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
rng = np.random.default_rng(3)
V = torch.from_numpy(rng.standard_normal((op.n, 16))).cuda()
ref = op.apply_device(V, _lib.APPLY_WINDOW_SUM, 16, pixel_major=True).clone()
cells = []
for w in wins:
    pts = np.ascontiguousarray(feats[:, w])
    plan = O.WindowPlan(pts, 1 / synth.SIGMA**2, n_expansion=32, cutoff=4, oversampling=2.0)
    b = np.floor(plan.torus(pts) * 64).astype(np.int64)
    key = b[:, 0] * 4096 + b[:, 1] * 64 + b[:, 2]
    u, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
    cells.append((inv, cnt))
for r in range(3):
    y = op.apply_device(V, _lib.APPLY_WINDOW_SUM, 16, pixel_major=True)
    d = (y != ref).cpu().numpy()
    px = np.nonzero(d.any(1))[0]
    print(f"run {r}: {d.sum()} entries, {len(px)} pixels; rhs hist",
          np.bincount(np.nonzero(d)[1], minlength=16).tolist(), flush=True)
    if len(px):
        dd = (y - ref).abs().cpu().numpy()[px]
        print("   max |diff| per pixel (first 10):", dd.max(1)[:10])
        for w in range(len(wins)):
            inv, cnt = cells[w]
            uc, cc = np.unique(inv[px], return_counts=True)
            print(f"   window {w}: {len(uc)} cells, sizes {cnt[uc][:10].tolist()}, diff px per cell {cc[:10].tolist()}")
        print("   pixel ids", px[:20].tolist())

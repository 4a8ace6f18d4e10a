"""Are all outputs written?  Fused 16-rhs product into an output pre-filled
with NaN (the first window's gather must overwrite every entry)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld
from paper_2407_06834_b200 import _lib
import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
feats, wins, _ = synth.make_problem(cfg)
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
op.degree_device()
print([op.window_info(w)["n_edge"] for w in range(len(wins))], flush=True)
rng = np.random.default_rng(3)
V = torch.from_numpy(rng.standard_normal((op.n, 16))).cuda()
for r in range(3):
    out = torch.full_like(V, float("nan"))
    op.apply_device(V, _lib.APPLY_WINDOW_SUM, 16, out=out, pixel_major=True)
    bad = torch.isnan(out)
    rows = torch.nonzero(bad.any(1)).flatten().cpu().numpy()
    print(f"run {r}: NaN entries {int(bad.sum())} in {len(rows)} pixels; rhs hist",
          bad.sum(0).cpu().numpy().tolist(), "first pixels", rows[:10].tolist(), flush=True)

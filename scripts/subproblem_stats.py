"""Cell / subproblem size statistics of a config's windows (CPU, numpy):
how many 128-node tiles and 32-node chunks the sliced kernels process
versus N / 128 (padding overhead of small cells)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import synth
from oracle import nfft_oracle as O

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
feats, wins, _ = synth.make_problem(cfg)
N = feats.shape[0]
for w in wins:
    p = feats[:, w]
    wp = O.WindowPlan(p, 2 * 0 + synth.SIGMA ** 2 / 1.0, n_expansion=32, cutoff=4)
    q = wp.torus(p)
    base = np.floor(q * wp.n).astype(np.int64) - 4
    key = base[:, 0] * 1 << 40 if False else (base[:, 0] + 100) * 1000000 + (base[:, 1] + 100) * 1000 + (base[:, -1] + 100)
    _, counts = np.unique(key, return_counts=True)
    subs = []
    for c in counts:
        while c > 2048:
            subs.append(2048); c -= 2048
        subs.append(c)
    subs = np.array(subs)
    tiles = np.ceil(subs / 128).sum()
    chunks = np.ceil(subs / 32).sum()
    print(f"{cfg} window {w.tolist()}: cells {len(counts)}, subproblems {len(subs)}, "
          f"tiles {int(tiles)} (N/128 = {N/128:.0f}, x{tiles/(N/128):.3f}), chunks {int(chunks)} "
          f"(x{chunks/(N/32):.3f}); subs<128: {(subs<128).sum()}, median {np.median(subs):.0f}")

"""Golden alpha sweep at config 1, made by running the REAL reference.

    python tests/golden/make_sweep_golden.py       # writes tests/golden/c1_sweep.npz

16 reference ``deflated_solve`` calls (linops.py:263-300, prec="jacobi",
tol 1e-6) on the c1 image, alpha log-spaced over [1, 100] / mean(eta) -- the
BASELINE config-4 sweep rule at a size the reference finishes in minutes.
The operator is the reference's own AnovaOperator with the BASELINE NFFT
parameters (make_golden.PinnedOperator).  Stored: per alpha the
iteration count, convergence flag, relative residual and residual history;
the full solution for four alphas; and for all 16 a seeded 4096-entry
subsample plus the norm, sum and the dot product with a fixed random vector.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import PinnedOperator, ref_linops, save, synth  # noqa: E402

FULL = (0, 5, 10, 15)


def main():
    feats, wins, f = synth.make_problem("c1")
    n = feats.shape[0]
    op = PinnedOperator(feats, wins, synth.SIGMA)
    eta = op.degree()
    alphas = synth.alpha_sweep(float(eta.mean()), 16)
    idx = np.sort(np.random.default_rng(98).choice(n, 4096, replace=False))
    probe = np.random.default_rng(97).standard_normal(n)
    out = dict(alphas=alphas, idx=idx, f=f[:, 0])
    its, conv, relres, hists, sub, norms, sums, dots = [], [], [], [], [], [], [], []
    t0 = time.perf_counter()
    for k, a in enumerate(alphas):
        system = ref_linops.ShiftedSystem(op, 1.0, float(a))
        res = ref_linops.deflated_solve(system, f[:, 0], prec="jacobi",
                                        tol=synth.CG_TOL, maxit=200)
        its.append(res.iterations)
        conv.append(res.converged)
        relres.append(res.relative_residual)
        hists.append(np.asarray(res.residual_history))
        sub.append(res.x[idx])
        norms.append(np.linalg.norm(res.x))
        sums.append(res.x.sum())
        dots.append(res.x @ probe)
        if k in FULL:
            out[f"u{k}"] = res.x
        print(f"alpha[{k}] = {a:.6g}: {res.iterations} its, relres "
              f"{res.relative_residual:.3e} ({time.perf_counter() - t0:.0f} s)", flush=True)
    width = max(len(h) for h in hists)
    hist = np.full((16, width), np.nan)
    for k, h in enumerate(hists):
        hist[k, :len(h)] = h
    out.update(iters=np.array(its), converged=np.array(conv),
               relres=np.array(relres), history=hist, u_idx=np.array(sub),
               u_norm=np.array(norms), u_sum=np.array(sums), u_dot=np.array(dots),
               probe_seed=np.array(97))
    save("c1_sweep", **out)


if __name__ == "__main__":
    main()

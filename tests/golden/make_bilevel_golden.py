"""Golden vectors for the bilevel driver, made by running the REAL reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_bilevel_golden.py

Writes tests/golden/bilevel.npz: the reference ``brent_minimize`` on the test
functions of its own test_bilevel.py (iterate history included), and a tiny
training set (two 20 x 20 synthetic images, NoiseSpec(30, seed=50), patch 5 --
test_bilevel.py:42-45) with the reference ``ReducedObjective`` values at a few
lambdas (exact and fast kernel modes) and its ``train`` result.  The GPU
tests rebuild the same problem from the stored pixels; nothing on the GPU box
reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from nldenoise import bilevel as B  # noqa: E402
from nldenoise import imaging as I  # noqa: E402

FUNCS = {
    "quadratic": (lambda x: (x - 1.25) ** 2, 0.0, 3.0, {}),
    "cosine": (np.cos, 0.0, 6.0, {"maxit": 40}),
    "linear": (lambda x: x, 0.0, 1.0, {"maxit": 60}),
    "wiggly": (lambda x: np.sin(50 * x) + x * x, -2.0, 2.0, {"maxit": 3}),
    "wiggly_long": (lambda x: np.sin(50 * x) + x * x, -2.0, 2.0, {"maxit": 30}),
    "quartic": (lambda x: (x * x - 2.0) ** 2 + 0.1 * x, 0.0, 3.0, {"tol": 1e-12}),
}
LAMS = np.array([0.05, 0.5, 1.0, 2.0])


def main():
    out = {}
    for name, (fn, a, b, kw) in FUNCS.items():
        res = B.brent_minimize(fn, a, b, **kw)
        out[f"brent_{name}"] = np.array([res.x, res.fx, res.iterations, float(res.converged)])
        out[f"brent_{name}_hist"] = np.array(res.history, np.float64)
    imgs = [I.synthetic_image((20, 20), seed=s) for s in range(2)]
    ts = B.TrainingSet.from_clean_images(imgs, I.NoiseSpec(30.0, seed=50), patch_size=5)
    out["clean"] = np.stack([p.clean.pixels for p in ts.pairs])
    out["noisy"] = np.stack([p.noisy.pixels for p in ts.pairs])
    out["settings"] = np.array([ts.patch_size, ts.sigma, ts.mu, ts.inner_tol, ts.inner_maxit])
    obj = B.ReducedObjective(ts)
    out["j_exact"] = np.array([obj(l) for l in LAMS])
    out["lams"] = LAMS
    ts_fast = B.TrainingSet.from_clean_images(imgs, I.NoiseSpec(30.0, seed=50), patch_size=5,
                                              kernel_mode="fast")
    obj_f = B.ReducedObjective(ts_fast)
    out["j_fast"] = np.array([obj_f(l) for l in LAMS])
    rep = B.train(ts)
    out["train"] = np.array([rep.lambda_opt, rep.objective_opt, rep.brent_iterations,
                             float(rep.brent_converged), *rep.objective_at_bounds])
    out["train_hist"] = np.array(rep.history, np.float64)
    np.savez_compressed(os.path.join(HERE, "bilevel.npz"), **out)
    print({k: v.shape for k, v in out.items()})
    print("train", out["train"])


if __name__ == "__main__":
    main()

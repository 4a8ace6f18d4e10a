"""Generate golden vectors by running the REAL reference (`nldenoise`).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py            # c0, c1, small cases
    python tests/golden/make_golden.py c2 c3 c4   # subsampled large configs

The reference's AnovaOperator hard-codes FastsumPlan defaults
(kernel.py:74); BASELINE pins n_expansion=32, cutoff=4, oversampling=2, so
``PinnedOperator`` overrides ``_build_plans`` exactly as SURVEY.md §8(c)
prescribes.  Everything else (apply, degree, ShiftedSystem, deflated_solve)
is the reference's unmodified code.  Outputs go to tests/golden/*.npz and are
committed; nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from nldenoise import kernel as ref_kernel  # noqa: E402
from nldenoise import linops as ref_linops  # noqa: E402
from nldenoise import transform as ref_transform  # noqa: E402

import synth  # noqa: E402

PLAN_KW = dict(n_expansion=synth.N_EXPANSION, cutoff=synth.CUTOFF,
               oversampling=synth.OVERSAMPLING)


class PinnedOperator(ref_kernel.AnovaOperator):
    """AnovaOperator with the BASELINE NFFT parameters."""

    def _build_plans(self, sigbar):
        plans = []
        for w in self.windows:
            pts = np.ascontiguousarray(self.features[:, w])
            plan = ref_transform.FastsumPlan.build(pts, sigbar, **PLAN_KW)
            plans.append((pts, plan, plan.tables_for(pts)))
        return plans


def feature_digest(feats: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(feats).tobytes()).hexdigest()


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def full_config(name, store_full=True, trim=()):
    feats, wins, f = synth.make_problem(name)
    n = feats.shape[0]
    v = synth.random_vector(n)
    t0 = time.perf_counter()
    op = PinnedOperator(feats, wins, synth.SIGMA)
    gv = op.apply(v)
    t_first = time.perf_counter() - t0
    eta = op.degree()
    mu = synth.ALPHA_SCALE / float(eta.mean())
    system = ref_linops.ShiftedSystem(op, 1.0, mu)
    av = system.apply(v)
    g2v = op.apply_squared(v)
    out = dict(digest=np.array(feature_digest(feats)), v_seed=np.array(1234),
               sigma=np.array(synth.SIGMA), gv=gv, eta=eta, av=av, g2v=g2v,
               mu=np.array(mu), t_first_apply=np.array(t_first))
    plans = op._plans
    out["centers"] = np.array([p.center for _, p, _ in plans], dtype=object) \
        if len({p.center.size for _, p, _ in plans}) > 1 else \
        np.array([p.center for _, p, _ in plans])
    out["scales"] = np.array([p.scale for _, p, _ in plans])
    coeffs0 = plans[0][1].kernel_coeffs
    out["coeffs0_axis"] = coeffs0[(slice(None),) + (16,) * (coeffs0.ndim - 1)]
    base0, w0 = plans[0][2]
    out["base0_head"] = base0[:64]
    out["weights0_head"] = w0[:64]
    if store_full:
        f1 = f[:, 0]
        res = ref_linops.deflated_solve(system, f1, prec="jacobi",
                                        tol=synth.CG_TOL, maxit=200)
        out.update(f=f1, u=res.x, iters=np.array(res.iterations),
                   converged=np.array(res.converged),
                   relres=np.array(res.relative_residual),
                   history=np.array(res.residual_history))
        if n <= 5000:
            exact = ref_kernel.AnovaOperator(feats, wins, synth.SIGMA,
                                             mode="exact")
            out["gv_dense"] = exact.apply(v)
    else:
        # keep only a seeded subsample plus global reductions
        idx = np.sort(np.random.default_rng(99).choice(n, 4096, replace=False))
        for key in ("gv", "eta", "av", "g2v"):
            vec = out.pop(key)
            out[key + "_idx"] = vec[idx]
            out[key + "_norm"] = np.array(np.linalg.norm(vec))
            out[key + "_sum"] = np.array(vec.sum())
        out["idx"] = idx
        out.pop("centers")
    for key in trim:
        out.pop(key, None)
    save(name, **out)


def default_param_cases():
    """Reference-default plans (m=5, adaptive N_d) on test_kernel-like data."""
    rng = np.random.default_rng(0)
    feats = rng.uniform(0, 255, size=(300, 7))
    wins = [np.arange(0, 3), np.arange(3, 6), np.arange(6, 7)]
    v = np.random.default_rng(4).standard_normal(300)
    op = ref_kernel.AnovaOperator(feats, wins, 40.0)
    gv = op.apply(v)
    eta = op.degree()
    g2v = op.apply_squared(v)
    nd = np.array([p.nfft_plan.bandwidth[0] for _, p, _ in op._plans])
    exact = ref_kernel.AnovaOperator(feats, wins, 40.0, mode="exact").apply(v)
    system = ref_linops.ShiftedSystem(op, 1e-2, 1e-2)
    f = rng.uniform(0, 255, size=300)
    res = ref_linops.deflated_solve(system, f, prec="jacobi", tol=1e-10,
                                    maxit=300)
    res_l2 = ref_linops.deflated_solve(system, f, prec="l2", tol=1e-10,
                                       maxit=300)
    res_none = ref_linops.plain_solve(system, f, prec="none", tol=1e-10,
                                      maxit=300)
    fgt = {}
    for d in (1, 2, 3):
        r = np.random.default_rng(20 + d)
        pts = r.uniform(0, 255, size=(400, d))
        alpha = r.standard_normal(400)
        plan = ref_transform.FastsumPlan.build(pts, 1.0 / 40.0 ** 2)
        fgt[f"fgt{d}_pts"] = pts
        fgt[f"fgt{d}_alpha"] = alpha
        fgt[f"fgt{d}_out"] = ref_transform.gauss_transform_fast(
            pts, pts, alpha, plan)
        fgt[f"fgt{d}_nd"] = np.array(plan.nfft_plan.bandwidth[0])
    save("default_params", feats=feats, v=v, gv=gv, eta=eta, g2v=g2v, nd=nd,
         gv_exact=exact, f=f, u=res.x, iters=np.array(res.iterations),
         history=np.array(res.residual_history), u_l2=res_l2.x,
         iters_l2=np.array(res_l2.iterations), u_plain=res_none.x,
         iters_plain=np.array(res_none.iterations), **fgt)


def edge_case():
    """Nodes on exact grid lines: 9 nonzero KB weights per dimension.

    center = 0 and radius = 0.21875 make scale == 1.0 exactly, so x*n = 64 p
    is exact; p = j/64 gives frac == 0 (weights i = 0..8 nonzero) and
    p = nextafter(j, 0)/64 gives frac = 1 - ulp (weights i = 1..9 nonzero).
    """
    rng = np.random.default_rng(7)
    r = 0.21875
    anchors = np.array([[r, 0, 0], [-r, 0, 0], [0, 0.1, 0], [0, -0.1, 0],
                        [0, 0, 0.1], [0, 0, -0.1]])
    body = rng.uniform(-0.1, 0.1, size=(400, 3))
    on_grid = rng.integers(-6, 7, size=(60, 3)) / 64.0
    below = np.nextafter(rng.integers(-6, 7, size=(60, 3)).astype(float),
                         -np.inf) / 64.0
    mixed = body[:60].copy()
    mixed[:, 1] = rng.integers(-6, 7, size=60) / 64.0
    pts = np.concatenate([anchors, body, on_grid, below, mixed])
    pts = np.clip(pts, -r, r)
    feats = np.concatenate([pts, pts[:, :1] * 0.5], axis=1)  # + a 1-D window
    wins = [np.arange(3), np.array([3])]
    v = np.random.default_rng(8).standard_normal(feats.shape[0])
    op = PinnedOperator(feats, wins, 0.1)
    gv = op.apply(v)
    _, plan, (base, w) = op._plans[0]
    nz = (w != 0).sum(axis=2)
    save("edge_nodes", feats=feats, v=v, gv=gv, scale0=np.array(plan.scale),
         nnz_max=np.array(nz.max()), eta=op.degree())


if __name__ == "__main__":
    todo = sys.argv[1:] or ["small"]
    for item in todo:
        t0 = time.perf_counter()
        if item == "small":
            full_config("c0")
            full_config("c1", trim=("f", "av", "g2v"))
            default_param_cases()
            edge_case()
        else:
            full_config(item, store_full=False)
        print(item, f"{time.perf_counter() - t0:.1f}s")

"""Brent minimiser (host logic of the bilevel driver) against the reference.

tests/golden/bilevel.npz holds the REAL reference's brent_minimize results and
iterate histories (tests/golden/make_bilevel_golden.py); the known-answer cases
are those of the reference's test_bilevel.py:12-38.
"""

import numpy as np
import pytest

from paper_2407_06834_b200 import bilevel as B

FUNCS = {
    "quadratic": (lambda x: (x - 1.25) ** 2, 0.0, 3.0, {}),
    "cosine": (np.cos, 0.0, 6.0, {"maxit": 40}),
    "linear": (lambda x: x, 0.0, 1.0, {"maxit": 60}),
    "wiggly": (lambda x: np.sin(50 * x) + x * x, -2.0, 2.0, {"maxit": 3}),
    "wiggly_long": (lambda x: np.sin(50 * x) + x * x, -2.0, 2.0, {"maxit": 30}),
    "quartic": (lambda x: (x * x - 2.0) ** 2 + 0.1 * x, 0.0, 3.0, {"tol": 1e-12}),
}


@pytest.mark.parametrize("name", sorted(FUNCS))
def test_brent_matches_reference_history(golden, name):
    g = golden("bilevel")
    fn, a, b, kw = FUNCS[name]
    res = B.brent_minimize(fn, a, b, **kw)
    want = g[f"brent_{name}"]
    hist = np.array(res.history, np.float64)
    # identical arithmetic in the identical order: bit-for-bit iterates
    assert hist.shape == g[f"brent_{name}_hist"].shape
    assert np.array_equal(hist, g[f"brent_{name}_hist"])
    assert res.x == want[0] and res.fx == want[1]
    assert res.iterations == int(want[2]) and res.converged == bool(want[3])


def test_known_answers():
    res = B.brent_minimize(lambda x: (x - 1.25) ** 2, 0.0, 3.0)
    assert res.converged and abs(res.x - 1.25) < 1e-8 and res.iterations <= 10
    res = B.brent_minimize(np.cos, 0.0, 6.0, maxit=40)
    assert res.converged and abs(res.x - np.pi) < 1e-7
    res = B.brent_minimize(lambda x: x, 0.0, 1.0, maxit=60)
    assert abs(res.x) < 1e-6
    res = B.brent_minimize(lambda x: (x - 2.0) ** 2, 0.0, 3.0)
    assert len(res.history) >= 2 and min(f for _, f in res.history) == res.fx
    res = B.brent_minimize(lambda x: np.sin(50 * x) + x * x, -2.0, 2.0, maxit=3)
    assert res.iterations <= 3


def test_bad_bracket():
    with pytest.raises(ValueError):
        B.brent_minimize(lambda x: x, 1.0, 1.0)


def test_training_set_defaults():
    ts = B.TrainingSet.from_arrays([np.zeros((4, 4))], [np.ones((4, 4))])
    assert (ts.patch_size, ts.sigma, ts.mu, ts.kernel_mode) == (7, 40.0, 0.01, "exact")
    assert (ts.inner_tol, ts.inner_maxit) == (B.DEFAULT_INNER_TOL, B.DEFAULT_INNER_MAXIT)
    assert B.DEFAULT_LAMBDA_RANGE == (1e-9, 3.0)

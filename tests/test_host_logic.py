"""CPU: host-side validation, error mapping and input generation."""

import numpy as np
import pytest

import paper_2407_06834_b200 as nld
from paper_2407_06834_b200 import _lib
import synth


class TestValidation:
    """Same exceptions, same order as kernel.py:30-48 / linops.py:31-37."""

    def test_wide_window_rejected(self):
        with pytest.raises(nld.WindowSizeError):
            nld.AnovaOperator(np.zeros((5, 4)), [np.arange(4)], 1.0)

    def test_window_index_out_of_range(self):
        with pytest.raises(nld.DimensionMismatchError):
            nld.AnovaOperator(np.zeros((5, 2)), [np.array([2])], 1.0)

    def test_bad_sigma(self):
        with pytest.raises(ValueError):
            nld.AnovaOperator(np.zeros((5, 2)), [np.arange(2)], 0.0)

    def test_empty_features_rejected(self):
        with pytest.raises(nld.DimensionMismatchError):
            nld.AnovaOperator(np.zeros((0, 3)), [np.arange(3)], 1.0)

    def test_features_must_be_2d(self):
        with pytest.raises(nld.DimensionMismatchError):
            nld.AnovaOperator(np.zeros(5), [np.arange(1)], 1.0)

    def test_no_windows(self):
        with pytest.raises(ValueError):
            nld.AnovaOperator(np.zeros((5, 2)), [], 1.0)

    def test_unknown_mode(self):
        with pytest.raises(ValueError):
            nld.AnovaOperator(np.zeros((5, 2)), [np.arange(2)], 1.0,
                              mode="approx")

    def test_odd_expansion(self):
        with pytest.raises(ValueError):
            nld.AnovaOperator(np.zeros((5, 2)), [np.arange(2)], 1.0,
                              n_expansion=31)

    def test_errors_share_the_reference_hierarchy(self):
        for exc in (nld.DimensionMismatchError, nld.ScalingOverflowError,
                    nld.WindowSizeError, nld.DenseLimitError,
                    nld.SolverBreakdownError):
            assert issubclass(exc, nld.NldenoiseError)


def test_status_codes_map_to_reference_exceptions():
    for code, exc in [(_lib.ERR_DIMENSION, nld.DimensionMismatchError),
                      (_lib.ERR_SCALING, nld.ScalingOverflowError),
                      (_lib.ERR_WINDOW, nld.WindowSizeError),
                      (_lib.ERR_DENSE_LIMIT, nld.DenseLimitError),
                      (_lib.ERR_BREAKDOWN, nld.SolverBreakdownError),
                      (_lib.ERR_VALUE, ValueError)]:
        with pytest.raises(exc):
            _lib.check(code)
    _lib.check(0)


@pytest.mark.parametrize("name,n,d,nwin", [("c0", 4096, 9, 3),
                                           ("c2", 1048576, 25, 9),
                                           ("c3", 262144, 27, 9)])
def test_generator_shapes(name, n, d, nwin):
    feats, wins, f = synth.make_problem(name)
    assert feats.shape == (n, d) and len(wins) == nwin
    assert feats.min() >= -0.2 and feats.max() <= 0.2
    assert f.min() >= 0.0 and f.max() <= 1.0
    sizes = [w.size for w in wins]
    assert sizes[:-1] == [3] * (nwin - 1) and sizes[-1] in (1, 3)
    # windows cover the features once, in row-major patch order
    assert np.array_equal(np.concatenate(wins), np.arange(d))


def test_generator_is_deterministic():
    a = synth.make_problem("c0")[0]
    b = synth.make_problem("c0")[0]
    assert np.array_equal(a, b)


def test_alpha_sweep():
    al = synth.alpha_sweep(100.0, 16)
    assert al.size == 16 and np.isclose(al[0], 0.01) and np.isclose(al[-1], 1.0)


class TestTransformValidation:
    """transform.py validation (no GPU needed)."""

    def test_plan_rules(self):
        from paper_2407_06834_b200 import transform as T
        with pytest.raises(ValueError):
            T.NfftPlan((15,))
        with pytest.raises(ValueError):
            T.NfftPlan((16,), oversampling=1.0)
        with pytest.raises(ValueError):
            T.NfftPlan((16,), cutoff=0)
        plan = T.NfftPlan((32, 32), oversampling=2.0, cutoff=4)
        assert plan.nos == (64, 64) and plan.dim == 2
        assert abs(plan._shape_b[0] - 1.5 * np.pi) < 1e-15

    def test_nodes_rules(self):
        from paper_2407_06834_b200 import transform as T
        with pytest.raises(nld.DimensionMismatchError):
            T.NodeSet(np.zeros((3, 4)))
        with pytest.raises(ValueError):
            T.NodeSet(np.array([0.5]))
        ns = T.NodeSet(np.array([[0.0, 0.1], [-0.5, 0.49]]))
        assert ns.dim == 2 and len(ns) == 2

    def test_expansion_degree(self):
        from oracle import nfft_oracle as O
        from paper_2407_06834_b200 import transform as T
        assert T.expansion_degree(1.0) == 16
        assert T.expansion_degree(1000.0) > T.expansion_degree(100.0)
        assert T.expansion_degree(1e9) == T.MAX_EXPANSION
        for s in (0.5, 3.0, 250.77, 1e4):
            assert T.expansion_degree(s) == O.expansion_degree(s)


def test_cell_partition_covers_and_keeps_cells_whole():
    """sharding.partition: every pixel on exactly one rank, balanced to
    within one pixel, and window-0 cells split across at most world - 1 rank
    boundaries (the point of the partition)."""
    from paper_2407_06834_b200 import sharding as S
    feats, wins, _ = synth.make_problem("c1")
    n = feats.shape[0]
    for world in (1, 2, 3, 8):
        parts = S.partition(feats, wins, world)
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
        allix = np.concatenate(parts)
        assert len(allix) == n and len(np.unique(allix)) == n
        p = feats[:, wins[0]]
        c = 0.5 * (p.min(0) + p.max(0))
        r = np.sqrt(((p - c) ** 2).sum(1).max())
        cell = np.floor((p - c) * ((0.25 - 1 / 32) / r) * 64).astype(np.int64)
        key = (cell[:, 0] * 1000 + cell[:, 1]) * 1000 + cell[:, 2]
        owners = {}
        for rank, ix in enumerate(parts):
            for k in np.unique(key[ix]):
                owners.setdefault(k, set()).add(rank)
        assert sum(len(o) - 1 for o in owners.values()) <= world - 1

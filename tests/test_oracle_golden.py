"""Pin the CPU oracle against the REAL reference's outputs (tests/golden).

The golden vectors were produced by tests/golden/make_golden.py, which runs
the unmodified reference (`nldenoise`) with BASELINE's NFFT parameters.
"""

import hashlib

import numpy as np
import pytest

from oracle import nfft_oracle as O
import synth

PIN = dict(n_expansion=32, cutoff=4, oversampling=2.0)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def test_generator_matches_golden_inputs(golden):
    for name in ("c0", "c1"):
        feats, _, _ = synth.make_problem(name)
        digest = hashlib.sha256(feats.tobytes()).hexdigest()
        assert digest == str(golden(name)["digest"]), name


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_oracle_matvec_matches_reference(golden, name):
    g = golden(name)
    feats, wins, _ = synth.make_problem(name)
    v = synth.random_vector(feats.shape[0])
    op = O.AnovaOracle(feats, wins, synth.SIGMA, **PIN)
    assert rel(op.apply(v), g["gv"]) < 1e-12
    assert rel(op.degree(), g["eta"]) < 1e-12
    plans = op.plans()
    assert np.array_equal([p.scale for _, p, _ in plans], g["scales"])
    base, w = plans[0][2]
    assert np.array_equal(base[:64], g["base0_head"])
    np.testing.assert_allclose(w[:64], g["weights0_head"], rtol=1e-14,
                               atol=0)
    sysm = O.SystemOracle(op, 1.0, float(g["mu"]))
    if "av" in g:
        assert rel(sysm.apply(v), g["av"]) < 1e-12
        assert rel(op.apply(v, squared=True), g["g2v"]) < 1e-12


def test_oracle_cg_matches_reference(golden):
    g = golden("c0")
    feats, wins, f = synth.make_problem("c0")
    op = O.AnovaOracle(feats, wins, synth.SIGMA, **PIN)
    sysm = O.SystemOracle(op, 1.0, float(g["mu"]))
    u, it, conv, relres, hist = O.deflated_solve(sysm, f[:, 0], "jacobi",
                                                 synth.CG_TOL, 200)
    assert it == int(g["iters"]) and conv
    assert rel(u, g["u"]) < 1e-12
    np.testing.assert_allclose(hist, g["history"], rtol=1e-8)


def test_oracle_dense_matches_reference_exact_mode(golden):
    g = golden("c0")
    feats, wins, _ = synth.make_problem("c0")
    v = synth.random_vector(feats.shape[0])
    op = O.AnovaOracle(feats, wins, synth.SIGMA)
    assert rel(op.dense() @ v, g["gv_dense"]) < 1e-13
    # the reference's own NFFT error at config 0 (~2.8e-6)
    assert rel(g["gv"], g["gv_dense"]) < 5e-6


def test_oracle_default_params(golden):
    g = golden("default_params")
    op = O.AnovaOracle(g["feats"], [np.arange(0, 3), np.arange(3, 6),
                                    np.arange(6, 7)], 40.0)
    assert rel(op.apply(g["v"]), g["gv"]) < 1e-12
    assert [p.bandwidth for _, p, _ in op.plans()] == list(g["nd"])
    assert rel(op.apply(g["v"], squared=True), g["g2v"]) < 1e-12
    sysm = O.SystemOracle(op, 1e-2, 1e-2)
    u, it, _, _, _ = O.deflated_solve(sysm, g["f"], "jacobi", 1e-10, 300)
    assert it == int(g["iters"]) and rel(u, g["u"]) < 1e-10
    u2, it2, _, _, _ = O.deflated_solve(sysm, g["f"], "l2", 1e-10, 300)
    assert it2 == int(g["iters_l2"]) and rel(u2, g["u_l2"]) < 1e-10
    u3, it3, _, _, _ = O.plain_solve(sysm, g["f"], "none", 1e-10, 300)
    assert it3 == int(g["iters_plain"]) and rel(u3, g["u_plain"]) < 1e-9
    for d in (1, 2, 3):
        pts, alpha = g[f"fgt{d}_pts"], g[f"fgt{d}_alpha"]
        plan = O.WindowPlan(pts, 1.0 / 40.0 ** 2)
        assert plan.bandwidth == int(g[f"fgt{d}_nd"])
        assert rel(plan.transform(pts, pts, alpha), g[f"fgt{d}_out"]) < 1e-12


def test_oracle_edge_nodes(golden):
    g = golden("edge_nodes")
    op = O.AnovaOracle(g["feats"], [np.arange(3), np.array([3])], 0.1, **PIN)
    _, plan, (base, w) = op.plans()[0]
    assert plan.scale == float(g["scale0"]) == 1.0
    assert (w != 0).sum(axis=2).max() == 9
    assert rel(op.apply(g["v"]), g["gv"]) < 1e-12


def test_known_answers():
    # test_linops.py:30-38 frozen SCS vectors
    x = np.array([2.0, 3.0, 5.0, 7.0])
    assert np.array_equal(O.scs_up(x), [17.0, 14.0, 9.0, 2.0])
    assert np.array_equal(O.scs_down(x), [17.0, 2.0, 5.0, 10.0])
    # test_linops.py:88-94 U columns for v = 1
    b = O.Basis(np.ones(4))
    assert np.allclose(b.apply(np.eye(4)[:, 0]), 0.5, atol=1e-13)
    assert np.allclose(b.apply(np.eye(4)[:, 1]),
                       [np.sqrt(0.5), -np.sqrt(0.5), 0, 0], atol=1e-13)
    # test_transform.py:26-31 ndft phase and :123-127 direct sum
    c = np.zeros(8, complex)
    c[5] = 1.0
    assert np.allclose(O.ndft(c, np.array([0.25])), [-1j], atol=1e-14)
    assert np.allclose(O.gauss_direct([0.0, 1.0], [0.0], [1.0, 1.0], 1.0),
                       [1.0 + np.exp(-1.0)], atol=1e-14)


def test_cpu_port_matches_reference(golden):
    from oracle.cpu_port import CpuPort
    g = golden("c0")
    feats, wins, _ = synth.make_problem("c0")
    v = synth.random_vector(feats.shape[0])
    port = CpuPort(feats, wins, synth.SIGMA, **PIN)
    assert rel(port.apply(v), g["gv"]) < 1e-12
    assert rel(port.system_apply(v, 1.0, float(g["mu"])), g["av"]) < 1e-12
    one = CpuPort(feats, wins, synth.SIGMA, nthreads=1, **PIN)
    assert rel(one.apply(v), g["gv"]) < 1e-12

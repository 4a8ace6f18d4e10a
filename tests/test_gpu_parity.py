"""GPU parity: the CUDA path (through the C-ABI) against the reference.

Expected values are the REAL reference's outputs (tests/golden, made by
tests/golden/make_golden.py) or the pinned CPU oracle at sizes it finishes in
seconds.  Tolerances (north star): 1e-10 relative l2 for the fp64 matvec
against the reference's own fast summation; the reference's NFFT error bound
against the dense kernel sum at config 0; CG to 1e-8 relative within +-1
iteration.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import GOLDEN  # noqa: E402

import paper_2407_06834_b200 as nld  # noqa: E402
from oracle import nfft_oracle as O  # noqa: E402
import synth  # noqa: E402

PIN = dict(n_expansion=synth.N_EXPANSION, cutoff=synth.CUTOFF,
           oversampling=synth.OVERSAMPLING)
MATVEC_TOL = 1e-10
CG_TOL_U = 1e-8


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def have(name):
    return os.path.exists(os.path.join(GOLDEN, f"{name}.npz"))


_OPS = {}


def operator(name):
    if name not in _OPS:
        feats, wins, f = synth.make_problem(name)
        _OPS[name] = (nld.AnovaOperator(feats, wins, synth.SIGMA, **PIN),
                      feats, wins, f)
    return _OPS[name]


# ---------------------------------------------------------------- config 0/1

@pytest.mark.parametrize("name", ["c0", "c1"])
def test_matvec_matches_reference(golden, name):
    g = golden(name)
    op, feats, _, _ = operator(name)
    v = synth.random_vector(op.n)
    assert rel(op.apply(v), g["gv"]) < MATVEC_TOL
    assert rel(op.degree(), g["eta"]) < MATVEC_TOL
    info = op.window_info(0)
    assert info["scale"] == float(g["scales"][0])
    assert info["bandwidth"] == 32 and info["grid"] == 64
    system = nld.ShiftedSystem(op, 1.0, float(g["mu"]))
    av = system.apply(v)
    if "av" in g:
        assert rel(av, g["av"]) < MATVEC_TOL
        assert rel(op.apply_squared(v), g["g2v"]) < MATVEC_TOL
    # the fused epilogue equals the composition of the reference's formulas
    want = 1.0 * v + float(g["mu"]) * (g["eta"] * v - g["gv"])
    assert rel(av, want) < MATVEC_TOL


def test_config0_against_dense_kernel_sum(golden):
    g = golden("c0")
    op, feats, wins, _ = operator("c0")
    v = synth.random_vector(op.n)
    fast = op.apply(v)
    # within the reference's own NFFT error (2.8e-6 rel l2)
    ref_err = rel(g["gv"], g["gv_dense"])
    assert rel(fast, g["gv_dense"]) < 1.5 * ref_err
    exact = nld.AnovaOperator(feats, wins, synth.SIGMA, mode="exact")
    assert rel(exact.apply(v), g["gv_dense"]) < 1e-12


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_deflated_cg_matches_reference(golden, name):
    g = golden(name)
    op, _, _, f = operator(name)
    system = nld.ShiftedSystem(op, 1.0, float(g["mu"]))
    res = nld.deflated_solve(system, f[:, 0], prec="jacobi", tol=synth.CG_TOL,
                             maxit=200)
    assert res.converged
    assert abs(res.iterations - int(g["iters"])) <= 1
    assert rel(res.x, g["u"]) < CG_TOL_U
    if res.iterations == int(g["iters"]):
        np.testing.assert_allclose(res.residual_history, g["history"],
                                   rtol=1e-6)
    # deflation preserves the mean (test_linops.py:182-185)
    assert abs(res.x.mean() - f[:, 0].mean()) < 1e-8


# ------------------------------------------------ large configs (subsampled)

@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_large_config_matvec_subsample(golden, name):
    if not have(name):
        pytest.skip(f"no golden for {name}")
    g = golden(name)
    op, feats, _, _ = operator(name)
    v = synth.random_vector(op.n)
    idx = g["idx"]
    vt = torch.from_numpy(v).cuda()
    gv = op.apply(vt)
    eta = op.degree_device()
    system = nld.ShiftedSystem(op, 1.0, float(g["mu"]))
    av = system.apply(vt)
    g2v = op.apply_squared(vt)
    for key, vec in (("gv", gv), ("eta", eta), ("av", av), ("g2v", g2v)):
        h = vec.cpu().numpy()
        assert rel(h[idx], g[key + "_idx"]) < MATVEC_TOL, key
        assert abs(np.linalg.norm(h) / float(g[key + "_norm"]) - 1) < MATVEC_TOL
    _OPS.pop(name, None)


# ------------------------------------------------ reference-default plans

def test_default_parameters(golden):
    """m=5, adaptive N_d (66/70/42 -> grids 132/140/84), exact mode, CG."""
    g = golden("default_params")
    wins = [np.arange(0, 3), np.arange(3, 6), np.arange(6, 7)]
    op = nld.AnovaOperator(g["feats"], wins, 40.0)
    assert rel(op.apply(g["v"]), g["gv"]) < MATVEC_TOL
    assert [op.window_info(w)["bandwidth"] for w in range(3)] == list(g["nd"])
    assert rel(op.apply_squared(g["v"]), g["g2v"]) < MATVEC_TOL
    assert rel(op.degree(), g["eta"]) < MATVEC_TOL
    exact = nld.AnovaOperator(g["feats"], wins, 40.0, mode="exact")
    assert rel(exact.apply(g["v"]), g["gv_exact"]) < 1e-12
    system = nld.ShiftedSystem(op, 1e-2, 1e-2)
    res = nld.deflated_solve(system, g["f"], prec="jacobi", tol=1e-10,
                             maxit=300)
    assert abs(res.iterations - int(g["iters"])) <= 1
    assert rel(res.x, g["u"]) < CG_TOL_U
    res = nld.deflated_solve(system, g["f"], prec="l2", tol=1e-10, maxit=300)
    assert abs(res.iterations - int(g["iters_l2"])) <= 1
    assert rel(res.x, g["u_l2"]) < CG_TOL_U
    res = nld.plain_solve(system, g["f"], prec="none", tol=1e-10, maxit=300)
    assert abs(res.iterations - int(g["iters_plain"])) <= 1
    assert rel(res.x, g["u_plain"]) < CG_TOL_U


@pytest.mark.parametrize("d", [1, 2, 3])
def test_fast_gauss_transform(golden, d):
    """gauss_transform_fast on 400 nodes in [0,255]^d (test_transform.py:142-151)."""
    g = golden("default_params")
    pts, alpha = g[f"fgt{d}_pts"], g[f"fgt{d}_alpha"]
    op = nld.AnovaOperator(pts, [np.arange(d)], 40.0)
    assert rel(op.window_sum(alpha), g[f"fgt{d}_out"]) < MATVEC_TOL
    assert op.window_info(0)["bandwidth"] == int(g[f"fgt{d}_nd"])


def test_edge_nodes(golden):
    """Nodes on grid lines carry 2m+1 nonzero weights (transform.py:168)."""
    g = golden("edge_nodes")
    op = nld.AnovaOperator(g["feats"], [np.arange(3), np.array([3])], 0.1,
                           **PIN)
    assert rel(op.apply(g["v"]), g["gv"]) < MATVEC_TOL
    assert rel(op.degree(), g["eta"]) < MATVEC_TOL
    assert op.window_info(0)["n_edge"] > 0
    assert op.window_info(0)["scale"] == 1.0


# ------------------------------------------------ other cutoffs (generic path)

@pytest.mark.parametrize("cutoff", [2, 3, 4, 5, 6])
def test_cutoffs_against_oracle(cutoff):
    rng = np.random.default_rng(cutoff)
    feats = rng.uniform(-1, 1, size=(700, 5))
    wins = [np.arange(0, 3), np.arange(3, 5)]
    v = rng.standard_normal(700)
    kw = dict(n_expansion=16, cutoff=cutoff, oversampling=2.0)
    op = nld.AnovaOperator(feats, wins, 0.5, **kw)
    ref = O.AnovaOracle(feats, wins, 0.5, **kw)
    assert rel(op.apply(v), ref.apply(v)) < MATVEC_TOL


# ------------------------------------------------ size-independent properties

def test_properties_full_size():
    op, _, _, _ = operator("c2")
    rng = np.random.default_rng(5)
    u = torch.from_numpy(rng.standard_normal(op.n)).cuda()
    w = torch.from_numpy(rng.standard_normal(op.n)).cuda()
    gu, gw = op.apply(u), op.apply(w)
    # linearity
    comb = op.apply(2.0 * u - 3.0 * w)
    assert rel(comb.cpu(), (2.0 * gu - 3.0 * gw).cpu()) < 1e-12
    # near-symmetry of the fast operator (test_kernel.py:136-144)
    lhs = float(u @ gw)
    rhs = float(gu @ w)
    assert abs(lhs - rhs) <= 1e-4 * max(abs(lhs), 1.0)
    # L 1 = 0 and A 1 = lam 1 (test_linops.py:262-269)
    system = nld.ShiftedSystem(op, 0.5, 1e-3)
    ones = torch.ones(op.n, dtype=torch.float64, device="cuda")
    assert float((system.apply(ones) - 0.5).abs().max()) < 1e-8
    # batched = stacked single products
    both = op.apply(torch.stack([u, w]))
    assert rel(both[0].cpu(), gu.cpu()) < 1e-15
    assert rel(both[1].cpu(), gw.cpu()) < 1e-15
    # determinism
    assert torch.equal(op.apply(u), gu)


def test_batched_alpha_sweep_matches_single_solves(golden):
    g = golden("c1")
    op, _, _, f = operator("c1")
    eta = op.degree()
    alphas = synth.alpha_sweep(float(eta.mean()), 4)
    batch = nld.deflated_solve_batched(op, f[:, 0], 1.0, alphas,
                                       tol=synth.CG_TOL, maxit=200)
    for a, res in zip(alphas, batch):
        single = nld.deflated_solve(nld.ShiftedSystem(op, 1.0, a), f[:, 0],
                                    tol=synth.CG_TOL, maxit=200)
        assert res.iterations == single.iterations
        assert rel(res.x, single.x) < 1e-12


# ------------------------------------------------ basis / pcg / errors

def test_deflating_basis_against_oracle():
    rng = np.random.default_rng(2)
    for n in (2, 30, 301, 5000):
        v = rng.standard_normal(n)
        v[0] += np.sign(v[0]) + 0.1
        x = rng.standard_normal(n)
        ob = O.Basis(v)
        b = nld.DeflatingBasis(v)
        assert np.abs(b.apply(x) - ob.apply(x)).max() < 1e-11
        assert np.abs(b.apply_adjoint(x) - ob.apply_adjoint(x)).max() < 1e-11
        assert np.abs(b.apply_adjoint(b.apply(x)) - x).max() < 1e-11
    x = np.array([2.0, 3.0, 5.0, 7.0])
    assert np.array_equal(nld.scs_up(x), [17.0, 14.0, 9.0, 2.0])
    assert np.array_equal(nld.scs_down(x), [17.0, 2.0, 5.0, 10.0])
    with pytest.raises(ValueError):
        nld.DeflatingBasis(np.array([0.0, 1.0, 2.0]))


def test_generic_pcg():
    rng = np.random.default_rng(3)
    m = rng.standard_normal((30, 30))
    a = m @ m.T + 30 * np.eye(30)
    b = rng.standard_normal(30)
    res = nld.pcg(lambda x: a @ x, b, tol=1e-12, maxit=200)
    assert res.converged
    assert np.abs(res.x - np.linalg.solve(a, b)).max() < 1e-9
    d = np.array([1.0, 4.0, 9.0])
    res = nld.pcg(lambda x: d * x, np.ones(3), prec=lambda r: r / d,
                  tol=1e-14, maxit=10)
    assert res.converged and res.iterations == 1
    with pytest.raises(nld.SolverBreakdownError):
        nld.pcg(lambda x: np.diag([1.0, -1.0]) @ x, np.array([1.0, 1.0]),
                maxit=10)


def test_solver_edge_cases(golden):
    op, _, _, f = operator("c0")
    system = nld.ShiftedSystem(op, 1.0, 1e-3)
    res = nld.deflated_solve(system, f[:, 0], maxit=0)
    assert not res.converged and res.iterations == 0
    # zero right-hand side (test_linops.py:162-164)
    res = nld.deflated_solve(system, np.zeros(op.n))
    assert res.converged and res.iterations == 0
    assert res.relative_residual == 0.0 and np.abs(res.x).max() == 0.0
    with pytest.raises(ValueError):
        nld.deflated_solve(system, f[:, 0], prec="ilu")
    with pytest.raises(nld.DimensionMismatchError):
        op.apply(np.ones(3))


def test_dense_limit():
    rng = np.random.default_rng(0)
    op = nld.AnovaOperator(rng.random((6000, 3)), [np.arange(3)], 40.0,
                           mode="exact")
    with pytest.raises(nld.DenseLimitError):
        op.apply(np.ones(6000))


# ------------------------------------------------ pixel sharding (emulated)

def test_sharded_ranks_match_single_gpu(golden):
    """2 ranks as host threads on one GPU (sharding.ThreadComm): the sharded
    matvec, degree and batched CG equal the unsharded operator's."""
    import threading

    from paper_2407_06834_b200 import sharding as S
    g = golden("c1")
    full, feats, wins, f = operator("c1")
    n = feats.shape[0]
    v = synth.random_vector(n)
    want_gv = full.apply(v)
    want_eta = full.degree()
    mus = [float(g["mu"]), 3.0 * float(g["mu"])]
    want_cg = nld.deflated_solve_batched(full, f[:, 0], 1.0, mus,
                                         tol=synth.CG_TOL, maxit=200)
    world = 2
    comm = S.ThreadComm(world, device=torch.device("cuda", 0))
    out, errs = {}, []

    def rank_main(rank):
        try:
            lo, hi = S.shard_range(n, rank, world)
            op = nld.AnovaOperator(torch.from_numpy(feats[lo:hi]).cuda(), wins,
                                   synth.SIGMA, **PIN)
            S.attach(op, comm, rank, n)
            gv = op.apply(v[lo:hi])
            eta = op.degree().cpu().numpy()
            res = nld.deflated_solve_batched(op, f[lo:hi, 0], 1.0, mus,
                                             tol=synth.CG_TOL, maxit=200)
            out[rank] = (gv, eta, res, op.window_info(0))
        except Exception as exc:  # pragma: no cover - reported below
            errs.append(exc)
            comm.barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errs, errs
    gv = np.concatenate([out[r][0] for r in range(world)])
    eta = np.concatenate([out[r][1] for r in range(world)])
    assert rel(gv, want_gv) < 1e-12
    assert rel(eta, want_eta) < 1e-12
    assert out[0][3]["scale"] == full.window_info(0)["scale"]
    assert out[0][3]["box_w"] == full.window_info(0)["box_w"]
    for k in range(len(mus)):
        its = {out[r][2][k].iterations for r in range(world)}
        assert its == {want_cg[k].iterations}
        x = np.concatenate([out[r][2][k].x for r in range(world)])
        assert rel(x, want_cg[k].x) < 1e-10


def test_torchcomm_nccl_single_rank(golden):
    """The NCCL hook path (zero-copy CAI views, ExternalStream ordering) with a
    one-rank process group gives the unsharded result bit for bit."""
    import socket

    import torch.distributed as dist

    from paper_2407_06834_b200 import sharding as S
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}",
                            rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        full, feats, wins, f = operator("c0")
        op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA,
                               **PIN)
        S.attach(op, S.TorchComm(device=torch.device("cuda", 0)), 0, op.n)
        v = synth.random_vector(op.n)
        assert np.array_equal(op.apply(v), full.apply(v))
        r1 = nld.deflated_solve_batched(op, f[:, 0], 1.0, [0.01, 0.02],
                                        tol=synth.CG_TOL)
        r0 = nld.deflated_solve_batched(full, f[:, 0], 1.0, [0.01, 0.02],
                                        tol=synth.CG_TOL)
        for a, b in zip(r0, r1):
            assert a.iterations == b.iterations
            assert np.array_equal(a.x, b.x)
    finally:
        dist.destroy_process_group()


def test_pixel_major_layout_matches_rhs_major():
    """NLD_LAYOUT_PIXEL_MAJOR: (n, nrhs) batches give the same products."""
    from paper_2407_06834_b200 import _lib
    op, _, _, _ = operator("c1")
    rng = np.random.default_rng(21)
    V = torch.from_numpy(rng.standard_normal((5, op.n))).cuda()
    coef = np.tile([1.0, 0.003], 5)
    a = op.apply_device(V, _lib.APPLY_SYSTEM, 5, coef)
    b = op.apply_device(V.T.contiguous(), _lib.APPLY_SYSTEM, 5, coef, pixel_major=True)
    assert torch.allclose(a, b.T, rtol=1e-14, atol=0)
    g = op.apply_device(V, _lib.APPLY_GAMMA, 5)
    h = op.apply_device(V.T.contiguous(), _lib.APPLY_GAMMA, 5, pixel_major=True)
    assert torch.allclose(g, h.T, rtol=1e-14, atol=0)


def _edge_two_windows():
    """Two 3-D windows whose nodes include exact grid-line (edge) nodes:
    the golden edge set (make_golden.edge_case) and its half-scaled copy."""
    rng = np.random.default_rng(7)
    r = 0.21875
    anchors = np.array([[r, 0, 0], [-r, 0, 0], [0, 0.1, 0], [0, -0.1, 0],
                        [0, 0, 0.1], [0, 0, -0.1]])
    body = rng.uniform(-0.1, 0.1, size=(400, 3))
    on_grid = rng.integers(-6, 7, size=(60, 3)) / 64.0
    pts = np.clip(np.concatenate([anchors, body, on_grid]), -r, r)
    return np.concatenate([pts, pts * 0.5], axis=1), [np.arange(3), np.arange(3, 6)]


@pytest.mark.parametrize("nrhs", [16, 24])
@pytest.mark.parametrize("case", ["c1", "edges"])
def test_fused_gather_epilogue(case, nrhs):
    """Pixel-major batches of >= 8 rhs take the fused gather epilogue (window
    sum + degree/shift inside the last window's gather); it must equal the
    rhs-major path with its separate epilogue, for every product kind."""
    from paper_2407_06834_b200 import _lib
    if case == "c1":
        op = operator("c1")[0]
    else:
        feats, wins = _edge_two_windows()
        op = nld.AnovaOperator(feats, wins, 0.1, **PIN)
    rng = np.random.default_rng(nrhs)
    V = torch.from_numpy(rng.standard_normal((nrhs, op.n))).cuda()
    coef = np.stack([rng.uniform(0.5, 2, nrhs), rng.uniform(0, 0.01, nrhs)], 1).ravel()
    for kind in (_lib.APPLY_GAMMA, _lib.APPLY_GAMMA_SQUARED, _lib.APPLY_SYSTEM,
                 _lib.APPLY_LAPLACIAN, _lib.APPLY_WINDOW_SUM):
        c = coef if kind == _lib.APPLY_SYSTEM else None
        a = op.apply_device(V, kind, nrhs, c)
        b = op.apply_device(V.T.contiguous(), kind, nrhs, c, pixel_major=True)
        err = float((a - b.T).norm() / a.norm())
        assert err < 1e-14, (kind, err)
    if case == "edges":
        assert op.window_info(0)["n_edge"] > 0 and op.window_info(1)["n_edge"] > 0
        # not only self-consistent: the fused sliced product (edge nodes'
        # extra stencil slices included) against the CPU oracle, every column
        ref = O.AnovaOracle(feats, wins, 0.1, **PIN)
        Vh = V.cpu().numpy()
        g = op.apply_device(V.T.contiguous(), _lib.APPLY_GAMMA, nrhs, pixel_major=True)
        g = g.cpu().numpy()
        for k in range(nrhs):
            want = ref.apply(Vh[k])
            assert rel(g[:, k], want) < 1e-10, (k, rel(g[:, k], want))
        y = op.apply_device(V.T.contiguous(), _lib.APPLY_SYSTEM, nrhs, coef,
                            pixel_major=True).cpu().numpy()
        eta = ref.degree()
        for k in (0, nrhs - 1):
            lam, mu = coef[2 * k], coef[2 * k + 1]
            want = lam * Vh[k] + mu * (eta * Vh[k] - ref.apply(Vh[k]))
            assert rel(y[:, k], want) < 1e-10


# ------------------------------ integer-sliced tensor-core path (16k rhs)

def test_sliced_products_match_reference(golden):
    """Batches of 16 rhs take the tcgen05 integer-sliced spread/gather
    (nld_ozaki.cu); the golden vector rides in column 0 and must match the
    reference's own outputs at the fp64 parity bar."""
    from paper_2407_06834_b200 import _lib
    g = golden("c1")
    op = operator("c1")[0]
    v = synth.random_vector(op.n)
    rng = np.random.default_rng(16)
    V = rng.standard_normal((op.n, 16))
    V[:, 0] = v
    Vd = torch.from_numpy(V).cuda()
    gam = op.apply_device(Vd, _lib.APPLY_GAMMA, 16, pixel_major=True).cpu().numpy()
    assert rel(gam[:, 0], g["gv"]) < MATVEC_TOL
    mu = float(g["mu"])
    coef = np.tile([1.0, mu], 16)
    av = op.apply_device(Vd, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True).cpu().numpy()
    want = v + mu * (g["eta"] * v - g["gv"])
    assert rel(av[:, 0], want) < MATVEC_TOL
    # every column equals its own single-rhs (fp64 DMMA) product
    for k in (1, 7, 15):
        one = op.apply_device(torch.from_numpy(V[:, k].copy()).cuda(), _lib.APPLY_GAMMA, 1)
        assert rel(gam[:, k], one.cpu().numpy()) < 1e-12


def test_sliced_scale_extremes():
    """Per-rhs scaling of the digit slices: columns of very different
    magnitude (and an all-zero column) in one batch keep their accuracy."""
    from paper_2407_06834_b200 import _lib
    op = operator("c0")[0]
    rng = np.random.default_rng(3)
    V = rng.standard_normal((op.n, 16))
    scales = np.array([1e-200, 1e200, 0.0, 1.0, 1e-30, 1e30, 2.0 ** -600, 3.0] * 2)
    V *= scales
    gam = op.apply_device(torch.from_numpy(V).cuda(), _lib.APPLY_GAMMA, 16,
                          pixel_major=True).cpu().numpy()
    for k in range(8):
        one = op.apply_device(torch.from_numpy(V[:, k].copy()).cuda(), _lib.APPLY_GAMMA, 1)
        one = one.cpu().numpy()
        if scales[k] == 0.0:
            assert np.all(gam[:, k] == 0.0)
        else:
            # compare at unit scale (norms of 1e-200 vectors underflow)
            assert rel(gam[:, k] / scales[k], one / scales[k]) < 1e-12, (k, scales[k])


def test_sliced_alpha_sweep_matches_single_solves(golden):
    """16 alphas share every product on the sliced path; each solve matches
    the single-rhs fp64 solve (same iterations within one, 1e-9)."""
    op, _, _, f = operator("c1")
    eta = op.degree()
    alphas = synth.alpha_sweep(float(eta.mean()), 16)
    batch = nld.deflated_solve_batched(op, f[:, 0], 1.0, alphas,
                                       tol=synth.CG_TOL, maxit=200)
    for a, res in list(zip(alphas, batch))[::5]:
        single = nld.deflated_solve(nld.ShiftedSystem(op, 1.0, a), f[:, 0],
                                    tol=synth.CG_TOL, maxit=200)
        assert abs(res.iterations - single.iterations) <= 1
        assert rel(res.x, single.x) < 1e-9


def test_sharded_sliced_path_matches_single_gpu():
    """2 ranks (ThreadComm on one GPU) with 16-rhs batches: the sliced
    tcgen05 spread/gather + grid allreduce equal the unsharded products; the
    ranks' digit scales differ (local max |v|) but the fp64 results agree."""
    import threading

    from paper_2407_06834_b200 import _lib
    from paper_2407_06834_b200 import sharding as S
    full, feats, wins, f = operator("c1")
    n = feats.shape[0]
    rng = np.random.default_rng(17)
    V = rng.standard_normal((n, 16))
    V[: n // 2] *= 1e3                     # rank 0 and rank 1 see different scales
    coef = np.stack([np.ones(16), rng.uniform(0, 0.01, 16)], 1).ravel()
    want = full.apply_device(torch.from_numpy(V).cuda(), _lib.APPLY_SYSTEM, 16, coef,
                             pixel_major=True).cpu().numpy()
    world = 2
    comm = S.ThreadComm(world, device=torch.device("cuda", 0))
    out, errs = {}, []

    def rank_main(rank):
        try:
            lo, hi = S.shard_range(n, rank, world)
            op = nld.AnovaOperator(torch.from_numpy(feats[lo:hi]).cuda(), wins,
                                   synth.SIGMA, **PIN)
            S.attach(op, comm, rank, n)
            op.degree()
            y = op.apply_device(torch.from_numpy(V[lo:hi].copy()).cuda(), _lib.APPLY_SYSTEM,
                                16, coef, pixel_major=True)
            out[rank] = y.cpu().numpy()
        except Exception as exc:  # pragma: no cover - reported below
            errs.append(exc)
            comm.barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errs, errs
    got = np.concatenate([out[0], out[1]])
    assert rel(got, want) < 1e-12


def test_sharded_cell_partition_matches_single_gpu():
    """2 ranks (ThreadComm on one GPU) holding the window-0 cell-ownership
    partition (sharding.partition) instead of contiguous ranges: with the
    per-window grid allreduce on the aux stream, the 16-rhs sliced product
    and a batched deflated CG equal the unsharded operator's."""
    import threading

    from paper_2407_06834_b200 import _lib
    from paper_2407_06834_b200 import sharding as S
    full, feats, wins, f = operator("c1")
    n = feats.shape[0]
    rng = np.random.default_rng(23)
    V = rng.standard_normal((n, 16))
    coef = np.stack([np.ones(16), rng.uniform(0, 0.01, 16)], 1).ravel()
    want = full.apply_device(torch.from_numpy(V).cuda(), _lib.APPLY_SYSTEM, 16, coef,
                             pixel_major=True).cpu().numpy()
    mus = [10.0 / float(full.degree().mean()), 0.5]
    want_cg = nld.deflated_solve_batched(full, f[:, 0], 1.0, mus, tol=synth.CG_TOL, maxit=200)
    world = 2
    parts = S.partition(feats, wins, world)
    assert sorted(np.concatenate(parts).tolist()) == list(range(n))
    comm = S.ThreadComm(world, device=torch.device("cuda", 0))
    out, errs = {}, []

    def rank_main(rank):
        try:
            ix = parts[rank]
            op = nld.AnovaOperator(torch.from_numpy(feats[ix]).cuda(), wins, synth.SIGMA, **PIN)
            S.attach(op, comm, rank, n)
            op.degree()
            y = op.apply_device(torch.from_numpy(V[ix].copy()).cuda(), _lib.APPLY_SYSTEM,
                                16, coef, pixel_major=True)
            res = nld.deflated_solve_batched(op, f[ix, 0], 1.0, mus, tol=synth.CG_TOL, maxit=200)
            out[rank] = (y.cpu().numpy(), res)
        except Exception as exc:  # pragma: no cover - reported below
            errs.append(exc)
            comm.barrier.abort()

    threads = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errs, errs
    got = np.empty_like(want)
    for r in range(world):
        got[parts[r]] = out[r][0]
    assert rel(got, want) < 1e-12
    for k in range(len(mus)):
        assert {out[r][1][k].iterations for r in range(world)} == {want_cg[k].iterations}
        x = np.empty(n)
        for r in range(world):
            x[parts[r]] = out[r][1][k].x
        assert rel(x, want_cg[k].x) < 1e-10


@pytest.mark.parametrize("nrhs", [32, 48])
def test_sliced_multiple_rhs_groups(nrhs):
    """nrhs = 16k runs k rhs groups through the same sliced kernels (G digits,
    row scales and accumulators per group): every column equals its own
    single-rhs fp64 product, for each product kind."""
    from paper_2407_06834_b200 import _lib
    op = operator("c1")[0]
    rng = np.random.default_rng(nrhs)
    V = rng.standard_normal((op.n, nrhs)) * rng.uniform(0.1, 10.0, nrhs)
    coef = np.stack([rng.uniform(0.5, 2, nrhs), rng.uniform(0, 0.01, nrhs)], 1).ravel()
    Vd = torch.from_numpy(V).cuda()
    for kind in (_lib.APPLY_GAMMA, _lib.APPLY_SYSTEM):
        c = coef if kind == _lib.APPLY_SYSTEM else None
        got = op.apply_device(Vd, kind, nrhs, c, pixel_major=True).cpu().numpy()
        for k in (0, 17, nrhs - 1):
            ck = None if c is None else c[2 * k:2 * k + 2]
            one = op.apply_device(torch.from_numpy(V[:, k].copy()).cuda(), kind, 1, ck)
            assert rel(got[:, k], one.cpu().numpy()) < 1e-12, (kind, k)


@pytest.mark.parametrize("tol", [1e-12, 1e-13, 3e-14, 1e-14])
def test_true_residual_confirmation_near_roundoff(tol):
    """The explicit-residual confirmation (linops.py:218-231) rides in the
    next product's batch; near round-off the recursive residual can pass
    while the explicit one fails, and the solve must then continue exactly
    as the reference does (checked against the oracle's restatement, batched
    and single)."""
    op, _, _, f = operator("c0")
    eta = op.degree()
    mu = synth.ALPHA_SCALE / float(np.mean(eta))
    system = nld.ShiftedSystem(op, 1.0, mu)
    ref = O.AnovaOracle(*operator("c0")[1:3], synth.SIGMA, **PIN)
    u, it, conv, relres, hist = O.deflated_solve(O.SystemOracle(ref, 1.0, mu), f[:, 0],
                                                 "jacobi", tol, 80)
    res = nld.deflated_solve(system, f[:, 0], prec="jacobi", tol=tol, maxit=80)
    assert res.converged == conv
    assert abs(res.iterations - it) <= 1
    assert rel(res.x, u) < 1e-8
    batch = nld.deflated_solve_batched(op, f[:, 0], 1.0, [mu, 2 * mu, mu], prec="jacobi",
                                       tol=tol, maxit=80)
    for r in (0, 2):
        assert batch[r].iterations == res.iterations
        assert batch[r].converged == res.converged
        assert rel(batch[r].x, res.x) < 1e-12

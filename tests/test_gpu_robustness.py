"""Memory-safety and race checks of the sliced tcgen05 path without
compute-sanitizer (closed on this GPU pool):

* races: the spread, assemble and gather sum in a fixed order, so a product
  repeated many times must be bit-for-bit identical -- a lost stage release,
  a WAR hazard on a TMEM/shared-memory stage or a stale mbarrier phase shows
  up as run-to-run differences;
* uninitialised reads (initcheck): every workspace buffer is filled with NaN
  bytes (`nld_op_debug_poison`) between two products; the second must equal
  the first bit for bit, so no kernel reads workspace it did not write;
* out-of-bounds writes (memcheck): the output and input batches sit inside
  larger allocations whose guard rows hold a sentinel pattern; after the
  products the guards are untouched and the input is unchanged.

Run at config 1 (65,536 pixels: ~200 subproblems per window, partial tiles
and chunks, several items per CTA) and at config 4 for the schedule that the
benchmark times (11k subproblems per window, every CTA streaming items).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2407_06834_b200 as nld  # noqa: E402
from paper_2407_06834_b200 import _lib  # noqa: E402
import synth  # noqa: E402

PIN = dict(n_expansion=synth.N_EXPANSION, cutoff=synth.CUTOFF,
           oversampling=synth.OVERSAMPLING)
SENTINEL = -1.2345678e300


def _operator(name):
    feats, wins, _ = synth.make_problem(name)
    op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA, **PIN)
    op.degree()
    return op


def _batch(n, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.randn((n, 16), dtype=torch.float64, device="cuda", generator=g)


@pytest.mark.parametrize("name,reps", [("c1", 12), ("c4", 4)])
def test_products_bitwise_repeatable(name, reps):
    op = _operator(name)
    V = _batch(op.n, 5)
    coef = np.stack([np.ones(16), np.linspace(1e-4, 1e-2, 16)], 1).ravel()
    for kind, cf in ((_lib.APPLY_SYSTEM, coef), (_lib.APPLY_GAMMA, None)):
        first = op.apply_device(V, kind, 16, cf, pixel_major=True)
        for _ in range(reps):
            again = op.apply_device(V, kind, 16, cf, pixel_major=True)
            assert torch.equal(again, first), "run-to-run difference (race)"
        del first, again
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_poisoned_workspace_does_not_leak(name):
    op = _operator(name)
    V = _batch(op.n, 6)
    coef = np.stack([np.ones(16), np.full(16, 3e-3)], 1).ravel()
    want_sys = op.apply_device(V, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True)
    want_gam = op.apply_device(V, _lib.APPLY_GAMMA, 16, pixel_major=True)
    v1 = V[:, 0].contiguous()
    want_one = op.apply_device(v1, _lib.APPLY_GAMMA, 1)
    for kind, cf, want, vin, nr in ((_lib.APPLY_SYSTEM, coef, want_sys, V, 16),
                                    (_lib.APPLY_GAMMA, None, want_gam, V, 16),
                                    (_lib.APPLY_GAMMA, None, want_one, v1, 1)):
        op.debug_poison_workspace()
        got = op.apply_device(vin, kind, nr, cf, pixel_major=nr > 1)
        assert torch.isfinite(got).all()
        assert torch.equal(got, want), "a kernel read workspace it did not write"
    # the solver's persistent vectors too
    f = torch.from_numpy(synth.make_problem(name)[2][:, 0].copy()).cuda()
    ref = nld.deflated_solve_batched(op, f, 1.0, [0.5, 2.0], tol=1e-8, maxit=100)
    op.debug_poison_workspace()
    res = nld.deflated_solve_batched(op, f, 1.0, [0.5, 2.0], tol=1e-8, maxit=100)
    for a, b in zip(ref, res):
        assert a.iterations == b.iterations
        assert torch.equal(torch.as_tensor(a.x), torch.as_tensor(b.x))


def test_guard_rows_untouched_and_input_unchanged():
    op = _operator("c1")
    n, g = op.n, 4096
    vbuf = torch.full((n + 2 * g, 16), SENTINEL, dtype=torch.float64, device="cuda")
    obuf = torch.full((n + 2 * g, 16), SENTINEL, dtype=torch.float64, device="cuda")
    V = vbuf[g:g + n]
    V.copy_(_batch(n, 7))
    keep = V.clone()
    coef = np.stack([np.ones(16), np.full(16, 1e-3)], 1).ravel()
    for kind, cf in ((_lib.APPLY_SYSTEM, coef), (_lib.APPLY_GAMMA, None),
                     (_lib.APPLY_LAPLACIAN, None), (_lib.APPLY_WINDOW_SUM, None)):
        op.apply_device(V, kind, 16, cf, out=obuf[g:g + n], pixel_major=True)
        assert torch.equal(V, keep), "the input batch was modified"
        for buf in (vbuf, obuf):
            assert bool((buf[:g] == SENTINEL).all()) and bool((buf[g + n:] == SENTINEL).all()), \
                "a kernel wrote outside its batch"
        assert torch.isfinite(obuf[g:g + n]).all()

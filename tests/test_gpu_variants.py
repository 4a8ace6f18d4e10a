"""The fp64 DMMA alternative of the sliced path and the product build's immunity to
the A/B switches.

* ``sliced=False`` runs 16-rhs batches of 3-D m = 4 windows on the fp64 DMMA
  kernels instead of the tcgen05 integer-sliced ones.  Both must match the reference's own matvec
  (tests/golden/c1.npz, kernel.py:79-93) at the fp64 parity bar in column 0,
  and agree with each other in EVERY column (1e-12).
* The product library compiles the experiment switches (nld_switch.cuh) to
  their defaults: setting them in the environment changes nothing, bit for bit.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2407_06834_b200 as nld  # noqa: E402
from paper_2407_06834_b200 import _lib  # noqa: E402
import synth  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIN = dict(n_expansion=synth.N_EXPANSION, cutoff=synth.CUTOFF,
           oversampling=synth.OVERSAMPLING)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def batch(n):
    V = np.random.default_rng(16).standard_normal((n, 16)) * np.logspace(-3, 3, 16)
    V[:, 0] = synth.random_vector(n)
    return V


def test_dmma_alternative_matches_reference(golden):
    g = golden("c1")
    feats, wins, _ = synth.make_problem("c1")
    mu = float(g["mu"])
    coef = np.tile([1.0, mu], 16)
    out = {}
    for tables in (True, False):
        op = nld.AnovaOperator(feats, wins, synth.SIGMA, sliced=tables, **PIN)
        Vd = torch.from_numpy(batch(op.n)).cuda()
        gam = op.apply_device(Vd, _lib.APPLY_GAMMA, 16, pixel_major=True).cpu().numpy()
        av = op.apply_device(Vd, _lib.APPLY_SYSTEM, 16, coef, pixel_major=True).cpu().numpy()
        v = Vd[:, 0].cpu().numpy()
        assert rel(gam[:, 0], g["gv"]) < 1e-10, tables
        assert rel(av[:, 0], v + mu * (g["eta"] * v - g["gv"])) < 1e-10, tables
        out[tables] = (gam, av)
        op.close()
    for k in range(16):
        assert rel(out[True][0][:, k], out[False][0][:, k]) < 1e-12, k
        assert rel(out[True][1][:, k], out[False][1][:, k]) < 1e-12, k


SCRIPT = r"""
import sys
import numpy as np, torch
sys.path.insert(0, %r)
import paper_2407_06834_b200 as nld
from paper_2407_06834_b200 import _lib
import synth
feats, wins, _ = synth.make_problem("c1")
op = nld.AnovaOperator(feats, wins, synth.SIGMA, n_expansion=32, cutoff=4, oversampling=2.0)
V = np.random.default_rng(16).standard_normal((op.n, 16))
y = op.apply_device(torch.from_numpy(V).cuda(), _lib.APPLY_GAMMA, 16, pixel_major=True)
np.save(sys.argv[1], y.cpu().numpy())
"""


def test_environment_switches_have_no_effect(tmp_path):
    code = SCRIPT % REPO
    res = {}
    for tag, env in (("plain", {}),
                     ("switched", {"NLD_OZAKI": "0", "NLD_NO_MMA": "1", "NLD_NO_OVERLAP": "1",
                                   "NLD_NO_FUSED_EPILOGUE": "1", "NLD_OZAKI_NO_SPREAD": "1"})):
        path = str(tmp_path / f"{tag}.npy")
        run = subprocess.run([sys.executable, "-c", code, path], env=dict(os.environ, **env),
                             capture_output=True, text=True, timeout=600)
        assert run.returncode == 0, run.stderr[-2000:]
        res[tag] = np.load(path)
    assert np.array_equal(res["plain"], res["switched"])

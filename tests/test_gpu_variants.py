"""The sliced path's alternative kernel configurations stay correct.

The library picks its variants once per process from environment switches
(plan-time Y digits for the spread, the persistent gather and its precomputed
G digits, the fp64 DMMA kernels), so each configuration runs in its own
subprocess on the c1 problem with 16 right-hand sides and must match the
reference's own matvec (tests/golden/c1.npz) at the fp64 parity bar.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %r)
import paper_2407_06834_b200 as nld
from paper_2407_06834_b200 import _lib
import synth
g = dict(np.load(%r))
feats, wins, _ = synth.make_problem("c1")
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA,
                       n_expansion=synth.N_EXPANSION, cutoff=synth.CUTOFF,
                       oversampling=synth.OVERSAMPLING)
v = synth.random_vector(op.n)
V = np.random.default_rng(16).standard_normal((op.n, 16))
V[:, 0] = v
Vd = torch.from_numpy(V).cuda()
gam = op.apply_device(Vd, _lib.APPLY_GAMMA, 16, pixel_major=True).cpu().numpy()
mu = float(g["mu"])
av = op.apply_device(Vd, _lib.APPLY_SYSTEM, 16, np.tile([1.0, mu], 16),
                     pixel_major=True).cpu().numpy()
want = v + mu * (g["eta"] * v - g["gv"])
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print(json.dumps({"gamma": rel(gam[:, 0], g["gv"]), "system": rel(av[:, 0], want)}))
"""

VARIANTS = {
    "default": {},
    "spread_on_the_fly_y": {"NLD_SPREAD_PREY": "0"},
    "spread_per_subproblem": {"NLD_SPREAD_PERSIST": "0"},
    "gather_in_kernel_g": {"NLD_GATHER_PREG": "0"},
    "gather_per_subproblem": {"NLD_GATHER_PERSIST": "0"},
    "gather_on_the_fly_y": {"NLD_GATHER_PREY": "0"},
    "fp64_dmma": {"NLD_OZAKI": "0"},
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_matches_reference(name):
    env = dict(os.environ, **VARIANTS[name])
    code = SCRIPT % (REPO, os.path.join(REPO, "tests", "golden", "c1.npz"))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["gamma"] < 1e-10 and res["system"] < 1e-10, res

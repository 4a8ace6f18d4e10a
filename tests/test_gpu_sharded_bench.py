"""GPU: bench.py's pixel-sharded mode end to end with 2 torchrun processes.

Both ranks share cuda:0 over gloo (NLD_TEST_SHARED_GPU=1): the host blocks in
the collectives, no kernel waits on another rank.  Checks the sharded CG
reproduces the single-GPU iteration counts and the JSON contract holds.
"""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

from conftest import REPO  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(args, env_extra=None, nproc=1):
    env = dict(os.environ, **(env_extra or {}))
    cmd = [sys.executable]
    if nproc > 1:
        cmd += ["-m", "torch.distributed.run", "--nnodes=1",
                f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
                "--master-port", str(_port())]
    cmd += [os.path.join(REPO, "bench.py")] + args
    out = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_sharded_bench_matches_single_gpu():
    common = ["--config", "c1", "--nrhs", "4", "--steps", "3", "--warmup", "3",
              "--no-cpu"]
    one = _bench(common + ["--gpus", "1"])
    two = _bench(common + ["--gpus", "2"], {"NLD_TEST_SHARED_GPU": "1"}, nproc=2)
    for line in (one, two):
        for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup",
                    "ms_per_step", "higher_is_better", "scaling", "dtype",
                    "config", "roofline", "e2e", "gpu_launches", "clocks"):
            assert key in line
        assert line["cg"]["converged"]
    assert two["n_gpus"] == 2 and two["config"]["nodes_per_rank"] == 32768
    assert two["cg"]["iterations"] == one["cg"]["iterations"]
    assert abs(two["cg"]["relres_max"] / one["cg"]["relres_max"] - 1) < 1e-6

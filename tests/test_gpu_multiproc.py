"""The product's angle-sharded solve in 2 and 4 processes on one
GPU: solvers.run on each rank's mirror-closed shard with a gloo all-reduce of
the CUDA partial backprojections (tools/multiproc_check.py). x must be
bit-identical across ranks (every rank applies the same reduced bits) and
match the single-GPU solve; each rank's dual rows match the single solve's."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("world,n_angles", [(2, 180), (4, 180), (2, 90), (2, 360)])  # 360 on 2 ranks: block-cyclic shards
def test_sharded_solve_in_processes(world, n_angles):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(REPO, "tools", "multiproc_check.py"), "--n-angles", str(n_angles)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert res.returncode == 0, res.stderr[-4000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    assert out["world"] == world and out["quad_shards"] == (n_angles % 4 == 0), out
    assert out["x_identical_across_ranks"] and out["rows_identical_across_ranks"], out
    assert out["levels_match_single"], out
    assert out["rel_x_vs_single"] <= 1e-5 and out["rel_y_vs_single"] <= 1e-5, out

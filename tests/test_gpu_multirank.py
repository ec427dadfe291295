"""The N>1 bench path (bench.py under torchrun: a ring of producer->consumer
pairs, rank r storing on GPU r and fetching into GPU r+1 through its own tube)
run with 2 ranks on the one GPU of the test box (both pairs then land on the
same GPU): both ranks finish, the delivered bytes are checked inside, and
rank 0 prints one JSON line with the whole-job value."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_ring_on_one_gpu():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29547", "bench.py", "--gpus", "2", "--steps", "10",
           "--warmup", "3", "--no-extras"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 10
    assert "cross_gpu_error" not in d["config"], d["config"]

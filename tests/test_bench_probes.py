"""bench.py's child-process probes (CPU): a probe that exits 0 reports nothing, one
that fails reports why — the N>1 rank then runs as a same-GPU replica and the
headline run falls back to one PCIe link instead of dying on a peer-path fault."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import pytest  # noqa: E402


def test_child_success_and_failure():
    why, out = bench._child(["--help"], 120, "help")
    assert why is None and "--gpus" in out
    why, _ = bench._child(["--impl", "bogus"], 120, "bad flag")
    assert why.startswith("bad flag exit 2")


def test_peer_and_stripe_probes_report_a_failing_path():
    import torch
    if torch.cuda.is_available():
        pytest.skip("the probes succeed on a GPU box (the GPU bench covers that side)")
    # no GPU here: the probes' children fail, and the failure comes back as a reason
    why = bench.probe_peer_path(0, 1)
    assert why is not None and why.startswith("peer probe 0->1")
    why = bench.probe_striping()
    assert why is not None and why.startswith("striping probe")

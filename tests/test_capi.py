"""The C-ABI boundary: libfaastube.so loads without a GPU and exports every
symbol include/faastube.h declares; the ctypes table covers them all."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "faastube.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ft_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_header():
    from paper_2411_01830_b200 import _lib
    dll = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in header_symbols() if not hasattr(dll, s)]
    assert not missing, missing


def test_ctypes_table_matches_header():
    from paper_2411_01830_b200 import _lib
    assert sorted(_lib.HEADER_SYMBOLS) == header_symbols()


def test_version_and_error_plumbing():
    from paper_2411_01830_b200 import TopologyError
    from paper_2411_01830_b200._lib import LIB
    assert b"sm_100a" in LIB.ft_version()
    from paper_2411_01830_b200 import topology
    with pytest.raises(TopologyError):
        topology.from_dict({"gpu_count": 1, "nodes": [], "links": [], "pcie_groups": {}})


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2411_01830_b200 import device
    with pytest.raises(RuntimeError):
        device.require_cuda()


def test_missing_library_is_loud(tmp_path, monkeypatch):
    from paper_2411_01830_b200 import _lib
    lib = _lib._Lib()
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(_lib.LibraryMissing):
        lib.load()


def test_device_entry_points_fail_cleanly_without_a_gpu():
    """Without a GPU every device entry point returns a status (raised as an
    exception) — no crash, no CPU fallback: the pacer, raw streams/events,
    batched copies and the VMM pool."""
    import ctypes as C

    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2411_01830_b200._lib import LIB, FaasTubeError, RouteC, SegmentC
    h = C.c_void_p()
    for call in (lambda: LIB.ft_pacer_create(50.0, 1, 5, 2_000_000, 4, 0, 0, C.byref(h)),
                 lambda: LIB.ft_stream_create(0, C.byref(h)),
                 lambda: LIB.ft_event_create(0, C.byref(h)),
                 lambda: LIB.ft_vmm_pool_create(0, 1 << 30, C.byref(h)),
                 lambda: LIB.ft_copy_batch((SegmentC * 1)(SegmentC(None, None, 16)), 1, 0, None)):
        with pytest.raises((FaasTubeError, RuntimeError, ValueError)):
            call()
    # argument validation happens before any device work
    with pytest.raises(ValueError):
        LIB.ft_pacer_submit(None, b"", 1, 1e9, 0.0, 50.0, None, 0, None, 16, 1, 1, (RouteC * 1)(), None,
                            C.byref(C.c_uint64()))

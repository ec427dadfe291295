"""Alg. 1 contention-aware NVLink path selection — mirror of tubesim
``nvlink_sched.py`` over libfaastube (``ft_select_paths`` et al.).

On a B200 NVSwitch box every pair has one direct 900 GB/s path and Alg. 1
returns exactly it; the multipath machinery is kept for
non-uniform fabrics and for decision parity with the reference.
"""

from __future__ import annotations

import ctypes as C
import threading
import json
from dataclasses import dataclass, field

from ._lib import LIB, MAX_PATH, NvPathC, enc, json_out
from .topology import BandwidthMatrix, Topology

MAX_HOPS = 4
MAX_CANDIDATES = 1000


@dataclass
class NvPath:
    gpus: list
    b_min_gbps: float
    held_by: str | None = None

    @property
    def hops(self) -> int:
        return len(self.gpus) - 1


@dataclass
class PathQuery:
    func: str
    g_s: int
    g_d: int
    matrix: BandwidthMatrix
    allow_busy: bool = True
    trace: dict = field(default_factory=dict)


def candidate_paths(topo: Topology, g_s: int, g_d: int, max_hops: int = MAX_HOPS) -> list:
    """nvlink_sched.py:42-57"""
    cap = 64
    while True:
        buf = (NvPathC * cap)()
        n = C.c_int()
        rc = LIB.raw("ft_candidate_paths")(topo.handle, g_s, g_d, max_hops, buf, cap, C.byref(n))
        if rc == 9:
            cap = n.value
            continue
        if rc:
            from ._lib import raise_status
            raise_status(rc)
        return [list(buf[i].gpus[: buf[i].n]) for i in range(n.value)]


_candidate_paths = candidate_paths


_tls = threading.local()


def select_paths(query: PathQuery) -> list:
    """nvlink_sched.py:64-133"""
    cap = MAX_CANDIDATES
    bufs = getattr(_tls, "bufs", None)
    if bufs is None:
        # per-thread output buffers (1000 paths + a 64 KiB trace: allocating and
        # zeroing them on every call cost more than the selection itself)
        bufs = _tls.bufs = ((NvPathC * cap)(), C.create_string_buffer(1 << 16))
    buf, tbuf = bufs
    tcap = len(tbuf)
    n = C.c_int()
    LIB.ft_select_paths(query.matrix.handle, enc(query.func), int(query.g_s), int(query.g_d),
                        1 if query.allow_busy else 0, buf, cap, C.byref(n), tbuf, tcap)
    tr = json.loads(tbuf.value.decode())
    query.trace.clear()
    query.trace.update({"candidates_examined": tr["candidates_examined"],
                        "phase1": [(p, r) for p, r in tr["phase1"]],
                        "phase2": [(p, r) for p, r in tr["phase2"]]})
    if "shared_fallback" in tr:
        query.trace["shared_fallback"] = tr["shared_fallback"]
    return [NvPath(list(buf[i].gpus[: buf[i].n]), buf[i].b_min_gbps, query.func if buf[i].held else None)
            for i in range(n.value)]


def release_paths(matrix: BandwidthMatrix, func: str):
    """nvlink_sched.py:228-230"""
    LIB.ft_release_paths(matrix.handle, enc(func))


def claim_direct_for_workflow(matrix: BandwidthMatrix, gpu_pairs, workflow_func: str):
    """nvlink_sched.py:233-259 -> (reservations, degraded)"""
    pairs = [int(x) for p in gpu_pairs for x in p]
    arr = (C.c_int32 * max(1, len(pairs)))(*pairs)
    out = json_out("ft_claim_direct", matrix.handle, arr, len(pairs) // 2, enc(workflow_func))
    return [(tuple(e), r) for e, r in out["reservations"]], out["degraded"]


def distribute_chunks(chunk_count: int, paths: list) -> list:
    """nvlink_sched.py:288-302"""
    w = [p.b_min_gbps if isinstance(p, NvPath) else float(p) for p in paths]
    arr = (C.c_double * max(1, len(w)))(*w)
    out = (C.c_int64 * max(1, len(w)))()
    LIB.ft_distribute_chunks(int(chunk_count), arr, len(w), out)
    return list(out[: len(w)])


assert MAX_PATH >= MAX_HOPS + 1

"""TEST INFRASTRUCTURE ONLY — the reference's CPU host-memory data path.

The reference's baseline strategy ``infless_plus`` (``strategies.py:35-38``)
is host-oriented: ``store`` lands a producer's output in host shared memory
(``engine.py:361-381``) and ``fetch`` copies it out of host memory to the
consumer over the consumer's single PCIe link, in sequential stages
(``dataplane.py:190-201, 264-272``). The reference only simulates this; its
byte semantics are identity (``SPEC.md:8``). This module restates it on host
cores with numpy so that

* tests have a byte oracle (the consumer must receive exactly the producer's
  bytes, compared as uint8), and
* ``bench.py`` can time the CPU host-memory path as the reported
  ``cpu_baseline`` and as the ``--impl reference`` arm.

The copy is chunked at the reference's 2 MB transfer granularity
(``pcie_sched.py:14``) and spread over ``threads`` host threads (numpy releases
the GIL inside ``copyto``).
"""

from __future__ import annotations

import itertools
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

CHUNK = 2 * 10**6  # pcie_sched.py:14


def _copy(dst: np.ndarray, src: np.ndarray, pool: ThreadPoolExecutor | None, chunk: int = CHUNK):
    n = src.nbytes
    d = dst.reshape(-1).view(np.uint8)
    s = src.reshape(-1).view(np.uint8)
    if pool is None or n <= chunk:
        np.copyto(d, s)
        return
    # one contiguous span per worker, walked in 2 MB chunks
    spans = pool._max_workers  # noqa: SLF001 - executor sizing is ours
    per = -(-n // spans)
    per = -(-per // chunk) * chunk

    def work(lo):
        hi = min(n, lo + per)
        for a in range(lo, hi, chunk):
            b = min(hi, a + chunk)
            np.copyto(d[a:b], s[a:b])

    list(pool.map(work, range(0, n, per)))


class HostMemoryStore:
    """unique_id / store / fetch over host memory (the infless_plus path)."""

    def __init__(self, threads: int | None = None):
        self.threads = threads or len(os.sched_getaffinity(0))
        self._pool = ThreadPoolExecutor(self.threads) if self.threads > 1 else None
        self._ids = itertools.count(1)  # dataplane.py:65,69-70
        self._objs: dict[int, np.ndarray] = {}

    def unique_id(self) -> int:
        return next(self._ids)

    def store(self, data_id: int, payload: np.ndarray) -> None:
        """Producer output -> host shared memory (engine.py:361-381)."""
        if data_id in self._objs:
            raise KeyError(f"data id {data_id} already stored")  # DuplicateStore
        seg = np.empty(payload.nbytes, dtype=np.uint8)
        _copy(seg, payload, self._pool)
        self._objs[data_id] = seg

    def put_resident(self, data_id: int, seg: np.ndarray) -> None:
        """Register bytes already in host memory (a cFunc's output / request input)."""
        self._objs[data_id] = seg.reshape(-1).view(np.uint8)

    def fetch(self, data_id: int, out: np.ndarray | None = None) -> np.ndarray:
        """host shared memory -> consumer buffer (dataplane.py:190-201)."""
        seg = self._objs.get(data_id)
        if seg is None:
            raise KeyError(f"data id {data_id} not found")  # MissingData
        dst = np.empty(seg.nbytes, dtype=np.uint8) if out is None else out
        _copy(dst, seg, self._pool)
        return dst

    def drop(self, data_id: int) -> None:
        self._objs.pop(data_id, None)

    def close(self):
        if self._pool is not None:
            self._pool.shutdown()

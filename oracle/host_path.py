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


class PcieHostMemoryStore:
    """The reference's CPU host-memory path with its PCIe legs (BASELINE.md §4,
    ``infless_plus``): the bytes of a GPU producer's output go

    * ``store`` — D2H on the producer GPU's own link into a POSIX shared-memory
      segment (``engine.py:361-381``: host-oriented store -> ``fetch_plan(gpu,
      host)`` = one ``_host_gpu`` stage, ``dataplane.py:190-197``);
    * ``fetch`` — shm -> H2D on the consumer GPU's own link
      (``dataplane.py:190-197``; GPU->GPU is the two stages of
      ``dataplane.py:265-272``).

    Each stage moves through pinned staging allocated per transfer, as every
    non-scheduler strategy does (``engine.py:518-533``): ``_staging_bytes`` =
    min(size, 2 x 2 MB chunks) (``dataplane.py:199-201``), pinned with
    ``cudaHostRegister`` at the start of the stage and released at its end
    (the cold-pin cost the reference models), double buffered: one chunk on
    the link while the host copies the other in or out of the segment.
    Single link, sequential stages, no pool, no NVLink, no striping.

    Only torch's copy engine path is used (``Tensor.copy_`` between pinned and
    device memory) — none of the product's kernels or its library.
    """

    def __init__(self, device: int = 0, chunk: int = CHUNK, threads: int | None = None):
        import torch
        self.torch = torch
        self.device = device
        self.chunk = int(chunk)
        self.threads = threads or len(os.sched_getaffinity(0))
        torch.set_num_threads(self.threads)              # host memcpy of the chunks (intra-op)
        self.stream = torch.cuda.Stream(device)
        self._ids = itertools.count(1)
        self._objs = {}                                  # id -> (SharedMemory, nbytes)

    def unique_id(self) -> int:
        return next(self._ids)

    def _staging(self, nbytes):
        """min(size, 2 chunks) of host memory pinned for this transfer only."""
        torch = self.torch
        n = max(1, min(nbytes, 2 * self.chunk))
        buf = np.empty(n + 4096, dtype=np.uint8)
        off = (-buf.ctypes.data) % 4096
        buf = buf[off:off + n]
        rc = torch._C._cudart.cudaHostRegister(buf.ctypes.data, n, 0)
        if int(rc) != 0:
            raise RuntimeError(f"cudaHostRegister failed ({rc})")
        return buf, torch.from_numpy(buf)

    def _unpin(self, buf):
        self.torch._C._cudart.cudaHostUnregister(buf.ctypes.data)

    def store(self, data_id: int, t) -> None:
        """GPU tensor -> D2H (own link) -> shm segment."""
        from multiprocessing import shared_memory
        torch = self.torch
        if data_id in self._objs:
            raise KeyError(f"data id {data_id} already stored")  # DuplicateStore
        src = t.detach().reshape(-1).view(torch.uint8)
        n = src.numel()
        shm = shared_memory.SharedMemory(create=True, size=max(1, n))
        seg = torch.frombuffer(shm.buf, dtype=torch.uint8, count=n) if n else torch.empty(0, dtype=torch.uint8)
        buf, stg = self._staging(n)
        c = self.chunk
        ev = [torch.cuda.Event(), torch.cuda.Event()]
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        try:
            pend = []                                     # (event, slot view, lo, hi) on the link
            for j, lo in enumerate(range(0, n, c)):
                hi = min(n, lo + c)
                k = j % 2
                if len(pend) == 2:                        # slot k's previous chunk: host copy out
                    e, v, a, b = pend.pop(0)
                    e.synchronize()
                    seg[a:b].copy_(v)
                view = stg[k * c:k * c + (hi - lo)]
                with torch.cuda.stream(self.stream):
                    view.copy_(src[lo:hi], non_blocking=True)
                    ev[k].record(self.stream)
                pend.append((ev[k], view, lo, hi))
            for e, v, a, b in pend:
                e.synchronize()
                seg[a:b].copy_(v)
        finally:
            self._unpin(buf)
        del seg
        self._objs[data_id] = (shm, n)

    def fetch(self, data_id: int, out) -> None:
        """shm segment -> H2D (own link) -> the consumer's device buffer."""
        torch = self.torch
        ent = self._objs.get(data_id)
        if ent is None:
            raise KeyError(f"data id {data_id} not found")  # MissingData
        shm, n = ent
        seg = torch.frombuffer(shm.buf, dtype=torch.uint8, count=n) if n else torch.empty(0, dtype=torch.uint8)
        dst = out.reshape(-1).view(torch.uint8)
        buf, stg = self._staging(n)
        c = self.chunk
        ev = [torch.cuda.Event(), torch.cuda.Event()]
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        try:
            for j, lo in enumerate(range(0, n, c)):
                hi = min(n, lo + c)
                k = j % 2
                if j >= 2:
                    ev[k].synchronize()                  # the H2D that used slot k has read it
                view = stg[k * c:k * c + (hi - lo)]
                view.copy_(seg[lo:hi])
                with torch.cuda.stream(self.stream):
                    dst[lo:hi].copy_(view, non_blocking=True)
                    ev[k].record(self.stream)
            self.stream.synchronize()
        finally:
            self._unpin(buf)
        del seg
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def drop(self, data_id: int) -> None:
        ent = self._objs.pop(data_id, None)
        if ent is not None:
            ent[0].close()
            ent[0].unlink()

    def close(self):
        for did in list(self._objs):
            self.drop(did)

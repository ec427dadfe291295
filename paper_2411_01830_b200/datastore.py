"""Elastic data-store policy — mirror of tubesim ``datastore.py`` over
libfaastube (``ft_pool_policy_*``, ``ft_hist_*``, ``ft_migration_plan``).

``MemoryPool`` here is the POLICY (which size-class block to reuse, when to
grow, which idle blocks to drop); ``device.DevicePool`` binds each policy
block to real VMM-mapped HBM on a B200 and releases it when the policy drops
it.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from ._lib import LIB, destroyer, MAX_CONSUMERS, HardPressure, StoredObjectC, enc, json_out

HISTOGRAM_WINDOW = 1000          # datastore.py:17
POOL_FLOOR_BYTES = 300 * 10**6   # datastore.py:18
CAPACITY_LIMIT_BYTES = 10**9     # datastore.py:19
NATIVE_ALLOC_MS = 1.0            # datastore.py:20
MODES = {"autoscale": 0, "cache_all": 1, "none": 2}

__all__ = ["size_class", "p99", "FuncHistogram", "reservation", "pool_target", "Block", "MemoryPool",
           "StoredObject", "HardPressure", "migration_plan", "prefetch_back"]


def size_class(size_bytes: float) -> int:
    """datastore.py:24-29"""
    x = C.c_int64()
    LIB.ft_size_class(float(size_bytes), C.byref(x))
    return x.value


def p99(samples) -> float:
    """datastore.py:32-35"""
    xs = [float(s) for s in samples]
    x = C.c_double()
    LIB.ft_p99((C.c_double * max(1, len(xs)))(*xs), len(xs), C.byref(x))
    return x.value


class FuncHistogram:
    """datastore.py:38-72"""

    def __init__(self, func: str, window: int = HISTOGRAM_WINDOW):
        self.func = func
        h = C.c_void_p()
        LIB.ft_hist_create(enc(func), int(window), C.byref(h))
        self._h = h

    def __del__(self, _destroy=destroyer("ft_hist_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    def _get(self):
        a, b, c, d = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        LIB.ft_hist_get(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
        return a.value, b.value, c.value, (None if d.value != d.value else d.value)

    r_window_ms = property(lambda s: s._get()[0])
    r_size_bytes = property(lambda s: s._get()[1])
    r_con = property(lambda s: s._get()[2])
    last_request_ms = property(lambda s: s._get()[3])

    def record_execution(self, now_ms: float, size_bytes: float, concurrency: float):
        LIB.ft_hist_record(self._h, float(now_ms), float(size_bytes), float(concurrency))

    def reservation_bytes(self) -> float:
        x = C.c_double()
        LIB.ft_hist_reservation(self._h, C.byref(x))
        return x.value

    def window_active(self, now_ms: float) -> bool:
        x = C.c_int()
        LIB.ft_hist_window_active(self._h, float(now_ms), C.byref(x))
        return bool(x.value)


def reservation(hist: FuncHistogram) -> float:
    return hist.reservation_bytes()


def pool_target(histograms, now_ms: float, floor_bytes: float = POOL_FLOOR_BYTES) -> float:
    """datastore.py:79-82"""
    hs = list(histograms)
    arr = (C.c_void_p * max(1, len(hs)))(*[h._h.value for h in hs])
    x = C.c_double()
    LIB.ft_pool_target(arr, len(hs), float(now_ms), float(floor_bytes), C.byref(x))
    return x.value


@dataclass(eq=False)
class Block:
    class_bytes: int
    in_use: bool = False
    block_id: int = 0


class MemoryPool:
    """Size-class block pool policy for one GPU (datastore.py:91-166)."""

    def __init__(self, gpu: int, mode: str = "autoscale", floor_bytes: float = POOL_FLOOR_BYTES,
                 native_alloc_ms: float = NATIVE_ALLOC_MS, physical_bytes: float = 32 * 10**9):
        if mode not in MODES:
            raise ValueError(f"unknown pool mode {mode!r}")
        self.gpu, self.mode, self.floor_bytes = gpu, mode, floor_bytes
        self.native_alloc_ms, self.physical_bytes = native_alloc_ms, physical_bytes
        h = C.c_void_p()
        LIB.ft_pool_policy_create(int(gpu), MODES[mode], float(floor_bytes), float(native_alloc_ms),
                                  float(physical_bytes), C.byref(h))
        self._h = h
        self._blocks = {}
        self.histograms = {}
        self._out = (C.c_int64(), C.c_int64(), C.c_double())

    def __del__(self, _destroy=destroyer("ft_pool_policy_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    def state(self) -> dict:
        return json_out("ft_pool_policy_state_json", self._h)

    @property
    def blocks(self) -> list:
        out = []
        for cls, used, bid in self.state()["blocks"]:
            b = self._blocks.get(bid)
            if b is None:
                b = self._blocks[bid] = Block(cls, used, bid)
            b.in_use = used
            out.append(b)
        return out

    @property
    def pool_bytes(self) -> float:
        return self.state()["pool_bytes"]

    @property
    def in_use_bytes(self) -> float:
        return self.state()["in_use_bytes"]

    def hist_window(self, func: str):
        """(R_window, last_request_ms or None) of func's histogram."""
        rw, last = C.c_double(), C.c_double()
        LIB.ft_pool_policy_hist(self._h, enc(func), C.byref(rw), C.byref(last))
        return rw.value, (None if last.value != last.value else last.value)

    def histogram(self, func: str) -> "_PolicyHist":
        if func not in self.histograms:
            self.histograms[func] = _PolicyHist(self, func)
        return self.histograms[func]

    def target(self, now_ms: float) -> float:
        x = C.c_double()
        LIB.ft_pool_policy_target(self._h, float(now_ms), C.byref(x))
        return x.value

    def allocate(self, size_bytes: float):
        """-> (block, latency_ms)   datastore.py:130-144"""
        bid, cls, cost = self._out                      # reused out-params (callers serialise)
        LIB.ft_pool_policy_allocate(self._h, float(size_bytes), bid, cls, cost)
        b = self._blocks.get(bid.value)
        if b is None:
            b = self._blocks[bid.value] = Block(cls.value, True, bid.value)
        b.in_use = True
        return b, cost.value

    def free(self, block: Block):
        LIB.ft_pool_policy_free(self._h, block.block_id)
        block.in_use = False
        if self.mode == "none":
            self._blocks.pop(block.block_id, None)

    def shrink(self, now_ms: float) -> list:
        """Drops idle blocks per the policy; returns the dropped Block objects."""
        cap = 4096
        ids = (C.c_int64 * cap)()
        n = C.c_int()
        LIB.ft_pool_policy_shrink(self._h, float(now_ms), ids, cap, C.byref(n))
        return [self._blocks.pop(i, Block(0, False, i)) for i in ids[: n.value]]


class _PolicyHist:
    """FuncHistogram owned by a MemoryPool (records go to the C pool)."""

    def __init__(self, pool: MemoryPool, func: str):
        self.pool, self.func = pool, func
        self.last_request_ms = None

    def record_execution(self, now_ms: float, size_bytes: float, concurrency: float):
        LIB.ft_pool_policy_record(self.pool._h, enc(self.func), float(now_ms), float(size_bytes),
                                  float(concurrency))
        self.last_request_ms = now_ms


@dataclass
class StoredObject:
    """datastore.py:169-185"""

    data_id: int
    size_bytes: float
    producer: str
    gpu: int
    stored_at_ms: float
    location: str = "gpu"
    consumers: dict = field(default_factory=dict)
    live: bool = True
    block: Block | None = None

    def nearest_queue_pos(self):
        return min(self.consumers.values()) if self.consumers else None

    def farthest_queue_pos(self):
        return max(self.consumers.values()) if self.consumers else None


_LOC = {"gpu": 0, "host": 1, "both": 2}


def _objs(objects):
    arr = (StoredObjectC * max(1, len(objects)))()
    for i, o in enumerate(objects):
        pos = list(o.consumers.values())
        if len(pos) > MAX_CONSUMERS:
            raise ValueError(f"at most {MAX_CONSUMERS} consumers per object")
        arr[i].data_id, arr[i].size_bytes, arr[i].stored_at_ms = o.data_id, o.size_bytes, o.stored_at_ms
        arr[i].location, arr[i].live, arr[i].n_consumers = _LOC[o.location], int(o.live), len(pos)
        for j, p in enumerate(pos):
            arr[i].consumer_pos[j] = p
    return arr


def migration_plan(objects: list, pressure_bytes: float, policy: str = "queue_aware") -> list:
    """datastore.py:192-222 -> [("reclaim"|"migrate", obj)]"""
    if policy not in ("queue_aware", "lru"):
        raise ValueError(f"unknown migration policy {policy!r}")
    n = len(objects)
    acts, idx, cnt = (C.c_int32 * max(1, n))(), (C.c_int32 * max(1, n))(), C.c_int()
    LIB.ft_migration_plan(_objs(objects), n, float(pressure_bytes), 0 if policy == "queue_aware" else 1, acts,
                          idx, max(1, n), C.byref(cnt))
    return [("reclaim" if acts[i] == 0 else "migrate", objects[idx[i]]) for i in range(cnt.value)]


def prefetch_back(objects: list, free_bytes: float) -> list:
    """datastore.py:225-238"""
    n = len(objects)
    idx, cnt = (C.c_int32 * max(1, n))(), C.c_int()
    LIB.ft_prefetch_back(_objs(objects), n, float(free_bytes), idx, max(1, n), C.byref(cnt))
    return [objects[idx[i]] for i in range(cnt.value)]

"""SLO-aware PCIe bandwidth partition, batch triggering and pinned ring —
mirror of tubesim ``pcie_sched.py`` over libfaastube (``ft_partition`` et al.).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from ._lib import LIB, destroyer, InfeasibleDemand, enc

CHUNK_BYTES = 2 * 10**6      # pcie_sched.py:14
BATCH_CHUNKS = 5             # pcie_sched.py:15
PINNED_COST_MS_PER_MB = 0.7  # pcie_sched.py:16

__all__ = ["CHUNK_BYTES", "BATCH_CHUNKS", "PINNED_COST_MS_PER_MB", "InfeasibleDemand", "min_rate",
           "RateDemand", "PcieSchedulerState", "partition", "trigger_batches", "PinnedRing", "pinned_cost",
           "default_ring_capacity"]


def min_rate(data_size_bytes: float, slo_ms: float, infer_ms: float) -> float:
    """pcie_sched.py:23-33"""
    x = C.c_double()
    LIB.ft_min_rate(float(data_size_bytes), float(slo_ms), float(infer_ms), C.byref(x))
    return x.value


@dataclass
class RateDemand:
    """pcie_sched.py:36-55"""

    func: str
    data_size_bytes: float
    slo_ms: float
    infer_ms: float
    arrival_ms: float = 0.0
    rate_least_gbps: float = field(init=False)
    slo_at_risk: bool = field(default=False, init=False)

    def __post_init__(self):
        self.rate_least_gbps = min_rate(self.data_size_bytes, self.slo_ms, self.infer_ms)

    def slack_ms(self, now_ms: float) -> float:
        least, slack = C.c_double(), C.c_double()
        LIB.ft_rate_demand(float(self.data_size_bytes), float(self.slo_ms), float(self.infer_ms),
                           float(self.arrival_ms), float(now_ms), C.byref(least), C.byref(slack))
        return slack.value


class PcieSchedulerState:
    """pcie_sched.py:58-77 (demands live in the C state, insertion ordered)."""

    def __init__(self, bw_all_gbps: float, batch_chunks: int = BATCH_CHUNKS, chunk_bytes: int = CHUNK_BYTES):
        self.bw_all_gbps = float(bw_all_gbps)
        self.batch_chunks = int(batch_chunks)
        self.chunk_bytes = int(chunk_bytes)
        self.demands = {}
        h = C.c_void_p()
        LIB.ft_pcie_state_create(self.bw_all_gbps, self.batch_chunks, self.chunk_bytes, C.byref(h))
        self._h = h

    def __del__(self, _destroy=destroyer("ft_pcie_state_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    @property
    def batch_bytes(self) -> int:
        return self.batch_chunks * self.chunk_bytes

    def rate_idle_gbps(self) -> float:
        x = C.c_double()
        LIB.ft_pcie_rate_idle(self._h, C.byref(x))
        return x.value

    def add(self, demand: RateDemand):
        LIB.ft_pcie_state_add(self._h, enc(demand.func), float(demand.data_size_bytes), float(demand.slo_ms),
                              float(demand.infer_ms), float(demand.arrival_ms))
        self.demands[demand.func] = demand

    def remove(self, func: str):
        LIB.ft_pcie_state_remove(self._h, enc(func))
        self.demands.pop(func, None)


def partition(state: PcieSchedulerState, now_ms: float = 0.0) -> dict:
    """pcie_sched.py:80-104"""
    n = len(state.demands)
    if n == 0:
        return {}
    rates = (C.c_double * n)()
    risk = (C.c_int32 * n)()
    cnt = C.c_int()
    LIB.ft_partition(state._h, float(now_ms), rates, risk, n, C.byref(cnt))
    out = {}
    for i, (f, d) in enumerate(state.demands.items()):
        out[f] = rates[i]
        d.slo_at_risk = bool(risk[i])
    return out


def trigger_batches(total_bytes: float, state: PcieSchedulerState) -> list:
    """pcie_sched.py:107-119"""
    cap = 1024
    while True:
        buf = (C.c_double * cap)()
        n = C.c_int()
        rc = LIB.raw("ft_trigger_batches")(float(total_bytes), state.chunk_bytes, state.batch_chunks, buf, cap,
                                           C.byref(n))
        if rc == 9:
            cap = n.value
            continue
        if rc:
            from ._lib import raise_status
            raise_status(rc)
        return list(buf[: n.value])


class PinnedRing:
    """pcie_sched.py:122-150"""

    def __init__(self, capacity_bytes: float, cost_ms_per_mb: float = PINNED_COST_MS_PER_MB,
                 prewarmed: bool = False):
        self.capacity_bytes = capacity_bytes
        self.cost_ms_per_mb = cost_ms_per_mb
        h = C.c_void_p()
        LIB.ft_ring_create(float(capacity_bytes), float(cost_ms_per_mb), 1 if prewarmed else 0, C.byref(h))
        self._h = h

    def __del__(self, _destroy=destroyer("ft_ring_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    def _state(self):
        w, c = C.c_double(), C.c_double()
        LIB.ft_ring_state(self._h, C.byref(w), C.byref(c))
        return w.value, c.value

    @property
    def warm_bytes(self) -> float:
        return self._state()[0]

    @property
    def cold_allocated_bytes(self) -> float:
        return self._state()[1]

    def acquire(self, bytes_needed: float) -> float:
        x = C.c_double()
        LIB.ft_ring_acquire(self._h, float(bytes_needed), C.byref(x))
        return x.value


def pinned_cost(bytes_needed: float, ring: PinnedRing) -> float:
    return ring.acquire(bytes_needed)


def default_ring_capacity(pcie_link_count: int, batch_bytes: int = BATCH_CHUNKS * CHUNK_BYTES) -> int:
    """pcie_sched.py:159-162"""
    return int(LIB.ft_default_ring_capacity(int(pcie_link_count), int(batch_bytes)))

"""Data-passing strategy presets — mirror of tubesim ``strategies.py:15-62``."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

from ._lib import LIB, StrategyC, enc

STRATEGY_NAMES = ("faastube", "faastube_star", "infless_plus", "deepplan_plus")
_POOL = ("autoscale", "cache_all", "none")
_MIG = ("queue_aware", "lru", "none")


@dataclass(frozen=True)
class Strategy:
    name: str
    host_oriented: bool
    parallel_pcie: bool
    unified_interface: bool
    pcie_sched: bool
    nvlink_sched: bool
    pool: str
    migration: str

    def gpu_store(self) -> bool:
        return not self.host_oriented

    def with_toggles(self, **kwargs) -> "Strategy":
        return replace(self, **kwargs)

    def to_c(self) -> StrategyC:
        return StrategyC(int(self.host_oriented), int(self.parallel_pcie), int(self.unified_interface),
                         int(self.pcie_sched), int(self.nvlink_sched), _POOL.index(self.pool),
                         _MIG.index(self.migration))


def strategy_preset(name: str, **overrides) -> Strategy:
    """strategies.py:58-62 (preset table lives in the C library)"""
    s = StrategyC()
    LIB.ft_strategy_preset(enc(name), C.byref(s))
    strat = Strategy(name, bool(s.host_oriented), bool(s.parallel_pcie), bool(s.unified_interface),
                     bool(s.pcie_sched), bool(s.nvlink_sched), _POOL[s.pool], _MIG[s.migration])
    return strat.with_toggles(**overrides) if overrides else strat

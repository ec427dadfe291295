"""Unified data-passing interface: data index and transfer-plan dispatch —
mirror of tubesim ``dataplane.py`` over libfaastube (``ft_index_*``,
``ft_fetch_plan``, ``ft_plan_*``).

Plans carry the reference's fields (method, stages, branches, links, byte
shares, reserved rates, fill terms) and a handle to the C plan, which the
device movers in ``tube.py`` execute on real links.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field

from ._lib import LIB, destroyer, DuplicateStore, MissingData, enc, json_out
from .strategies import Strategy
from .topology import BandwidthMatrix, Topology

LOCAL_LOOKUP_MS = 0.005   # dataplane.py:20
GLOBAL_LOOKUP_MS = 0.2    # dataplane.py:21
SYNC_PERIOD_MS = 10.0     # dataplane.py:22
INTRA_GPU_MAP_MS = 0.05   # dataplane.py:23

__all__ = ["MissingData", "DuplicateStore", "Location", "DataIndexEntry", "DataIndex", "Branch", "Stage",
           "TransferPlan", "Dataplane", "plan_latency_model", "h2d", "d2h", "nv", "net"]


@dataclass(frozen=True)
class Location:
    node: int
    gpu: int | None = None

    @property
    def on_host(self) -> bool:
        return self.gpu is None


@dataclass
class DataIndexEntry:
    data_id: int
    size_bytes: float
    location: Location
    created_ms: float = 0.0
    producer: str = ""
    response: bool = False
    global_visible_ms: float = 0.0


class DataIndex:
    """Two-level mapping: per-node local tables + global table (dataplane.py:55-107)."""

    def __init__(self, sync_period_ms: float = SYNC_PERIOD_MS, local_lookup_ms: float = LOCAL_LOOKUP_MS,
                 global_lookup_ms: float = GLOBAL_LOOKUP_MS):
        self.sync_period_ms, self.local_lookup_ms, self.global_lookup_ms = (
            sync_period_ms, local_lookup_ms, global_lookup_ms)
        h = C.c_void_p()
        LIB.ft_index_create(float(sync_period_ms), float(local_lookup_ms), float(global_lookup_ms), C.byref(h))
        self._h = h
        self._meta = {}

    def __del__(self, _destroy=destroyer("ft_index_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    def unique_id(self) -> int:
        x = C.c_int64()
        LIB.ft_index_unique_id(self._h, C.byref(x))
        return x.value

    def store(self, data_id: int, location: Location, size_bytes: float, now_ms: float, producer: str,
              response: bool = False) -> DataIndexEntry:
        vis = C.c_double()
        gpu = -1 if location.gpu is None else location.gpu
        LIB.ft_index_store(self._h, int(data_id), location.node, gpu, float(size_bytes), float(now_ms),
                           enc(producer), int(bool(response)), C.byref(vis))
        e = DataIndexEntry(data_id, size_bytes, location, now_ms, producer, response, vis.value)
        self._meta[data_id] = e
        return e

    def resolve(self, data_id: int, node: int, now_ms: float):
        """-> (entry, lookup_cost_ms, ready_ms)"""
        en, eg, cost, ready, size = C.c_int(), C.c_int(), C.c_double(), C.c_double(), C.c_double()
        LIB.ft_index_resolve(self._h, int(data_id), int(node), float(now_ms), C.byref(en), C.byref(eg),
                             C.byref(cost), C.byref(ready), C.byref(size))
        e = self._meta.get(data_id) or DataIndexEntry(data_id, size.value, Location(en.value))
        e.location = Location(en.value, None if eg.value < 0 else eg.value)
        return e, cost.value, ready.value

    def drop(self, data_id: int):
        LIB.ft_index_drop(self._h, int(data_id))
        self._meta.pop(data_id, None)

    def relocate(self, data_id: int, location: Location):
        LIB.ft_index_relocate(self._h, int(data_id), location.node, -1 if location.gpu is None else location.gpu)
        if data_id in self._meta:
            self._meta[data_id].location = location


def h2d(node: int, root: int) -> tuple:
    return ("h2d", node, root)


def d2h(node: int, root: int) -> tuple:
    return ("d2h", node, root)


def nv(u: int, v: int) -> tuple:
    return ("nv", u, v)


def net(a: int, b: int) -> tuple:
    return ("net", a, b)


@dataclass
class Branch:
    links: list
    bytes_share: float
    cap_gbps: float | None = None
    reserved_gbps: float | None = None
    fill_ms: float = 0.0
    hop_caps: list = field(default_factory=list)


@dataclass
class Stage:
    branches: list
    managed: bool = False
    pinned_bytes: float = 0.0


_LINK_KINDS = ("h2d", "d2h", "nv", "nvp_out", "nvp_in", "net")   # ft_link_kind
_tls = threading.local()


class TransferPlan:
    """dataplane.py:153-160, backed by a C plan (``_h``)."""

    _METHODS = ("intra_gpu", "inter_gpu", "host_gpu", "inter_node")

    def __init__(self, handle):
        self._h = handle
        m = C.c_int()
        LIB.ft_plan_method(handle, C.byref(m), None, None)
        self.method = self._METHODS[m.value]
        self._d = None  # full plan parsed lazily (the same-GPU fast path never needs it)

    def _full(self):
        if self._d is None:
            d = json_out("ft_plan_json", self._h)
            d["stages"] = [Stage([Branch([tuple(l) for l in b["links"]], b["bytes_share"], b["cap_gbps"],
                                         b["reserved_gbps"], b["fill_ms"], b["hop_caps"]) for b in s["branches"]],
                                 s["managed"], s["pinned_bytes"]) for s in d["stages"]]
            if "_stages" in self.__dict__:
                d["stages"] = self._stages          # one set of objects per plan
            self._d = d
        return self._d

    size_bytes = property(lambda self: self._full()["size_bytes"])
    claimed_func = property(lambda self: self._full()["claimed_func"])
    note = property(lambda self: self._full()["note"])

    @property
    def stages(self) -> list:
        """Stages read through the struct accessors (ft_plan_stage/_branch): the
        request path needs only these, and a JSON round trip of the whole plan
        cost more than building it."""
        if self._d is not None:
            return self._d["stages"]
        st = self.__dict__.get("_stages")
        if st is None:
            buf = getattr(_tls, "buf", None)
            if buf is None:
                buf = _tls.buf = (C.c_double * 4096)()
            need = C.c_size_t()
            if LIB.raw("ft_plan_pack")(self._h, buf, len(buf), C.byref(need)):
                buf = (C.c_double * need.value)()
                LIB.ft_plan_pack(self._h, buf, len(buf), C.byref(need))
            v = memoryview(buf).cast("B")[:8 * need.value].cast("d").tolist()   # one C-level conversion
            st, i = [], 1
            for _ in range(int(v[0])):
                managed, pinned, nb = v[i] != 0.0, v[i + 1], int(v[i + 2])
                i += 3
                brs = []
                for _ in range(nb):
                    nl = int(v[i])
                    i += 1
                    links = []
                    for _ in range(nl):
                        k = int(v[i])
                        links.append((_LINK_KINDS[k], int(v[i + 1])) if k in (3, 4)
                                     else (_LINK_KINDS[k], int(v[i + 1]), int(v[i + 2])))
                        i += 3
                    nc = int(v[i])
                    caps = v[i + 1:i + 1 + nc]
                    i += 1 + nc
                    share, cap, res, fill = v[i:i + 4]
                    i += 4
                    brs.append(Branch(links, share, None if cap != cap else cap, None if res != res else res, fill,
                                      caps))
                st.append(Stage(brs, managed, pinned))
            self._stages = st
        return st

    def __del__(self, _destroy=destroyer("ft_plan_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    @property
    def fixed_ms(self) -> float:
        f = C.c_double()
        LIB.ft_plan_method(self._h, None, C.byref(f), None)
        return f.value

    @fixed_ms.setter
    def fixed_ms(self, value: float):
        LIB.ft_plan_add_fixed_ms(self._h, float(value) - self.fixed_ms)

    def to_dict(self) -> dict:
        return json_out("ft_plan_json", self._h)


class Dataplane:
    """Builds transfer plans (dataplane.py:163-348)."""

    def __init__(self, topo: Topology, strategy: Strategy, matrix: BandwidthMatrix, chunk_bytes: float,
                 intra_gpu_map_ms: float = INTRA_GPU_MAP_MS):
        self.topo, self.strategy, self.matrix = topo, strategy, matrix
        self.chunk_bytes, self.intra_gpu_map_ms = chunk_bytes, intra_gpu_map_ms
        s = strategy.to_c()
        h = C.c_void_p()
        LIB.ft_plane_create(topo.handle, C.byref(s), matrix.handle, float(chunk_bytes), float(intra_gpu_map_ms),
                            C.byref(h))
        self._h = h

    def __del__(self, _destroy=destroyer("ft_plane_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    def fetch_plan(self, entry_loc: Location, dest: Location, size_bytes: float) -> TransferPlan:
        """dataplane.py:176-186"""
        h = C.c_void_p()
        LIB.ft_fetch_plan(self._h, entry_loc.node, -1 if entry_loc.gpu is None else entry_loc.gpu, dest.node,
                          -1 if dest.gpu is None else dest.gpu, float(size_bytes), C.byref(h))
        return TransferPlan(h)

    def release_claim(self, plan: TransferPlan):
        """dataplane.py:346-348"""
        LIB.ft_release_claim(self._h, plan._h)


def plan_latency_model(plan: TransferPlan) -> float:
    """dataplane.py:351-369"""
    x = C.c_double()
    LIB.ft_plan_latency(plan._h, C.byref(x))
    return x.value


assert math.isfinite(INTRA_GPU_MAP_MS)

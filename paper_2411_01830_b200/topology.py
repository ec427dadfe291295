"""Topology and bandwidth matrix — host-side mirror of tubesim ``topology.py``
backed by libfaastube (``ft_topo_*`` / ``ft_matrix_*``).

Same names, argument meaning and exceptions as the reference
(``topology.py:65-449``); every query is answered by the C library.
"""

from __future__ import annotations

import ctypes as C
import json

from ._lib import LIB, destroyer, TopologyError, enc, json_out

__all__ = ["Topology", "TopologyError", "BandwidthMatrix", "build_preset", "b200_doc", "from_dict",
           "load_custom", "snapshot_matrix", "PRESET_NAMES"]

# reference calibration points (topology.py:17-22) — preset data only
NVLINK_LANE_GBPS = 24.0
PCIE_PINNED_GBPS = 12.0
NVSWITCH_PAIR_GBPS = 300.0
# B200 HGX: NVLink 5 through NVSwitch, 900 GB/s per direction per GPU
B200_NVLINK_GBPS = 900.0
PRESET_NAMES = ("dgx_v100", "dgx_a100", "quad_a10", "b200")

_CUBE_MESH = ((0, 1, 2), (0, 2, 1), (0, 3, 1), (0, 4, 2), (1, 2, 1), (1, 3, 2), (1, 5, 1), (2, 3, 2),
              (2, 6, 2), (3, 7, 1), (4, 5, 2), (4, 6, 1), (4, 7, 1), (5, 6, 1), (5, 7, 2), (6, 7, 2))


class Topology:
    """Immutable connectivity model (topology.py:65-152)."""

    def __init__(self, doc: dict):
        self._doc = json.loads(json.dumps(doc))
        h = C.c_void_p()
        LIB.ft_topo_create(enc(json.dumps(self._doc)), C.byref(h))
        self._h = h
        n = C.c_int()
        LIB.ft_topo_gpu_count(h, C.byref(n))
        self.gpu_count = n.value
        self.name = self._doc.get("name", "custom")
        self.nodes = self._doc["nodes"]
        self.pcie_groups = {int(k): list(v) for k, v in self._doc["pcie_groups"].items()}
        rates = []
        for i in range(4):
            x = C.c_double()
            LIB.ft_topo_rate(h, i, C.byref(x))
            rates.append(x.value)
        self.pcie_gbps, self.pcie_pageable_gbps, self.pcie_peer_gbps, self.network_gbps = rates

    def __del__(self, _destroy=destroyer("ft_topo_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    @property
    def handle(self):
        return self._h

    def _d(self, fn, *args):
        x = C.c_double()
        getattr(LIB, fn)(self._h, *args, C.byref(x))
        return x.value

    def _i(self, fn, *args):
        x = C.c_int()
        getattr(LIB, fn)(self._h, *args, C.byref(x))
        return x.value

    def gpus(self) -> list:
        return list(range(self.gpu_count))

    def node_of(self, gpu: int) -> int:
        return self._i("ft_topo_node_of", int(gpu))

    def pcie_root_of(self, gpu: int) -> int:
        return self._i("ft_topo_root_of", int(gpu))

    def nvlink_gbps(self, u: int, v: int) -> float:
        return self._d("ft_topo_nvlink_gbps", int(u), int(v))

    def nvlink_neighbors(self, gpu: int) -> list:
        buf = (C.c_int32 * max(1, self.gpu_count))()
        n = C.c_int()
        LIB.ft_topo_neighbors(self._h, int(gpu), buf, len(buf), C.byref(n))
        return list(buf[: n.value])

    def nvlink_pairs(self) -> dict:
        out = {}
        for u in range(self.gpu_count):
            for v in range(u + 1, self.gpu_count):
                c = self.nvlink_gbps(u, v)
                if c > 0:
                    out[(u, v)] = c
        return out

    def pair_kind(self, u: int, v: int):
        return {0: None, 1: "nvlink", 2: "nvswitch"}[self._i("ft_topo_pair_kind", int(u), int(v))]

    def switch_port_gbps(self, gpu: int) -> float:
        return self._d("ft_topo_switch_port_gbps", int(gpu))

    def nvlink_degree_gbps(self, gpu: int) -> float:
        return self._d("ft_topo_degree_gbps", int(gpu))

    def pair_bandwidth(self, u: int, v: int) -> float:
        return self._d("ft_topo_pair_bandwidth", int(u), int(v))

    def roots(self) -> list:
        buf = (C.c_int32 * 64)()
        n = C.c_int()
        LIB.ft_topo_roots(self._h, buf, 64, C.byref(n))
        return list(buf[: n.value])

    def to_dict(self) -> dict:
        return json.loads(json.dumps(self._doc))


def from_dict(doc: dict) -> Topology:
    """topology.py:327-355"""
    return Topology(doc)


def load_custom(path: str) -> Topology:
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except (OSError, json.JSONDecodeError) as exc:
        raise TopologyError(f"cannot read topology file {path}: {exc}") from exc
    return from_dict(doc)


def _single(name, n, links, groups, **rates):
    return {"name": name, "gpu_count": n, "nodes": [{"id": 0, "gpus": list(range(n))}],
            "links": links, "pcie_groups": {str(k): v for k, v in groups.items()}, "rates": rates}


def b200_doc(n_gpus: int = 8, pcie_gbps: float = 55.0, groups: dict | None = None,
             nvlink_gbps: float = B200_NVLINK_GBPS, name: str = "b200") -> dict:
    """B200 HGX box: every GPU on the NVSwitch fabric at ``nvlink_gbps`` per
    direction, one PCIe Gen5 x16 root per GPU unless ``groups`` says otherwise.
    ``pcie_gbps`` should be the MEASURED per-link pinned H2D rate."""
    groups = groups if groups is not None else {g: [g] for g in range(n_gpus)}
    links = [{"kind": "pcie", "endpoints": ["host:0", r], "bandwidth_gbps": pcie_gbps} for r in sorted(groups)]
    links += [{"kind": "nvswitch", "endpoints": [u, v], "bandwidth_gbps": nvlink_gbps}
              for u in range(n_gpus) for v in range(u + 1, n_gpus)]
    return _single(name, n_gpus, links, groups, pcie_gbps=pcie_gbps)


def build_preset(name: str, **kw) -> Topology:
    """topology.py:269-274, plus the ``b200`` preset this build targets."""
    pcie4 = [{"kind": "pcie", "endpoints": ["host:0", r], "bandwidth_gbps": PCIE_PINNED_GBPS} for r in range(4)]
    g4 = {0: [0, 1], 1: [2, 3], 2: [4, 5], 3: [6, 7]}
    if name == "dgx_v100":
        links = pcie4 + [{"kind": "nvlink", "endpoints": [u, v], "bandwidth_gbps": NVLINK_LANE_GBPS,
                          "multiplicity": m} for u, v, m in _CUBE_MESH]
        return from_dict(_single("dgx_v100", 8, links, g4))
    if name == "dgx_a100":
        links = pcie4 + [{"kind": "nvswitch", "endpoints": [u, v], "bandwidth_gbps": NVSWITCH_PAIR_GBPS}
                         for u in range(8) for v in range(u + 1, 8)]
        return from_dict(_single("dgx_a100", 8, links, g4))
    if name == "quad_a10":
        return from_dict(_single("quad_a10", 4, pcie4, {r: [r] for r in range(4)}))
    if name == "b200":
        return from_dict(b200_doc(**kw))
    raise TopologyError(f"unknown topology preset {name!r} (known: {sorted(PRESET_NAMES)})")


class BandwidthMatrix:
    """Residual directed NVLink bandwidth + per-GPU budgets (topology.py:358-443)."""

    def __init__(self, topo: Topology):
        self.topo = topo
        h = C.c_void_p()
        LIB.ft_matrix_create(topo.handle, C.byref(h))
        self._h = h

    def __del__(self, _destroy=destroyer("ft_matrix_destroy")):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            _destroy(h)

    @property
    def handle(self):
        return self._h

    def state(self) -> dict:
        return json_out("ft_matrix_state_json", self._h)

    @property
    def residual(self) -> dict:
        return {(u, v): r for u, v, r in self.state()["residual"]}

    @property
    def egress_budget(self) -> dict:
        return dict(enumerate(self.state()["egress"]))

    @property
    def ingress_budget(self) -> dict:
        return dict(enumerate(self.state()["ingress"]))

    @property
    def held(self) -> dict:
        return {f: [(p, r) for p, r in lst] for f, lst in self.state()["held"].items()}

    def edge_residual(self, u: int, v: int) -> float:
        x = C.c_double()
        LIB.ft_matrix_residual(self._h, u, v, C.byref(x))
        return x.value

    def hold(self, func: str, path: list, rate: float):
        arr = (C.c_int32 * len(path))(*path)
        LIB.ft_matrix_hold(self._h, enc(func), arr, len(path), float(rate))

    def release(self, func: str):
        LIB.ft_matrix_release(self._h, enc(func))

    def release_path(self, func: str, path: list):
        arr = (C.c_int32 * len(path))(*path)
        LIB.ft_matrix_release_path(self._h, enc(func), arr, len(path))

    def aggregate_of(self, func: str) -> float:
        x = C.c_double()
        LIB.ft_matrix_aggregate_of(self._h, enc(func), C.byref(x))
        return x.value


def snapshot_matrix(topo: Topology) -> BandwidthMatrix:
    """topology.py:446-449"""
    return BandwidthMatrix(topo)

"""Workflow inputs for the live runtime: workflow DAG documents, the seeded
arrival traces and per-request draws, placement and SLO calibration.

These restate the reference's experiment inputs (``harness.py:45-208``,
``workflow.py:24-438``) so a live run on B200 replays EXACTLY the request
trace and per-function SLOs (hence Rate_least) the simulator would use on the
same seed — checked against golden traces in ``tests/golden/harness.json``.
Workflow presets are the reference's own documents, stored as data in
``workflows.json`` (``Workflow.to_dict`` schema, ``workflow.py:139-162``).
"""

from __future__ import annotations

import json
import math
import os
import random
from dataclasses import dataclass, field

from .dataplane import Dataplane, Location, plan_latency_model
from .strategies import strategy_preset
from .topology import Topology, snapshot_matrix

MB = 10**6
BURST_FACTOR, BURST_FRACTION, PERIODIC_JITTER = 10.0, 0.05, 0.05   # harness.py:24-27
_PRESETS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "workflows.json")


# ----------------------------------------------------------------- arrivals
def gen_workload(pattern: str, mean_rate_rps: float, duration_s: float, seed: int) -> list:
    """Arrival times (ms) — same RNG stream as harness.gen_workload (harness.py:45-88)."""
    if pattern not in ("sporadic", "periodic", "bursty"):
        raise ValueError(f"unknown pattern {pattern!r}")
    if mean_rate_rps <= 0:
        raise ValueError("mean rate must be > 0")
    rng = random.Random(f"workload:{pattern}:{mean_rate_rps}:{duration_s}:{seed}")
    end = duration_s * 1000.0
    times = []
    if pattern == "periodic":
        gap = 1000.0 / mean_rate_rps
        t = gap * rng.uniform(1 - PERIODIC_JITTER, 1 + PERIODIC_JITTER)
        while t < end:
            times.append(t)
            t += gap * rng.uniform(1 - PERIODIC_JITTER, 1 + PERIODIC_JITTER)
        return times
    bursts = []
    if pattern == "bursty":
        length = min(1000.0, BURST_FRACTION * end)
        n = max(1, round(BURST_FRACTION * end / length))
        span = end / n
        for i in range(n):
            a = i * span + rng.uniform(0, max(0.0, span - length))
            bursts.append((a, a + length))
    peak = mean_rate_rps * (BURST_FACTOR if pattern == "bursty" else 1.0)
    t = 0.0
    while True:
        t += rng.expovariate(peak / 1000.0)
        if t >= end:
            return times
        rate = mean_rate_rps * BURST_FACTOR if any(a <= t < b for a, b in bursts) else mean_rate_rps
        if rng.random() <= rate / peak:
            times.append(t)


# ----------------------------------------------------------------- workflow model
@dataclass
class Size:
    const: float = 0.0
    per_object: float = 0.0
    lo: int = 1
    hi: int = 1

    @classmethod
    def parse(cls, d):
        if isinstance(d, (int, float)):
            return cls(const=float(d) * MB)
        if "per_object_mb" in d:
            lo, hi = d.get("count_range", [1, 1])
            return cls(per_object=float(d["per_object_mb"]) * MB, lo=int(lo), hi=int(hi))
        return cls(const=float(d["const_mb"]) * MB)

    def expected(self) -> float:
        return self.per_object * (self.lo + self.hi) / 2.0 if self.per_object else self.const

    def draw(self, rng) -> float:
        return self.per_object * rng.randint(self.lo, self.hi) if self.per_object else self.const


@dataclass
class Func:
    id: str
    kind: str
    compute_ms: float
    slo_ms: float | None = None
    infer_ms: float | None = None


@dataclass
class Flow:
    src: str
    dst: str
    size: Size
    p: float = 1.0


@dataclass
class Workflow:
    name: str
    funcs: list
    flows: list
    input_size: Size = field(default_factory=lambda: Size(const=MB))
    response_size: Size = field(default_factory=lambda: Size(const=MB))
    slo_ms: float | None = None

    @classmethod
    def parse(cls, doc: dict) -> "Workflow":
        funcs = []
        for f in doc["functions"]:
            c = float(f["compute_latency_ms"])
            inf = f.get("infer_latency_ms")
            funcs.append(Func(f["id"], f["kind"], c, f.get("slo_ms"), c if inf is None else inf))
        flows = [Flow(e["src"], e["dst"], Size.parse(e["size"]), float(e.get("probability", 1.0)))
                 for e in doc["edges"]]
        return cls(doc["name"], funcs, flows, Size.parse(doc.get("input_size", {"const_mb": 1})),
                   Size.parse(doc.get("response_size", {"const_mb": 1})), doc.get("slo_ms"))

    def func(self, fid) -> Func:
        return next(f for f in self.funcs if f.id == fid)

    def gfuncs(self):
        return [f.id for f in self.funcs if f.kind == "gFunc"]

    def entries(self):
        dsts = {e.dst for e in self.flows}
        return [f.id for f in self.funcs if f.id not in dsts]

    def sinks(self):
        srcs = {e.src for e in self.flows}
        return [f.id for f in self.funcs if f.id not in srcs]

    def ins(self, fid):
        return [e for e in self.flows if e.dst == fid]

    def outs(self, fid):
        return [e for e in self.flows if e.src == fid]

    def order(self):
        """Kahn order, ties by name (workflow.py:122-137)."""
        deg = {f.id: 0 for f in self.funcs}
        for e in self.flows:
            deg[e.dst] += 1
        ready = sorted(k for k, v in deg.items() if v == 0)
        out = []
        while ready:
            k = ready.pop(0)
            out.append(k)
            for e in self.outs(k):
                deg[e.dst] -= 1
                if deg[e.dst] == 0:
                    ready.append(e.dst)
            ready.sort()
        if len(out) != len(self.funcs):
            raise ValueError(f"{self.name}: cycle")
        return out


def preset_workflow(name: str) -> Workflow:
    with open(_PRESETS) as fh:
        docs = json.load(fh)
    if name not in docs:
        raise ValueError(f"unknown workflow preset {name!r} (known: {sorted(docs)})")
    return Workflow.parse(docs[name])


@dataclass
class Request:
    rid: int
    workflow: str
    arrival_ms: float
    edge_bytes: dict
    fired: set
    input_bytes: float
    response_bytes: float


def build_requests(wf: Workflow, arrivals: list, seed: int, rid_start: int = 0) -> list:
    """Pre-drawn branch firing and payload sizes (harness.py:130-149)."""
    rng = random.Random(f"requests:{wf.name}:{seed}")
    out = []
    for i, t in enumerate(arrivals):
        fired, sizes = set(), {}
        for e in wf.flows:
            hit = e.p >= 1.0 or rng.random() < e.p
            n = e.size.draw(rng)
            if hit:
                fired.add((e.src, e.dst))
                sizes[(e.src, e.dst)] = n
        out.append(Request(rid_start + i, wf.name, t, sizes, fired, wf.input_size.draw(rng),
                           wf.response_size.draw(rng)))
    return out


# ----------------------------------------------------------------- placement + SLOs
def place(wf: Workflow, topo: Topology, occupancy: dict | None = None, limit: int = 1,
          colocate: bool = False) -> dict:
    """Greedy NVLink-aware placement (workflow.py:375-438): heaviest gFunc edges
    onto the best free pair, leftovers onto the GPUs with the most NVLink.

    The reference gives every gFunc of a workflow its own GPU, so it cannot
    place a multi-gFunc workflow on a box with fewer GPUs. ``colocate=True``
    (used when the box is smaller, e.g. one B200) shares GPUs round-robin
    instead — same-GPU edges then take the zero-copy intra-GPU method."""
    if colocate:
        gpus = topo.gpus()
        where = {fid: ("gpu", gpus[i % len(gpus)]) for i, fid in enumerate(wf.gfuncs())}
        home = topo.node_of(gpus[0])
        where.update({f.id: ("host", home) for f in wf.funcs if f.kind == "cFunc"})
        return where
    occ = dict(occupancy or {})
    free = [g for g in topo.gpus() if occ.get(g, 0) < limit]
    if len(wf.gfuncs()) > len(free):
        raise RuntimeError(f"{wf.name}: {len(wf.gfuncs())} gFuncs but only {len(free)} free GPUs")
    where = {}

    def take(g, fid):
        where[fid] = ("gpu", g)
        free.remove(g)

    heavy = [e for e in wf.flows if wf.func(e.src).kind == "gFunc" and wf.func(e.dst).kind == "gFunc"]
    heavy.sort(key=lambda e: (-e.size.expected() * e.p, e.src, e.dst))
    for e in heavy:
        a, b = e.src in where, e.dst in where
        if a and b:
            continue
        if not a and not b:
            best = None
            for u in free:
                for v in free:
                    if u != v:
                        bw = topo.pair_bandwidth(u, v)
                        if best is None or bw > best[0] + 1e-12:
                            best = (bw, u, v)
            if best is None:
                raise RuntimeError(f"{wf.name}: no free GPU pair for {e.src}->{e.dst}")
            take(best[1], e.src)
            take(best[2], e.dst)
        else:
            anchor = where[e.src][1] if a else where[e.dst][1]
            todo = e.dst if a else e.src
            best = None
            for g in free:
                bw = topo.pair_bandwidth(anchor, g)
                if best is None or bw > best[0] + 1e-12:
                    best = (bw, g)
            if best is None:
                raise RuntimeError(f"{wf.name}: no free GPU for {todo}")
            take(best[1], todo)
    for fid in wf.gfuncs():
        if fid not in where:
            take(max(free, key=lambda g: (topo.nvlink_degree_gbps(g), -g)), fid)
    nodes = sorted(topo.node_of(w[1]) for w in where.values() if w[0] == "gpu")
    home = max(set(nodes), key=lambda n: (nodes.count(n), -n)) if nodes else 0
    for f in wf.funcs:
        if f.kind == "cFunc":
            where[f.id] = ("host", home)
    return where


def _loc(topo, where, fid) -> Location:
    kind, w = where[fid]
    return Location(topo.node_of(w), w) if kind == "gpu" else Location(w, None)


def unloaded_runtime_ms(wf: Workflow, topo: Topology, where: dict, chunk: float = 2 * MB,
                        map_ms: float = 0.05) -> float:
    """Critical path of one request on an idle box under the faastube model (harness.py:154-195)."""
    plane = Dataplane(topo, strategy_preset("faastube"), snapshot_matrix(topo), chunk, map_ms)

    def xfer(a, b, n):
        p = plane.fetch_plan(a, b, n)
        t = plan_latency_model(p)
        plane.release_claim(p)
        return t

    done = {}
    for fid in wf.order():
        here = _loc(topo, where, fid)
        ins = wf.ins(fid)
        if not ins:
            ready = 0.0 if here.on_host else xfer(Location(here.node, None), here, wf.input_size.expected())
        else:
            ready = max(done[e.src] + xfer(_loc(topo, where, e.src), here, e.size.expected()) for e in ins)
        done[fid] = ready + wf.func(fid).compute_ms
    finish = 0.0
    for fid in wf.sinks():
        here = _loc(topo, where, fid)
        resp = 0.0 if here.on_host else xfer(here, Location(here.node, None), wf.response_size.expected())
        finish = max(finish, done[fid] + resp)
    return finish


def calibrate_slo(wf: Workflow, topo: Topology, where: dict, scale: float = 1.5, chunk: float = 2 * MB) -> float:
    """Workflow SLO = scale x unloaded runtime, split over functions by compute (harness.py:198-208)."""
    runtime = unloaded_runtime_ms(wf, topo, where, chunk)
    wf.slo_ms = scale * runtime
    total = sum(f.compute_ms for f in wf.funcs) or 1.0
    for f in wf.funcs:
        f.slo_ms = wf.slo_ms * f.compute_ms / total
        f.infer_ms = f.compute_ms
    return runtime


assert math.isfinite(BURST_FACTOR)

"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's decision
functions on the data-passing path (see ``oracle/__init__.py``).

Every function cites the reference ``file:line`` it restates; paths are
relative to ``/root/reference/pkg/src/tubesim/``. Arithmetic is Python float
(IEEE binary64) with the reference's summation order, tie-breaks and
epsilons, so results are bit-identical to the reference on the same inputs.
Units: GB/s = 1e9 B/s, bytes, milliseconds (``topology.py:3-5``).
"""

from __future__ import annotations

import itertools
import math
from collections import deque

# ----------------------------------------------------------------------------
# constants (topology.py:17-22, pcie_sched.py:14-16, datastore.py:17-21,
# dataplane.py:20-23, nvlink_sched.py:17-18)
# ----------------------------------------------------------------------------
LANE_GBPS = 24.0
PCIE_GBPS = 12.0
PAGEABLE_GBPS = 3.0
PEER_GBPS = 7.9
SWITCH_PAIR_GBPS = 300.0
NET_GBPS = 10.0

CHUNK = 2 * 10**6
BATCH = 5
PIN_MS_PER_MB = 0.7

HIST_WINDOW = 1000
FLOOR = 300 * 10**6
STORE_CAP = 10**9
ALLOC_MS = 1.0
CLASS = 2 * 10**6

LOOKUP_LOCAL_MS = 0.005
LOOKUP_GLOBAL_MS = 0.2
SYNC_MS = 10.0
MAP_MS = 0.05

HOP_LIMIT = 4
CANDIDATE_LIMIT = 1000


class OracleError(Exception):
    """Base; ``kind`` names the reference exception it stands for."""

    kind = "error"


class TopoErr(OracleError):
    kind = "TopologyError"


class Infeasible(OracleError):
    kind = "InfeasibleDemand"


class Missing(OracleError):
    kind = "MissingData"


class Duplicate(OracleError):
    kind = "DuplicateStore"


class Pressure(OracleError):
    kind = "HardPressure"


class PoolFull(OracleError):
    kind = "MemoryError"


# ----------------------------------------------------------------------------
# topology (topology.py:65-152, 327-355)
# ----------------------------------------------------------------------------
class Fabric:
    """Restates ``Topology`` built from a JSON document (``from_dict``)."""

    def __init__(self, doc: dict):
        try:
            rates = doc.get("rates", {})
            self.name = doc.get("name", "custom")
            self.gpu_count = int(doc["gpu_count"])
            self.nodes = doc["nodes"]
            self.links = []
            for ent in doc["links"]:
                bw = float(ent["bandwidth_gbps"])
                mult = int(ent.get("multiplicity", 1))
                if bw <= 0 or mult < 1:
                    raise TopoErr(f"bad link {ent}")
                self.links.append((ent["kind"], tuple(ent["endpoints"]), bw, mult))
            self.groups = {int(k): list(v) for k, v in doc["pcie_groups"].items()}
            self.pcie = float(rates.get("pcie_gbps", PCIE_GBPS))
            self.pageable = float(rates.get("pcie_pageable_gbps", PAGEABLE_GBPS))
            self.peer = float(rates.get("pcie_peer_gbps", PEER_GBPS))
            self.net = float(rates.get("network_gbps", NET_GBPS))
        except (KeyError, TypeError, ValueError) as exc:
            raise TopoErr(f"malformed topology document: {exc}") from exc
        # per unordered pair: summed capacity and kind (last link wins kind)
        self.cap = {}
        self.kinds = {}
        for kind, ends, bw, mult in self.links:
            if kind in ("nvlink", "nvswitch"):
                a, b = ends
                key = (min(a, b), max(a, b))
                self.cap[key] = self.cap.get(key, 0.0) + bw * mult
                self.kinds[key] = kind
        self.node = {}
        for nd in self.nodes:
            for g in nd["gpus"]:
                self.node[g] = nd["id"]
        self.root = {}
        for r, gs in self.groups.items():
            for g in gs:
                self.root[g] = r
        bad = self.problems()
        if bad:
            raise TopoErr(f"invalid topology: {bad}")

    def problems(self):  # topology.py:160-185
        out = []
        seen = {}
        for nd in self.nodes:
            for g in nd["gpus"]:
                if g in seen:
                    out.append(f"gpu {g} assigned to nodes {seen[g]} and {nd['id']}")
                seen[g] = nd["id"]
        out += [f"gpu {g} belongs to no node" for g in range(self.gpu_count) if g not in seen]
        seen_r = {}
        for r, gs in self.groups.items():
            for g in gs:
                if g in seen_r:
                    out.append(f"gpu {g} in PCIe groups {seen_r[g]} and {r}")
                seen_r[g] = r
        out += [f"gpu {g} has no PCIe group" for g in range(self.gpu_count) if g not in seen_r]
        for _, ends, _, _ in self.links:
            for e in ends:
                if isinstance(e, int) and e not in seen:
                    out.append(f"link {ends} references unknown gpu {e}")
        return out

    def check(self, g):  # topology.py:154-156
        if not isinstance(g, int) or isinstance(g, bool) or g not in self.node:
            raise TopoErr(f"unknown GPU id {g!r}")

    def gpus(self):
        return list(range(self.gpu_count))

    def node_of(self, g):
        self.check(g)
        return self.node[g]

    def root_of(self, g):
        self.check(g)
        return self.root[g]

    def nv(self, u, v):  # topology.py:110-114
        self.check(u)
        self.check(v)
        return self.cap.get((min(u, v), max(u, v)), 0.0)

    def neighbors(self, g):  # topology.py:116-119
        self.check(g)
        return sorted(b if a == g else a for (a, b) in self.cap if g in (a, b))

    def kind(self, u, v):
        return self.kinds.get((min(u, v), max(u, v)))

    def port(self, g):  # topology.py:127-132
        caps = [c for (a, b), c in self.cap.items()
                if g in (a, b) and self.kinds[(a, b)] == "nvswitch"]
        return max(caps) if caps else 0.0

    def degree(self, g):  # topology.py:134-140
        p = self.port(g)
        if p > 0:
            return p
        return sum(c for (a, b), c in self.cap.items() if g in (a, b))

    def pair_bw(self, u, v):  # topology.py:142-152
        if u == v:
            raise TopoErr("pair_bandwidth needs two distinct GPUs")
        c = self.nv(u, v)
        if c > 0:
            return c
        if self.node_of(u) != self.node_of(v):
            return self.net
        return self.peer


def fabric_doc_switch(n_gpus=8, pair_gbps=900.0, groups=None, pcie_gbps=55.0, name="b200"):
    """JSON document of an NVSwitch box (same schema as ``topology.py:327-355``)."""
    groups = groups if groups is not None else {r: [r] for r in range(n_gpus)}
    links = [{"kind": "pcie", "endpoints": ["host:0", r], "bandwidth_gbps": pcie_gbps}
             for r in sorted(groups)]
    links += [{"kind": "nvswitch", "endpoints": [u, v], "bandwidth_gbps": pair_gbps}
              for u in range(n_gpus) for v in range(u + 1, n_gpus)]
    return {"name": name, "gpu_count": n_gpus,
            "nodes": [{"id": 0, "gpus": list(range(n_gpus))}],
            "links": links,
            "pcie_groups": {str(k): list(v) for k, v in groups.items()},
            "rates": {"pcie_gbps": pcie_gbps}}


# ----------------------------------------------------------------------------
# bandwidth matrix (topology.py:358-443)
# ----------------------------------------------------------------------------
class Residuals:
    def __init__(self, fab: Fabric):
        self.fab = fab
        self.capacity = {}
        self.residual = {}
        for (u, v), c in fab.cap.items():
            for e in ((u, v), (v, u)):
                self.capacity[e] = c
                self.residual[e] = c
        budget = {g: fab.degree(g) for g in fab.gpus()}
        self.egress = dict(budget)
        self.ingress = dict(budget)
        self.owners = {e: [] for e in self.residual}
        self.held = {}

    def res(self, u, v):
        return self.residual.get((u, v), 0.0)

    def idle(self, u, v):
        e = (u, v)
        return e in self.residual and self.residual[e] == self.capacity[e]

    def hold(self, func, path, rate):  # topology.py:390-401
        edges = list(zip(path, path[1:]))
        for e in edges:
            if self.residual.get(e, 0.0) + 1e-12 < rate:
                raise TopoErr(f"hold over capacity on edge {e}")
        for e in edges:
            self.residual[e] -= rate
            self.owners[e].append(func)
        self.egress[path[0]] -= rate
        self.ingress[path[-1]] -= rate
        self.held.setdefault(func, []).append((list(path), rate))

    def _give_back(self, func, path, rate):
        for e in zip(path, path[1:]):
            self.residual[e] += rate
            self.owners[e].remove(func)
        self.egress[path[0]] += rate
        self.ingress[path[-1]] += rate

    def release(self, func):  # topology.py:403-412
        if func not in self.held:
            raise TopoErr(f"release without claim for {func!r}")
        for path, rate in self.held.pop(func):
            self._give_back(func, path, rate)

    def release_path(self, func, path):  # topology.py:414-428
        lst = self.held.get(func, [])
        for i, (p, rate) in enumerate(lst):
            if p == path:
                lst.pop(i)
                self._give_back(func, path, rate)
                if not lst:
                    del self.held[func]
                return
        raise TopoErr(f"{func!r} does not hold path {path}")

    def holders(self, u, v):
        return list(self.owners.get((u, v), []))

    def aggregate(self, func):
        return sum(r for _, r in self.held.get(func, []))

    def consistent(self):  # topology.py:436-443
        return [e for e, c in self.capacity.items()
                if self.residual[e] < -1e-9 or self.residual[e] > c + 1e-9]


# ----------------------------------------------------------------------------
# Alg. 1 path selection (nvlink_sched.py:42-302)
# ----------------------------------------------------------------------------
def candidates(fab: Fabric, src, dst, max_hops=HOP_LIMIT):  # nvlink_sched.py:42-57
    found = []
    todo = [(src, [src])]
    while todo:
        at, walk = todo.pop()
        for nxt in reversed(fab.neighbors(at)):
            if nxt in walk:
                continue
            if nxt == dst:
                found.append(walk + [nxt])
            elif len(walk) <= max_hops - 1:
                todo.append((nxt, walk + [nxt]))
    found.sort(key=lambda p: (len(p), p))
    return found


def bottleneck(mx: Residuals, path):  # nvlink_sched.py:60-61
    return min(mx.res(u, v) for u, v in zip(path, path[1:]))


def _grant(mx, src, dst, b):  # nvlink_sched.py:136-139
    return min(b, mx.egress[src], mx.ingress[dst])


def select(mx: Residuals, func, src, dst, allow_busy=True, trace=None):
    """nvlink_sched.py:64-133. Returns [(gpus, b_min, held: bool)]."""
    fab = mx.fab
    if src == dst:
        raise TopoErr("select_paths needs two distinct GPUs")
    fab.check(src)
    fab.check(dst)
    cands = candidates(fab, src, dst)
    tr = trace if trace is not None else {}
    tr["candidates_examined"] = len(cands)
    tr["phase1"] = []
    tr["phase2"] = []
    if len(cands) > CANDIDATE_LIMIT:
        raise TopoErr("path search exceeded its candidate bound")
    if not cands:
        return []
    picked = []

    def open_budgets():
        return mx.egress[src] > 1e-9 and mx.ingress[dst] > 1e-9

    while open_budgets():
        free = [p for p in cands if all(mx.idle(u, v) for u, v in zip(p, p[1:]))]
        if not free:
            break
        free.sort(key=lambda p: (len(p), -bottleneck(mx, p), p))
        best = free[0]
        rate = _grant(mx, src, dst, bottleneck(mx, best))
        if rate <= 1e-9:
            break
        mx.hold(func, best, rate)
        picked.append((best, rate, True))
        tr["phase1"].append((list(best), rate))

    if open_budgets() and allow_busy:
        for p in cands:
            if not open_budgets():
                break
            if any(q[0] == p for q in picked):
                continue
            got = _adopt(mx, func, src, dst, p)
            if got is not None:
                picked.append(got)
                tr["phase2"].append((list(got[0]), got[1]))

    if not picked:
        best = max(cands, key=lambda p: (min(fab.nv(u, v) for u, v in zip(p, p[1:])), -len(p)))
        cap = min(fab.nv(u, v) for u, v in zip(best, best[1:]))
        picked.append((best, cap, False))
        tr["shared_fallback"] = list(best)
    return picked


def _adopt(mx, func, src, dst, path):  # nvlink_sched.py:142-170
    edges = list(zip(path, path[1:]))
    busy = [e for e in edges if not mx.idle(*e)]
    if not busy:
        return None
    owners = sorted({f for e in busy for f in mx.holders(*e)})
    if not owners or func in owners or len(owners) > 1:
        return None
    other = owners[0]
    theirs = [(list(p), r) for p, r in mx.held.get(other, [])
              if any(tuple(e) in list(zip(p, p[1:])) for e in busy)]
    if not theirs:
        return None
    if _move_holder(mx, other, theirs, busy):
        rate = _grant(mx, src, dst, bottleneck(mx, path))
        if rate > 1e-9:
            mx.hold(func, path, rate)
            return (path, rate, True)
        return None
    return _halve(mx, func, src, dst, path, other, theirs)


def _move_holder(mx, other, theirs, forbidden):  # nvlink_sched.py:173-201
    fab = mx.fab
    before = sum(r for _, r in theirs)
    for p, _ in theirs:
        mx.release_path(other, p)
    placed = []
    total = 0.0
    a, b = theirs[0][0][0], theirs[0][0][-1]
    for c in candidates(fab, a, b):
        if any((u, v) in forbidden or (v, u) in forbidden for u, v in zip(c, c[1:])):
            continue
        if not all(mx.idle(u, v) for u, v in zip(c, c[1:])):
            continue
        r = bottleneck(mx, c)
        if r <= 1e-9:
            continue
        mx.hold(other, c, r)
        placed.append((c, r))
        total += r
        if total >= before - 1e-9:
            break
    if total >= before - 1e-9:
        return True
    for p, _ in placed:
        mx.release_path(other, p)
    for p, r in theirs:
        mx.hold(other, p, r)
    return False


def _halve(mx, func, src, dst, path, other, theirs):  # nvlink_sched.py:204-225
    fab = mx.fab
    mine_direct = fab.nv(src, dst)
    their_direct = fab.nv(theirs[0][0][0], theirs[0][0][-1])
    after = mx.aggregate(other) - sum(r / 2 for _, r in theirs)
    if after + 1e-9 < their_direct:
        return None
    freed = min(r / 2 for _, r in theirs)
    gain = _grant(mx, src, dst, freed)
    now_mine = sum(r for _, r in mx.held.get(func, []))
    if now_mine + gain + 1e-9 < mine_direct:
        return None
    if gain <= 1e-9:
        return None
    for p, r in theirs:
        mx.release_path(other, p)
        mx.hold(other, p, r / 2)
    mx.hold(func, path, gain)
    return (path, gain, True)


def claim_direct(mx, pairs, wf_func):  # nvlink_sched.py:233-259
    booked = []
    hurt = {}
    for a, b in pairs:
        if mx.fab.nv(a, b) <= 0:
            continue
        for u, v in ((a, b), (b, a)):
            for f in list(mx.holders(u, v)):
                if f == wf_func:
                    continue
                hurt.setdefault(f, 0.0)
                hurt[f] += _evict(mx, f, (u, v))
        r = min(mx.res(a, b), mx.res(b, a))
        if r > 1e-9:
            mx.hold(wf_func, [a, b], r)
            mx.hold(wf_func, [b, a], r)
            booked.append(((a, b), r))
    return booked, {f: x for f, x in hurt.items() if x > 1e-9}


def _evict(mx, func, edge):  # nvlink_sched.py:262-285
    victims = [(list(p), r) for p, r in mx.held.get(func, []) if edge in list(zip(p, p[1:]))]
    lost = 0.0
    for p, r in victims:
        mx.release_path(func, p)
        got = 0.0
        for c in candidates(mx.fab, p[0], p[-1]):
            if edge in list(zip(c, c[1:])):
                continue
            if not all(mx.idle(u, v) for u, v in zip(c, c[1:])):
                continue
            x = min(bottleneck(mx, c), r - got)
            if x <= 1e-9:
                continue
            mx.hold(func, c, x)
            got += x
            if got >= r - 1e-9:
                break
        lost += max(0.0, r - got)
    return lost


def split_chunks(n, weights):  # nvlink_sched.py:288-302
    if not weights:
        raise ValueError("distribute_chunks needs at least one path")
    tot = sum(weights)
    if tot <= 0:
        raise ValueError("paths carry no bandwidth")
    raw = [n * w / tot for w in weights]
    cnt = [int(x) for x in raw]
    short = n - sum(cnt)
    for i in sorted(range(len(weights)), key=lambda i: (-(raw[i] - cnt[i]), i))[:short]:
        cnt[i] += 1
    return cnt


# ----------------------------------------------------------------------------
# PCIe policy (pcie_sched.py:23-162)
# ----------------------------------------------------------------------------
def least_rate(nbytes, slo, infer):  # pcie_sched.py:23-33
    if nbytes < 0:
        raise ValueError("data size must be >= 0")
    if nbytes == 0:
        return 0.0
    w = slo - infer
    if w <= 0:
        raise Infeasible(f"slo {slo} <= infer {infer}")
    return nbytes / (w * 1e6)


class Demand:  # pcie_sched.py:36-55
    def __init__(self, func, nbytes, slo, infer, arrival=0.0):
        self.func, self.nbytes, self.slo, self.infer, self.arrival = func, nbytes, slo, infer, arrival
        self.least = least_rate(nbytes, slo, infer)
        self.at_risk = False

    def slack(self, now):
        deadline = self.arrival + self.slo - self.infer
        if self.least <= 0:
            return deadline - now
        return (deadline - now) - self.nbytes / (self.least * 1e6)


class LinkShare:  # pcie_sched.py:58-77
    def __init__(self, bw_all, batch_chunks=BATCH, chunk=CHUNK):
        self.bw_all, self.batch_chunks, self.chunk = bw_all, batch_chunks, chunk
        self.demands = {}

    @property
    def batch_bytes(self):
        return self.batch_chunks * self.chunk

    def idle(self):
        return max(0.0, self.bw_all - sum(d.least for d in self.demands.values()))


def split_rates(st: LinkShare, now=0.0):  # pcie_sched.py:80-104
    ds = list(st.demands.values())
    if not ds:
        return {}
    least = {d.func: d.least for d in ds}
    tot = sum(least.values())
    if tot > st.bw_all:
        k = st.bw_all / tot
        out = {}
        for d in ds:
            d.at_risk = True
            out[d.func] = least[d.func] * k
        return out
    for d in ds:
        d.at_risk = False
    out = dict(least)
    spare = st.bw_all - tot
    if spare > 0:
        t = min(ds, key=lambda d: (d.slack(now), d.arrival, d.func))
        out[t.func] += spare
    return out


def batches(total, st: LinkShare):  # pcie_sched.py:107-119
    if total <= 0:
        return []
    n = max(1, math.ceil(total / st.chunk))
    out = []
    left = total
    for _ in range(math.ceil(n / st.batch_chunks)):
        x = min(left, st.batch_bytes)
        out.append(x)
        left -= x
    return out


class Ring:  # pcie_sched.py:122-150
    def __init__(self, capacity, ms_per_mb=PIN_MS_PER_MB, prewarmed=False):
        self.capacity, self.ms_per_mb = capacity, ms_per_mb
        self.warm = capacity if prewarmed else 0.0
        self.cold = 0.0

    def acquire(self, need):
        if need < 0:
            raise ValueError("bytes must be >= 0")
        usable = min(need, self.capacity)
        short = max(0.0, usable - self.warm) + max(0.0, need - self.capacity)
        if usable > self.warm:
            self.warm = usable
        if short > 0:
            self.cold += short
            return self.ms_per_mb * short / 1e6
        return 0.0


def ring_capacity(links, batch_bytes=BATCH * CHUNK):  # pcie_sched.py:159-162
    return 2 * batch_bytes * links


# ----------------------------------------------------------------------------
# latency model and percentile (simcore.py:21-50, 247-252)
# ----------------------------------------------------------------------------
def ms_for(nbytes, gbps):
    return nbytes / (gbps * 1e6)


def pipe_latency(size, hops, chunk):  # simcore.py:25-42
    if not hops:
        raise ValueError("pipeline_latency needs at least one hop")
    if any(b <= 0 for b in hops):
        raise ValueError("hop bandwidths must be > 0")
    if chunk <= 0 or chunk > size:
        chunk = size
    slow = min(range(len(hops)), key=lambda i: hops[i])
    t = ms_for(size, hops[slow])
    for i, b in enumerate(hops):
        if i != slow:
            t += ms_for(chunk, b)
    return t


def pipe_fill(hops, chunk):  # simcore.py:45-50
    if len(hops) <= 1:
        return 0.0
    slow = min(range(len(hops)), key=lambda i: hops[i])
    return sum(ms_for(chunk, b) for i, b in enumerate(hops) if i != slow)


def rank_pct(sorted_vals, pct):  # simcore.py:247-252
    if not sorted_vals:
        raise ValueError("empty sample")
    return sorted_vals[max(1, math.ceil(pct / 100.0 * len(sorted_vals))) - 1]


# ----------------------------------------------------------------------------
# elastic store policy (datastore.py:24-238)
# ----------------------------------------------------------------------------
def block_class(nbytes):  # datastore.py:24-29
    if nbytes <= 0:
        raise ValueError("allocation size must be > 0")
    return CLASS * max(1, math.ceil(nbytes / CLASS))


def p99(xs):  # datastore.py:32-35
    v = sorted(xs)
    return v[max(1, math.ceil(0.99 * len(v))) - 1]


class Hist:  # datastore.py:38-72
    def __init__(self, func, window=HIST_WINDOW):
        self.func = func
        self.gaps = deque(maxlen=window)
        self.sizes = deque(maxlen=window)
        self.conc = deque(maxlen=window)
        self.last = None
        self.r_window = 0.0
        self.r_size = 0.0
        self.r_con = 0.0

    def record(self, now, size, conc):
        if size < 0 or conc < 0:
            raise ValueError("histogram samples must be >= 0")
        if self.last is not None:
            self.gaps.append(now - self.last)
        self.last = now
        self.sizes.append(size)
        self.conc.append(conc)
        if self.gaps:
            self.r_window = p99(self.gaps)
        self.r_size = p99(self.sizes)
        self.r_con = p99(self.conc)

    def reserve(self):
        if not self.sizes:
            return 0.0
        return self.r_size * max(1.0, self.r_con)

    def active(self, now):
        if self.last is None:
            return False
        return now - self.last <= max(self.r_window, 0.0)


def target_bytes(hists, now, floor=FLOOR):  # datastore.py:79-82
    return max(sum(h.reserve() for h in hists if h.active(now)), floor)


class PoolPolicy:  # datastore.py:91-166; blocks are [class_bytes, in_use]
    def __init__(self, gpu, mode="autoscale", floor=FLOOR, alloc_ms=ALLOC_MS, physical=32 * 10**9):
        if mode not in ("autoscale", "cache_all", "none"):
            raise ValueError(f"unknown pool mode {mode!r}")
        self.gpu, self.mode, self.floor, self.alloc_ms, self.physical = gpu, mode, floor, alloc_ms, physical
        self.blocks = []
        self.hists = {}
        self._ids = itertools.count(1)

    def hist(self, func):
        if func not in self.hists:
            self.hists[func] = Hist(func)
        return self.hists[func]

    @property
    def pool_bytes(self):
        return float(sum(b[0] for b in self.blocks))

    @property
    def in_use_bytes(self):
        return float(sum(b[0] for b in self.blocks if b[1]))

    def target(self, now):
        return target_bytes(self.hists.values(), now, self.floor)

    def allocate(self, nbytes):
        """-> (block, cost_ms); block = [class_bytes, in_use, id]"""
        cls = block_class(nbytes)
        if self.pool_bytes + cls > self.physical and not any(
                b[0] == cls and not b[1] for b in self.blocks):
            raise PoolFull(f"gpu {self.gpu}: pool would exceed physical memory")
        if self.mode != "none":
            for b in self.blocks:
                if not b[1] and b[0] == cls:
                    b[1] = True
                    return b, 0.0
        b = [cls, True, next(self._ids)]
        self.blocks.append(b)
        return b, self.alloc_ms

    def free(self, b):
        b[1] = False
        if self.mode == "none":
            self.blocks.remove(b)

    def shrink(self, now):
        """Returns the dropped blocks (the reference drops them silently)."""
        dropped = []
        if self.mode != "autoscale":
            return dropped
        limit = self.target(now)
        if not any(h.active(now) for h in self.hists.values()):
            limit = min(limit, self.floor)
        for b in sorted((b for b in self.blocks if not b[1]), key=lambda b: -b[0]):
            if self.pool_bytes - b[0] < min(limit, self.floor):
                break
            if self.pool_bytes <= limit:
                break
            self.blocks.remove(b)
            dropped.append(b)
        return dropped


class Obj:  # datastore.py:169-185
    def __init__(self, data_id, size, producer, gpu, stored_at, location="gpu", consumers=None, live=True):
        self.data_id, self.size, self.producer, self.gpu = data_id, size, producer, gpu
        self.stored_at, self.location = stored_at, location
        self.consumers = dict(consumers or {})
        self.live = live

    def nearest(self):
        return min(self.consumers.values()) if self.consumers else None


def evict_order(objs, pressure, policy="queue_aware"):  # datastore.py:192-222
    if pressure <= 0:
        raise ValueError("pressure must be > 0")
    if policy not in ("queue_aware", "lru"):
        raise ValueError(f"unknown migration policy {policy!r}")
    plan = []
    freed = 0.0
    here = [o for o in objs if o.location == "gpu"]
    for o in sorted((o for o in here if not o.live), key=lambda o: o.data_id):
        plan.append(("reclaim", o))
        freed += o.size
        if freed >= pressure:
            return plan
    cand = [o for o in here if o.live and o.consumers]
    if policy == "queue_aware":
        cand.sort(key=lambda o: (-o.nearest(), o.data_id))
    else:
        cand.sort(key=lambda o: (o.stored_at, o.data_id))
    for o in cand:
        plan.append(("migrate", o))
        freed += o.size
        if freed >= pressure:
            return plan
    raise Pressure(f"need {pressure} bytes but only {freed} reclaimable/migratable")


def reload_order(objs, free_bytes):  # datastore.py:225-238
    if free_bytes <= 0:
        raise ValueError("free_bytes must be > 0")
    back = [o for o in objs if o.location == "host" and o.live and o.consumers]
    back.sort(key=lambda o: (o.nearest(), o.data_id))
    out = []
    room = free_bytes
    for o in back:
        if o.size <= room:
            out.append(o)
            room -= o.size
    return out


# ----------------------------------------------------------------------------
# strategies (strategies.py:15-62)
# ----------------------------------------------------------------------------
STRATEGIES = {
    # name: (host_oriented, parallel_pcie, unified_interface, pcie_sched, nvlink_sched, pool, migration)
    "infless_plus": (True, False, True, False, False, "none", "none"),
    "deepplan_plus": (True, True, True, False, False, "none", "none"),
    "faastube_star": (False, True, True, False, False, "none", "none"),
    "faastube": (False, True, True, True, True, "autoscale", "queue_aware"),
}
STRATEGY_FIELDS = ("host_oriented", "parallel_pcie", "unified_interface", "pcie_sched",
                   "nvlink_sched", "pool", "migration")


def strategy(name, **over):
    if name not in STRATEGIES:
        raise ValueError(f"unknown strategy {name!r}")
    s = dict(zip(STRATEGY_FIELDS, STRATEGIES[name]))
    s.update(over)
    s["name"] = name
    return s


# ----------------------------------------------------------------------------
# data index + fetch plans (dataplane.py:55-369)
# ----------------------------------------------------------------------------
def _floordiv(a, b):
    return a // b  # Python float floor division, as dataplane.py:78


class Index:  # dataplane.py:55-107; entries are dicts
    def __init__(self, sync=SYNC_MS, local=LOOKUP_LOCAL_MS, glob=LOOKUP_GLOBAL_MS):
        self.sync, self.local_ms, self.global_ms = sync, local, glob
        self._ids = itertools.count(1)
        self.local = {}
        self.table = {}

    def unique_id(self):
        return next(self._ids)

    def store(self, did, node, gpu, size, now, producer, response=False):
        t = self.local.setdefault(node, {})
        if did in t or did in self.table:
            raise Duplicate(f"data id {did} already stored")
        vis = (int(_floordiv(now, self.sync)) + 1) * self.sync if self.sync > 0 else now
        e = {"id": did, "size": size, "node": node, "gpu": gpu, "created": now,
             "producer": producer, "response": response, "visible": vis}
        t[did] = e
        self.table[did] = e
        return e

    def resolve(self, did, node, now):
        t = self.local.get(node, {})
        if did in t:
            return t[did], self.local_ms, now
        e = self.table.get(did)
        if e is None:
            raise Missing(f"data id {did} not found in local or global table")
        return e, self.local_ms + self.global_ms, max(now, e["visible"])

    def drop(self, did):
        e = self.table.pop(did, None)
        if e is not None:
            self.local.get(e["node"], {}).pop(did, None)

    def relocate(self, did, node, gpu):
        e = self.table[did]
        self.local.get(e["node"], {}).pop(did, None)
        e["node"], e["gpu"] = node, gpu
        self.local.setdefault(node, {})[did] = e


def hop_links(fab, u, v):  # dataplane.py:128-133
    if fab.kind(u, v) == "nvswitch":
        return [("nvp_out", u), ("nvp_in", v)]
    return [("nv", u, v)]


def branch(links, share, cap=None, reserved=None, fill=0.0, hop_caps=None):  # dataplane.py:136-143
    return {"links": links, "bytes_share": share, "cap_gbps": cap, "reserved_gbps": reserved,
            "fill_ms": fill, "hop_caps": list(hop_caps or [])}


def stage(branches, managed=False, pinned=0.0):  # dataplane.py:146-150
    return {"branches": branches, "managed": managed, "pinned_bytes": pinned}


def plan(method, size, stages=None, fixed=0.0, claimed=None, note=""):  # dataplane.py:153-160
    return {"method": method, "size_bytes": size, "stages": stages or [], "fixed_ms": fixed,
            "claimed_func": claimed, "note": note}


class Plane:  # dataplane.py:163-348
    def __init__(self, fab, strat, mx, chunk, map_ms=MAP_MS):
        self.fab, self.strat, self.mx, self.chunk, self.map_ms = fab, strat, mx, chunk, map_ms
        self._claims = itertools.count(1)

    def fetch_plan(self, src, dst, size):
        """src/dst = (node, gpu-or-None)."""
        if src[0] != dst[0]:
            return self._inter_node(src, dst, size)
        if src[1] is None and dst[1] is None:
            return plan("intra_gpu", size, fixed=0.0, note="host-to-host shared memory")
        if (src[1] is None) != (dst[1] is None):
            return self._host_gpu(src, dst, size)
        if src[1] == dst[1]:
            return plan("intra_gpu", size, fixed=self.map_ms)
        return self._inter_gpu(src, dst, size)

    def _host_gpu(self, src, dst, size):
        into = src[1] is None
        gpu = dst[1] if into else src[1]
        brs = self._pcie_branches(dst[0], gpu, size, into)
        return plan("host_gpu", size, stages=[stage(brs, self.strat["pcie_sched"], self._staging(size))])

    def _staging(self, size):
        return min(size, 2 * self.chunk)

    def _pcie_branches(self, node, gpu, size, into):
        fab = self.fab
        own = fab.root_of(gpu)
        tag = "h2d" if into else "d2h"
        routes = [[(tag, node, own)]]
        if self.strat["parallel_pcie"]:
            for r, gs in sorted(fab.groups.items()):
                if r == own or not any(fab.node_of(g) == node for g in gs):
                    continue
                d = self._detour(node, r, gpu, into)
                if d is not None:
                    routes.append(d)
        share = size / len(routes)
        out = []
        for links in routes:
            caps = [self._cap(l) for l in links]
            out.append(branch(links, share, hop_caps=caps, fill=pipe_fill(caps, min(self.chunk, share))))
        return out

    def _detour(self, node, r, gpu, into):
        fab = self.fab
        best = None
        for sg in [g for g in sorted(fab.groups[r]) if fab.node_of(g) == node]:
            p = self._nv_route(sg, gpu, into)
            if p and (best is None or len(p) < len(best[1])):
                best = (sg, p)
        if best is None:
            return None
        pcie = ("h2d" if into else "d2h", node, r)
        nvl = [l for u, v in zip(best[1], best[1][1:]) for l in hop_links(fab, u, v)]
        return [pcie] + nvl if into else nvl + [pcie]

    def _nv_route(self, a, b, into):
        s, d = (a, b) if into else (b, a)
        for p in candidates(self.fab, s, d, max_hops=2):
            if all(self.mx.res(u, v) > 0 for u, v in zip(p, p[1:])):
                return p
        return None

    def _cap(self, link):
        k = link[0]
        if k in ("h2d", "d2h"):
            return self.fab.pcie
        if k == "nv":
            return self.fab.nv(link[1], link[2])
        if k in ("nvp_out", "nvp_in"):
            return self.fab.port(link[1])
        return self.fab.net

    def _inter_gpu(self, src, dst, size):
        if self.strat["host_oriented"]:
            pin = self._staging(size)
            down = stage(self._pcie_branches(src[0], src[1], size, False), pinned=pin)
            up = stage(self._pcie_branches(dst[0], dst[1], size, True), pinned=pin)
            return plan("inter_gpu", size, stages=[down, up], note="staged through host memory")
        func = f"xfer{next(self._claims)}"
        if self.strat["nvlink_sched"]:
            paths = select(self.mx, func, src[1], dst[1], allow_busy=False)
        else:
            c = self.fab.nv(src[1], dst[1])
            paths = [([src[1], dst[1]], c, False)] if c > 0 else []
        if not paths:
            return self._pcie_peer(src, dst, size)
        tot = sum(p[1] for p in paths)
        claimed = any(p[2] for p in paths)
        brs = []
        for gpus, bmin, held in paths:
            links = [l for u, v in zip(gpus, gpus[1:]) for l in hop_links(self.fab, u, v)]
            share = size * bmin / tot
            caps = [self.fab.nv(u, v) for u, v in zip(gpus, gpus[1:])]
            brs.append(branch(links, share, hop_caps=caps, reserved=bmin if held else None,
                              fill=pipe_fill(caps, min(self.chunk, share))))
        return plan("inter_gpu", size, stages=[stage(brs)], claimed=func if claimed else None)

    def _pcie_peer(self, src, dst, size):
        # dataplane.py:304-324. The reference raises NameError here (SURVEY
        # Appendix A1: pipeline_latency not imported); restated as intended.
        links = [("d2h", src[0], self.fab.root_of(src[1])), ("h2d", dst[0], self.fab.root_of(dst[1]))]
        peer, pcie = self.fab.peer, self.fab.pcie
        ch = min(self.chunk, size)
        if pipe_latency(size, [peer], ch) <= pipe_latency(size, [pcie, pcie], ch):
            br = branch(links, size, cap=peer, hop_caps=[peer, peer], fill=pipe_fill([peer, peer], ch))
            note = "pcie peer fallback"
        else:
            br = branch(links, size, hop_caps=[pcie, pcie], fill=pipe_fill([pcie, pcie], ch))
            note = "pipelined host staging fallback"
        return plan("inter_gpu", size, stages=[stage([br])], note=note)

    def _inter_node(self, src, dst, size):
        hops = []
        if src[1] is not None:
            hops.append(("d2h", src[0], self.fab.root_of(src[1])))
        hops.append(("net", src[0], dst[0]))
        if dst[1] is not None:
            hops.append(("h2d", dst[0], self.fab.root_of(dst[1])))
        caps = [self._cap(l) for l in hops]
        if self.strat["host_oriented"]:
            return plan("inter_node", size, stages=[stage([branch([l], size, hop_caps=[c])])
                                                    for l, c in zip(hops, caps)],
                        note="sequential copies through both hosts")
        br = branch(hops, size, hop_caps=caps, fill=pipe_fill(caps, min(self.chunk, size)))
        return plan("inter_node", size, stages=[stage([br])], note="pipelined across nodes")

    def release_claim(self, p):
        if p["claimed_func"] and p["claimed_func"] in self.mx.held:
            self.mx.release(p["claimed_func"])


def plan_latency(p):  # dataplane.py:351-369
    t = p["fixed_ms"]
    for st in p["stages"]:
        worst = 0.0
        for br in st["branches"]:
            if br["reserved_gbps"] is not None:
                r = br["reserved_gbps"]
            elif br["cap_gbps"] is not None:
                r = br["cap_gbps"]
            else:
                r = min(br["hop_caps"])
            worst = max(worst, ms_for(br["bytes_share"], r) + br["fill_ms"])
        t += worst
    return t

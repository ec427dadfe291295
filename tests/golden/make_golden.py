"""Generate golden decision vectors from the REFERENCE implementation.

Run in the build container only (it imports ``/root/reference/pkg/src/tubesim``,
which does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes ``tests/golden/*.json``. Every vector is an op sequence with the
reference's result recorded after each op, replayed by
``tests/golden_replay.py`` against the oracle and against the product's
C-ABI library. Seeds are fixed, so regenerating is byte-identical.
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = os.environ.get("FT_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from tubesim import datastore, dataplane, nvlink_sched, pcie_sched, simcore, topology  # noqa: E402
from tubesim import engine as engine_mod  # noqa: E402
from tubesim import harness  # noqa: E402
from tubesim.strategies import strategy_preset  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def b200_doc(n=8, pair=900.0, groups=None, pcie=55.0, name="b200"):
    groups = groups if groups is not None else {r: [r] for r in range(n)}
    links = [{"kind": "pcie", "endpoints": ["host:0", r], "bandwidth_gbps": pcie} for r in sorted(groups)]
    links += [{"kind": "nvswitch", "endpoints": [u, v], "bandwidth_gbps": pair}
              for u in range(n) for v in range(u + 1, n)]
    return {"name": name, "gpu_count": n, "nodes": [{"id": 0, "gpus": list(range(n))}],
            "links": links, "pcie_groups": {str(k): v for k, v in groups.items()},
            "rates": {"pcie_gbps": pcie}}


def topo_docs():
    docs = {
        "dgx_v100": topology.build_preset("dgx_v100").to_dict(),
        "dgx_a100": topology.build_preset("dgx_a100").to_dict(),
        "quad_a10": topology.build_preset("quad_a10").to_dict(),
        "b200_k8": b200_doc(),
        "b200_k4": b200_doc(groups={r: [2 * r, 2 * r + 1] for r in range(4)}, name="b200_k4"),
        "b200_k2": b200_doc(groups={r: list(range(4 * r, 4 * r + 4)) for r in range(2)}, name="b200_k2"),
        "b200_k1": b200_doc(groups={0: list(range(8))}, name="b200_k1"),
        "b200_2gpu": b200_doc(n=2, name="b200_2gpu"),
        "b200_4gpu": b200_doc(n=4, name="b200_4gpu"),
        "cluster_a100_x2": topology.build_cluster("dgx_a100", 2).to_dict(),
    }
    # build_cluster docs carry int endpoints and "host:n" strings already
    return docs


def err_name(exc):
    return type(exc).__name__


# ---------------------------------------------------------------- topology
def gen_topology(docs):
    cases = []
    for name, doc in docs.items():
        t = topology.from_dict(doc)
        n = t.gpu_count
        q = {"name": name, "doc": doc, "gpu_count": n,
             "node_of": [t.node_of(g) for g in range(n)],
             "root_of": [t.pcie_root_of(g) for g in range(n)],
             "nvlink": [[t.nvlink_gbps(u, v) for v in range(n)] for u in range(n)],
             "neighbors": [t.nvlink_neighbors(g) for g in range(n)],
             "port": [t.switch_port_gbps(g) for g in range(n)],
             "degree": [t.nvlink_degree_gbps(g) for g in range(n)],
             "pair_bw": [[(t.pair_bandwidth(u, v) if u != v else None) for v in range(n)] for u in range(n)],
             "kind": [[t.pair_kind(u, v) for v in range(n)] for u in range(n)]}
        cases.append(q)
    bad = []
    base = b200_doc(n=4)
    d1 = json.loads(json.dumps(base)); d1["links"].append({"kind": "nvswitch", "endpoints": [0, 9], "bandwidth_gbps": 1.0})
    d2 = json.loads(json.dumps(base)); d2["pcie_groups"]["0"] = [0, 1]
    d3 = json.loads(json.dumps(base)); d3["links"][0]["bandwidth_gbps"] = 0
    d4 = json.loads(json.dumps(base)); del d4["nodes"]
    d5 = json.loads(json.dumps(base)); d5["nodes"] = [{"id": 0, "gpus": [0, 1, 2]}]
    for d in (d1, d2, d3, d4, d5):
        try:
            topology.from_dict(d)
            bad.append({"doc": d, "error": None})
        except Exception as exc:  # noqa: BLE001
            bad.append({"doc": d, "error": err_name(exc)})
    return {"cases": cases, "invalid": bad}


# ---------------------------------------------------------------- nvlink
def matrix_state(m):
    return {"residual": sorted([[u, v, r] for (u, v), r in m.residual.items()]),
            "egress": [m.egress_budget[g] for g in sorted(m.egress_budget)],
            "ingress": [m.ingress_budget[g] for g in sorted(m.ingress_budget)],
            "held": {f: [[p, r] for p, r in lst] for f, lst in m.held.items()}}


def gen_nvlink(docs):
    seqs = []
    rng = random.Random(1830)
    for name in ("dgx_v100", "dgx_a100", "b200_k8", "b200_4gpu", "quad_a10", "b200_2gpu"):
        doc = docs[name]
        for rep in range(6 if name == "dgx_v100" else 3):
            t = topology.from_dict(doc)
            m = topology.snapshot_matrix(t)
            ops = []
            funcs = 0
            for _ in range(40):
                r = rng.random()
                holders = sorted(m.held)
                if r < 0.55 or not holders:
                    funcs += 1
                    f = f"f{funcs}"
                    s, d = rng.sample(range(t.gpu_count), 2)
                    ab = rng.random() < 0.6
                    q = nvlink_sched.PathQuery(f, s, d, m, allow_busy=ab)
                    try:
                        ps = nvlink_sched.select_paths(q)
                        res = {"paths": [[p.gpus, p.b_min_gbps, p.held_by == f] for p in ps],
                               "trace": {k: v for k, v in q.trace.items()}}
                    except Exception as exc:  # noqa: BLE001
                        res = {"error": err_name(exc)}
                    ops.append({"op": "select", "func": f, "src": s, "dst": d, "allow_busy": ab,
                                "expect": res, "state": matrix_state(m)})
                elif r < 0.85:
                    f = rng.choice(holders + ["nobody"])
                    try:
                        nvlink_sched.release_paths(m, f)
                        res = {"ok": True}
                    except Exception as exc:  # noqa: BLE001
                        res = {"error": err_name(exc)}
                    ops.append({"op": "release", "func": f, "expect": res, "state": matrix_state(m)})
                else:
                    funcs += 1
                    f = f"wf{funcs}"
                    npairs = rng.randint(0, 3)
                    pairs = [rng.sample(range(t.gpu_count), 2) for _ in range(npairs)]
                    try:
                        resv, deg = nvlink_sched.claim_direct_for_workflow(m, [tuple(p) for p in pairs], f)
                        res = {"reservations": [[list(e), r] for e, r in resv], "degraded": deg}
                    except Exception as exc:  # noqa: BLE001
                        res = {"error": err_name(exc)}
                    ops.append({"op": "claim_direct", "func": f, "pairs": pairs, "expect": res,
                                "state": matrix_state(m)})
            seqs.append({"topology": name, "ops": ops})
    # candidate enumeration
    cands = []
    for name in ("dgx_v100", "dgx_a100", "b200_k8", "b200_4gpu", "b200_2gpu", "quad_a10"):
        t = topology.from_dict(docs[name])
        for s in range(t.gpu_count):
            for d in range(t.gpu_count):
                if s != d:
                    for mh in (2, 4):
                        cands.append({"topology": name, "src": s, "dst": d, "max_hops": mh,
                                      "paths": nvlink_sched._candidate_paths(t, s, d, mh)})
    chunks = []
    for _ in range(300):
        k = rng.randint(1, 6)
        w = [rng.choice([24.0, 48.0, 300.0, 900.0, rng.uniform(0.5, 900.0)]) for _ in range(k)]
        n = rng.randint(0, 600)
        ps = [nvlink_sched.NvPath([0, 1], x) for x in w]
        chunks.append({"n": n, "weights": w, "counts": nvlink_sched.distribute_chunks(n, ps)})
    chunks.append({"n": 30, "weights": [48.0, 24.0], "counts": [20, 10]})
    chunks.append({"n": 10, "weights": [24.0, 24.0, 24.0], "counts": [4, 3, 3]})
    return {"sequences": seqs, "candidates": cands, "distribute": chunks}


# ---------------------------------------------------------------- pcie
def gen_pcie():
    rng = random.Random(2411)
    mr = []
    for _ in range(200):
        b = rng.choice([0, rng.uniform(0, 1e9), rng.randint(1, 10**9)])
        slo = rng.uniform(0, 200)
        inf = rng.choice([rng.uniform(0, 200), slo, slo * 0.5])
        try:
            mr.append({"args": [b, slo, inf], "rate": pcie_sched.min_rate(b, slo, inf)})
        except Exception as exc:  # noqa: BLE001
            mr.append({"args": [b, slo, inf], "error": err_name(exc)})
    parts = []
    for _ in range(300):
        st = pcie_sched.PcieSchedulerState(bw_all_gbps=rng.choice([12.0, 48.0, 55.0, 440.0, rng.uniform(1, 500)]))
        ds = []
        for i in range(rng.randint(0, 8)):
            slo = rng.uniform(5, 300)
            d = pcie_sched.RateDemand(f"m{i}", rng.uniform(1e5, 6e8), slo, rng.uniform(0, slo * 0.9),
                                      arrival_ms=rng.choice([0.0, rng.uniform(0, 100)]))
            st.add(d)
            ds.append([d.func, d.data_size_bytes, d.slo_ms, d.infer_ms, d.arrival_ms])
        now = rng.uniform(0, 150)
        rates = pcie_sched.partition(st, now)
        parts.append({"bw_all": st.bw_all_gbps, "demands": ds, "now": now, "rates": rates,
                      "at_risk": {d.func: d.slo_at_risk for d in st.demands.values()},
                      "idle": st.rate_idle_gbps(),
                      "slack": {d.func: d.slack_ms(now) for d in st.demands.values()}})
    trig = []
    for _ in range(100):
        st = pcie_sched.PcieSchedulerState(bw_all_gbps=48.0, batch_chunks=rng.randint(1, 8),
                                           chunk_bytes=rng.choice([2 * 10**6, 1 << 20, 4 * 10**6]))
        tot = rng.choice([0, -5, rng.uniform(1, 5e8), 20 * 10**6, 1 * 10**6, 1 << 30])
        trig.append({"total": tot, "batch_chunks": st.batch_chunks, "chunk": st.chunk_bytes,
                     "batches": pcie_sched.trigger_batches(tot, st)})
    rings = []
    for _ in range(40):
        cap = rng.choice([0.0, 20e6, 160e6, rng.uniform(1e6, 2e8)])
        pre = rng.random() < 0.5
        ring = pcie_sched.PinnedRing(cap, prewarmed=pre)
        seq = []
        for _ in range(10):
            need = rng.choice([0.0, rng.uniform(0, 3e8), 4e6, 1e8])
            seq.append([need, ring.acquire(need), ring.warm_bytes, ring.cold_allocated_bytes])
        rings.append({"capacity": cap, "prewarmed": pre, "seq": seq})
    rc = [[k, b, pcie_sched.default_ring_capacity(k, b)] for k in (1, 2, 4, 8) for b in (10 * 10**6, 4 * 10**6)]
    return {"min_rate": mr, "partition": parts, "trigger": trig, "rings": rings, "ring_capacity": rc}


# ---------------------------------------------------------------- simcore
def gen_simcore():
    rng = random.Random(7)
    pl = []
    for _ in range(200):
        hops = [rng.choice([12.0, 24.0, 48.0, 55.0, 900.0, rng.uniform(0.1, 1000)]) for _ in range(rng.randint(1, 5))]
        size = rng.choice([1 << 30, 96e6, 2e6, rng.uniform(1, 2e9)])
        ch = rng.choice([2e6, 0, size * 2, rng.uniform(1, 4e6)])
        pl.append({"size": size, "hops": hops, "chunk": ch,
                   "latency": simcore.pipeline_latency(size, hops, ch),
                   "fill": simcore.pipeline_fill_ms(hops, ch)})
    nr = []
    for _ in range(100):
        xs = sorted(rng.uniform(0, 100) for _ in range(rng.randint(1, 300)))
        pct = rng.choice([50, 90, 99, 99.9, 100, rng.uniform(0, 100)])
        nr.append({"values": xs, "pct": pct, "result": simcore.nearest_rank(xs, pct)})
    nr.append({"values": [float(i) for i in range(1, 101)], "pct": 99, "result": 99.0})
    return {"pipeline": pl, "nearest_rank": nr}


# ---------------------------------------------------------------- datastore
def gen_datastore():
    rng = random.Random(99)
    sc = []
    for x in [1, 2e6, 2e6 + 1, 4e6 - 1, 130e6, 1 << 30, 0.5, 64 * 1024 * 1024] + [rng.uniform(1, 1e9) for _ in range(50)]:
        sc.append([x, datastore.size_class(x)])
    hists = []
    for _ in range(40):
        h = datastore.FuncHistogram("f", window=rng.choice([1000, 5]))
        t = 0.0
        seq = []
        for _ in range(rng.randint(1, 40)):
            t += rng.choice([0.0, rng.uniform(0, 50)])
            size = rng.choice([rng.uniform(1e6, 5e8), 128e6, 64 * 10**6])
            con = rng.choice([1, 2, 3, rng.uniform(0, 4)])
            h.record_execution(t, size, con)
            probe = t + rng.uniform(0, 80)
            seq.append({"now": t, "size": size, "con": con, "r_window": h.r_window_ms, "r_size": h.r_size_bytes,
                        "r_con": h.r_con, "reservation": h.reservation_bytes(), "probe": probe,
                        "active": h.window_active(probe)})
        hists.append({"window": h.intervals.maxlen, "seq": seq})
    pools = []
    for mode in ("autoscale", "cache_all", "none"):
        for rep in range(8):
            floor = rng.choice([300 * 10**6, 50e6, 0.0])
            phys = rng.choice([32 * 10**9, 1e9])
            p = datastore.MemoryPool(0, mode, floor, 1.0, phys)
            ops = []
            t = 0.0
            for _ in range(60):
                r = rng.random()
                t += rng.uniform(0, 20)
                used = [i for i, b in enumerate(p.blocks) if b.in_use]
                if r < 0.4:
                    size = rng.choice([1e6, 4e6, 64e6, 128e6, 256e6, 512e6, rng.uniform(1, 6e8)])
                    try:
                        b, cost = p.allocate(size)
                        res = {"index": p.blocks.index(b) if b in p.blocks else None, "cost": cost}
                        # identity index (first equal block may differ; record by identity)
                        res["index"] = next(i for i, x in enumerate(p.blocks) if x is b)
                    except Exception as exc:  # noqa: BLE001
                        res = {"error": err_name(exc)}
                    ops.append({"op": "allocate", "size": size, "expect": res})
                elif r < 0.7 and used:
                    k = rng.randrange(len(used))
                    p.free(p.blocks[used[k]])
                    ops.append({"op": "free", "nth_in_use": k, "expect": {}})
                elif r < 0.85:
                    f = rng.choice(["a", "b", "c"])
                    size = rng.choice([1e6, 64e6, 128e6, 512e6])
                    con = rng.choice([1, 2, 3])
                    p.histogram(f).record_execution(t, size, con)
                    ops.append({"op": "record", "func": f, "now": t, "size": size, "con": con, "expect": {}})
                else:
                    probe = t + rng.choice([0.0, 5.0, 100.0, 1e4])
                    tgt = p.target(probe)
                    p.shrink(probe)
                    ops.append({"op": "shrink", "now": probe, "expect": {"target": tgt}})
                ops[-1]["state"] = {"blocks": [[b.class_bytes, b.in_use] for b in p.blocks],
                                    "pool_bytes": p.pool_bytes, "in_use_bytes": p.in_use_bytes}
            pools.append({"mode": mode, "floor": floor, "physical": phys, "ops": ops})
    migs = []
    for _ in range(150):
        objs = []
        for i in range(rng.randint(0, 8)):
            cons = {(0, f"c{j}"): rng.randint(1, 50) for j in range(rng.randint(0, 3))}
            o = datastore.StoredObject(i + 1 + rng.randint(0, 3) * 10, rng.choice([1e6, 64e6, 256e6, rng.uniform(1, 5e8)]),
                                       "p", 0, rng.uniform(0, 100), location=rng.choice(["gpu", "gpu", "host", "both"]),
                                       consumers=cons, live=rng.random() < 0.8)
            objs.append(o)
        ser = [[o.data_id, o.size_bytes, o.stored_at_ms, o.location, sorted(o.consumers.values()), o.live] for o in objs]
        pressure = rng.choice([1e6, 1e8, 5e8, 2e9])
        pol = rng.choice(["queue_aware", "lru"])
        try:
            plan = datastore.migration_plan(objs, pressure, pol)
            res = {"plan": [[a, o.data_id, objs.index(o)] for a, o in plan]}
        except Exception as exc:  # noqa: BLE001
            res = {"error": err_name(exc)}
        free = rng.choice([1e6, 1e8, 5e8, 2e9])
        sched = datastore.prefetch_back(objs, free)
        migs.append({"objects": ser, "pressure": pressure, "policy": pol, "expect": res, "free": free,
                     "prefetch": [objs.index(o) for o in sched]})
    targets = []
    for _ in range(60):
        hs = []
        desc = []
        for j in range(rng.randint(0, 4)):
            h = datastore.FuncHistogram(f"f{j}")
            t = 0.0
            recs = []
            for _ in range(rng.randint(1, 6)):
                t += rng.uniform(0, 30)
                s, c = rng.choice([64e6, 130e6, 260e6]), rng.choice([1, 2])
                h.record_execution(t, s, c)
                recs.append([t, s, c])
            hs.append(h)
            desc.append(recs)
        now = rng.uniform(0, 200)
        floor = rng.choice([300 * 10**6, 0.0])
        targets.append({"hists": desc, "now": now, "floor": floor, "target": datastore.pool_target(hs, now, floor)})
    return {"size_class": sc, "histograms": hists, "pools": pools, "migration": migs, "targets": targets}


# ---------------------------------------------------------------- dataplane
def ser_plan(p):
    return {"method": p.method, "size_bytes": p.size_bytes, "fixed_ms": p.fixed_ms,
            "claimed_func": p.claimed_func, "note": p.note,
            "stages": [{"managed": s.managed, "pinned_bytes": s.pinned_bytes,
                        "branches": [{"links": [list(l) for l in b.links], "bytes_share": b.bytes_share,
                                      "cap_gbps": b.cap_gbps, "reserved_gbps": b.reserved_gbps,
                                      "fill_ms": b.fill_ms, "hop_caps": b.hop_caps}
                                     for b in s.branches]} for s in p.stages],
            "latency": dataplane.plan_latency_model(p)}


def gen_dataplane(docs):
    rng = random.Random(4242)
    seqs = []
    for name in ("b200_k8", "b200_k4", "b200_k2", "b200_k1", "dgx_v100", "dgx_a100", "quad_a10", "cluster_a100_x2", "b200_2gpu"):
        for sname in ("faastube", "faastube_star", "infless_plus", "deepplan_plus"):
            t = topology.from_dict(docs[name])
            strat = strategy_preset(sname)
            m = topology.snapshot_matrix(t)
            dp = dataplane.Dataplane(t, strat, m, rng.choice([2 * 10**6, 2 * 10**6, 1 << 20]), 0.05)
            ops = []
            live = []
            nodes = sorted({n["id"] for n in t.nodes})
            for _ in range(30):
                if live and rng.random() < 0.3:
                    i = rng.randrange(len(live))
                    pid = live.pop(i)
                    dp.release_claim(pid[1])
                    ops.append({"op": "release", "plan": pid[0], "state": matrix_state(m)})
                    continue

                def loc():
                    nd = rng.choice(nodes)
                    gs = [g for g in range(t.gpu_count) if t.node_of(g) == nd]
                    return [nd, rng.choice(gs + [None])]
                src, dst = loc(), loc()
                size = rng.choice([4096, 64 * 2**20, 1 << 30, 2e6, rng.uniform(1, 1e9), 256e6])
                try:
                    p = dp.fetch_plan(dataplane.Location(*src), dataplane.Location(*dst), size)
                    res = ser_plan(p)
                    live.append((len(ops), p))
                except Exception as exc:  # noqa: BLE001
                    res = {"error": err_name(exc)}
                ops.append({"op": "fetch_plan", "src": src, "dst": dst, "size": size, "expect": res,
                            "state": matrix_state(m)})
            seqs.append({"topology": name, "strategy": sname, "chunk": dp.chunk_bytes, "ops": ops})
    idx = []
    for rep in range(10):
        di = dataplane.DataIndex(rng.choice([10.0, 0.0, 3.3]), 0.005, 0.2)
        ops = []
        ids = []
        for _ in range(50):
            r = rng.random()
            now = rng.uniform(0, 100)
            if r < 0.2:
                i = di.unique_id()
                ids.append(i)
                ops.append({"op": "unique_id", "expect": i})
            elif r < 0.45 and ids:
                i = rng.choice(ids + [999])
                node, gpu = rng.randint(0, 1), rng.choice([None, 0, 3])
                size, resp = rng.uniform(1, 1e9), rng.random() < 0.3
                try:
                    e = di.store(i, dataplane.Location(node, gpu), size, now, "p", resp)
                    res = {"visible": e.global_visible_ms}
                except Exception as exc:  # noqa: BLE001
                    res = {"error": err_name(exc)}
                ops.append({"op": "store", "id": i, "node": node, "gpu": gpu, "size": size,
                            "now": now, "response": resp, "expect": res})
            elif r < 0.8 and ids:
                i = rng.choice(ids + [999])
                node = rng.randint(0, 1)
                try:
                    e, cost, ready = di.resolve(i, node, now)
                    res = {"cost": cost, "ready": ready, "node": e.location.node, "gpu": e.location.gpu}
                except Exception as exc:  # noqa: BLE001
                    res = {"error": err_name(exc)}
                ops.append({"op": "resolve", "id": i, "node": node, "now": now, "expect": res})
            elif r < 0.9 and ids:
                i = rng.choice(ids)
                di.drop(i)
                ops.append({"op": "drop", "id": i, "expect": {}})
            elif ids:
                i = rng.choice(ids)
                node, gpu = rng.randint(0, 1), rng.choice([None, 1])
                try:
                    di.relocate(i, dataplane.Location(node, gpu))
                    res = {}
                except Exception as exc:  # noqa: BLE001
                    res = {"error": err_name(exc)}
                ops.append({"op": "relocate", "id": i, "node": node, "gpu": gpu, "expect": res})
        idx.append({"sync": di.sync_period_ms, "ops": ops})
    return {"sequences": seqs, "index": idx}


# ---------------------------------------------------------------- arbiter traces
class _Recorder:
    def __init__(self):
        self.calls = []
        self.cur = None
        self.engine = None


def _snapshot(eng):
    out = {}
    for k, m in eng._managed.items():
        out[k] = [m.rate_gbps, m.started, m.pending_rate, m.anchor_ms, m.armed_ms]
    return out


def record_engine(cfg):
    rec = _Recorder()
    E = engine_mod.Engine
    orig_start, orig_boundary, orig_set, orig_arm = (E._start_managed_stage, E._on_boundary,
                                                       E._set_stage_rate, E._arm_boundary)
    orig_remove = pcie_sched.PcieSchedulerState.remove
    orig_partition = pcie_sched.partition
    stage_dir = {}

    def open_call(kind, eng, **kw):
        if rec.cur is not None:
            rec.cur["state_after"] = _snapshot(eng)
        rec.cur = {"kind": kind, "now": eng.now, **kw, "decisions": []}
        rec.calls.append(rec.cur)

    def start(self, req, stage, consumer, begin, branch_done):
        wf = req.wf
        func = wf.function(consumer) if consumer in wf._by_id else None
        total = sum(br.bytes_share for br in stage.branches)
        node, direction = 0, "h2d"
        for br in stage.branches:
            for l in br.links:
                if l[0] in ("h2d", "d2h"):
                    node, direction = l[1], l[0]
        slo = func.slo_ms if func is not None and func.slo_ms else 1e9
        infer = func.infer_latency_ms if func is not None else 0.0
        per_branch = min(min(br.hop_caps) for br in stage.branches)
        before = set(self._managed)
        open_call("start", self, key=None, total=total, slo=slo, infer=infer, arrival=begin,
                  per_branch_cap=per_branch, n_branches=len(stage.branches), node=node, direction=direction)
        call = rec.cur
        r = orig_start(self, req, stage, consumer, begin, branch_done)
        (key,) = set(self._managed) - before
        call["key"] = key
        stage_dir[key] = (node, direction)
        return r

    def boundary(self, m):
        open_call("boundary", self, key=m.key, node=m.node, direction=m.direction)
        return orig_boundary(self, m)

    def remove(self, func):
        eng = rec.engine
        nd = stage_dir.get(func, (None, None))
        open_call("finish", eng, key=func, node=nd[0], direction=nd[1])
        return orig_remove(self, func)

    def set_rate(self, m, rate):
        rec.cur["decisions"].append(["set_rate", m.key, rate, rate / len(m.flows)])
        assert m.key in self._managed or rec.cur["kind"] == "start"
        return orig_set(self, m, rate)

    def arm(self, m, t):
        before = m.armed_ms
        r = orig_arm(self, m, t)
        if m.armed_ms is not None and m.armed_ms != before or (before is None and m.armed_ms is not None):
            rec.cur["decisions"].append(["arm", m.key, m.armed_ms])
        return r

    def part(state, now=0.0):
        r = orig_partition(state, now)
        if rec.cur is not None:
            rec.cur["decisions"].append(["partition", dict(r)])
        return r

    E._start_managed_stage, E._on_boundary, E._set_stage_rate, E._arm_boundary = start, boundary, set_rate, arm
    pcie_sched.PcieSchedulerState.remove = remove
    pcie_sched.partition = part
    try:
        eng = harness.prepare_engine(cfg)
        rec.engine = eng
        eng.run_until(cfg.duration_s * 1000.0 + cfg.drain_ms)
        if rec.cur is not None:
            rec.cur["state_after"] = _snapshot(eng)
        summ = eng.metrics.summary(cfg.duration_s * 1000.0)
        bw = {f"{n}:{d}": s.bw_all_gbps for (n, d), s in eng._pcie.items()}
    finally:
        E._start_managed_stage, E._on_boundary, E._set_stage_rate, E._arm_boundary = orig_start, orig_boundary, orig_set, orig_arm
        pcie_sched.PcieSchedulerState.remove = orig_remove
        pcie_sched.partition = orig_partition
    return {"calls": rec.calls, "bw_all": bw, "batch_chunks": cfg.engine.batch_chunks,
            "chunk": cfg.engine.chunk_bytes, "summary": summ, "risk_flags": eng.metrics.slo_risk_flags}


def gen_arbiter(docs):
    scen = []
    specs = [
        ("b200_k8", [("traffic", "bursty", 20.0), ("yelp", "sporadic", 30.0)], 1.0, 0),
        ("b200_k4", [("traffic", "sporadic", 15.0), ("social", "bursty", 10.0)], 1.0, 1),
        ("b200_k2", [("image", "bursty", 20.0), ("yelp", "periodic", 40.0)], 1.0, 2),
        ("dgx_a100", [("traffic", "bursty", 8.0), ("yelp", "sporadic", 10.0)], 1.0, 3),
        ("b200_k8", [("traffic", "bursty", 60.0)], 0.5, 4),
    ]
    for topo_name, wfs, dur, seed in specs:
        doc = {"topology": {}, "strategy": {"name": "faastube"},
               "workflows": [{"preset": w, "pattern": pat, "mean_rate_rps": r} for w, pat, r in wfs],
               "trace": {"duration_s": dur}, "seed": seed, "placement": {"occupancy_limit": 2}}
        cfg = harness.ExperimentConfig.from_dict(doc)
        cfg.topology = topology.from_dict(docs[topo_name])
        cfg.drain_ms = 2000.0
        r = record_engine(cfg)
        r["name"] = f"{topo_name}:{'+'.join(w for w, _, _ in wfs)}:seed{seed}"
        scen.append(r)
        print(r["name"], len(r["calls"]), "calls", r["summary"].get("requests_completed"), "done", file=sys.stderr)
    return {"scenarios": scen}


def gen_harness(docs):
    """Workflow presets (as data for the package), arrival traces, per-request
    draws, placement and SLO calibration — the live runtime's inputs."""
    from tubesim import workflow
    presets = {n: workflow.preset_workflow(n).to_dict() for n in workflow.PRESET_NAMES}
    pkg = os.path.join(os.path.dirname(os.path.dirname(OUT)), "paper_2411_01830_b200", "workflows.json")
    with open(pkg, "w") as fh:
        json.dump(presets, fh, indent=1, sort_keys=True)
    traces = []
    for pattern in ("sporadic", "periodic", "bursty"):
        for rate in (5.0, 20.0):
            for dur in (1.0, 5.0):
                for seed in (0, 1, 2):
                    tr = harness.gen_workload(pattern, rate, dur, seed)
                    traces.append({"pattern": pattern, "rate": rate, "duration": dur, "seed": seed,
                                   "times": tr.timestamps_ms})
    reqs = []
    for name in workflow.PRESET_NAMES:
        wf = workflow.preset_workflow(name)
        tr = harness.gen_workload("bursty", 20.0, 2.0, 3)
        specs = harness.build_requests(wf, tr, 3, rid_start=100)
        reqs.append({"workflow": name, "requests": [
            {"rid": s.rid, "arrival": s.arrival_ms, "fired": sorted(list(map(list, s.fired))),
             "edge_bytes": sorted([[a, b, v] for (a, b), v in s.edge_bytes.items()]),
             "input": s.input_bytes, "response": s.response_bytes} for s in specs]})
    calib = []
    for tname in ("b200_k8", "b200_k4", "dgx_v100", "dgx_a100"):
        t = topology.from_dict(docs[tname])
        for name in workflow.PRESET_NAMES:
            for limit in (1, 2):
                wf = workflow.preset_workflow(name)
                try:
                    pl = workflow.place(wf, t, {}, limit)
                except Exception as exc:  # noqa: BLE001
                    calib.append({"topology": tname, "workflow": name, "limit": limit, "error": err_name(exc)})
                    continue
                rt = harness.calibrate_slo(wf, t, pl, engine_mod.EngineConfig(), 1.5)
                calib.append({"topology": tname, "workflow": name, "limit": limit,
                              "placement": {k: list(v) for k, v in pl.mapping.items()},
                              "runtime": rt, "slo": wf.slo_ms,
                              "funcs": {f.id: [f.slo_ms, f.infer_latency_ms] for f in wf.functions}})
    return {"traces": traces, "requests": reqs, "calibration": calib}


def main():
    docs = topo_docs()
    parts = {
        "topology": lambda: gen_topology(docs),
        "nvlink": lambda: gen_nvlink(docs),
        "pcie": gen_pcie,
        "simcore": gen_simcore,
        "datastore": gen_datastore,
        "dataplane": lambda: gen_dataplane(docs),
        "arbiter": lambda: gen_arbiter(docs),
        "harness": lambda: gen_harness(docs),
    }
    only = sys.argv[1:] or list(parts)
    for name in only:
        data = parts[name]()
        with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
            json.dump(data, fh, separators=(",", ":"), sort_keys=True)
        print("wrote", name, os.path.getsize(os.path.join(OUT, f"{name}.json")), "bytes", file=sys.stderr)


if __name__ == "__main__":
    main()

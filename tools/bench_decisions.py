"""Per-call host time of the decision functions on the path (SURVEY §8a rows
a5-a20): the reference's Python (imported from /root/reference — build
container only) vs this build's C ABI through its Python mirror, same inputs,
same machine. Results must agree (asserted); prints a JSON summary.

    python tools/bench_decisions.py > profiles/r01/decisions_speed.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("FT_REFERENCE_SRC", "/root/reference/pkg/src"))

import tubesim.dataplane as r_dp  # noqa: E402
import tubesim.datastore as r_ds  # noqa: E402
import tubesim.nvlink_sched as r_nv  # noqa: E402
import tubesim.pcie_sched as r_pc  # noqa: E402
import tubesim.topology as r_tp  # noqa: E402
from tubesim.strategies import strategy_preset as r_strategy  # noqa: E402

from paper_2411_01830_b200 import dataplane as o_dp  # noqa: E402
from paper_2411_01830_b200 import datastore as o_ds  # noqa: E402
from paper_2411_01830_b200 import nvlink_sched as o_nv  # noqa: E402
from paper_2411_01830_b200 import pcie_sched as o_pc  # noqa: E402
from paper_2411_01830_b200 import topology as o_tp  # noqa: E402
from paper_2411_01830_b200.strategies import strategy_preset as o_strategy  # noqa: E402
b200_doc = o_tp.b200_doc


def per_call_us(fn, min_s=0.5):
    fn()
    n, t0 = 0, time.perf_counter()
    while True:
        fn()
        n += 1
        dt = time.perf_counter() - t0
        if dt >= min_s and n >= 20:
            return 1e6 * dt / n


def both(name, ref_fn, our_fn, note):
    r, o = per_call_us(ref_fn), per_call_us(our_fn)
    return {"row": name, "reference_us": round(r, 2), "ours_us": round(o, 2), "speedup": round(r / o, 1),
            "case": note}


rows = []

# a8 Alg. 1: select + release, B200 (NVSwitch, 1 candidate) and the V100 cube mesh
for tname, doc, s, d in (("b200_k8", b200_doc(), 0, 3),
                         ("dgx_v100", r_tp.build_preset("dgx_v100").to_dict(), 0, 7)):
    rm, om = r_tp.snapshot_matrix(r_tp.from_dict(doc)), o_tp.snapshot_matrix(o_tp.from_dict(doc))

    def ref_sel(rm=rm, s=s, d=d):
        ps = r_nv.select_paths(r_nv.PathQuery("f", s, d, rm, allow_busy=False))
        r_nv.release_paths(rm, "f")
        return ps

    def our_sel(om=om, s=s, d=d):
        ps = o_nv.select_paths(o_nv.PathQuery("f", s, d, om, allow_busy=False))
        o_nv.release_paths(om, "f")
        return ps
    assert [(p.gpus, p.b_min_gbps) for p in ref_sel()] == [(p.gpus, p.b_min_gbps) for p in our_sel()]
    rows.append(both("a8 select_paths + release_paths", ref_sel, our_sel, f"{tname}, GPU {s} -> {d}"))

# a15 partition: 16 demands (config 5's tenants)
def demands(mod, st):
    for i in range(16):
        slo = 20.0 + 7.0 * i
        st.add(mod.RateDemand(f"m{i}", (1 + i) * 16e6, slo, 0.3 * slo, arrival_ms=float(i)))
    return st


r_st, o_st = demands(r_pc, r_pc.PcieSchedulerState(55.0)), demands(o_pc, o_pc.PcieSchedulerState(55.0))
assert r_pc.partition(r_st, 5.0) == o_pc.partition(o_st, 5.0)
rows.append(both("a15 partition", lambda: r_pc.partition(r_st, 5.0), lambda: o_pc.partition(o_st, 5.0),
                 "16 demands, BW_all 55 GB/s"))

# a5/a12 fetch_plan: host -> GPU 0 striped over 8 roots; GPU 0 -> GPU 5 (claim + release)
doc = b200_doc()
r_t, o_t = r_tp.from_dict(doc), o_tp.from_dict(doc)
r_m, o_m = r_tp.snapshot_matrix(r_t), o_tp.snapshot_matrix(o_t)
r_plane = r_dp.Dataplane(r_t, r_strategy("faastube"), r_m, 2e6)
o_plane = o_dp.Dataplane(o_t, o_strategy("faastube"), o_m, 2e6)
for case, src, dst in (("host -> GPU 0, 8 PCIe roots", (0, None), (0, 0)), ("GPU 0 -> GPU 5", (0, 0), (0, 5))):
    def ref_plan(src=src, dst=dst):
        p = r_plane.fetch_plan(r_dp.Location(*src), r_dp.Location(*dst), 64 * 2.0**20)
        st = p.stages
        r_plane.release_claim(p)
        return st

    def our_plan(src=src, dst=dst):
        p = o_plane.fetch_plan(o_dp.Location(*src), o_dp.Location(*dst), 64 * 2.0**20)
        st = p.stages
        o_plane.release_claim(p)
        return st
    rs, os_ = ref_plan(), our_plan()
    assert [[(b.links, b.bytes_share) for b in s.branches] for s in rs] == \
        [[([tuple(x) for x in b.links], b.bytes_share) for b in s.branches] for s in os_]
    rows.append(both("a5/a7/a12 fetch_plan (+ stages, release)", ref_plan, our_plan, case + ", 64 MiB"))

# a19/a20 pool: allocate + free of a cached class, with histogram records
r_pool, o_pool = r_ds.MemoryPool(0), o_ds.MemoryPool(0)
r_pool.histogram("f").record_execution(0.0, 64e6, 1.0)
o_pool.histogram("f").record_execution(0.0, 64e6, 1.0)


def ref_alloc():
    b, _ = r_pool.allocate(64e6)
    r_pool.free(b)


def our_alloc():
    b, _ = o_pool.allocate(64e6)
    o_pool.free(b)


rows.append(both("a20 MemoryPool.allocate + free", ref_alloc, our_alloc, "64 MB class, warm"))
clock = [0.0]


rows.append(both("a19 FuncHistogram.record_execution", lambda: r_pool.histogram("f").record_execution(
    clock.__setitem__(0, clock[0] + 1.0) or clock[0], 64e6, 2.0),
    lambda: o_pool.histogram("f").record_execution(clock.__setitem__(0, clock[0] + 1.0) or clock[0], 64e6, 2.0),
    "1000-sample windows (p99 of interval/size/concurrency)"))

print(json.dumps({"machine": f"build container, {len(os.sched_getaffinity(0))} cores (same machine for both)",
                  "rows": rows}, indent=1))

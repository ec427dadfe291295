import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import workload
from paper_2411_01830_b200.runtime import Runtime
from paper_2411_01830_b200.tube import FaaSTube
for strategy in ("faastube", "infless_plus", "faastube"):
    tube = FaaSTube(strategy)
    wf = workload.preset_workflow("yelp")
    where = workload.place(wf, tube.topo, {}, colocate=True)
    workload.calibrate_slo(wf, tube.topo, where, 1.5)
    reqs = workload.build_requests(wf, workload.gen_workload("sporadic", 20.0, 1.0, 0), 0)
    rt = Runtime(tube, compute="sleep")
    out = rt.run([(wf, where, reqs)], 1.0, drain_s=60)
    print(strategy, json.dumps({k: out.get(k) for k in ("p50_ms", "p99_ms", "phase_p99_ms", "peak_pool_bytes", "pool_after_idle_bytes")}))
    print("  stats", tube.stats, "grow", {g: p.grow_events for g, p in tube.pools.items()})
    for r in rt.records[:6]:
        print("   ", r.rid, round(r.end_ms - r.arrival_ms, 2), {k: round(v, 2) for k, v in r.phases.items()})
    tube.close()

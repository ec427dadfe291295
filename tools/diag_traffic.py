import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import workload
from paper_2411_01830_b200.runtime import Runtime
from paper_2411_01830_b200.tube import FaaSTube
tube = FaaSTube("faastube")
wf = workload.preset_workflow("traffic")
where = workload.place(wf, tube.topo, {}, colocate=True)
workload.calibrate_slo(wf, tube.topo, where, 1.5)
print("slo", wf.slo_ms, {f.id: (f.slo_ms, f.infer_ms) for f in wf.funcs})
reqs = workload.build_requests(wf, workload.gen_workload("bursty", 10.0, 2.0, 0), 0)
rt = Runtime(tube, compute="model")
out = rt.run([(wf, where, reqs)], 2.0, drain_s=60)
print(json.dumps({k: out.get(k) for k in ("p50_ms", "p99_ms", "phase_p99_ms")}))
for r in rt.records[:12]:
    print("  ", r.rid, round(r.arrival_ms, 1), round(r.end_ms - r.arrival_ms, 1), {k: round(v, 1) for k, v in r.phases.items()})
tr = tube.pacer.trace()
t0 = tr[0][0] if tr else 0
for t, k, ev, v in tr[:120]:
    if ev != "issue":
        print(f"{t - t0:9.3f} {k} {ev} {v}")
tube.close()

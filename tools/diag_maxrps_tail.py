"""The first max-throughput trial (traffic DAG, rate 1 rps, sleep compute) run
several times on one warm tube: every request's latency and phases, so the
request that breaks the SLO can be read off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_01830_b200 import workload  # noqa: E402
from paper_2411_01830_b200.runtime import Runtime, build_requests_for  # noqa: E402
from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

strategy = sys.argv[1] if len(sys.argv) > 1 else "faastube"
tube = FaaSTube(strategy)
wf = workload.preset_workflow("traffic")
where = workload.place(wf, tube.topo, {}, colocate=tube.topo.gpu_count < len(wf.gfuncs()))
workload.calibrate_slo(wf, tube.topo, where, 1.5)
print("slo_ms", round(wf.slo_ms, 2))
for rep_i in range(3):
    reqs = build_requests_for(wf, "sporadic", 1.0, 10.0, 0)
    Runtime.warm_daemon(tube, [(wf, where, build_requests_for(wf, "sporadic", 4.0, 0.5, 1))], "sleep", 0.5)
    rt = Runtime(tube, compute="sleep")
    rep = rt.run([(wf, where, reqs)], 10.0, drain_s=30, idle_s=0.0)
    recs = sorted((r for r in rt.records if r.end_ms is not None), key=lambda r: r.arrival_ms)
    print(f"run {rep_i}: p99 {rep['p99_ms']:.2f}")
    for r in recs:
        lat = r.end_ms - r.arrival_ms
        flag = " <-- over SLO" if lat > wf.slo_ms else ""
        print(f"  rid {r.rid:3d} t={r.arrival_ms:8.1f} lat {lat:7.2f} ms",
              {k: round(v, 2) for k, v in r.phases.items() if v}, flag)
tube.close()

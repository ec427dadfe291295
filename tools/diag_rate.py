"""Why does a lone managed stage get half the link? Dump the arbiter log."""
import json, os, sys
os.environ["FT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import workload
from paper_2411_01830_b200.runtime import Runtime
from paper_2411_01830_b200.tube import FaaSTube
tube = FaaSTube("faastube")
wf = workload.preset_workflow("traffic")
where = workload.place(wf, tube.topo, {}, colocate=True)
workload.calibrate_slo(wf, tube.topo, where, 1.5)
print("pcie", tube.topo.pcie_gbps, "funcs", [(f.fid if hasattr(f, "fid") else getattr(f, "id", "?"), getattr(f, "slo_ms", None), getattr(f, "infer_ms", None)) for f in wf.gfuncs()] if hasattr(wf, "gfuncs") else "")
reqs = workload.build_requests(wf, workload.gen_workload("bursty", 10.0, 2.0, 0), 0)
Runtime.warm_daemon(tube, [(wf, where, reqs)], "sleep", 0.5)
print("after warm: state", tube.pacer.state(), "stats", tube.pacer.stats())
n0 = len(tube.pacer.log())
Runtime(tube, compute="sleep").run([(wf, where, reqs)], 1.0, drain_s=60)
for e in tube.pacer.log()[n0:n0 + 12]:
    print(json.dumps(e)[:400])
tube.close()

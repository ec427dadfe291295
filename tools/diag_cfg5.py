"""Config 5 (faastube) with marks for every slow call (> 5 ms)."""
import functools, json, os, sys, threading, time
os.environ["FT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2411_01830_b200 import device, runtime as rt_mod, tube as tube_mod
marks = []
def timed(name, fn):
    @functools.wraps(fn)
    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            d = time.perf_counter() - t0
            if d > 0.005:
                marks.append((round(t0 % 1000, 4), round(d * 1e3, 2), threading.current_thread().name[-6:], name))
    return w
for n in ("_maybe_free", "_retire", "fetch", "store", "_out", "_respond", "response", "release", "_store_locked", "_pinned"):
    setattr(tube_mod.FaaSTube, n, timed(n, getattr(tube_mod.FaaSTube, n)))
device.Pacer.submit = timed("submit", device.Pacer.submit)
device.DevicePool.allocate = timed("allocate", device.DevicePool.allocate)
device.DevicePool.shrink = timed("shrink", device.DevicePool.shrink)
device.LIB.ft_vmm_block_unmap  # resolve
_unmap = device.LIB.ft_vmm_block_unmap
device.LIB.ft_vmm_block_unmap = timed("vmm_unmap", _unmap)
_map = device.LIB.ft_vmm_block_map
device.LIB.ft_vmm_block_map = timed("vmm_map", _map)
rt_mod.Runtime._compute = timed("_compute", rt_mod.Runtime._compute)
torch.cuda.Stream.synchronize = timed("stream.sync", torch.cuda.Stream.synchronize)
torch.cuda.Event.synchronize = timed("event.sync", torch.cuda.Event.synchronize)
orig_run = rt_mod.Runtime._run
def run(self, *a, **k):
    marks.clear()
    out = orig_run(self, *a, **k)
    print("RUN", json.dumps({k2: out.get(k2) for k2 in ("p50_ms", "p99_ms", "phase_p99_ms")}), flush=True)
    for m in sorted(marks, key=lambda m: -m[1])[:25]:
        print("  mark", m)
    tr = self.tube.pacer.trace()
    st = {}
    for t, tk, kind, v in tr:
        if tk:
            st.setdefault(tk, []).append((round(t, 2), kind, round(v, 2) if isinstance(v, float) else v))
    durs = sorted(((ev[-1][0] - ev[0][0]), tk) for tk, ev in st.items() if ev[-1][1] == "land")
    for d, tk in durs[-2:]:
        ev = st[tk]
        print("  stage", tk, round(d, 2), "ms", ev, "n", len(ev))
    print("  guards", sum(1 for x in tr if x[2] == "guard"), "stages", len(st))
    slow = sorted(self.records, key=lambda r: -(r.end_ms - r.arrival_ms))[:5]
    for r in slow:
        print("  slow", r.rid, r.workflow, round(r.arrival_ms, 1), round(r.end_ms - r.arrival_ms, 2), {k2: round(v, 2) for k2, v in r.phases.items()})
    return out
rt_mod.Runtime._run = run
if len(sys.argv) > 1:
    # config 4 only, faastube only
    from paper_2411_01830_b200 import workload
    from paper_2411_01830_b200.runtime import Runtime
    from paper_2411_01830_b200.tube import FaaSTube
    for rep in range(2):
        tube = FaaSTube("faastube")
        wf = workload.preset_workflow("traffic")
        where = workload.place(wf, tube.topo, {}, colocate=True)
        workload.calibrate_slo(wf, tube.topo, where, 1.5)
        reqs = workload.build_requests(wf, workload.gen_workload("bursty", 10.0, 2.0, 0), 0)
        Runtime.warm_daemon(tube, [(wf, where, reqs)], "model", 0.5)
        Runtime(tube, compute="model").run([(wf, where, reqs)], 2.0, drain_s=60)
        print("stats", tube.stats)
        tube.close()
else:
    out = bench.run_workflows()

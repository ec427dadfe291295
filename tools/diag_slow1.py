"""Traffic at 1 rps Poisson for 10 s (faastube): where does a 700 ms request come from?"""
import functools, json, os, sys, threading, time
os.environ["FT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import workload, device, tube as tube_mod
from paper_2411_01830_b200.runtime import Runtime, build_requests_for
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
                marks.append((round(t0 % 1000, 3), round(d * 1e3, 2), threading.current_thread().name[-6:], name))
    return w
for n in ("fetch", "store", "_out", "_respond", "response", "release", "_store_locked", "_pinned", "_check_pressure", "_migrate_out", "_maybe_prefetch"):
    setattr(tube_mod.FaaSTube, n, timed(n, getattr(tube_mod.FaaSTube, n)))
device.Pacer.submit = timed("submit", device.Pacer.submit)
device.Pacer.submit_d2h = timed("submit_d2h", device.Pacer.submit_d2h)
device.Pacer.wait = timed("pacer.wait", device.Pacer.wait)
device.DevicePool.allocate = timed("allocate", device.DevicePool.allocate)
device.DevicePool.shrink = timed("shrink", device.DevicePool.shrink)
device.DevicePool.reclaim = timed("reclaim", device.DevicePool.reclaim)
torch.cuda.Stream.synchronize = timed("stream.sync", torch.cuda.Stream.synchronize)
tube = tube_mod.FaaSTube("faastube")
wf = workload.preset_workflow("traffic")
where = workload.place(wf, tube.topo, {}, colocate=True)
workload.calibrate_slo(wf, tube.topo, where, 1.5)
print("slo", wf.slo_ms, [(f.fid if hasattr(f,'fid') else None) for f in []])
Runtime.warm_daemon(tube, [(wf, where, build_requests_for(wf, "sporadic", 4.0, 0.5, 1))], "sleep", 0.5)
if len(sys.argv) > 1:   # the max-throughput trial's own warm-up
    time.sleep(1.5)
    Runtime.warm_daemon(tube, [(wf, where, build_requests_for(wf, "sporadic", 4.0, 0.5, 1))], "sleep", 0.5)
marks.clear()
reqs = build_requests_for(wf, "sporadic", 1.0, 10.0, 0)
rt = Runtime(tube, compute="sleep")
t0 = time.perf_counter()
out = rt.run([(wf, where, reqs)], 10.0, drain_s=30, idle_s=0.0)
print(json.dumps({k: out.get(k) for k in ("p50_ms", "p99_ms", "phase_p99_ms")}))
for r in sorted(rt.records, key=lambda r: -(r.end_ms - r.arrival_ms))[:4]:
    print("slow", r.rid, round(r.arrival_ms, 1), round(r.end_ms - r.arrival_ms, 1), {k: round(v, 1) for k, v in r.phases.items()})
slowest = max(rt.records, key=lambda r: r.end_ms - r.arrival_ms)
print("slowest window", round(slowest.arrival_ms, 1), round(slowest.end_ms, 1))
for m in sorted(marks, key=lambda m: -m[1])[:20]:
    print("mark", m)
print("stats", tube.stats, tube.pacer.stats())
tr = tube.pacer.trace()
st = {}
for t, tk, kind, v in tr:
    if tk: st.setdefault(tk, []).append((round(t, 1), kind, v))
durs = sorted(((ev[-1][0] - ev[0][0]), tk) for tk, ev in st.items() if ev[-1][1] == "land")
for d, tk in durs[-3:]:
    print("stage", tk, d, st[tk][:5], st[tk][-3:])
print("guards", sum(1 for x in tr if x[2] == "guard"))
tube.close()

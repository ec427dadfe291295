"""Yelp runtime after heavy pacer traffic, with pacer traces of slow stages."""
import json, os, sys, time
os.environ["FT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from paper_2411_01830_b200 import workload, device
from paper_2411_01830_b200.runtime import Runtime
from paper_2411_01830_b200.tube import FaaSTube
if len(sys.argv) > 1 and sys.argv[1] == "pre":
    import subprocess
    # run the GPU test files that precede test_gpu_runtime, in this process
    import pytest
    rc = pytest.main(["-q", "-m", "gpu", "-x", "tests/test_gpu_ipc.py", "tests/test_gpu_migration.py",
                      "tests/test_gpu_movers.py", "tests/test_gpu_pacer.py", "tests/test_gpu_pairs.py"])
    print("pre done", rc, flush=True)
import threading, functools
from paper_2411_01830_b200 import tube as tube_mod, runtime as rt_mod
marks = []
def timed(name, fn):
    @functools.wraps(fn)
    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            d = time.perf_counter() - t0
            if d > 0.01:
                marks.append((threading.current_thread().name, name, round(t0 % 1000, 4), round(d * 1e3, 2)))
    return w
for n in ("fetch", "store", "_out", "_host_to_gpu", "_respond", "_execute", "_maybe_free", "response", "release"):
    setattr(tube_mod.FaaSTube, n, timed(n, getattr(tube_mod.FaaSTube, n)))
device.Pacer.submit = timed("submit", device.Pacer.submit)
device.DevicePool.allocate = timed("allocate", device.DevicePool.allocate)
device.DevicePool.shrink = timed("shrink", device.DevicePool.shrink)
_sync = torch.cuda.Stream.synchronize
torch.cuda.Stream.synchronize = timed("stream.sync", _sync)
for strategy in ("faastube", "infless_plus", "faastube"):
    marks.clear()
    print("pinned cache / torch mem", torch.cuda.memory_reserved() >> 20, "MiB reserved", flush=True)
    tube = FaaSTube(strategy)
    wf = workload.preset_workflow("yelp")
    where = workload.place(wf, tube.topo, {}, colocate=True)
    workload.calibrate_slo(wf, tube.topo, where, 1.5)
    reqs = workload.build_requests(wf, workload.gen_workload("sporadic", 20.0, 1.0, 0), 0)
    rt = Runtime(tube, compute="sleep")
    out = rt.run([(wf, where, reqs)], 1.0, drain_s=60)
    print(strategy, "pcie", tube.topo.pcie_gbps, json.dumps({k: out.get(k) for k in ("p50_ms", "p99_ms", "phase_p99_ms")}), flush=True)
    print("  funcs", {f.id: (round(f.slo_ms, 2) if f.slo_ms else None, f.infer_ms) for f in wf.functions} if hasattr(wf, "functions") else "")
    recs = sorted(rt.records, key=lambda r: -(r.end_ms - r.arrival_ms))[:4]
    for r in recs:
        print("   slow", r.rid, round(r.end_ms - r.arrival_ms, 2), {k: round(v, 2) for k, v in r.phases.items()})
    tr = tube.pacer.trace()
    st = {}
    for t, tk, kind, v in tr:
        st.setdefault(tk, []).append((round(t, 3), kind, v))
    durs = sorted(((ev[-1][0] - ev[0][0]), tk) for tk, ev in st.items() if tk and ev[-1][1] == "land")
    for d, tk in durs[-3:]:
        print("   stage", tk, round(d, 2), "ms", st[tk][:6], "...", st[tk][-2:])
    print("   guards", sum(1 for x in tr if x[2] == "guard"), "log tail", tube.pacer.log()[-3:])
    for m in marks[:40]:
        print("   mark", m)
    tube.close()

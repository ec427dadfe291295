"""Isolation scenario with the pacer's arbiter log (FT_TRACE)."""
import json, os, sys
os.environ["FT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_sched as T
from paper_2411_01830_b200 import tube as tube_mod
from paper_2411_01830_b200.tube import measure_pcie_gbps
orig = tube_mod.FaaSTube.close
logs = []
def close(self):
    logs.append((self.pacer.log(), self.pacer.trace()))
    return orig(self)
tube_mod.FaaSTube.close = close
import threading, time, functools
marks = []
def timed(name, fn):
    @functools.wraps(fn)
    def w(*a, **k):
        t0 = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            marks.append((threading.current_thread().name, name, t0, time.perf_counter()))
    return w
tube_mod.FaaSTube.fetch = timed("fetch", tube_mod.FaaSTube.fetch)
tube_mod.FaaSTube._out = timed("_out", tube_mod.FaaSTube._out)
tube_mod.FaaSTube._host_to_gpu = timed("_host_to_gpu", tube_mod.FaaSTube._host_to_gpu)
from paper_2411_01830_b200 import device as devmod
devmod.Pacer.submit = timed("submit", devmod.Pacer.submit)
link = measure_pcie_gbps([0])
print("link", link)
for s in ("faastube", "faastube_star"):
    print(s, T._contend(s, link))
m0 = min(m[2] for m in marks)
for th, name, a, b in sorted(marks, key=lambda m: m[2])[:60]:
    print(f"{th:12s} {name:14s} {1e3*(a-m0):9.3f} -> {1e3*(b-m0):9.3f}")
log, tr = logs[0]
t0 = log[0][0] if log else 0
for t, call, key, dec, *_ in log[:80]:
    short = []
    for d in dec:
        if d[0] == "partition":
            short.append("P" + json.dumps({k: round(v, 3) for k, v in d[1].items()}))
        else:
            short.append(json.dumps([round(x, 3) if isinstance(x, float) else x for x in d]))
    print(f"{t - t0:9.3f} {call:8s} {key:4s} " + " ".join(short))
print("trace")
last = {}
for t, tk, kind, v in tr:
    if kind != "issue" or t - last.get(tk, -1e9) > 3.0:
        print(f"{t - t0:9.3f} {tk} {kind} {v}")
    if kind == "issue":
        last[tk] = t

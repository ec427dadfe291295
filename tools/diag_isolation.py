import json, os, sys, time, threading
os.environ["FT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import test_gpu_sched as T
from paper_2411_01830_b200 import tube as tube_mod
orig = tube_mod.FaaSTube.close
traces = []
def close(self):
    traces.append(list(self._trace or []))
    return orig(self)
tube_mod.FaaSTube.close = close
for s in ("faastube", "faastube_star", "faastube"):
    print(s, T._contend(s))
tr = traces[-1]
t0 = tr[0][0] if tr else 0
last = {}
for t, k, ev, v in tr:
    if ev != "issue" or k not in last or t - last[k] > 2.0:
        print(f"{t - t0:8.3f} {k} {ev} {v}")
    if ev == "issue":
        last[k] = t

import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200.tube import FaaSTube
h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
t0 = time.perf_counter()
for _ in range(1000):
    h.is_pinned()
print("is_pinned us", (time.perf_counter() - t0) * 1e3)
for strat in ("faastube", "faastube_star", "faastube"):
    tube = FaaSTube(strat)
    for i in range(3):
        d = tube.unique_id()
        tube.store(d, h)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x = tube.fetch(d, device=0, slo_ms=100.0, infer_ms=10.0)
        torch.cuda.synchronize()
        print(strat, "256MB fetch ms", round((time.perf_counter() - t0) * 1e3, 3), tube.stats.get("managed_stages"))
    tube.close()

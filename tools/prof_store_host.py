import sys, time, statistics, cProfile, pstats
sys.path.insert(0, "/root/repo")
import torch
from paper_2411_01830_b200.tube import FaaSTube
tube = FaaSTube("faastube", gpus=[0], pcie_gbps=55.0)
host = torch.empty(1 << 20, dtype=torch.uint8).pin_memory()
ts = []
ids = []
for i in range(3000):
    d = tube.unique_id()
    t0 = time.perf_counter(); tube.store(d, host); ts.append(time.perf_counter() - t0)
    ids.append(d)
    if len(ids) > 100:
        tube.release(ids.pop(0))
print("store pinned host us p50", round(1e6 * statistics.median(ts[300:]), 2))
pr = cProfile.Profile(); pr.enable()
for i in range(2000):
    d = tube.unique_id(); tube.store(d, host); tube.release(d)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
tube.close()

import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200.tube import FaaSTube
tube = FaaSTube("faastube")
x = torch.ones(4096, dtype=torch.uint8, device="cuda:0")
def loop(n):
    ts_s, ts_f = [], []
    for _ in range(n):
        d = tube.unique_id()
        t0 = time.perf_counter(); tube.store(d, x); t1 = time.perf_counter()
        v = tube.fetch(d, device=0); t2 = time.perf_counter()
        del v
        ts_s.append(t1 - t0); ts_f.append(t2 - t1)
    ts_s.sort(); ts_f.sort()
    return 1e6 * ts_s[n // 2], 1e6 * ts_f[n // 2]
loop(500)
print("store us p50 %.1f  view-fetch us p50 %.1f" % loop(3000))
pr = cProfile.Profile(); pr.enable(); loop(3000); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

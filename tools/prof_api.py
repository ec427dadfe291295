"""Host-side cost of the put/get API (run on the GPU box): per-call latency of
store+fetch for small payloads, plus a cProfile of the hot Python frames."""
import cProfile
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

tube = FaaSTube("faastube")
x = torch.ones(4096, dtype=torch.uint8, device="cuda:0")
out = torch.empty_like(x)


def loop(n, zero_copy):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        d = tube.unique_id()
        tube.store(d, x)
        v = tube.fetch(d, device=0) if zero_copy else tube.fetch(d, device=0, out=out)
        ts.append(time.perf_counter() - t0)
        del v
    return ts


loop(200, False)
loop(200, True)
for zc in (False, True):
    ts = sorted(loop(2000, zc))
    print(f"zero_copy={zc}: store+fetch host us p50 {1e6 * ts[len(ts) // 2]:.1f} p99 {1e6 * ts[int(len(ts) * .99)]:.1f}")
pr = cProfile.Profile()
pr.enable()
loop(2000, False)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
torch.cuda.synchronize()

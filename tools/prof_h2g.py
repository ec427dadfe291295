"""Host cost of the e2e step's API calls on the GPU box: store(host payload)
and fetch(host -> GPU) for a small payload (the fixed cost in front of the
first DMA), plus a cProfile of the hot Python frames."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

tube = FaaSTube("faastube")
n = int(os.environ.get("N", 4096))
host = torch.ones(n, dtype=torch.uint8).pin_memory()
out = torch.empty(n, dtype=torch.uint8, device="cuda:0")


def loop(k):
    a, b = [], []
    for _ in range(k):
        t0 = time.perf_counter()
        d = tube.unique_id()
        tube.store(d, host, producer="decode")
        t1 = time.perf_counter()
        tube.fetch(d, device=0, out=out, consumer="producer")
        t2 = time.perf_counter()
        torch.cuda.current_stream().synchronize()
        a.append(t1 - t0)
        b.append(t2 - t1)
    return sorted(a), sorted(b)


loop(200)
a, b = loop(2000)
print(f"store(host) us p50 {1e6 * a[len(a) // 2]:.1f}   fetch(h2g submit) us p50 {1e6 * b[len(b) // 2]:.1f} "
      f"p99 {1e6 * b[int(len(b) * .99)]:.1f}")
pr = cProfile.Profile()
pr.enable()
loop(2000)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
tube.close()

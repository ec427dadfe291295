"""Host cost of the same-GPU put/get API (profile for the small-message path):
per-call wall time of store / fetch(out=) / zero-copy fetch / fetch_many, and a
cProfile of the store+fetch loop.   python tools/prof_api.py [bytes]"""
import cProfile
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
tube = FaaSTube("faastube", gpus=[0], pcie_gbps=55.0)
x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
y = torch.empty_like(x)
torch.cuda.synchronize()


def loop(k, fetch_mode="out"):
    st, ft = [], []
    for _ in range(k):
        d = tube.unique_id()
        t0 = time.perf_counter()
        tube.store(d, x)
        t1 = time.perf_counter()
        if fetch_mode == "out":
            tube.fetch(d, device=0, out=y)
        else:
            v = tube.fetch(d, device=0)
            del v
        t2 = time.perf_counter()
        st.append(t1 - t0)
        ft.append(t2 - t1)
    torch.cuda.synchronize()
    return statistics.median(st) * 1e6, statistics.median(ft) * 1e6


loop(200)
print(f"bytes={n} store_us={loop(2000)[0]:.1f} fetch_out_us={loop(2000)[1]:.1f} "
      f"fetch_view_us={loop(2000, 'view')[1]:.1f}")
xs = torch.randint(0, 256, (64, n), dtype=torch.uint8, device="cuda:0")
ys = torch.empty_like(xs)
ts = []
for r in range(20):
    ids = []
    for j in range(64):
        d = tube.unique_id()
        tube.store(d, xs[j])
        ids.append(d)
    items = [(d, ys[j]) for j, d in enumerate(ids)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tube.fetch_many(items)
    ts.append(time.perf_counter() - t0)
torch.cuda.synchronize()
assert torch.equal(xs, ys)
print(f"fetch_many 64 x {n}: host {statistics.median(ts) * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
loop(2000)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
pr = cProfile.Profile()
for r in range(10):
    ids = []
    for j in range(64):
        d = tube.unique_id()
        tube.store(d, xs[j])
        ids.append(d)
    items = [(d, ys[j]) for j, d in enumerate(ids)]
    torch.cuda.synchronize()
    pr.enable()
    tube.fetch_many(items)
    pr.disable()
print("---- fetch_many profile")
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
tube.close()

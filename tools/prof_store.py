"""Host time of a same-GPU store (1 MiB) split into its pieces (pool allocate, the
native store_local call, record_stream, the shrink timer, _after_store) and of a
fetch(out=) (the native fetch_local call vs the rest).   python tools/prof_store.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402
from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

tube = FaaSTube("faastube", gpus=[0], pcie_gbps=55.0)
x = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device="cuda:0")
y = torch.empty_like(x)
acc = {}


def timed(name, fn):
    def w(*a, **kw):
        t0 = time.perf_counter()
        try:
            return fn(*a, **kw)
        finally:
            acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
    return w


pool = tube.pools[0]
for name in ("allocate", "store_local", "fetch_local"):
    setattr(pool, name, timed(name, getattr(pool, name)))
for name in ("_push_due", "_after_store", "_reap", "_store_locked", "_fetch_local"):
    setattr(tube, name, timed(name, getattr(tube, name)))
dev.LIB.ft_store_local = timed("ft_store_local(native)", dev.LIB.ft_store_local)
dev.LIB.ft_fetch_local = timed("ft_fetch_local(native)", dev.LIB.ft_fetch_local)
rows = {"store": [], "fetch": []}
parts = {"store": [], "fetch": []}
for i in range(3000):
    d = tube.unique_id()
    acc.clear()
    t0 = time.perf_counter()
    tube.store(d, x)
    t1 = time.perf_counter()
    ps = dict(acc)
    acc.clear()
    t2 = time.perf_counter()
    tube.fetch(d, device=0, out=y)
    t3 = time.perf_counter()
    if i >= 300:
        rows["store"].append(t1 - t0)
        rows["fetch"].append(t3 - t2)
        parts["store"].append(ps)
        parts["fetch"].append(dict(acc))
    if i % 64 == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
med = statistics.median
for op in ("store", "fetch"):
    names = sorted({k for p in parts[op] for k in p})
    print(f"{op}: {1e6 * med(rows[op]):.1f} us; " +
          ", ".join(f"{k} {1e6 * med(p.get(k, 0.0) for p in parts[op]):.1f}" for k in names))
tube.close()

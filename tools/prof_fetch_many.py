"""Host time of fetch_many (64 x 1 MiB same-GPU objects) split into its native
pieces (wait_events, copy_batch_flat, retire_many) and the Python remainder.
python tools/prof_fetch_many.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402
from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

tube = FaaSTube("faastube", gpus=[0], pcie_gbps=55.0)
n, k = 1 << 20, 64
xs = torch.randint(0, 256, (k, n), dtype=torch.uint8, device="cuda:0")
ys = torch.empty_like(xs)
acc = {}


def timed(name, fn):
    def w(*a, **kw):
        t0 = time.perf_counter()
        try:
            return fn(*a, **kw)
        finally:
            acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
    return w


dev.wait_events = timed("wait_events", dev.wait_events)
dev.copy_batch_flat = timed("copy_batch_flat", dev.copy_batch_flat)
dev.DevicePool.retire_many = timed("retire_many", dev.DevicePool.retire_many)
dev.LIB.ft_retire_many = timed("ft_retire_many(native)", dev.LIB.ft_retire_many)
dev.LIB.ft_copy_batch = timed("ft_copy_batch(native)", dev.LIB.ft_copy_batch)
tube._push_due = timed("_push_due", tube._push_due)
tube._reap = timed("_reap", tube._reap)
tot, parts = [], []
for r in range(60):
    ids = []
    for j in range(k):
        d = tube.unique_id()
        tube.store(d, xs[j])
        ids.append(d)
    items = [(d, ys[j]) for j, d in enumerate(ids)]
    torch.cuda.synchronize()
    acc.clear()
    t0 = time.perf_counter()
    tube.fetch_many(items)
    t = time.perf_counter() - t0
    if r >= 10:
        tot.append(t)
        parts.append(dict(acc))
torch.cuda.synchronize()
assert torch.equal(xs, ys)
med = statistics.median
print(f"fetch_many {k} x {n}: host {1e6 * med(tot):.1f} us; " +
      ", ".join(f"{name} {1e6 * med(p.get(name, 0.0) for p in parts):.1f}" for name in
                ("_reap", "wait_events", "copy_batch_flat", "ft_copy_batch(native)", "retire_many",
                 "ft_retire_many(native)", "_push_due")))
tube.close()

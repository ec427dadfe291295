"""Device time of the copy engines at small sizes (pre-queued behind a device
spin, so events time the kernel, not the launch):  k_copy_bulk vs k_copy_vec
vs k_copy_multi (64 segments) and the CE, 4 KiB .. 16 MiB."""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402

s = torch.cuda.current_stream(0)


def spin(ns):
    dev.LIB.ft_spin_ns(int(ns), 0, C.c_void_p(s.cuda_stream))


def timed(fn, reps=30):
    ts = []
    for _ in range(reps):
        spin(50_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        ts.append((a, b))
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ts[3:]) * 1e3   # us


for lg in range(12, 25):
    n = 1 << lg
    x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    y = torch.empty_like(x)
    row = {"bytes": n}
    row["bulk_us"] = timed(lambda: dev.copy(y.data_ptr(), x.data_ptr(), n, 0, s, dev.ENGINE_BULK))
    row["vec_us"] = timed(lambda: dev.copy(y.data_ptr(), x.data_ptr(), n, 0, s, dev.ENGINE_VEC))
    row["ce_us"] = timed(lambda: y.copy_(x))
    row["empty_spin_us"] = timed(lambda: None)
    assert torch.equal(x, y)
    print(" ".join(f"{k}={v:.2f}" if isinstance(v, float) else f"{k}={v}" for k, v in row.items()), flush=True)
for lg in (12, 16, 20):
    m = 1 << lg
    xs = torch.randint(0, 256, (64, m), dtype=torch.uint8, device="cuda:0")
    ys = torch.empty_like(xs)
    segs = [(ys[j].data_ptr(), xs[j].data_ptr(), m) for j in range(64)]
    us = timed(lambda: dev.copy_batch(segs, 0, s))
    assert torch.equal(xs, ys)
    print(f"multi 64 x {m}: {us:.2f} us = {64 * m / us / 1e3:.1f} GB/s", flush=True)

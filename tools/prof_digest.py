"""Digest kernel (k_fingerprint) over 64 MiB: event-timed, for ncu capture."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
n = 64 << 20
x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
fp = dev.Fingerprint(0)
s = torch.cuda.current_stream()
ts = []
for i in range(30):
    flush.fill_(i & 0xFF)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); fp.launch(x.data_ptr(), n, s); b.record(s)
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(a.elapsed_time(b))
assert fp.value() == dev.fingerprint_host(x.cpu())
ms = statistics.median(ts)
print(f"k_fingerprint 64 MiB: {ms*1e3:.2f} us -> {n / ms / 1e6:.0f} GB/s")

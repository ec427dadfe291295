"""Where does the pacer's per-stage overhead go? (64 MiB pinned H2D)"""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev

n = 64 << 20
host = torch.empty(n, dtype=torch.uint8).pin_memory(); host.fill_(5)
dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
s0 = torch.cuda.current_stream(0)
ce, fw = torch.cuda.Stream(0), torch.cuda.Stream(0)
p = dev.Pacer(55.0, 5, 2 * 10**6)

def wall(name, fn, reps=20, warm=3):
    ts = []
    for i in range(warm + reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); t1 = time.perf_counter()
        if i >= warm: ts.append((t1 - t0) * 1e3)
    ts.sort()
    print(f"{name:40s} p50 {ts[len(ts)//2]:.3f} ms  min {ts[0]:.3f}  -> {n/ts[len(ts)//2]/1e6:.1f} GB/s", flush=True)

wall("pcie_copy on default stream", lambda: dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, 0, s0))
wall("pcie_copy on torch side stream", lambda: dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, 0, ce))
wall("pcie_copy 10MB ops side stream", lambda: dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, 0, ce, 10**7))
r = [(0, 0, 0, n, ce.cuda_stream, fw.cuda_stream)]
wall("pacer unmanaged", lambda: p.submit("", False, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True, r, s0.cuda_stream))
wall("pacer managed", lambda: p.submit("", True, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True, r, s0.cuda_stream))
def timed_submit(managed):
    t0 = time.perf_counter()
    t = p.submit("", managed, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True, r, s0.cuda_stream)
    t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    p.wait(t); t3 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t0) * 1e3, (t3 - t0) * 1e3
for m in (False, True):
    xs = [timed_submit(m) for _ in range(10)]
    print("managed" if m else "unmanaged", "submit/sync/landed ms", [tuple(round(v, 3) for v in x) for x in xs[-4:]], flush=True)
# device-side duration of the DMA on the CE stream
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for m in (False, True):
    torch.cuda.synchronize()
    a.record(ce)
    p.submit("", m, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True, r, s0.cuda_stream)
    b.record(ce)
    torch.cuda.synchronize()
    print("device time on ce", m, round(a.elapsed_time(b), 3), flush=True)
p.close()

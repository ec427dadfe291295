"""GPU -> host through FaaSTube.fetch(device=None) (managed d2h stage) vs the CE peak."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
from paper_2411_01830_b200.tube import FaaSTube
tube = FaaSTube("faastube", capacity_limit_bytes=64e9)
for n in (1 << 20, 64 << 20, 1 << 30):
    x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    out = torch.empty(n, dtype=torch.uint8).pin_memory()
    s = torch.cuda.current_stream(0)
    ce = []
    for _ in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        dev.pcie_copy(out.data_ptr(), x.data_ptr(), n, False, 0, s); s.synchronize()
        ce.append(time.perf_counter() - t0)
    ts = []
    for i in range(6):
        did = tube.unique_id(); tube.store(did, x, producer="p")
        torch.cuda.synchronize(); t0 = time.perf_counter()
        tube.fetch(did, device=None, out=out, consumer="sink")
        ts.append(time.perf_counter() - t0)
    assert torch.equal(out[-4096:], x[-4096:].cpu())
    print(f"{n:>11d} B  CE {n / min(ce) / 1e9:6.2f} GB/s   tube d2h p50 {n / sorted(ts)[len(ts) // 2] / 1e9:6.2f} GB/s "
          f"({1e3 * sorted(ts)[len(ts) // 2]:.3f} ms)")
tube.close()

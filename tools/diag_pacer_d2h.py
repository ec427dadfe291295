"""Pacer d2h stages (GPU -> pinned host) vs one CE op: managed/unmanaged, 64 MiB and 1 GiB."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
for n in (64 << 20, 1 << 30):
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    s0 = torch.cuda.current_stream(0)
    ce, fw = dev.new_stream(0), dev.new_stream(0)
    p = dev.Pacer(55.0, 5, 2 * 10**6)
    r = [(0, 0, 0, n, ce.cuda_stream, fw.cuda_stream)]
    def wall(name, fn, reps=6):
        ts = []
        for i in range(reps + 2):
            torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); t1 = time.perf_counter()
            if i >= 2: ts.append(t1 - t0)
        ts.sort(); print(f"{n:>11d} {name:28s} {n / ts[len(ts) // 2] / 1e9:6.2f} GB/s", flush=True)
    wall("CE one op", lambda: dev.pcie_copy(host.data_ptr(), src.data_ptr(), n, False, 0, ce))
    wall("CE 10 MB ops", lambda: dev.pcie_copy(host.data_ptr(), src.data_ptr(), n, False, 0, ce, 10**7))
    wall("CE 20 MB ops", lambda: dev.pcie_copy(host.data_ptr(), src.data_ptr(), n, False, 0, ce, 2 * 10**7))
    for m in (False, True):
        wall(f"pacer d2h managed={m}", lambda: p.wait(p.submit_d2h("", m, 1e9, 0.0, 55.0, host.data_ptr(),
                                                                   src.data_ptr(), 0, n, r, s0.cuda_stream)))
    assert torch.equal(host[-4096:], src[-4096:].cpu())
    p.close()

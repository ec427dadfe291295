"""Why does the start-up PCIe calibration read low? variants of the same 64 MiB H2D loop."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
n = 64 << 20
def run(name, host, s, reps=12):
    dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    for _ in range(4):
        dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, 0, s)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(s)
    for i in range(reps):
        dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, 0, s)
        ev[i + 1].record(s)
    ev[-1].synchronize()
    ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]
    print(f"{name:40s} best {n / min(ts) / 1e6:6.1f} GB/s  median {n / sorted(ts)[reps // 2] / 1e6:6.1f}", flush=True)
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
run("pin_memory() of empty, torch stream", h1, torch.cuda.Stream(0))
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
run("empty(pin_memory=True), torch stream", h2, torch.cuda.Stream(0))
h2.fill_(3)
run("  same after fill_", h2, torch.cuda.Stream(0))
run("pin_memory() of empty, private stream", h1, dev.new_stream(0))
h1.fill_(7)
run("pin_memory() after fill_", h1, torch.cuda.Stream(0))
run("pin_memory() after fill_, again", h1, torch.cuda.Stream(0))

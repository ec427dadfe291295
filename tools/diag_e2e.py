"""Where does the e2e pass time go? (run on the GPU box)"""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
from paper_2411_01830_b200.tube import FaaSTube

g = 0
n = 64 << 20
host = torch.empty(n, dtype=torch.uint8).pin_memory(); host.fill_(5)
dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
inp = torch.empty_like(dst)
s = torch.cuda.current_stream(0)

def wall(fn, reps=20, warm=3):
    ts = []
    for i in range(warm + reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); t1 = time.perf_counter()
        if i >= warm: ts.append((t1 - t0) * 1e3)
    ts.sort()
    return f"p50 {ts[len(ts)//2]:.3f} ms  mean {statistics.mean(ts):.3f} ms  -> {n/statistics.mean(ts)/1e6:.1f} GB/s"

print("CE one op   ", wall(lambda: dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, g, s)))
print("CE 10MB ops ", wall(lambda: dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, g, s, 10 * 10**6)))
print("CE 2MB ops  ", wall(lambda: dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, g, s, 2 * 10**6)))
for strat in ("faastube", "faastube_star"):
    tube = FaaSTube(strat)
    def h2g():
        d = tube.unique_id(); tube.store(d, host, producer="decode"); tube.fetch(d, device=0, out=dst, consumer="p")
    print(strat, "fetch H2G  ", wall(h2g))
    fp = dev.Fingerprint(0)
    def e2e():
        d = tube.unique_id(); tube.store(d, host, producer="decode"); tube.fetch(d, device=0, out=dst, consumer="p")
        d = tube.unique_id(); tube.store(d, dst, producer="p"); tube.fetch(d, device=0, out=inp, consumer="c")
        fp.launch(inp.data_ptr(), n, s); fp.value()
    print(strat, "e2e        ", wall(e2e))
    if os.environ.get("FT_TRACE"):
        for t in tube.pacer.trace()[-30:]: print("  ", t)
    tube.close()

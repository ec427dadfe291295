"""Pageable host payload -> GPU through the pacer's pinned ring (workers memcpy + DMA)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200.tube import FaaSTube
tube = FaaSTube("faastube")
n = 1 << 30
pg = torch.randint(0, 256, (n,), dtype=torch.uint8)          # pageable
pn = pg.clone().pin_memory()
out = torch.empty(n, dtype=torch.uint8, device="cuda:0")
for name, h in (("pinned", pn), ("pageable", pg)):
    ts = []
    for i in range(4):
        d = tube.unique_id(); tube.store(d, h, producer="gw")
        torch.cuda.synchronize(); t0 = time.perf_counter()
        tube.fetch(d, out=out); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    assert torch.equal(out[:4096].cpu(), h[:4096]) and torch.equal(out[-4096:].cpu(), h[-4096:])
    print(name, [round(n / t / 1e9, 1) for t in ts], "GB/s", flush=True)
t0 = time.perf_counter(); x = pg.clone(); t1 = time.perf_counter()
print("host memcpy 1 thread (clone)", round(n / (t1 - t0) / 1e9, 1), "GB/s; cores", len(os.sched_getaffinity(0)))
tube.close()

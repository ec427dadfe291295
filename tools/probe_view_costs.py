import os, statistics, sys, time, weakref
sys.path.insert(0, "/root/repo")
import torch
from paper_2411_01830_b200.tube import FaaSTube
tube = FaaSTube("faastube", gpus=[0], pcie_gbps=55.0)
x = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device="cuda:0")
fv, rel, fin, sl = [], [], [], []
blk_view = None
for i in range(3000):
    d = tube.unique_id(); tube.store(d, x)
    t0 = time.perf_counter(); v = tube.fetch(d, device=0); t1 = time.perf_counter()
    del v; t2 = time.perf_counter()
    if i >= 300: fv.append(t1 - t0); rel.append(t2 - t1)
    if i % 64 == 0: torch.cuda.synchronize()
o = tube._objs  # noqa
def cb(): pass
for i in range(3000):
    t = x[:10]
    t0 = time.perf_counter(); weakref.finalize(t, cb); t1 = time.perf_counter()
    fin.append(t1 - t0)
    t0 = time.perf_counter(); y = x[:4096].view(torch.uint8).view((4096,)); t1 = time.perf_counter()
    sl.append(t1 - t0)
med = statistics.median
print(f"fetch view {1e6*med(fv):.1f} us, release {1e6*med(rel):.1f} us, weakref.finalize {1e6*med(fin):.2f} us, slice+views {1e6*med(sl):.2f} us")
tube.close()

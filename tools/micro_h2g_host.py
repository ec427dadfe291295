import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2411_01830_b200 import device as dev
from paper_2411_01830_b200.tube import FaaSTube
tube = FaaSTube("faastube", gpus=[0], pcie_gbps=55.0)
s = torch.cuda.Stream(0); torch.cuda.set_stream(s)
host = torch.empty(1<<20, dtype=torch.uint8, pin_memory=True)
dst = torch.empty(1<<20, dtype=torch.uint8, device="cuda:0")
def t(name, fn, n=20000):
    for _ in range(200): fn()
    t0=time.perf_counter()
    for _ in range(n): fn()
    print(f"{name}: {(time.perf_counter()-t0)/n*1e6:.2f} us")
t("is_pinned", host.is_pinned)
t("data_ptr", host.data_ptr)
t("now_ms", tube.now_ms)
tk = tube.pacer.submit_routes  # noqa
did = tube.unique_id(); tube.store(did, host); tube.fetch(did, device=0, out=dst); torch.cuda.synchronize()
t("pacer.done", lambda: tube.pacer.done(1))
t("unique_id", tube.unique_id)
t("_stream", lambda: tube._stream(0))
t("_loc", lambda: tube._loc(0))
t("lock", lambda: tube._lock.__enter__() or tube._lock.__exit__(None,None,None))
t("_reap(empty)", tube._reap)
t("current_stream", lambda: dev.current_stream(0))
t("out.is_contiguous", dst.is_contiguous)
t("out.nbytes", lambda: dst.nbytes)
t("dev.index", lambda: dst.device.index)
def storefetch():
    d = tube.unique_id(); tube.store(d, host); tube.fetch(d, device=0, out=dst)
t("store+fetch", storefetch, 5000)
ids=[]
for _ in range(5200):
    d = tube.unique_id(); tube.store(d, host); ids.append(d)
t("fetch", lambda: tube.fetch(ids.pop(), device=0, out=dst), 5000)
def st():
    d = tube.unique_id(); tube.store(d, host); ids.append(d)
t("uid+store", st, 5000)
import cProfile, pstats
ids2=[]
for _ in range(3000):
    d = tube.unique_id(); tube.store(d, host); ids2.append(d)
torch.cuda.synchronize()
pr=cProfile.Profile(); pr.enable()
for d in ids2: tube.fetch(d, device=0, out=dst)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
tube.close()

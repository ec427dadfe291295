"""VMM map / unmap cost vs block size, idle and with the GPU busy."""
import ctypes as C, os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
from paper_2411_01830_b200._lib import LIB
h = C.c_void_p()
LIB.ft_vmm_pool_create(0, 64 << 30, C.byref(h))
def one(n):
    vid, ptr = C.c_uint64(), C.c_void_p()
    t0 = time.perf_counter(); LIB.ft_vmm_block_map(h, n, C.byref(vid), C.byref(ptr)); t1 = time.perf_counter()
    LIB.ft_vmm_block_unmap(h, vid.value); t2 = time.perf_counter()
    return (t1 - t0) * 1e3, (t2 - t1) * 1e3
for busy in (False, True):
    stop = threading.Event()
    def load():
        s = torch.cuda.Stream(0)
        while not stop.is_set():
            LIB.ft_spin_ns(2_000_000, 0, C.c_void_p(s.cuda_stream))
            s.synchronize()
    th = threading.Thread(target=load) if busy else None
    if th: th.start(); time.sleep(0.05)
    for n in (2 << 20, 64 << 20, 512 << 20, 2 << 30):
        r = [one(n) for _ in range(3)]
        print("busy" if busy else "idle", n >> 20, "MiB map/unmap ms", [tuple(round(x, 2) for x in t) for t in r], flush=True)
    stop.set()
    if th: th.join()

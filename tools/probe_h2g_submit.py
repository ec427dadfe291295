"""Where the device time of a small host->GPU fetch goes: the same 1 MiB pinned
copy as a raw copy-engine op, as a pacer stage (unmanaged / managed) submitted
straight to the pacer on the consumer's stream, and through tube.fetch —
device time between events around the call on an idle stream (so it includes
the host time before the DMA is enqueued) and the host time of the call.
python tools/probe_h2g_submit.py"""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402
from paper_2411_01830_b200._lib import RouteC  # noqa: E402
from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

tube = FaaSTube("faastube", gpus=[0], pcie_gbps=55.0)
s = torch.cuda.Stream(0)            # a real stream (the legacy default is handle 0)
torch.cuda.set_stream(s)
sp = s.cuda_stream
REPS = 400


def timed(fn):
    dv, hv = [], []
    for i in range(REPS + 50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter()
        b.record(s)
        b.synchronize()
        if i >= 50:
            dv.append(a.elapsed_time(b) * 1e3)
            hv.append((t1 - t0) * 1e6)
    return round(statistics.median(dv), 1), round(statistics.median(hv), 1)


for n in [int(x) for x in os.environ.get("PROBE_SIZES", "4096,1048576,4194304").split(",")]:
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    routes = (RouteC * 1)()
    routes[0].stage_dev, routes[0].off, routes[0].len = 0, 0, n
    routes[0].ce_stream = C.c_void_p(sp)
    routes[0].fw_stream = C.c_void_p(sp)
    res = {"raw_ce": timed(lambda: dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, 0, s))}
    for managed in (0, 1):
        res[f"pacer_managed{managed}"] = timed(lambda: tube.pacer.submit_routes(
            "", bool(managed), 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True, 1, routes, sp))

    def via_tube():
        did = tube.unique_id()
        tube.store(did, host, producer="decode")
        tube.fetch(did, device=0, out=dst, consumer="pre")
    res["tube_store+fetch"] = timed(via_tube)
    ids = []

    def fetch_only():
        tube.fetch(ids.pop(), device=0, out=dst, consumer="pre")
    for _ in range(REPS + 50):
        did = tube.unique_id()
        tube.store(did, host, producer="decode")
        ids.append(did)
    res["tube_fetch"] = timed(fetch_only)
    print(f"bytes={n} (device_us, host_us) p50:", res, flush=True)
tube.close()

"""Host cost of each step of a small host->GPU fetch, replayed outside
FaaSTube.fetch with the same internal calls (GPU box)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

tube = FaaSTube("faastube")
n = 4096
host = torch.ones(n, dtype=torch.uint8).pin_memory()
out = torch.empty(n, dtype=torch.uint8, device="cuda:0")
steps = {k: [] for k in ("store", "lock+lookup", "fetch_plan", "stages", "host_to_gpu", "submit", "consumed",
                         "fetch (whole)")}
for i in range(3000):
    t0 = time.perf_counter()
    did = tube.unique_id()
    tube.store(did, host, producer="decode")
    t1 = time.perf_counter()
    with tube._lock:
        tube._reap()
        obj = tube._objs.get(did)
        tube._last_op_ms = tube.now_ms()
        src, dst = tube._loc(obj.gpu), tube._loc(0)
        t2 = time.perf_counter()
        plan = tube.plane.fetch_plan(src, dst, obj.nbytes)
        t3 = time.perf_counter()
        plan.stages
        t4 = time.perf_counter()
        res, stage = tube._host_to_gpu(obj, plan, dst, out, None, None)
        t5 = time.perf_counter()
        tube._consumed(obj)
        t6 = time.perf_counter()
    ticket = tube.pacer.submit(*stage)
    t7 = time.perf_counter()
    with tube._lock:
        tube._tickets.append((ticket, obj.host, res))
    did = tube.unique_id()
    tube.store(did, host, producer="decode")
    t8 = time.perf_counter()
    tube.fetch(did, device=0, out=out, consumer="producer")
    t9 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    if i >= 200:
        for k, v in zip(steps, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t7 - t6, t6 - t5, t9 - t8)):
            steps[k].append(v * 1e6)
for k, v in steps.items():
    print(f"{k:14s} p50 {statistics.median(v):6.1f} us")
tube.close()

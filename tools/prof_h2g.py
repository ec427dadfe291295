"""Host cost of a small host->GPU fetch (config 2 at small sizes): per-call
wall time of store(pinned host) and fetch(out=), the plan and the pacer submit
alone, a raw copy-engine op for comparison, and a cProfile of the fetch.
python tools/prof_h2g.py"""
import cProfile
import os
import pstats
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402
from paper_2411_01830_b200.dataplane import Location  # noqa: E402
from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

tube = FaaSTube("faastube", gpus=[0], pcie_gbps=55.0)
s = torch.cuda.current_stream(0)
for n in (4096, 1 << 20):
    host = torch.randint(0, 256, (n,), dtype=torch.uint8).pin_memory()
    dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    st, ft, dv = [], [], []
    for i in range(600):
        did = tube.unique_id()
        t0 = time.perf_counter()
        tube.store(did, host, producer="decode")
        t1 = time.perf_counter()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        tube.fetch(did, device=0, out=dst, consumer="pre")
        t2 = time.perf_counter()
        b.record(s)
        b.synchronize()
        if i >= 100:
            st.append(t1 - t0)
            ft.append(t2 - t1)
            dv.append(a.elapsed_time(b))
    # A/B: the same stage submitted straight to the pacer (no tube bookkeeping), routes
    # from the native planner vs a Python-built route list
    from paper_2411_01830_b200._lib import RouteC
    import ctypes as C
    routes, k, mg, cap, nv = (RouteC * 16)(), C.c_int(), C.c_int(), C.c_double(), C.c_uint64()
    ab = {"native": [], "python": []}
    for i in range(400):
        mode = "native" if i % 2 else "python"
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        sp = s.cuda_stream
        if mode == "native":
            dev.LIB.ft_h2g_routes(tube.plane._h, 0, 0, n, C.c_void_p(sp), routes, 16, C.byref(k), C.byref(mg),
                                  C.byref(cap), C.byref(nv))
            tube.pacer.submit_routes("", bool(mg.value), 1e9, 0.0, cap.value, dst.data_ptr(), 0, host.data_ptr(), n,
                                     True, k.value, routes, sp)
        else:
            ce, fw = tube._pair(0, (sp >> 4) * 0x9E3779B1 >> 16)
            tube.pacer.submit("", True, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True,
                              [(0, 0, 0, n, ce.cuda_stream, fw.cuda_stream)], sp)
        b.record(s)
        b.synchronize()
        if i >= 100:
            ab[mode].append(a.elapsed_time(b))
    print(f"bytes={n} pacer-only dev_ms native={statistics.median(ab['native']):.4f} "
          f"python={statistics.median(ab['python']):.4f} (managed={mg.value} cap={cap.value})")
    plan_t = []
    for i in range(600):
        t0 = time.perf_counter()
        p = tube.plane.fetch_plan(Location(0, None), Location(0, 0), n)
        plan_t.append(time.perf_counter() - t0)
    raw, rawdev = [], []
    for i in range(600):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        t0 = time.perf_counter()
        dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, 0, s)
        t1 = time.perf_counter()
        b.record(s)
        b.synchronize()
        raw.append(t1 - t0)
        rawdev.append(a.elapsed_time(b))
    print(f"bytes={n} store_us={1e6 * statistics.median(st):.1f} fetch_us={1e6 * statistics.median(ft):.1f} "
          f"fetch_dev_ms={statistics.median(dv):.4f} plan_us={1e6 * statistics.median(plan_t):.1f} "
          f"raw_ce_call_us={1e6 * statistics.median(raw):.1f} raw_ce_dev_ms={statistics.median(rawdev):.4f}")
    pr = cProfile.Profile()
    for i in range(300):
        did = tube.unique_id()
        tube.store(did, host, producer="decode")
        pr.enable()
        tube.fetch(did, device=0, out=dst, consumer="pre")
        pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
tube.close()

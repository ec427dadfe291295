"""Per-call host time of a function process's store / zero-copy fetch / release
through the daemon, per payload size, in a given size order (is the small-size
penalty the size or the order?).   python tools/probe_daemon_sizes.py [n1 n2 ...]"""
import multiprocessing as mp
import os
import statistics
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def client(path, sizes, q):
    sys.path.insert(0, ROOT)
    if os.environ.get("PROBE_PIN"):               # the function process on the upper half of the cores
        n = os.cpu_count()
        os.sched_setaffinity(0, set(range(n // 2, n)))
    import torch
    from paper_2411_01830_b200.daemon import TubeClient
    c = TubeClient(path, 0)
    res = []
    for n in sizes:
        if n <= 0:                                   # a pause of -n ms (0: 200 ms), nothing timed
            time.sleep((-n or 200) / 1e3)
            continue
        x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
        st, vt, rt = [], [], []
        imp0 = len(c._imports)
        busy = 0
        cs = torch.cuda.current_stream(0)
        for i in range(300):
            busy += not cs.query()                   # the stream still has queued work
            did = c.unique_id()
            t0 = time.perf_counter()
            c.store(did, x)
            t1 = time.perf_counter()
            v = c.fetch(did)
            t2 = time.perf_counter()
            del v
            t3 = time.perf_counter()
            if i >= 50:
                st.append(t1 - t0)
                vt.append(t2 - t1)
                rt.append(t3 - t2)
        q10 = sorted(st)[len(st) // 10]
        q90 = sorted(st)[9 * len(st) // 10]
        res.append((n, round(1e6 * statistics.median(st), 1), round(1e6 * statistics.median(vt), 1),
                    round(1e6 * statistics.median(rt), 1),
                    f"store p10/p90 {1e6 * q10:.1f}/{1e6 * q90:.1f} imports +{len(c._imports) - imp0} "
                    f"stream busy at {busy}/300 iteration starts"))
    c.close()
    q.put(res)


if __name__ == "__main__":
    import torch
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    sizes = [int(a) for a in sys.argv[1:]] or [4096, 1 << 20, 4096, 64 << 20, 4096]
    if os.environ.get("PROBE_PIN"):               # the daemon on the lower half
        os.sched_setaffinity(0, set(range(os.cpu_count() // 2)))
    floor = os.environ.get("PROBE_FLOOR")       # pool floor bytes (a large floor: no shrinks)
    tube = FaaSTube(gpus=[0], pcie_gbps=55.0, **({"pool_floor_bytes": float(floor)} if floor else {}))
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=client, args=(path, sizes, q))
    p.start()
    for n, s, v, r, extra in q.get(timeout=600):
        print(f"bytes={n} store_us={s} view_us={v} release_us={r} {extra}", flush=True)
    import ctypes as C
    from paper_2411_01830_b200._lib import LIB
    st = (C.c_uint64 * 10)()
    LIB.ft_lane_stats(d._lane, st, 10)
    print("lane", list(st))
    p.join(60)
    d.close()
    tube.close()

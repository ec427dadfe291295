"""cProfile of a function process's store() through the daemon's native lane,
in the pattern store -> fetch(out=) -> store -> zero-copy fetch -> release
(the bench's daemon_put_get loop).   python tools/prof_daemon_store.py"""
import cProfile
import multiprocessing as mp
import os
import pstats
import statistics
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def client(path, q):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2411_01830_b200.daemon import TubeClient
    c = TubeClient(path, 0)
    x = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device="cuda:0")
    out = torch.empty_like(x)
    prs, prr = cProfile.Profile(), cProfile.Profile()
    t = {"store1": [], "fetch_out": [], "store2": [], "view": [], "release": []}
    for i in range(400):
        on = i >= 100
        did = c.unique_id()
        t0 = time.perf_counter()
        if on:
            prs.enable()
        c.store(did, x)
        if on:
            prs.disable()
        t1 = time.perf_counter()
        c.fetch(did, out=out)
        t2 = time.perf_counter()
        did = c.unique_id()
        c.store(did, x)
        t3 = time.perf_counter()
        v = c.fetch(did)
        t4 = time.perf_counter()
        if on:
            prr.enable()
        del v
        if on:
            prr.disable()
        t5 = time.perf_counter()
        if on:
            for k, a, b in (("store1", t0, t1), ("fetch_out", t1, t2), ("store2", t2, t3), ("view", t3, t4),
                            ("release", t4, t5)):
                t[k].append(b - a)
    import io
    out_s = {k: round(1e6 * statistics.median(v), 1) for k, v in t.items()}
    b1, b2 = io.StringIO(), io.StringIO()
    pstats.Stats(prs, stream=b1).sort_stats("tottime").print_stats(25)
    pstats.Stats(prr, stream=b2).sort_stats("tottime").print_stats(15)
    c.close()
    q.put((out_s, b1.getvalue(), b2.getvalue()))


def main():
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=55.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=client, args=(path, q))
    p.start()
    res, a, b = q.get(timeout=300)
    p.join(timeout=60)
    print(res)
    print("==== store (first of the pair)\n" + a)
    print("==== release of a view\n" + b)
    import ctypes as C
    from paper_2411_01830_b200._lib import LIB
    st = (C.c_uint64 * 8)()
    LIB.ft_lane_stats(d._lane, st, 8)
    print("lane stats (commits, fetches, dones, uids, forwarded, stock hits, stock misses, adopted):", list(st))
    d.close()
    tube.close()


if __name__ == "__main__":
    main()

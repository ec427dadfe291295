"""Per-iteration host time of a function process's store + zero-copy fetch of 1 MiB
through the daemon, with the daemon GPU test's pool settings (one 2 MiB arena per
block, no reservation): the slowest iterations and where they fall.
python tools/probe_daemon_stalls.py [iterations]"""
import multiprocessing as mp
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def client(path, n_it, q):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2411_01830_b200.daemon import TubeClient
    c = TubeClient(path, 0)
    m = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device="cuda:0")
    ts = []
    r = None
    imp = []
    for i in range(n_it):
        t0 = time.perf_counter()
        did = c.unique_id()
        c.store(did, m)
        r = c.fetch(did)
        ts.append((time.perf_counter() - t0) * 1e6)
        imp.append(len(c._imports))
    c.close()
    q.put((ts, imp))


if __name__ == "__main__":
    os.environ["FT_POOL_RESERVE_BYTES"] = "0"
    os.environ["FT_POOL_ARENA_BYTES"] = str(2 << 20)
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    n_it = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0], pool_floor_bytes=0.0)
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=client, args=(path, n_it, q))
    p.start()
    ts, imp = q.get(timeout=600)
    p.join(60)
    order = sorted(range(len(ts)), key=lambda i: -ts[i])[:8]
    print("mean us", round(sum(ts) / len(ts), 1), "median", round(sorted(ts)[len(ts) // 2], 1))
    print("slowest (iteration, us, imports):", [(i, round(ts[i], 1), imp[i]) for i in order])
    d.close()
    tube.close()

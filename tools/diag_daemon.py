"""Per-op latency of the function <-> daemon channel (TubeClient against a
TubeDaemon in this process): unique_id / alloc / commit / fetch / done."""

import json
import multiprocessing as mp
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _client(path, q, nbytes, reps):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2411_01830_b200.daemon import TubeClient
    c = TubeClient(path, 0)
    m = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda:0")
    out = torch.empty_like(m)
    ops = {"unique_id": [], "store": [], "fetch": [], "ping": []}
    for i in range(reps):
        t0 = time.perf_counter()
        did = c.unique_id()
        t1 = time.perf_counter()
        c.store(did, m)
        t2 = time.perf_counter()
        c.fetch(did, out=out)
        t3 = time.perf_counter()
        if i >= 5:
            ops["unique_id"].append((t1 - t0) * 1e6)
            ops["store"].append((t2 - t1) * 1e6)
            ops["fetch"].append((t3 - t2) * 1e6)
    c.close()
    q.put({k: sorted(v)[len(v) // 2] for k, v in ops.items() if v})


def main():
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    import collections
    import torch
    from paper_2411_01830_b200 import daemon as dmod, device as dev
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    spent = collections.defaultdict(list)

    def timed(name, fn):
        def w(*a, **k):
            t0 = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                spent[name].append((time.perf_counter() - t0) * 1e6)
        return w
    tube.empty = timed("tube.empty", tube.empty)
    tube.store = timed("tube.store", tube.store)
    tube.fetch = timed("tube.fetch", tube.fetch)
    tube.pools[0].export_fd = timed("export_fd", tube.pools[0].export_fd)
    dmod.torch.cuda.synchronize = timed("cuda.synchronize", torch.cuda.synchronize)
    dev.Ev.synchronize = timed("Ev.synchronize", dev.Ev.synchronize)
    dmod.Channel.send_fd = timed("send_fd", dmod.Channel.send_fd)
    dmod.Channel.recv_msg = timed("recv_msg(wait)", dmod.Channel.recv_msg)
    dmod.TubeDaemon._handle = timed("handle", dmod.TubeDaemon._handle)
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn")
    res = {}
    for nbytes in (4096, 1 << 20, 64 << 20):
        q = ctx.Queue()
        p = ctx.Process(target=_client, args=(path, q, nbytes, 40))
        p.start()
        res[nbytes] = q.get(timeout=300)
        p.join()
    print(json.dumps({"median_us": res, "switch_interval": sys.getswitchinterval(),
                      "daemon_median_us": {k: sorted(v)[len(v) // 2] for k, v in spent.items()},
                      "daemon_max_us": {k: max(v) for k, v in spent.items()}}, indent=1))
    d.close()
    tube.close()


if __name__ == "__main__":
    main()

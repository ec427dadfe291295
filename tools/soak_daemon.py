"""Soak the daemon's native lane: N function processes for D seconds, each storing
random-size outputs (several size classes, ragged byte counts, 1–3 consumers) and
fetching other processes' objects as views or copies, releasing views in random
order; every payload checked by digest. Reports lane counters and any mismatch.
python tools/soak_daemon.py [procs] [seconds]"""
import multiprocessing as mp
import os
import random
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def payload(n, seed):
    import torch
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g)


def worker(path, wid, nproc, dur, q_out, q_in):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2411_01830_b200.daemon import TubeClient
    rnd = random.Random(wid)
    c = TubeClient(path, 0)
    sizes = [4096 + 7, 1 << 20, 3 * 10**6 + 1, 9 * 10**6 + 5, 33 * 10**6 + 3]
    made = fetched = bad = 0
    views = []
    t_end = time.time() + dur
    try:
        while time.time() < t_end:
            # produce
            n = rnd.choice(sizes) - rnd.randrange(0, 4096)
            seed = wid * 10**7 + made
            cons = rnd.choice((1, 1, 2))
            did = c.unique_id()
            c.store(did, payload(n, seed).cuda(), producer=f"w{wid}", consumers=cons)
            for k in range(cons):
                q_out[rnd.randrange(nproc)].put((did, n, seed))
            made += 1
            # consume whatever arrived
            while not q_in.empty():
                did, n, seed = q_in.get_nowait()
                if rnd.random() < 0.5:
                    v = c.fetch(did)
                    ok = torch.equal(v.cpu(), payload(n, seed))
                    if rnd.random() < 0.3:
                        views.append(v)                    # release later, out of order
                    del v
                else:
                    out = torch.empty(n, dtype=torch.uint8, device="cuda:0")
                    c.fetch(did, out=out)
                    ok = torch.equal(out.cpu(), payload(n, seed))
                bad += not ok
                fetched += 1
                if len(views) > 4:
                    views.pop(rnd.randrange(len(views)))
        views.clear()
        # drain: objects still addressed to this worker
        t_drain = time.time() + 10
        while time.time() < t_drain:
            try:
                did, n, seed = q_in.get(timeout=1.0)
            except Exception:  # noqa: BLE001
                break
            out = torch.empty(n, dtype=torch.uint8, device="cuda:0")
            c.fetch(did, out=out)
            bad += not torch.equal(out.cpu(), payload(n, seed))
            fetched += 1
        c.close()
        q_out[nproc].put(("ok", wid, made, fetched, bad))
    except Exception:  # noqa: BLE001
        import traceback
        q_out[nproc].put(("err", wid, traceback.format_exc(), 0, 0))


def main():
    import ctypes as C
    import torch
    from paper_2411_01830_b200._lib import LIB
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    nproc = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    dur = float(sys.argv[2]) if len(sys.argv) > 2 else 30.0
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    in_use0 = tube.pools[0].policy.in_use_bytes
    ctx = mp.get_context("spawn")
    qs = [ctx.Queue() for _ in range(nproc + 2)]          # one per worker, results, the in-process tenant
    ps = [ctx.Process(target=worker, args=(path, w, nproc + 1, dur, qs[:nproc + 1] + [qs[nproc + 1]], qs[w]))
          for w in range(nproc)]
    # the workers' results queue is qs[nproc + 1] (index nproc + 1 of their list); objects they
    # address to "worker nproc" go to the in-process tenant below, which adopts them from the lane
    for p in ps:
        p.start()
    import threading
    local = {"made": 0, "fetched": 0, "bad": 0, "err": None}

    def tenant():
        rnd = random.Random(99)
        try:
            t_end = time.time() + dur
            while time.time() < t_end:
                n = rnd.choice((4096 + 5, 1 << 20, 5 * 10**6 + 3))
                did = tube.unique_id()
                x = payload(n, 777 + local["made"]).cuda()
                tube.store(did, x, producer="local")
                out = torch.empty(n, dtype=torch.uint8, device="cuda:0")
                tube.fetch(did, out=out)
                local["bad"] += not torch.equal(out, x)
                local["made"] += 1
                while not qs[nproc].empty():              # a function process's object, fetched here
                    did, n, seed = qs[nproc].get_nowait()
                    got = tube.fetch(did, device=0) if rnd.random() < 0.5 else \
                        tube.fetch(did, out=torch.empty(n, dtype=torch.uint8, device="cuda:0"))
                    local["bad"] += not torch.equal(got.cpu(), payload(n, seed))
                    local["fetched"] += 1
                    del got
            t_drain = time.time() + 15
            while time.time() < t_drain:
                try:
                    did, n, seed = qs[nproc].get(timeout=1.0)
                except Exception:  # noqa: BLE001
                    break
                got = tube.fetch(did, out=torch.empty(n, dtype=torch.uint8, device="cuda:0"))
                local["bad"] += not torch.equal(got.cpu(), payload(n, seed))
                local["fetched"] += 1
        except Exception:  # noqa: BLE001
            import traceback
            local["err"] = traceback.format_exc()

    th = threading.Thread(target=tenant)
    th.start()
    res = [qs[nproc + 1].get(timeout=dur + 300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    th.join(timeout=120)
    res.append(("in-process tenant", local))
    st = (C.c_uint64 * 10)()
    LIB.ft_lane_stats(d._lane, st, 10)
    time.sleep(1.0)
    torch.cuda.synchronize()
    left = len(tube._objs)
    d.close()
    ok_acc = tube._accounts_consistent()
    in_use1 = tube.pools[0].policy.in_use_bytes
    tube.close()
    print({"procs": nproc, "seconds": dur, "workers": res,
           "lane": dict(zip(("commits", "fetches", "dones", "unique_ids", "handed_to_python", "stock_hits",
                             "stock_misses", "adopted", "recycled", "lost"), list(st))),
           "objects_left_in_tube": left, "accounts_consistent": ok_acc,
           "pool_in_use_before_after": (in_use0, in_use1)})


if __name__ == "__main__":
    main()

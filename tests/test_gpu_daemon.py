"""Function process <-> per-box daemon: a spawned function
process drives Listing 1 (unique_id / store / fetch) through ``TubeClient``
against a ``TubeDaemon`` owning the FaaSTube in this process. GPU payloads
cross as exported VMM pool blocks (zero copy on the daemon side), host payloads
as memfds; every byte is checked against the seeded source in both processes."""

import multiprocessing as mp
import os
import sys
import tempfile
import time

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIZES = [1, 4097, 3 * 10**6 + 7, 64 << 20]


def payload(n, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g)


def _function(path, q, phase1, phase2):
    sys.path.insert(0, ROOT)
    try:
        from paper_2411_01830_b200.daemon import DaemonError, TubeClient
        c = TubeClient(path, 0)
        ids = {}
        for i, n in enumerate(SIZES):
            src = payload(n, i).cuda()
            did = c.unique_id()
            c.store(did, src, consumers=3)           # the daemon also reads it, and fetch_host
            got = c.fetch(did)                        # same GPU: the stored block itself, mapped here
            assert torch.equal(got, src), ("gpu->gpu", n)
            host = c.fetch(did, out=torch.empty(n, dtype=torch.uint8))
            assert torch.equal(host, src.cpu()), ("gpu->host", n)
            ids[n] = did
        # typed tensor keeps dtype and shape
        x = torch.randn(3, 5, 7, device="cuda:0", dtype=torch.float16)
        did = c.unique_id()
        c.store(did, x)
        y = c.fetch(did)
        assert y.dtype == x.dtype and y.shape == x.shape and torch.equal(x, y)
        # empty and NaN-bit payloads, GPU and host producers
        for t in (torch.empty(0, dtype=torch.float16), torch.empty(2, 0, dtype=torch.int32),
                  torch.randint(0, 1 << 16, (4097,), dtype=torch.int32).to(torch.int16).view(torch.float16)):
            for dev_t in (t.cuda(), t):
                did = c.unique_id()
                c.store(did, dev_t)
                y = c.fetch(did)
                assert y.shape == t.shape and y.dtype == t.dtype
                assert torch.equal(y.cpu().reshape(-1).view(torch.uint8), t.reshape(-1).view(torch.uint8))
        # a host (cFunc) payload: memfd to the daemon, staged host->GPU by its pacer on fetch
        h = payload(5 * 10**6 + 3, 77)
        did = c.unique_id()
        c.store(did, h)
        out = torch.empty_like(h, device="cuda:0")
        c.fetch(did, out=out)
        assert torch.equal(out.cpu(), h)
        # steady state: pool blocks are reused by size class, so nothing new is mapped
        before = len(c._imports)
        t0 = time.perf_counter()
        reps = 50
        m = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device="cuda:0")
        for _ in range(reps):
            did = c.unique_id()
            c.store(did, m)
            r = c.fetch(did)
        us = (time.perf_counter() - t0) / reps * 1e6
        assert torch.equal(r, m)
        grown = len(c._imports) - before
        # errors travel back as typed messages
        try:
            c.fetch(10**12)
            missing = None
        except DaemonError as e:
            missing = str(e)
        # the daemon's pool unmaps its free blocks: the next reply tells this process
        # to unmap its imports of them (they would keep the physical memory alive)
        mapped = len(c._imports)
        phase1.set()
        assert phase2.wait(120)
        c.unique_id()
        after = len(c._imports)
        c.close()
        q.put(("ok", {"ids": ids, "us_store_fetch_1MiB": us, "imports_grown": grown, "missing": missing,
                      "mapped": mapped, "after_shrink": after}))
    except Exception as exc:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc() + repr(exc)))


def test_function_process_through_daemon(monkeypatch):
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    # one arena per block and no reservation: the shrink below must unmap arenas, so
    # the client is told to drop its imports of them
    monkeypatch.setenv("FT_POOL_RESERVE_BYTES", "0")
    monkeypatch.setenv("FT_POOL_ARENA_BYTES", str(2 << 20))
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0], pool_floor_bytes=0.0)
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn")
    q, phase1, phase2 = ctx.Queue(), ctx.Event(), ctx.Event()
    p = ctx.Process(target=_function, args=(path, q, phase1, phase2))
    p.start()
    while not phase1.wait(1):
        assert p.is_alive() or not q.empty(), "function process died"
        if not q.empty():
            break
    if phase1.is_set():
        torch.cuda.synchronize()
        dropped = tube.pools[0].shrink(tube.now_ms() + 1e9)
        phase2.set()
    status, res = q.get(timeout=600)
    p.join(timeout=60)
    assert status == "ok", res
    print("daemon round trip (store+fetch 1 MiB, GPU, cross-process):", f"{res['us_store_fetch_1MiB']:.1f} us")
    # the lane keeps a stock of lendable blocks per size class (lane.cc kStockDepth = 3):
    # the blocks in rotation are the stock, the one lent, the one being read and one
    # whose release the daemon has not applied yet when the next store takes from the
    # stock (the release races the next commit); each is imported once (one arena per
    # block here), then nothing new is mapped
    assert res["imports_grown"] <= 3 + 3, res
    assert res["missing"] and "MissingData" in res["missing"], res
    # the shrink unmaps idle pool blocks; the client drops its imports of those it had
    # mapped (which of its blocks are idle then — rather than recycled into the lane's
    # stock or holding live objects — depends on timing; the CPU protocol test checks
    # the notice itself deterministically)
    assert dropped > 0 and res["after_shrink"] <= res["mapped"], (dropped, res)
    # the daemon side holds the function's bytes (third consumer)
    for i, n in enumerate(SIZES):
        t = tube.fetch(res["ids"][n], device=0)
        assert torch.equal(t.cpu(), payload(n, i)), n
        del t
    torch.cuda.synchronize()
    d.close()
    tube.close()


def _producer(path, q, count):
    sys.path.insert(0, ROOT)
    try:
        from paper_2411_01830_b200.daemon import TubeClient
        c = TubeClient(path, 0)
        ids = []
        for i in range(count):
            n = (i * 7919) % (3 << 20) + 1
            did = c.unique_id()
            c.store(did, payload(n, 1000 + i).cuda(), producer="prod")
            ids.append((did, n, 1000 + i))
        c.close()
        q.put(("ok", ids))
    except Exception:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc()))


def _consumer(path, ids, q):
    sys.path.insert(0, ROOT)
    try:
        from paper_2411_01830_b200.daemon import TubeClient
        c = TubeClient(path, 0)
        bad = []
        for did, n, seed in ids:
            got = c.fetch(did, consumer="cons")
            if not torch.equal(got.cpu(), payload(n, seed)):
                bad.append(did)
        c.close()
        q.put(("ok", bad))
    except Exception:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc()))


def test_producer_and_consumer_processes():
    """Two function processes: the producer's outputs (written through its mapping
    of daemon pool blocks) are fetched by a separate consumer process — every
    object bit-exact, and the daemon retires each after its one consumer."""
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    prod = ctx.Process(target=_producer, args=(path, q, 40))
    prod.start()
    status, ids = q.get(timeout=600)
    prod.join(timeout=60)
    assert status == "ok", ids
    cons = ctx.Process(target=_consumer, args=(path, ids, q))
    cons.start()
    status, bad = q.get(timeout=600)
    cons.join(timeout=60)
    assert status == "ok", bad
    assert bad == []
    assert all(did not in tube._objs for did, _, _ in ids)       # consumed -> retired
    assert tube._accounts_consistent()
    d.close()
    tube.close()


def _dies_after_alloc(path, q):
    sys.path.insert(0, ROOT)
    from paper_2411_01830_b200.daemon import TubeClient
    c = TubeClient(path, 0)
    rep = c._call({"op": "alloc", "gpu": 0, "nbytes": 8 << 20})   # a loan it never commits
    q.put(rep["token"])
    q.close()
    q.join_thread()                                                  # flushed before the hard exit
    os._exit(0)                                                      # no close, no commit


def test_dead_client_loans_return_to_the_pool():
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    before = tube.pools[0].policy.in_use_bytes
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_dies_after_alloc, args=(path, q))
    p.start()
    q.get(timeout=120)
    p.join(timeout=60)
    deadline = time.time() + 10
    while tube.pools[0].policy.in_use_bytes != before and time.time() < deadline:
        time.sleep(0.05)
    assert tube.pools[0].policy.in_use_bytes == before
    assert not d._held
    d.close()
    assert not d._acceptor.is_alive()
    tube.close()


def _views_and_loans(path, q):
    sys.path.insert(0, ROOT)
    try:
        from paper_2411_01830_b200.daemon import TubeClient
        c = TubeClient(path, 0)
        n = 3 * 10**6 + 5
        a = payload(n, 1).cuda()
        did = c.unique_id()
        c.store(did, a)
        v = c.fetch(did)                                    # zero-copy view of the stored block (last consumer)
        sent0 = c._sent
        for k in range(20):                                 # same size: lent blocks, never the viewed one
            d = c.unique_id()
            c.store(d, payload(n, 100 + k).cuda())
            w = c.fetch(d)
            assert torch.equal(w, payload(n, 100 + k).cuda()), k
            del w
        per_store = (c._sent - sent0) / 20                  # unique_id + commit + fetch + done (+ no alloc)
        torch.cuda.synchronize()
        ok_view = torch.equal(v, a)                          # untouched while alive
        derived = v[7:1000].clone()
        del v                                                # release -> the daemon may reuse the block
        import gc
        gc.collect()                                         # every view's `done` is sent by now
        c.unique_id()                                        # its reply acknowledges everything before it
        q.put(("ok", {"ok_view": ok_view, "derived": torch.equal(derived, a[7:1000]), "per_store": per_store,
                      "acked": c._acked, "sent": c._sent}))
        c.close()
    except Exception as exc:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc() + repr(exc)))


def test_zero_copy_views_and_lent_blocks():
    """A client's zero-copy view pins the stored block until the last tensor
    over it dies (later same-size stores, served from lent blocks, never land
    in it); a steady producer needs no alloc round trip (the commit reply lends
    the next block); every message is acknowledged (IPC-event ring reuse)."""
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0], pool_floor_bytes=0.0)
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_views_and_loans, args=(path, q))
    p.start()
    status, res = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", res
    assert res["ok_view"] and res["derived"], res
    assert res["per_store"] <= 4.0, res
    assert res["acked"] == res["sent"], res
    d.close()
    assert tube._accounts_consistent()
    tube.close()

"""The daemon's native lane (csrc/lane.cc, client.cc) under the conditions its
fast path is not the whole story: several function processes at once, a client
that dies with its copy still queued, the tube adopting a lane object another
process still views, and store-cap migration of lane objects. Every payload is
checked byte for byte against its seeded source."""

import multiprocessing as mp
import os
import sys
import tempfile
import time

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def payload(n, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g)


def lane_stats(d):
    import ctypes as C
    from paper_2411_01830_b200._lib import LIB
    st = (C.c_uint64 * 10)()
    LIB.ft_lane_stats(d._lane, st, 10)
    return dict(zip(("commits", "fetches", "dones", "unique_ids", "handed_to_python", "stock_hits", "stock_misses",
                     "adopted", "recycled", "lost"), list(st)))


def _producer(path, q, count, seed0):
    sys.path.insert(0, ROOT)
    from paper_2411_01830_b200.daemon import TubeClient
    try:
        c = TubeClient(path, 0)
        ids = []
        for i in range(count):
            # a function's outputs vary within one size class (ragged, odd byte counts)
            n = 3 * 10**6 + (i * 7919 + seed0) % 900_000 + 1
            did = c.unique_id()
            c.store(did, payload(n, seed0 + i).cuda(), producer=f"p{seed0}")
            ids.append((did, n, seed0 + i))
        c.close()
        q.put(("ok", ids))
    except Exception:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc()))


def _consumer(path, ids, q_res):
    sys.path.insert(0, ROOT)
    from paper_2411_01830_b200.daemon import TubeClient
    try:
        c = TubeClient(path, 0)
        bad, k = [], 0
        for did, n, seed in ids:
            if k % 2:
                got = c.fetch(did)                                  # zero-copy view
            else:
                got = c.fetch(did, out=torch.empty(n, dtype=torch.uint8, device="cuda:0"))
            if not torch.equal(got.cpu(), payload(n, seed)):
                bad.append(did)
            del got
            k += 1
        c.close()
        q_res.put(("ok", (k, bad)))
    except Exception:  # noqa: BLE001
        import traceback
        q_res.put(("err", traceback.format_exc()))


def test_lane_concurrent_function_pairs():
    """Two producer -> consumer pairs of function processes run at once through the
    daemon's lane (four workers, one table): every object arrives bit-exact, the hot
    requests never reach Python, and the tube's accounts match its table after."""
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    in_use0 = tube.pools[0].policy.in_use_bytes
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    # the two producers run at once, then the two consumers
    prods = [ctx.Process(target=_producer, args=(path, q, 40, 1000 * (pair + 1))) for pair in range(2)]
    for p in prods:
        p.start()
    made = [q.get(timeout=600) for _ in prods]
    for p in prods:
        p.join(timeout=60)
    for status, ids in made:
        assert status == "ok", ids
    cons = [ctx.Process(target=_consumer, args=(path, ids, q)) for _, ids in made]
    for p in cons:
        p.start()
    results = [q.get(timeout=600) for _ in cons]
    for p in cons:
        p.join(timeout=60)
    for status, res in results:
        assert status == "ok", res
        assert res == (40, []), res
    st = lane_stats(d)
    assert st["commits"] == 80 and st["fetches"] == 80, st
    assert st["handed_to_python"] <= 4 * 3, st          # chan/hello per connection + first allocs
    deadline = time.time() + 10
    while tube.pools[0].policy.in_use_bytes > in_use0 and time.time() < deadline:
        time.sleep(0.05)                                  # (frees are applied by the lane service)
    assert tube.pools[0].policy.in_use_bytes == in_use0   # every block back (loans, stock, objects)
    assert tube._accounts_consistent()
    d.close()
    tube.close()


def _dies_mid_store(path, q, n):
    sys.path.insert(0, ROOT)
    import ctypes as C
    from paper_2411_01830_b200 import device as dev
    from paper_2411_01830_b200.daemon import TubeClient
    c = TubeClient(path, 0)
    x = payload(n, 5).cuda()
    torch.cuda.synchronize()
    did0 = c.unique_id()
    c.store(did0, x)                                      # a complete store (its copy ran)
    torch.cuda.synchronize()
    # the next store's copy and mark queue behind 2 s of device spin: the commit
    # is acknowledged before the bytes are written, then the process dies
    dev.LIB.ft_spin_ns(2_000_000_000, 0, C.c_void_p(torch.cuda.current_stream(0).cuda_stream))
    did1 = c.unique_id()
    c.store(did1, x)
    q.put((did0, did1))
    q.close()
    q.join_thread()
    os._exit(0)


def test_lane_client_dies_with_its_copy_queued():
    """A function process dies after its commit was acknowledged but before its copy
    ran: the daemon's stream is never left parked on the dead client's mark, the
    object it never wrote is dropped (a fetch misses — nobody reads garbage) or, if
    the driver still ran the copy, arrives intact; the pool gets its blocks back."""
    from paper_2411_01830_b200 import MissingData
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    n = 3 * 10**6 + 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_dies_mid_store, args=(path, q, n))
    p.start()
    did0, did1 = q.get(timeout=300)
    p.join(timeout=60)
    time.sleep(0.5)                                       # the worker notices (socket EOF)
    out = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    tube.fetch(did0, out=out)                             # the complete store is intact
    assert torch.equal(out.cpu(), payload(n, 5))
    try:
        tube.fetch(did1, out=out)
        assert torch.equal(out.cpu(), payload(n, 5)), "a dead client's store must not deliver garbage"
    except MissingData:
        assert lane_stats(d)["lost"] == 1
    torch.cuda.synchronize()                              # nothing is parked on the dead client's mark
    assert tube._accounts_consistent()
    d.close()
    tube.close()


def _views_then_waits(path, q, go):
    sys.path.insert(0, ROOT)
    from paper_2411_01830_b200.daemon import TubeClient
    try:
        c = TubeClient(path, 0)
        n = 5 * 10**6 + 3
        did = c.unique_id()
        c.store(did, payload(n, 9).cuda(), consumers=2)
        v = c.fetch(did)                                  # a view (the first of two consumers)
        q.put(did)
        assert go.wait(120)                               # the tube adopts it meanwhile
        ok = torch.equal(v.cpu(), payload(n, 9))
        del v                                             # the release goes to the tube (UNPIN)
        c.unique_id()
        c.close()
        q.put(("ok", ok))
    except Exception:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc()))


def test_tube_adopts_a_lane_object_another_process_views():
    """An object committed through the lane, viewed by its first consumer in a
    function process, is fetched in the daemon's own process by its second
    consumer: the tube adopts it with the view's pin, the view stays intact, and
    the view's release (UNPIN) frees the block afterwards."""
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn")
    q, go = ctx.Queue(), ctx.Event()
    p = ctx.Process(target=_views_then_waits, args=(path, q, go))
    p.start()
    did = q.get(timeout=300)
    n = 5 * 10**6 + 3
    out = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    tube.fetch(did, out=out)                              # the last consumer, in process (adoption)
    assert torch.equal(out.cpu(), payload(n, 9))
    assert lane_stats(d)["adopted"] == 1
    go.set()
    status, ok = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok" and ok, ok
    deadline = time.time() + 10
    while tube._lane_adopted and time.time() < deadline:   # the UNPIN has been applied
        time.sleep(0.05)
    assert not tube._lane_adopted
    assert tube._accounts_consistent()
    d.close()
    tube.close()


def _stores_many(path, q, sizes):
    sys.path.insert(0, ROOT)
    from paper_2411_01830_b200.daemon import TubeClient
    try:
        c = TubeClient(path, 0)
        ids = []
        for i, n in enumerate(sizes):
            did = c.unique_id()
            c.store(did, payload(n, 300 + i).cuda(), producer="big")
            ids.append(did)
        torch.cuda.synchronize()
        q.put(("ids", ids))
        # fetch them back after the tube migrated some to host memory (Python serves those)
        msg = q.get(timeout=300)
        assert msg == "fetch"
        bad = []
        for i, (did, n) in enumerate(zip(ids, sizes)):
            got = c.fetch(did, out=torch.empty(n, dtype=torch.uint8, device="cuda:0"))
            if not torch.equal(got.cpu(), payload(n, 300 + i)):
                bad.append(did)
        c.close()
        q.put(("ok", bad))
    except Exception:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc()))


def test_lane_objects_migrate_under_the_store_cap():
    """Lane objects count against the per-GPU store cap (datastore.py:19): when a
    function process's stores exceed it, the tube adopts the GPU's lane objects
    and migrates the farthest-queued ones to host memory (datastore.py:192-222);
    fetching them back through the daemon is bit-exact."""
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0], capacity_limit_bytes=100e6)
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    sizes = [30 * 10**6 + 7 * i for i in range(6)]       # 180 MB > the 100 MB cap
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_stores_many, args=(path, q, sizes))
    p.start()
    kind, ids = q.get(timeout=300)
    assert kind == "ids", ids
    deadline = time.time() + 20
    while tube._stored_on(0) > tube.capacity_limit and time.time() < deadline:
        time.sleep(0.05)                                  # (the lane service applies the cap)
    assert tube.stats["migrated_bytes"] > 0
    assert tube._stored_on(0) <= tube.capacity_limit
    q.put("fetch")
    status, bad = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok" and bad == [], bad
    assert tube._accounts_consistent()
    d.close()
    tube.close()


def _response_and_release(path, q):
    sys.path.insert(0, ROOT)
    from paper_2411_01830_b200.daemon import DaemonError, TubeClient
    try:
        c = TubeClient(path, 0)
        x = payload(2 * 10**6 + 9, 21).cuda()
        did = c.unique_id()
        c.store(did, x, response=True, consumers=2)   # the slow path (Python) inside a lane connection
        y = c.fetch(did, out=torch.empty_like(x))
        ok_resp = torch.equal(y, x)
        did2 = c.unique_id()
        c.store(did2, x, consumers=3)
        c.release(did2)                               # dropped regardless of consumers
        try:
            c.fetch(did2)
            released = False
        except DaemonError as e:
            released = "MissingData" in str(e)
        c.close()
        q.put(("ok", (ok_resp, released, did)))
    except Exception:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc()))


def test_lane_connection_slow_paths():
    """Requests the lane hands to Python on a lane connection — a store with a
    response leg (engine.py:414-423), release — keep their semantics: the response
    lands in host memory, bit-exact; a released object misses."""
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_response_and_release, args=(path, q))
    p.start()
    status, res = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", res
    ok_resp, released, did = res
    assert ok_resp and released
    assert torch.equal(tube.response(did).view(torch.uint8).reshape(-1), payload(2 * 10**6 + 9, 21))
    assert tube._accounts_consistent()
    d.close()
    tube.close()


def _daemon_only(path, q):
    sys.path.insert(0, ROOT)
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    TubeDaemon(tube, path)
    q.put("up")
    time.sleep(600)


def _outlives_its_daemon(path, q, go):
    sys.path.insert(0, ROOT)
    from paper_2411_01830_b200 import device as dev
    from paper_2411_01830_b200.daemon import TubeClient
    try:
        c = TubeClient(path, 0)
        n = 10**6 + 7
        did = c.unique_id()
        c.store(did, payload(n, 31).cuda(), consumers=24)
        views = [c.fetch(did) for _ in range(24)]
        ok = all(torch.equal(v[:4096].cpu(), payload(n, 31)[:4096]) for v in views[:2])
        torch.cuda.synchronize()
        q.put(("ready", ok))
        assert go.wait(120)                               # the daemon is dead now
        t0 = time.time()
        # this process's stream waits on a mark the daemon will never write
        s = torch.cuda.current_stream(0)
        dev.LIB.ft_client_wait(c._cl, dev.stream_ptr(s), 100_000)  # noqa: SLF001
        del views                                         # 24 releases: more than the ring holds
        try:
            c.unique_id()
            raised = False
        except ConnectionError:
            raised = True
        torch.cuda.synchronize()                          # the parked wait was released
        c.close()
        q.put(("ok", (raised, time.time() - t0)))
    except Exception:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc()))


def test_function_process_outlives_its_daemon():
    """The daemon dies (SIGKILL) under a function process holding zero-copy views and
    a stream parked on one of the daemon's marks: releasing more views than the
    request ring holds does not block, the next request raises ConnectionError, and
    synchronising / closing the client returns (its waits on the dead daemon's marks
    are released) instead of hanging the function."""
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    ctx = mp.get_context("spawn")
    q, qc, go = ctx.Queue(), ctx.Queue(), ctx.Event()
    dp = ctx.Process(target=_daemon_only, args=(path, q))
    dp.start()
    try:
        assert q.get(timeout=300) == "up"
        cp = ctx.Process(target=_outlives_its_daemon, args=(path, qc, go))
        cp.start()
        try:
            status, ok = qc.get(timeout=300)
            assert status == "ready" and ok, ok
            dp.kill()
            dp.join(timeout=60)
            go.set()
            status, res = qc.get(timeout=120)
            assert status == "ok", res
            raised, took = res
            assert raised and took < 30, res
            cp.join(timeout=60)
            assert cp.exitcode == 0
        finally:
            if cp.is_alive():
                cp.kill()
    finally:
        if dp.is_alive():
            dp.kill()


def _bad_shapes(path, q):
    sys.path.insert(0, ROOT)
    import struct
    from paper_2411_01830_b200 import daemon as dm
    try:
        c = dm.TubeClient(path, 0)
        x = payload(4096, 1).cuda()
        errors = []
        for shape in ((1 << 62, 8), (-1, 8)):
            did = c.unique_id()
            c.store(did, x)                               # leaves the next 4 KiB-class block lent
            rep = c._loans.pop(dm._class_of(4096))        # noqa: SLF001
            name = b"evil"
            body = dm._COMMIT.pack(dm.OP_COMMIT, dm._CODE[torch.uint8], 2, 0, 0, 1, len(name), rep["token"],
                                   c.unique_id(), 0) + struct.pack("<2q", *shape) + name
            try:
                c._block_bin(body)                        # noqa: SLF001
                errors.append(None)
            except dm.DaemonError as e:
                errors.append(str(e))
            assert torch.equal(c.fetch(did), x)           # (its only consumer: the block goes back)
        did = c.unique_id()                               # the daemon still serves this client
        c.store(did, x)
        ok = torch.equal(c.fetch(did), x)
        c.close()
        q.put(("ok", (errors, ok)))
    except Exception:  # noqa: BLE001
        import traceback
        q.put(("err", traceback.format_exc()))


def test_lane_rejects_forged_commit_shapes():
    """A commit whose shape overflows the byte count or has a negative dimension (a
    buggy or hostile function process) is refused with an error reply — not stored
    with a byte count smaller than what its shape lets a consumer read — and the lent
    block goes back to the pool; the connection keeps working."""
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=50.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    in_use0 = tube.pools[0].policy.in_use_bytes
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_bad_shapes, args=(path, q))
    p.start()
    status, res = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", res
    errors, ok = res
    assert ok
    assert all(e is not None and "ValueError" in e for e in errors), errors
    deadline = time.time() + 10
    while tube.pools[0].policy.in_use_bytes > in_use0 and time.time() < deadline:
        time.sleep(0.05)
    assert tube.pools[0].policy.in_use_bytes == in_use0
    assert tube._accounts_consistent()
    d.close()
    tube.close()

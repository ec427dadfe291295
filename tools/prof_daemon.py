"""Where a function process's put/get through the daemon spends its time:
transport ping (unique_id round trip), client-side segments of store/fetch,
daemon-side handler time per op, and the CUDA cost of interprocess vs plain
event records/waits.   python tools/prof_daemon.py"""
import multiprocessing as mp
import os
import statistics
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def med(xs):
    return round(1e6 * statistics.median(xs), 1) if xs else None


def client(path, q):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2411_01830_b200 import device as dev
    from paper_2411_01830_b200.daemon import TubeClient
    c = TubeClient(path, 0)
    res = {}
    ping = []
    for i in range(500):
        t0 = time.perf_counter()
        c.unique_id()
        ping.append(time.perf_counter() - t0)
    res["ping_unique_id_us"] = med(ping[50:])
    x = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device="cuda:0")
    out = torch.empty_like(x)
    st, ft, vt = [], [], []
    # the first loop's stores, step by step (store after a fetch(out=) copy)
    from paper_2411_01830_b200 import daemon as dmod
    first = {"alloc_call": [], "commit_call": [], "copy": [], "mark": [], "after_daemon": [], "sync": []}
    o_calls = (c._call, c._block_bin, dmod.dev.copy, c._mark, c._after_daemon)

    def tm(name, fn):
        def w(*a, **k):
            t0 = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                first[name].append(time.perf_counter() - t0)
        return w
    c._call, c._block_bin, dmod.dev.copy, c._mark, c._after_daemon = (
        tm("alloc_call", o_calls[0]), tm("commit_call", o_calls[1]), tm("copy", o_calls[2]), tm("mark", o_calls[3]),
        tm("after_daemon", o_calls[4]))
    for i in range(300):
        did = c.unique_id()
        t0 = time.perf_counter()
        c.store(did, x)
        t1 = time.perf_counter()
        c.fetch(did, out=out)
        t2 = time.perf_counter()
        did = c.unique_id()
        c.store(did, x)
        t3 = time.perf_counter()
        v = c.fetch(did)
        t4 = time.perf_counter()
        del v
        if i >= 50:
            st.append(t1 - t0)
            ft.append(t2 - t1)
            vt.append(t4 - t3)
    res["store_us"], res["fetch_out_us"], res["fetch_view_us"] = med(st), med(ft), med(vt)
    c._call, c._block_bin, dmod.dev.copy, c._mark, c._after_daemon = o_calls
    res["first_loop_steps"] = {k: (len(v), med(v[100:])) for k, v in first.items()}
    if hasattr(c, "_mine") and c._mine is not None:
        res["acked_vs_sent"] = (c._acked, c._sent)
    if getattr(c, "_bin", False):
        # per-step wall times of one zero-copy fetch + release, measured inside the client
        from paper_2411_01830_b200 import daemon as dmod
        steps = {"call": [], "after_daemon": [], "as_tensor": [], "mark": [], "done_send": []}
        o_call, o_after, o_as, o_mark, o_done = (c._block_bin, c._after_daemon, dmod.dev.as_tensor, c._mark,
                                                 c._done)

        def timed(name, fn):
            def w(*a, **k):
                t0 = time.perf_counter()
                try:
                    return fn(*a, **k)
                finally:
                    steps[name].append(time.perf_counter() - t0)
            return w
        c._block_bin, c._after_daemon, c._mark = timed("call", o_call), timed("after_daemon", o_after), \
            timed("mark", o_mark)
        c._done = timed("done_send", o_done)
        dmod.dev.as_tensor = timed("as_tensor", o_as)
        for i in range(300):
            did = c.unique_id()
            c.store(did, x)
            for k in steps:
                steps[k] = steps[k][:i] if k != "mark" else steps[k]
            v = c.fetch(did)
            del v
        c._block_bin, c._after_daemon, c._mark, c._done = o_call, o_after, o_mark, o_done
        dmod.dev.as_tensor = o_as
        res["client_fetch_steps_us"] = {k: med(v[50:]) for k, v in steps.items()}
        # the same for a store: alloc round trips (msgpack), the binary commit, copy, mark
        st_steps = {"alloc_call": [], "commit_call": [], "copy": [], "mark": [], "after_daemon": [], "total": []}
        o_callm, o_copy = c._call, dmod.dev.copy
        c._call = timed("alloc_call", o_callm)
        steps.update(st_steps)
        c._block_bin, c._mark, c._after_daemon = timed("commit_call", o_call), timed("mark", o_mark), \
            timed("after_daemon", o_after)
        dmod.dev.copy = timed("copy", o_copy)
        for i in range(300):
            did = c.unique_id()
            t0 = time.perf_counter()
            c.store(did, x)
            steps["total"].append(time.perf_counter() - t0)
            v = c.fetch(did)
            del v
        c._call, c._block_bin, c._mark, c._after_daemon = o_callm, o_call, o_mark, o_after
        dmod.dev.copy = o_copy
        res["client_store_steps"] = {k: (len(steps[k]), med(steps[k][50:])) for k in st_steps}
        # client-side split of a zero-copy fetch: the binary round trip alone vs the rest
        import cProfile
        import pstats
        pr = cProfile.Profile()
        for i in range(300):
            did = c.unique_id()
            c.store(did, x)
            pr.enable()
            v = c.fetch(did)
            del v
            pr.disable()
        import io
        buf = io.StringIO()
        pstats.Stats(pr, stream=buf).sort_stats("tottime").print_stats(16)
        res["client_fetch_profile"] = buf.getvalue()
    # CUDA cost of the ordering primitives in this process
    s = torch.cuda.current_stream(0).cuda_stream
    ring = dev.IpcEventRing(0, 4)
    plain = dev.Ev(0)
    rec_ipc, rec_plain, wait_ipc, wait_plain, copy = [], [], [], [], []
    for i in range(500):
        t0 = time.perf_counter()
        ring.record(i % 4, s)
        t1 = time.perf_counter()
        plain.record(s)
        t2 = time.perf_counter()
        dev.wait_events(s, [ring.h[i % 4]]) if False else dev.LIB.ft_stream_wait_events(
            dev.C.c_void_p(s), (dev.C.c_void_p * 1)(ring.h[i % 4]), 1)
        t3 = time.perf_counter()
        plain.wait(s)
        t4 = time.perf_counter()
        dev.copy(out.data_ptr(), x.data_ptr(), 4096, 0, s)
        t5 = time.perf_counter()
        rec_ipc.append(t1 - t0)
        rec_plain.append(t2 - t1)
        wait_ipc.append(t3 - t2)
        wait_plain.append(t4 - t3)
        copy.append(t5 - t4)
    torch.cuda.synchronize()
    res["cuda_us"] = {"record_ipc": med(rec_ipc), "record_plain": med(rec_plain), "wait_ipc": med(wait_ipc),
                      "wait_plain": med(wait_plain), "copy_4k_launch": med(copy)}
    import msgpack
    m = {"op": "commit", "token": 12, "id": 99, "dtype": "torch.uint8", "shape": [1 << 20], "producer": "func",
         "consumers": 1, "response": False, "ev": 3, "next": 1 << 20}
    pk, up = [], []
    for i in range(2000):
        t0 = time.perf_counter()
        b = msgpack.packb(m)
        t1 = time.perf_counter()
        msgpack.unpackb(b)
        t2 = time.perf_counter()
        pk.append(t1 - t0)
        up.append(t2 - t1)
    res["msgpack_us"] = {"pack": med(pk), "unpack": med(up)}
    c.close()
    q.put(res)


def main():
    import torch
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(pcie_gbps=55.0, gpus=[0])
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    times = {}
    orig = d._handle
    import cProfile
    import pstats
    prof, calls = {}, {}

    def timed(conn, msg):
        op = msg["op"]
        calls[op] = calls.get(op, 0) + 1
        pr = prof.setdefault(op, cProfile.Profile()) if calls[op] % 2 else None
        t0 = time.perf_counter()
        if pr is not None:
            pr.enable()
        try:
            return orig(conn, msg)
        finally:
            if pr is not None:
                pr.disable()
            else:
                times.setdefault(op, []).append(time.perf_counter() - t0)
    d._handle = timed
    ost, ofe = tube.store_block, tube.fetch_resident
    tin = {"tube.store_block": [], "tube.fetch_resident": [], "tube.lend_block": []}

    def st(*a, **k):
        t0 = time.perf_counter()
        try:
            return ost(*a, **k)
        finally:
            tin["tube.store_block"].append(time.perf_counter() - t0)

    def fr(*a, **k):
        t0 = time.perf_counter()
        try:
            return ofe(*a, **k)
        finally:
            tin["tube.fetch_resident"].append(time.perf_counter() - t0)
    oem = tube.lend_block

    def em(*a, **k):
        t0 = time.perf_counter()
        try:
            return oem(*a, **k)
        finally:
            tin["tube.lend_block"].append(time.perf_counter() - t0)
    tube.store_block, tube.fetch_resident, tube.lend_block = st, fr, em
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=client, args=(path, q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    res["daemon_handler_us"] = {k: med(v[50:]) for k, v in times.items()}
    res["daemon_tube_us"] = {k: med(v[50:]) for k, v in tin.items()}
    prof_txt = res.pop("client_fetch_profile", "")
    print(res)
    print(prof_txt)
    for op in ("commit", "fetch", "done"):
        if op in prof:
            print("==== daemon handler profile:", op)
            pstats.Stats(prof[op]).sort_stats("tottime").print_stats(14)
    d.close()
    tube.close()


if __name__ == "__main__":
    main()

"""GPU-side latency of a cross-process stream dependency: process A records an
interprocess event after a device spin; process B's stream waits on it and records
its own event. Both hosts poll their event and stamp completion on the shared
monotonic clock: B's completion minus A's is the time the dependency took to
resolve on the device (vs the same with two streams of one process).
python tools/probe_ipc_latency.py"""
import ctypes as C
import multiprocessing as mp
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def poll(ev):
    import ctypes as C
    from paper_2411_01830_b200 import device as dev
    d = C.c_int()
    q = dev.LIB.raw("ft_event_query")
    while True:
        q(C.c_void_p(ev), C.byref(d))
        if d.value:
            return time.perf_counter()


def side_a(q_h, q_go, q_t):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2411_01830_b200 import device as dev
    torch.cuda.init()
    ring = dev.IpcEventRing(0, 1)
    q_h.put(ring.handles[0])
    s = torch.cuda.Stream(0)
    while True:
        go = q_go.get()
        if go is None:
            return
        dev.LIB.ft_spin_ns(200_000, 0, C.c_void_p(s.cuda_stream))
        ring.record(0, s.cuda_stream)
        q_t.put(poll(ring.h[0]))


def main():
    import torch
    from paper_2411_01830_b200 import device as dev
    ctx = mp.get_context("spawn")
    q_h, q_go, q_t = ctx.Queue(), ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=side_a, args=(q_h, q_go, q_t))
    p.start()
    peer = dev.PeerEvents(0, [q_h.get(timeout=120)])
    s = torch.cuda.Stream(0)
    mine = dev.Ev(0)
    lat = []
    for i in range(60):
        q_go.put(1)
        time.sleep(0.00005)
        peer.wait(0, s.cuda_stream)
        mine.record(s.cuda_stream)
        tb = poll(mine.h)
        ta = q_t.get()
        lat.append(tb - ta)
    q_go.put(None)
    p.join(30)
    # one process, two streams
    s1, s2 = torch.cuda.Stream(0), torch.cuda.Stream(0)
    e1, e2 = dev.Ev(0), dev.Ev(0)
    loc = []
    for i in range(60):
        dev.LIB.ft_spin_ns(200_000, 0, C.c_void_p(s1.cuda_stream))
        e1.record(s1.cuda_stream)
        e1.wait(s2.cuda_stream)
        e2.record(s2.cuda_stream)
        ta = poll(e1.h)
        tb = poll(e2.h)
        loc.append(tb - ta)
    lat.sort()
    loc.sort()
    print(f"cross-process dependency: p50 {1e6 * lat[len(lat) // 2]:.1f} us  p90 {1e6 * lat[int(.9 * len(lat))]:.1f} us;"
          f" same process: p50 {1e6 * loc[len(loc) // 2]:.1f} us")


if __name__ == "__main__":
    main()

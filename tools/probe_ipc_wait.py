"""Does a stream wait on another process's CUDA event stall the host at the next
launch? Process A records an interprocess event after a device spin of S us;
process B makes its stream wait on it and launches a copy: the wall time of that
launch call, for spins of 0 / 50 / 200 us (and the same with a plain event of B's
own for comparison).   python tools/probe_ipc_wait.py"""
import ctypes as C
import multiprocessing as mp
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def side_a(q_h, q_go, q_done):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2411_01830_b200 import device as dev
    torch.cuda.init()
    ring = dev.IpcEventRing(0, 1)
    q_h.put(ring.handles[0])
    s = torch.cuda.Stream(0)
    while True:
        spin = q_go.get()
        if spin is None:
            return
        dev.LIB.ft_spin_ns(int(spin * 1000), 0, C.c_void_p(s.cuda_stream))
        ring.record(0, s.cuda_stream)
        q_done.put(1)
        s.synchronize()


def main():
    import torch
    from paper_2411_01830_b200 import device as dev
    ctx = mp.get_context("spawn")
    q_h, q_go, q_done = ctx.Queue(), ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=side_a, args=(q_h, q_go, q_done))
    p.start()
    peer = dev.PeerEvents(0, [q_h.get(timeout=120)])
    s = torch.cuda.Stream(0)
    x = torch.empty(1 << 20, dtype=torch.uint8, device="cuda:0")
    y = torch.empty_like(x)
    own = dev.Ev(0)
    s2 = torch.cuda.Stream(0)
    for spin in (0, 50, 200, 1000):
        ipc, loc = [], []
        for i in range(40):
            q_go.put(spin)
            q_done.get()                    # A has enqueued the spin and the record
            peer.wait(0, s.cuda_stream)
            t0 = time.perf_counter()
            dev.copy(y.data_ptr(), x.data_ptr(), x.nbytes, 0, s, dev.ENGINE_BULK)
            ipc.append(time.perf_counter() - t0)
            s.synchronize()
            # same with an event of this process recorded after a local spin
            dev.LIB.ft_spin_ns(int(spin * 1000), 0, C.c_void_p(s2.cuda_stream))
            own.record(s2.cuda_stream)
            own.wait(s.cuda_stream)
            t0 = time.perf_counter()
            dev.copy(y.data_ptr(), x.data_ptr(), x.nbytes, 0, s, dev.ENGINE_BULK)
            loc.append(time.perf_counter() - t0)
            s.synchronize()
        print(f"spin={spin}us launch after wait: ipc event {1e6 * statistics.median(ipc[5:]):.1f} us, "
              f"local event {1e6 * statistics.median(loc[5:]):.1f} us")
    q_go.put(None)
    p.join(30)


if __name__ == "__main__":
    main()

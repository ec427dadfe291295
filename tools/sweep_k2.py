"""K2 vs the event chain vs the direct route: 1 GiB pinned host -> GPU 0 through
one route of the pacer on one PCIe link, unmanaged and managed, for several
chunk sizes (pcie_sched.py:14's 2 MB and larger). Device-event time."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402

n = 1 << 30
host = torch.empty(n, dtype=torch.uint8).pin_memory()
host[::4093] = 7
dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
s = torch.cuda.current_stream(0)
streams = (torch.cuda.Stream(0), torch.cuda.Stream(0))


def run(kind, chunk, managed, reps=4):
    p = dev.Pacer(55.0, 5, chunk, staging_slots=4, host_ring_bytes=64 << 20, adapt=False)
    routes = [(0, int(kind == "staged"), 0, n, streams[0].cuda_stream, streams[1].cuda_stream)]
    ts = []
    for i in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        p.submit("", managed, 1e9, 0.0, 1e9, dst.data_ptr(), 0, host.data_ptr(), n, True, routes, s.cuda_stream)
        b.record(s)
        b.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    p.close()
    ok = torch.equal(dst.cpu(), host)
    return n / (statistics.median(ts) * 1e-3) / 1e9, ok


for managed in (False, True):
    g, ok = run("direct", 2_000_000, managed)
    print(f"managed={managed} direct: {g:.2f} GB/s ok={ok}", flush=True)
    for piece in ("2000000", "4000000", "8000000"):
        for k2, ce2 in (("1", "1"), ("0", "1")):
            os.environ["FT_K2"], os.environ["FT_K2_CE2"] = k2, ce2
            if piece:
                os.environ["FT_STAGE_CHUNK"] = piece
            else:
                os.environ.pop("FT_STAGE_CHUNK", None)
            g, ok = run("staged", 2_000_000, managed)
            print(f"managed={managed} staged piece={piece or 'auto(<=8MB)'} K2={k2} CE2={ce2}: {g:.2f} GB/s ok={ok}",
                  flush=True)
    os.environ["FT_K2"], os.environ["FT_K2_CE2"] = "1", "1"
    os.environ.pop("FT_STAGE_CHUNK", None)

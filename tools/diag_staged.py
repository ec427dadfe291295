"""A 1 GiB host->GPU stage carried entirely by a forced staging route (CE ->
chunk ring -> forward kernel) vs a direct route, on one GPU; FT_STAGE_CHUNK
sets the ring slot size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
n = 1 << 30
host = torch.randint(0, 256, (n,), dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
s0 = torch.cuda.current_stream(0)
p = dev.Pacer(55.0, 5, 2 * 10**6, staging_slots=int(os.environ.get("SLOTS", 4)))
ce, fw = dev.new_stream(0), dev.new_stream(0)
for kind in (0, 1):
    r = [(0, kind, 0, n, ce.cuda_stream, fw.cuda_stream)]
    ts = []
    for i in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        p.wait(p.submit("", True, 1e9, 0.0, 1e9, dst.data_ptr(), 0, host.data_ptr(), n, True, r, s0.cuda_stream))
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    assert torch.equal(dst[-8192:].cpu(), host[-8192:])
    print(f"stage_chunk={os.environ.get('FT_STAGE_CHUNK', '2000000')} slots={os.environ.get('SLOTS', 4)} "
          f"{'staged' if kind else 'direct'}: {n / sorted(ts)[2] / 1e9:.2f} GB/s", flush=True)
p.close()

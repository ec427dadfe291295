"""Config-1 pass (store copy + fetch copy, 64 MiB) under every L2 hint combination."""
import itertools, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64 << 20
x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
blk = torch.empty(n, dtype=torch.uint8, device="cuda:0")
inp = torch.empty_like(blk)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
s = torch.cuda.current_stream(0)
N, F, L = dev.L2_NORMAL, dev.L2_EVICT_FIRST, dev.L2_EVICT_LAST
res = []
for ss, sd, fs, fd in itertools.product((N, F), (N, L), (N, F), (N, F)):
    ts = []
    for i in range(40):
        flush.fill_(i & 0xFF); flush.amax()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        dev.copy_hint(blk.data_ptr(), x.data_ptr(), n, 0, s, ss, sd)
        dev.copy_hint(inp.data_ptr(), blk.data_ptr(), n, 0, s, fs, fd)
        b.record(s)
        b.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b))
    res.append((statistics.median(ts), (ss, sd, fs, fd)))
for ms, k in sorted(res)[:8]:
    print(f"pass {ms*1e3:.2f} us  store(src,dst)={k[:2]} fetch(src,dst)={k[2:]}  -> {n/(ms*1e-3)/1e9:.0f} GB/s")
print("current (F,L | F,N):", [f"{ms*1e3:.2f}" for ms, k in res if k == (F, L, F, N)])

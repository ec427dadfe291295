"""Small exercise of every device kernel, for compute-sanitizer (memcheck / racecheck)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
from paper_2411_01830_b200._lib import LIB
s = torch.cuda.current_stream(0)
for n, shift in ((1, 0), (17, 3), (4097, 0), ((1 << 20) + 5, 1), (3 << 20, 0)):
    x = torch.randint(0, 256, (n + 16,), dtype=torch.uint8, device="cuda:0")
    y = torch.zeros_like(x)
    for eng in (1, 2):
        dev.copy(y.data_ptr() + shift, x.data_ptr() + shift, n, 0, s, eng)
    dev.copy_hint(y.data_ptr(), x.data_ptr(), n, 0, s, dev.L2_EVICT_FIRST, dev.L2_EVICT_LAST)
    fp = dev.Fingerprint(0); fp.launch(x.data_ptr(), n, s)
torch.cuda.synchronize()
dev.copy_batch([(y.data_ptr(), x.data_ptr(), 1000), (y.data_ptr() + 2048, x.data_ptr() + 7, 70000)], 0, s)
w = torch.zeros(4, dtype=torch.int32, device="cuda:0")
LIB.ft_signal(C.c_void_p(w.data_ptr()), 3, 0, C.c_void_p(s.cuda_stream))
LIB.ft_wait_timeout(C.c_void_p(w.data_ptr()), 3, 10**9, C.c_void_p(w.data_ptr() + 8), 0, C.c_void_p(s.cuda_stream))
LIB.ft_spin_ns(100000, 0, C.c_void_p(s.cuda_stream))
torch.cuda.synchronize()
p = dev.Pacer(50.0, 5, 2 * 10**6, staging_slots=2)
h = torch.randint(0, 256, (5 * 10**6 + 3,), dtype=torch.uint8).pin_memory()
d = torch.zeros(h.numel(), dtype=torch.uint8, device="cuda:0")
st = [(torch.cuda.Stream(0), torch.cuda.Stream(0)) for _ in range(2)]
half = h.numel() // 2 // 256 * 256
r = [(0, 0, 0, half, st[0][0].cuda_stream, st[0][1].cuda_stream), (0, 1, half, h.numel() - half, st[1][0].cuda_stream, st[1][1].cuda_stream)]
t = p.submit("", True, 1e9, 0.0, 50.0, d.data_ptr(), 0, h.data_ptr(), h.numel(), True, r, s.cuda_stream)
p.wait(t)
t = p.submit_d2h("", True, 1e9, 0.0, 50.0, h.data_ptr(), d.data_ptr(), 0, h.numel(), r, s.cuda_stream)
p.wait(t)
torch.cuda.synchronize()
assert torch.equal(d.cpu(), h)
p.close()
# K2 forward (device flags + one forward kernel per batch), misaligned destination too
os.environ["FT_K2"] = "1"
p = dev.Pacer(50.0, 5, 2 * 10**6, staging_slots=2)
for off in (0, 3):
    d = torch.zeros(h.numel() + 16, dtype=torch.uint8, device="cuda:0")
    t = p.submit("", off == 0, 1e9, 0.0, 50.0, d.data_ptr() + off, 0, h.data_ptr(), h.numel(), True,
                 [(0, 1, 0, h.numel(), st[0][0].cuda_stream, st[0][1].cuda_stream)], s.cuda_stream)
    p.wait(t)
    torch.cuda.synchronize()
    assert torch.equal(d[off:off + h.numel()].cpu(), h)
p.close()
# fused request-path calls and the batched retire
from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402
tube = FaaSTube("faastube", gpus=[0], pcie_gbps=50.0, pool_floor_bytes=0.0)
xs = [torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0") for n in (1, 4097, 1 << 20)]
ids = []
for x in xs:
    ids.append(tube.unique_id())
    tube.store(ids[-1], x, consumers=2)
outs = [torch.empty_like(x) for x in xs]
for i, o in zip(ids, outs):
    tube.fetch(i, device=0, out=o)
tube.fetch_many([(i, torch.empty_like(x)) for i, x in zip(ids, xs)])
torch.cuda.synchronize()
assert all(torch.equal(a, b) for a, b in zip(xs, outs))
tube.close()
print("kernels exercised ok")

"""Driver for ncu captures of the data-path kernels (run under ncu, one GPU):
K1 k_copy_vec at 1 MiB and 64 MiB (the NVLink mover, here local), k_copy_bulk at
1 MiB and 64 MiB (the same-GPU store/fetch copy), k_copy_multi over 64 x 1 MiB
(fetch_many), and K2's k_forward on a staged 64 MiB stage (FT_K2=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402

s = torch.cuda.current_stream(0)
for n in (1 << 20, 64 << 20):
    x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    y = torch.empty_like(x)
    for _ in range(3):
        dev.copy(y.data_ptr(), x.data_ptr(), n, 0, s, dev.ENGINE_VEC)
    for _ in range(3):
        dev.copy(y.data_ptr(), x.data_ptr(), n, 0, s, dev.ENGINE_BULK)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
xs = torch.randint(0, 256, (64, 1 << 20), dtype=torch.uint8, device="cuda:0")
ys = torch.empty_like(xs)
for _ in range(3):
    dev.copy_batch([(ys[j].data_ptr(), xs[j].data_ptr(), 1 << 20) for j in range(64)], 0, s)
torch.cuda.synchronize()
assert torch.equal(xs, ys)
os.environ["FT_K2"] = "1"
p = dev.Pacer(55.0, 5, 2_000_000, staging_slots=4, host_ring_bytes=16 << 20)
n = 64 << 20
host = torch.randint(0, 256, (n,), dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
st = (torch.cuda.Stream(0), torch.cuda.Stream(0))
t = p.submit("", False, 1e9, 0.0, 1e9, dst.data_ptr(), 0, host.data_ptr(), n, True,
             [(0, 1, 0, n, st[0].cuda_stream, st[1].cuda_stream)], s.cuda_stream)
torch.cuda.synchronize()
p.wait(t)
assert torch.equal(dst.cpu(), host)
p.close()
print("ok")

"""Driver for ncu captures of the other kernels on their config sizes:
k_copy_vec (K1/K2 NVLink engine, here local 64 MiB), k_copy_multi (64 x 1 MiB
batched handoff), k_fingerprint (64 MiB digest)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402

n = 64 << 20
x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
y = torch.empty_like(x)
for _ in range(3):
    dev.copy(y.data_ptr(), x.data_ptr(), n, 0, None, dev.ENGINE_VEC)
segs = [(y.data_ptr() + i * (1 << 20), x.data_ptr() + i * (1 << 20), 1 << 20) for i in range(64)]
for _ in range(3):
    dev.copy_batch(segs, 0, torch.cuda.current_stream(0).cuda_stream)
fp = dev.Fingerprint(0)
for _ in range(3):
    fp.launch(x.data_ptr(), n, torch.cuda.current_stream(0))
torch.cuda.synchronize()
assert torch.equal(x, y) and fp.value() == dev.fingerprint_host(x.cpu())
print("ok")

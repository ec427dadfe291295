"""Minimal driver for ncu captures of the copy kernel (64 MiB config-1 payload)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64 << 20
engine = int(sys.argv[2]) if len(sys.argv) > 2 else dev.ENGINE_BULK
x = torch.empty(n, dtype=torch.uint8, device="cuda:0").fill_(5)
y = torch.empty_like(x)
for _ in range(5):
    dev.copy(y.data_ptr(), x.data_ptr(), n, 0, None, engine)
torch.cuda.synchronize()
assert torch.equal(x, y)
print("ok")

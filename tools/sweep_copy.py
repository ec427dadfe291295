"""Copy-kernel shape sweep (run on the GPU box): FT_BULK_* env variants in
subprocesses; clean-L2 CUDA-event timing at 64 MiB and 1 GiB."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, statistics, json
sys.path.insert(0, %r)
import torch
from paper_2411_01830_b200 import device as dev
res = {}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
for n in (4 << 20, 64 << 20, 1 << 30):
    x = torch.empty(n, dtype=torch.uint8, device="cuda:0").fill_(1); y = torch.empty_like(x)
    ts = []
    for i in range(25):
        flush.fill_(i); flush.amax()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); dev.copy(y.data_ptr(), x.data_ptr(), n, 0, None, int(os.environ.get("ENG", "1"))); b.record()
        b.synchronize()
        if i >= 5: ts.append(a.elapsed_time(b))
    assert torch.equal(x, y)
    res[n] = 2 * n / (statistics.median(ts) * 1e-3) / 1e9
print(json.dumps(res))
''' % ROOT
variants = [dict(ENG="2")]
for st in (2, 3, 4, 6):
    for tile in (16384, 32768, 49152):
        if st * tile > 200 * 1024:
            continue
        for per in (1, 2, 3, 4):
            if per * st * tile > 220 * 1024:
                continue
            variants.append(dict(FT_BULK_STAGES=str(st), FT_BULK_TILE=str(tile), FT_BULK_CTAS_PER_SM=str(per)))
out = []
for v in variants:
    env = dict(os.environ, **v)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-300:]
    print(v, line, flush=True)
    out.append({"env": v, "result": line})
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "sweep_copy.json"), "w"), indent=1)

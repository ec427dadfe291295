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
eng = int(os.environ.get("ENG", "1"))
for n in (4 << 20, 64 << 20, 256 << 20, 1 << 30):
    pairs = max(1, min(8, (1 << 30) // n))          # cycle >= 1 GiB of sources: nothing hits L2
    xs = [torch.empty(n, dtype=torch.uint8, device="cuda:0").fill_(i + 1) for i in range(pairs)]
    ys = [torch.empty_like(x) for x in xs]
    reps = 40
    for i in range(pairs):
        dev.copy(ys[i].data_ptr(), xs[i].data_ptr(), n, 0, None, eng)
    torch.cuda.synchronize()
    best = []
    for trial in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for r in range(reps):
            i = r %% pairs
            dev.copy(ys[i].data_ptr(), xs[i].data_ptr(), n, 0, None, eng)
        b.record(); b.synchronize()
        best.append(a.elapsed_time(b) / reps)
    for i in range(pairs):
        assert torch.equal(xs[i], ys[i])
    res[n] = round(2 * n / (min(best) * 1e-3) / 1e9, 1)
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

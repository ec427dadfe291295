"""Tail of the bench's e2e step (zero-copy flow): per-phase host timestamps of
the slowest steps out of 400."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01830_b200 import device as dev  # noqa: E402
from paper_2411_01830_b200.tube import FaaSTube  # noqa: E402

tube = FaaSTube("faastube")
n = 64 << 20
host_in = torch.randint(0, 256, (n,), dtype=torch.uint8).pin_memory()
fp = dev.Fingerprint(0)
s = torch.cuda.current_stream(0)
gcs = []
gc.callbacks.append(lambda phase, info: gcs.append((time.perf_counter(), phase, info.get("generation"))))
rows = []
nxt = tube.empty((n,), torch.uint8, device=0)
for i in range(420):
    t = [time.perf_counter()]
    out = nxt
    d_in = tube.unique_id()
    tube.store(d_in, host_in, producer="decode"); t.append(time.perf_counter())
    tube.fetch(d_in, device=0, out=out, consumer="producer"); t.append(time.perf_counter())
    nxt = tube.empty((n,), torch.uint8, device=0); t.append(time.perf_counter())
    did = tube.unique_id()
    tube.store(did, out, producer="producer"); del out
    view = tube.fetch(did, device=0, consumer="consumer"); t.append(time.perf_counter())
    fp.launch(view.data_ptr(), n, s); del view
    fp.value(); t.append(time.perf_counter())
    if i >= 20:
        rows.append((t[-1] - t[0], [1e3 * (t[k + 1] - t[k]) for k in range(len(t) - 1)], t[0], t[-1]))
rows.sort(key=lambda r: r[0])
print("p50 step ms %.4f  p99 %.4f  max %.4f" % (1e3 * rows[len(rows) // 2][0], 1e3 * rows[int(len(rows) * .99)][0],
                                                 1e3 * rows[-1][0]))
print("phases: store_host | fetch_h2g(submit) | empty | store+view | digest+sync")
print("median", [round(sorted(r[1][k] for r in rows)[len(rows) // 2], 4) for k in range(5)])
for r in rows[-6:]:
    g = [(ph, gen) for (tt, ph, gen) in gcs if r[2] <= tt <= r[3]]
    print(round(1e3 * r[0], 4), [round(x, 4) for x in r[1]], "gc:", g)
tube.close()

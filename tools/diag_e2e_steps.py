"""Per-phase host timestamps and device events of the bench's e2e step."""
import os, statistics, sys, time
os.environ.setdefault("FT_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
from paper_2411_01830_b200.tube import FaaSTube
tube = FaaSTube("faastube")
n = 64 << 20
x = torch.randn(32, 1024, 1024).half().cuda()
host_in = torch.empty(n, dtype=torch.uint8).pin_memory(); host_in.copy_(x.view(-1).view(torch.uint8).cpu())
prod_out = torch.empty_like(x); inp = torch.empty_like(x)
fp = dev.Fingerprint(0); s = torch.cuda.current_stream(0)
rows = []
for i in range(60):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t = [time.perf_counter()]
    d_in = tube.unique_id(); tube.store(d_in, host_in, producer="decode"); t.append(time.perf_counter())
    e[0].record(s)
    tube.fetch(d_in, device=0, out=prod_out.view(-1).view(torch.uint8), consumer="producer"); t.append(time.perf_counter())
    e[1].record(s)
    did = tube.unique_id(); tube.store(did, prod_out, producer="producer"); tube.fetch(did, device=0, out=inp, consumer="consumer"); t.append(time.perf_counter())
    e[2].record(s)
    fp.launch(inp.data_ptr(), n, s); e[3].record(s); t.append(time.perf_counter())
    fp.value(); t.append(time.perf_counter())
    torch.cuda.synchronize()
    if i >= 10:
        rows.append(([1e3 * (t[k + 1] - t[k]) for k in range(len(t) - 1)], [e[k].elapsed_time(e[k + 1]) for k in range(3)], 1e3 * (t[-1] - t[0])))
med = lambda xs: round(statistics.median(xs), 4)
print("host ms: store_host %.4f | fetch_h2g(submit) %.4f | store+fetch %.4f | fp.launch %.4f | fp.value(sync) %.4f" % tuple(med([r[0][k] for r in rows]) for k in range(5)))
print("gpu ms: h2g %.4f | store+fetch copies %.4f | digest %.4f" % tuple(med([r[1][k] for r in rows]) for k in range(3)))
print("step ms", med([r[2] for r in rows]), "-> GB/s", round(n / med([r[2] for r in rows]) / 1e6, 1))
tr = tube.pacer.trace()
st = {}
for tt, tk, kind, v in tr:
    if tk: st.setdefault(tk, []).append((tt, kind))
ds = []
for tk, ev in st.items():
    k = dict((b, a) for a, b in ev)
    if "start" in k and "land" in k:
        ds.append((k["land"] - k["start"], ev[1][0] - k["start"] if len(ev) > 1 else 0))
if ds:
    print("pacer stage start->land ms", med([d[0] for d in ds]), "start->first event ms", med([d[1] for d in ds]))
tube.close()
# the link itself: one 64 MiB pinned H2D per step (cudaMemcpyAsync), same box
raw = []
for i in range(40):
    t0 = time.perf_counter()
    prod_out.view(-1).view(torch.uint8).copy_(host_in, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    if i >= 5:
        raw.append(1e3 * (time.perf_counter() - t0))
print("raw 64 MiB H2D copy+sync ms", med(raw), "-> GB/s", round(n / med(raw) / 1e6, 1))

"""Reproduce the bench sequence up to the 1 GiB managed H2G fetch with a watchdog."""
import os, sys, threading, time, json, faulthandler
os.environ["FT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200 import device as dev
from paper_2411_01830_b200.tube import FaaSTube

tube = FaaSTube("faastube")
print("pcie", tube.topo.pcie_gbps, flush=True)

def watchdog():
    time.sleep(float(sys.argv[1]) if len(sys.argv) > 1 else 40)
    print("WATCHDOG", flush=True)
    res = {}
    def grab():
        res["stats"] = tube.pacer.stats()
        res["state"] = tube.pacer.state()
        res["trace"] = tube.pacer.trace()[-25:]
    t = threading.Thread(target=grab, daemon=True); t.start(); t.join(5)
    print(json.dumps(res, default=str)[:6000] if res else "pacer calls hung (mu held)", flush=True)
    faulthandler.dump_traceback(all_threads=True)
    os._exit(3)
threading.Thread(target=watchdog, daemon=True).start()

g = 0
s = torch.cuda.current_stream(0)
for n, reps in ((64 << 20, 30), (1 << 30, 4)):
    host = torch.empty(n, dtype=torch.uint8).pin_memory(); host.fill_(7)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    for _ in range(2):
        dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, g, s)
    torch.cuda.synchronize()
    for i in range(reps):
        t0 = time.perf_counter()
        did = tube.unique_id()
        tube.store(did, host, producer="decode")
        tube.fetch(did, device=g, out=dst, consumer="preproc")
        torch.cuda.synchronize()
        print(n, i, round((time.perf_counter() - t0) * 1e3, 3), "ms", flush=True)
print("done", tube.pacer.stats(), flush=True)
os._exit(0)

import os, sys, time, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2411_01830_b200 import device as dev
MB = 10**6
def run(n, kinds, managed, same=False):
    p = dev.Pacer(55.0, 5, 2 * MB, staging_slots=3, host_ring_bytes=8 * MB)
    k = len(kinds)
    bounds = [0] + [min(n, (n * (i + 1) // k) // 256 * 256) for i in range(k - 1)] + [n]
    streams = [(torch.cuda.Stream(0), torch.cuda.Stream(0)) for _ in kinds]
    routes = [(0, int(kd == "s"), bounds[i], bounds[i+1]-bounds[i], streams[i][0].cuda_stream, streams[i][1].cuda_stream) for i, kd in enumerate(kinds)]
    host = torch.from_numpy(np.random.default_rng(1).integers(0, 256, n, dtype=np.uint8)).pin_memory()
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    s = torch.cuda.current_stream(0)
    t0 = time.time()
    try:
        t = p.submit("", managed, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True, routes, s.cuda_stream)
        torch.cuda.synchronize()
        p.wait(t, 20000.0)
        ok = torch.equal(dst.cpu(), host)
        print(n, kinds, managed, "ok" if ok else "BYTES DIFFER", round(time.time()-t0, 3), flush=True)
    except Exception as e:
        print(n, kinds, managed, "ERR", repr(e)[:600], round(time.time()-t0, 3), flush=True)
    p.close()
for args in [(1, "d", False), (4097, "ds", False), (3*MB, "s", False), (11*MB, "s", False), (11*MB, "s", True), (22*MB, "ss", False), (33555209, "dss", False), (33555209, "dss", True), (64*MB, "s", False)]:
    run(*args)

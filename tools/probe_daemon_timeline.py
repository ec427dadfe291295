import multiprocessing as mp, os, statistics, sys, tempfile, time
ROOT = "/root/repo"
sys.path.insert(0, ROOT)
def client(path, q):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2411_01830_b200.daemon import TubeClient
    c = TubeClient(path, 0)
    out = []
    for n, k in ((4096, 1500), (64 << 20, 300), (4096, 2000)):
        x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
        st = []
        t00 = time.perf_counter()
        for i in range(k):
            did = c.unique_id()
            t0 = time.perf_counter()
            c.store(did, x)
            st.append(time.perf_counter() - t0)
            v = c.fetch(did); del v
        wins = [round(1e6 * statistics.median(st[j:j + 100]), 1) for j in range(0, k, 100)]
        out.append((n, round(time.perf_counter() - t00, 3), wins))
    c.close()
    q.put(out)
if __name__ == "__main__":
    from paper_2411_01830_b200.daemon import TubeDaemon
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(gpus=[0], pcie_gbps=55.0)
    path = os.path.join(tempfile.mkdtemp(), "s.sock")
    d = TubeDaemon(tube, path)
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    p = ctx.Process(target=client, args=(path, q)); p.start()
    for row in q.get(timeout=600): print(row, flush=True)
    p.join(60); d.close(); tube.close()

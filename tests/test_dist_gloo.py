"""Multi-process host logic on CPU (world_size 2, gloo): the function<->daemon
channel passes descriptors between ranks (SCM_RIGHTS), and the bench's
max-over-ranks aggregation is what the N>1 runs report."""

import os
import tempfile

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, sockdir, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2411_01830_b200.channel import Channel
    path = os.path.join(sockdir, "tube.sock")
    try:
        if rank == 0:
            srv = Channel.listen(path)
            dist.barrier()
            ch = Channel.accept(srv)
            fd, path_r = tempfile.mkstemp()
            os.write(fd, b"faastube-payload")
            ch.send_fd(fd, {"data_id": 7, "nbytes": 16})
            reply = ch.recv_msg()
            os.close(fd)
            q.put(("rank0", reply))
        else:
            dist.barrier()
            ch = Channel.connect(path)
            fd, meta = ch.recv_fd()
            os.lseek(fd, 0, 0)
            data = os.read(fd, meta["nbytes"])
            ch.send_msg({"ok": data == b"faastube-payload", "data_id": meta["data_id"]})
            os.close(fd)
        # max-over-ranks timing as bench.py reports it
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((f"max{rank}", t.item()))
    finally:
        dist.destroy_process_group()


def test_channel_and_max_over_ranks():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        procs = [ctx.Process(target=_worker, args=(r, 2, port, d, q)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=120)
        got = {}
        while not q.empty():
            k, v = q.get()
            got[k] = v
    assert all(p.exitcode == 0 for p in procs)
    assert got["rank0"] == {"ok": True, "data_id": 7}
    assert got["max0"] == 2.0 and got["max1"] == 2.0

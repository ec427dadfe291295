"""Cross-process producer->consumer ring with device doorbells (the N>1 bench
path), run as two processes on one GPU: fd exchange, peer mapping, RDY/ACK
ordering and bit-exact delivery over several steps."""

import multiprocessing as mp
import os
import socket
import sys
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank(rank, world, port, sock_dir, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_01830_b200.pairs import CrossPair
        from paper_2411_01830_b200.tube import FaaSTube
        tube = FaaSTube("faastube", pool_floor_bytes=0.0, gpus=[0])
        n = 8 << 20
        pair = CrossPair(tube, 0, rank, world, sock_dir, n, dist.barrier)
        out = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        ok = True
        for step in range(1, 6):
            x = torch.full((n,), (rank * 16 + step) & 0xFF, dtype=torch.uint8, device="cuda:0")
            pair.produce(x)
            pair.consume(out)
            torch.cuda.synchronize()
            want = (((rank - 1) % world) * 16 + step) & 0xFF      # previous rank's payload of this step
            ok = ok and int(out.min()) == want and int(out.max()) == want
        pair.close()
        tube.close()
        q.put((rank, ok))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_process_ring_bit_exact():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        ps = [ctx.Process(target=_rank, args=(r, 2, port, d, q)) for r in range(2)]
        for p in ps:
            p.start()
        res = dict(q.get(timeout=300) for _ in ps)
        for p in ps:
            p.join(timeout=60)
    assert res == {0: True, 1: True}, res

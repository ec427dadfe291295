"""Cross-process zero-copy handoff: a pool block exported as a POSIX fd
(cuMemExportToShareableHandle), passed over a Unix socket with SCM_RIGHTS,
imported and mapped by another process (the paper's CUDA-IPC channel between
function processes and the per-box daemon)."""

import multiprocessing as mp
import os
import socket
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _child(s, arena_bytes, off, nbytes, q):
    sys.path.insert(0, ROOT)
    try:
        from paper_2411_01830_b200 import device
        fd, tag = device.recv_fd(s)
        blk = device.ImportedBlock(0, fd, arena_bytes, off, nbytes)
        t = blk.tensor()
        fp = device.Fingerprint(0)
        fp.launch(t.data_ptr(), tag)
        val = fp.value()
        t[:16].fill_(0xAB)                       # write back through the mapping
        torch.cuda.synchronize()
        del t
        blk.close()
        q.put(("ok", val))
    except Exception as exc:  # noqa: BLE001
        q.put(("err", repr(exc)))


def test_export_import_across_processes():
    from paper_2411_01830_b200 import device
    pool = device.DevicePool(0, "cache_all", floor_bytes=0.0)
    n = 8 * 10**6 + 123
    blk = pool.allocate(n)
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    view = device.as_tensor(blk.ptr, n, 0)
    view.copy_(src)
    torch.cuda.synchronize()
    fd, arena_bytes, off = pool.export(blk)        # the block's arena + its offset there
    a, b = socket.socketpair(socket.AF_UNIX, socket.SOCK_STREAM)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_child, args=(b, arena_bytes, off, blk.nbytes, q))   # socket duplicated into the child
    p.start()
    device.send_fd(a, fd, n)
    status, val = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", val
    assert val == device.fingerprint_host(src.cpu())
    torch.cuda.synchronize()
    assert int(view[:16].min()) == 0xAB and int(view[:16].max()) == 0xAB   # child's write is visible
    os.close(fd)
    pool.free(blk)
    pool.close()

"""Host logic of the function <-> daemon protocol (daemon.py) on CPU: a
TubeDaemon over a stand-in tube (no GPU: pool blocks are host tensors, fds
are /dev/null) driven through the raw channel — loans, commits, zero-copy
fetches, fds sent once per connection, unmap notices, dead clients, host
payloads as memfds and typed errors."""

import itertools
import os
import tempfile
import time

import pytest
import torch


class _Blk:
    def __init__(self, vid, nbytes, device=0):
        self.vmm_id, self.nbytes, self.device = vid, nbytes, device
        self.data = torch.zeros(nbytes, dtype=torch.uint8)    # stands in for the device memory

    def wait_fences(self, stream):
        pass


class _Pool:
    def __init__(self):
        self.on_unmap, self.freed, self.exports, self._ids = [], [], 0, itertools.count(1)

    def locate(self, blk):
        return blk.vmm_id, 0, blk.nbytes             # one block per "arena" in the stand-in

    def export_fd(self, blk):
        self.exports += 1
        return os.open("/dev/null", os.O_RDONLY)

    def free(self, blk, fences=()):
        self.freed.append(blk.vmm_id)

    def unmap(self, vid):
        for fn in self.on_unmap:
            fn(vid)


class _Obj:
    def __init__(self, t, gpu, block):
        self.t, self.gpu, self.block = t, gpu, block
        self.nbytes, self.dtype, self.shape = t.nbytes, t.dtype, tuple(t.shape)


class _Tube:
    """The slice of FaaSTube the daemon uses."""

    def __init__(self):
        self.pools = {0: _Pool()}
        self._objs, self._ids, self.stored = {}, itertools.count(1), {}

    def unique_id(self):
        return next(self._ids)

    def empty(self, shape, dtype, device=0):
        blk = self.lend_block(device, torch.zeros((), dtype=dtype).element_size() * int(torch.tensor(shape).prod()))
        t = blk.data.view(dtype).view(shape)
        t._ft_block = blk
        return t

    def lend_block(self, device, nbytes):
        return _Blk(next(self.pools[device]._ids), nbytes, device)

    def store_block(self, did, blk, nbytes, dtype, shape, stream, response=False, producer="func", consumers=1):
        from paper_2411_01830_b200 import DuplicateStore
        if did in self._objs:
            raise DuplicateStore(f"data id {did} already stored")
        t = blk.data[:nbytes].view(dtype).view(shape)
        self._objs[did] = _Obj(t, blk.device, blk)
        self.stored[did] = t.clone()

    def sync_stream(self, g):
        pass

    def store(self, did, t, response=False, producer="func", consumers=1):
        from paper_2411_01830_b200 import DuplicateStore
        if did in self._objs:
            raise DuplicateStore(f"data id {did} already stored")
        blk = getattr(t, "_ft_block", None)
        if blk is not None:
            self._objs[did] = _Obj(t, 0, blk)
        self.stored[did] = t.clone()

    def fetch(self, did, device=None, out=None, consumer="func", slo_ms=None, infer_ms=None):
        from paper_2411_01830_b200 import MissingData
        if did not in self._objs:
            raise MissingData(f"data id {did} has no live payload")
        if device is None:
            return self.stored[did]
        return self._objs[did].t

    def peek(self, did):
        return self._objs.get(did)

    def fetch_resident(self, did, device, consumer="func", stream=None):
        o = self._objs.get(did)
        if o is None or o.gpu != device or o.block is None:
            return None
        t = self.fetch(did, device, consumer=consumer)
        return o.block, t.nbytes, t.dtype, tuple(t.shape), lambda stream=None: None

    def release(self, did):
        self._objs.pop(did, None)


@pytest.fixture(params=["socket", "shm"])
def daemon(request):
    """The daemon over a stand-in tube; connections speak over the socket or,
    after ``upgrade``, over the shared-memory rings (channel.py)."""
    from paper_2411_01830_b200.daemon import TubeDaemon
    tube = _Tube()
    d = TubeDaemon(tube, os.path.join(tempfile.mkdtemp(), "d.sock"))
    d.shm = request.param == "shm"
    yield d, tube
    d.close()


def _connect(d):
    from paper_2411_01830_b200.channel import Channel
    ch = Channel.connect(d.path)
    if d.shm:
        ch.upgrade()
        assert ch.recv_msg()["ok"]
    return ch


def _call(ch, msg):
    ch.send_msg(msg)
    rep = ch.recv_msg()
    if rep.get("fd"):
        fd, _ = ch.recv_fd()
        rep["_fd"] = fd
    return rep


def test_put_get_over_the_channel(daemon):
    d, tube = daemon
    ch = _connect(d)
    ids = [_call(ch, {"op": "unique_id"})["id"] for _ in range(3)]
    assert ids == sorted(ids) and len(set(ids)) == 3
    rep = _call(ch, {"op": "alloc", "gpu": 0, "nbytes": 24})
    assert rep["ok"] and rep["fd"] and rep["nbytes"] == 24
    os.close(rep["_fd"])
    blk = rep["block"]
    rep = _call(ch, {"op": "commit", "token": rep["token"], "id": ids[0], "dtype": "torch.float32", "shape": [2, 3],
                     "producer": "p", "consumers": 1})
    assert rep["ok"]
    assert tube.stored[ids[0]].dtype == torch.float32 and tuple(tube.stored[ids[0]].shape) == (2, 3)
    # same-GPU fetch: the stored block itself, already mapped by this connection -> no fd
    rep = _call(ch, {"op": "fetch", "id": ids[0], "gpu": 0})
    assert rep["ok"] and rep["block"] == blk and not rep["fd"]
    assert rep["dtype"] == "torch.float32" and rep["shape"] == [2, 3]
    ch.send_msg({"op": "done", "token": rep["token"]})            # fire and forget
    # a second connection has not mapped it: the fd crosses once for it too
    ch2 = _connect(d)
    rep2 = _call(ch2, {"op": "fetch", "id": ids[0], "gpu": 0})
    assert rep2["fd"] and rep2["block"] == blk
    os.close(rep2["_fd"])
    ch2.send_msg({"op": "done", "token": rep2["token"]})
    assert tube.pools[0].exports == 2
    # typed errors
    rep = _call(ch, {"op": "fetch", "id": 10**9, "gpu": 0})
    assert not rep["ok"] and rep["error"] == "MissingData"
    rep = _call(ch, {"op": "commit", "token": 12345, "id": 7, "dtype": "torch.uint8", "shape": [1]})
    assert not rep["ok"] and rep["error"] == "KeyError"
    rep = _call(ch, {"op": "bogus"})
    assert not rep["ok"] and rep["error"] == "ValueError"
    ch.close()
    ch2.close()


def test_unmap_notice_and_refetch(daemon):
    d, tube = daemon
    ch = _connect(d)
    rep = _call(ch, {"op": "alloc", "gpu": 0, "nbytes": 8})
    os.close(rep["_fd"])
    blk = rep["block"]
    did = _call(ch, {"op": "unique_id"})["id"]
    _call(ch, {"op": "commit", "token": rep["token"], "id": did, "dtype": "torch.uint8", "shape": [8]})
    tube.pools[0].unmap(blk)                      # the daemon's pool gives the block back
    rep = _call(ch, {"op": "unique_id"})          # any reply carries the notice
    assert rep["drop"] == [blk]
    rep = _call(ch, {"op": "fetch", "id": did, "gpu": 0})
    assert rep["fd"], "a dropped block is exported again"
    os.close(rep["_fd"])
    ch.close()


def test_duplicate_commit_returns_block_and_dead_client_loans(daemon):
    d, tube = daemon
    ch = _connect(d)
    did = _call(ch, {"op": "unique_id"})["id"]
    for i in range(2):
        rep = _call(ch, {"op": "alloc", "gpu": 0, "nbytes": 4})
        os.close(rep["_fd"])
        r = _call(ch, {"op": "commit", "token": rep["token"], "id": did, "dtype": "torch.uint8", "shape": [4]})
        if i == 1:
            assert not r["ok"] and r["error"] == "DuplicateStore"
            assert tube.pools[0].freed == [rep["block"]]          # the unpublished block went back
    rep = _call(ch, {"op": "alloc", "gpu": 0, "nbytes": 4})       # a loan the client never commits
    os.close(rep["_fd"])
    ch.close()                                                    # the function process dies
    deadline = time.time() + 5
    while rep["block"] not in tube.pools[0].freed and time.time() < deadline:
        time.sleep(0.01)
    assert rep["block"] in tube.pools[0].freed
    assert not d._held


def test_host_payload_as_memfd(daemon):
    from paper_2411_01830_b200.daemon import _from_memfd, _memfd
    d, tube = daemon
    ch = _connect(d)
    x = torch.arange(1000, dtype=torch.int16).reshape(10, 100)
    did = _call(ch, {"op": "unique_id"})["id"]
    fd = _memfd(x)
    ch.send_msg({"op": "store_host", "id": did, "nbytes": x.nbytes, "dtype": str(x.dtype), "shape": [10, 100]})
    ch.send_fd(fd, {})
    os.close(fd)
    assert ch.recv_msg()["ok"]
    assert torch.equal(tube.stored[did], x)
    e = torch.empty(0, 3, dtype=torch.float16)
    did2 = _call(ch, {"op": "unique_id"})["id"]
    fd = _memfd(e)
    ch.send_msg({"op": "store_host", "id": did2, "nbytes": 0, "dtype": str(e.dtype), "shape": [0, 3]})
    ch.send_fd(fd, {})
    os.close(fd)
    assert ch.recv_msg()["ok"]
    assert tube.stored[did2].shape == (0, 3) and tube.stored[did2].dtype == torch.float16
    # round trip of the memfd helpers
    fd = _memfd(x)
    y = _from_memfd(fd, x.nbytes)
    os.close(fd)
    assert torch.equal(y.view(torch.int16).view(10, 100), x)
    ch.close()

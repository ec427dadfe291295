"""Function <-> daemon put/get over the local channel — the paper's unified
interface: function processes call ``TubeClient.store`` /
``fetch`` (Listing 1); the per-box daemon (``TubeDaemon``) owns the FaaSTube
(index, pools, pacer). GPU payloads never cross the socket: pool blocks are
exported as POSIX fds (``cuMemExportToShareableHandle``, SCM_RIGHTS over
AF_UNIX, ``channel.py``) and mapped by the function process; host payloads
travel as a sealed memfd. The socket carries only small JSON messages.

Protocol: every request gets one reply message; a reply with ``"fd": true``
is followed by one descriptor (SCM_RIGHTS). Replies also carry ``"drop"``:
block ids the daemon's pool has unmapped since, which the client unmaps too
(its mappings would otherwise keep the physical memory alive).

  {"op": "unique_id"}                                -> {"id"}
  {"op": "alloc", "gpu", "nbytes"}                   -> {"token", "block", "fd"} [+ fd]
      a pool block for the producer's output; the client writes it and commits
  {"op": "commit", "token", "id", "dtype", "shape", "producer", "consumers", "response"}
      -> {}   (tube.store of the pool-backed block: zero copy)
  {"op": "store_host", "id", "nbytes", ...} + memfd  -> {}
  {"op": "fetch", "id", "gpu", "consumer", "slo_ms", "infer_ms"}
      -> {"token", "block", "nbytes", "dtype", "shape", "fd"} [+ fd]: a block
         holding the bytes on the consumer's GPU (the stored block itself for a
         same-GPU object — zero copy — else a pool block the daemon fetched into)
  {"op": "fetch_host", "id", ...}                    -> {"nbytes", "dtype", "shape"} + memfd
  {"op": "done", "token"}                            -> no reply (the client has read it)
  {"op": "release", "id"}                            -> {}

A block's fd is exported and sent once per connection
(``cuMemExportToShareableHandle`` costs ~1 ms): pool blocks are reused by
size class, so a steady stream of requests maps and exports nothing new.
Ordering across processes is by host synchronization: the client finishes
writing before ``commit``; the daemon's fetch has landed before it replies.
"""

from __future__ import annotations

import itertools
import math
import mmap
import os
import threading

import torch

from . import device as dev
from .channel import Channel

_DTYPES = {str(t): t for t in (torch.uint8, torch.int8, torch.int16, torch.int32, torch.int64, torch.float16,
                               torch.bfloat16, torch.float32, torch.float64, torch.bool)}


def _memfd(data: torch.Tensor) -> int:
    """A sealed-size anonymous file holding the bytes of a host tensor."""
    n = data.numel() * data.element_size()
    fd = os.memfd_create("faastube", os.MFD_CLOEXEC)
    os.ftruncate(fd, max(1, n))
    if n:
        with mmap.mmap(fd, n) as m:
            m[:] = memoryview(data.contiguous().view(torch.uint8).numpy()).cast("B")
    return fd


def _from_memfd(fd: int, nbytes: int) -> torch.Tensor:
    m = mmap.mmap(fd, max(1, nbytes))
    t = torch.frombuffer(m, dtype=torch.uint8, count=nbytes) if nbytes else torch.empty(0, dtype=torch.uint8)
    t._ft_mmap = m  # noqa: SLF001 - the mapping lives as long as the tensor
    return t


class _Conn:
    __slots__ = ("ch", "tokens", "mapped", "drop")

    def __init__(self, ch):
        self.ch = ch
        self.tokens = set()      # loans of this connection (dropped if the client dies)
        self.mapped = set()      # (gpu, block id) the client has mapped
        self.drop = []           # block ids to unmap, sent with the next reply


class TubeDaemon:
    """Serves the put/get API of ``tube`` to function processes on ``path``."""

    def __init__(self, tube, path: str):
        self.tube, self.path = tube, path
        self.server = Channel.listen(path)
        self._tokens = itertools.count(1)
        self._held = {}            # token -> tensor keeping a block (or a pinned view) alive
        self._lock = threading.Lock()
        self._closing = False
        self._threads = []
        self._conns = []
        for g, pool in tube.pools.items():
            pool.on_unmap.append(lambda vid, g=g: self._dropped(g, vid))
        self._acceptor = threading.Thread(target=self._accept_loop, name="faastube-daemon", daemon=True)
        self._acceptor.start()

    def _accept_loop(self):
        while not self._closing:
            try:
                ch = Channel.accept(self.server)
            except OSError:
                return
            th = threading.Thread(target=self._serve, args=(ch,), name="faastube-daemon-conn", daemon=True)
            th.start()
            self._threads = [t for t in self._threads if t.is_alive()] + [th]

    def _dropped(self, g, vid):
        with self._lock:
            for conn in self._conns:
                if (g, vid) in conn.mapped:
                    conn.mapped.discard((g, vid))
                    conn.drop.append(vid)

    def _hold(self, conn, t) -> int:
        tok = next(self._tokens)
        with self._lock:
            self._held[tok] = t
        conn.tokens.add(tok)
        return tok

    def _take(self, conn, tok):
        conn.tokens.discard(tok)
        with self._lock:
            return self._held.pop(tok, None)

    def _unhold(self, conn, tok):
        t = self._take(conn, tok)
        # a daemon-side fetch buffer, or an output block never committed (the client
        # died between alloc and commit), goes back to the pool
        keep = getattr(t, "_ft_keep", None) if not getattr(t, "_ft_alloc", False) else t
        del t
        if keep is not None:
            self._free(keep)

    def _free(self, t):
        blk = t._ft_block  # noqa: SLF001
        del t
        self.tube.pools[blk.device].free(blk)

    def _serve(self, ch: Channel):
        conn = _Conn(ch)
        with self._lock:
            self._conns.append(conn)
        try:
            while True:
                msg = ch.recv_msg()
                try:
                    self._handle(conn, msg)
                except Exception as exc:  # noqa: BLE001 - the error travels back to the caller
                    if msg.get("op") == "done":        # fire-and-forget: nobody waits for a reply
                        continue
                    ch.send_msg({"ok": False, "error": type(exc).__name__, "msg": str(exc)})
        except (ConnectionError, OSError):
            pass
        finally:
            with self._lock:
                self._conns.remove(conn)
            for tok in list(conn.tokens):      # a client that died drops its loans
                self._unhold(conn, tok)
            ch.close()

    def _reply(self, conn, meta, fd=None):
        with self._lock:
            drop, conn.drop = conn.drop, []
        conn.ch.send_msg(dict(meta, ok=True, fd=fd is not None, drop=drop))
        if fd is not None:
            conn.ch.send_fd(fd, {})

    def _reply_block(self, conn, g, blk, meta):
        key = (g, int(blk.vmm_id))
        meta = dict(meta, block=key[1], block_bytes=int(blk.nbytes))
        with self._lock:
            known = key in conn.mapped
            conn.mapped.add(key)
        if known:                              # the client has it mapped already
            self._reply(conn, meta)
            return
        fd = self.tube.pools[g].export_fd(blk)
        try:
            self._reply(conn, meta, fd)
        finally:
            os.close(fd)

    def _handle(self, conn, msg: dict):
        tube, op, ch = self.tube, msg["op"], conn.ch
        if op == "unique_id":
            self._reply(conn, {"id": tube.unique_id()})
        elif op == "alloc":
            g, n = int(msg["gpu"]), int(msg["nbytes"])
            t = tube.empty((max(1, n),), torch.uint8, device=g)              # pool-backed output
            t._ft_alloc = True  # noqa: SLF001
            tube.sync_stream(g)                # the block's previous users are done before the client writes
            self._reply_block(conn, g, t._ft_block, {"token": self._hold(conn, t), "nbytes": n})  # noqa: SLF001
        elif op == "commit":
            t = self._take(conn, int(msg["token"]))
            if t is None:
                raise KeyError(f"unknown token {msg['token']}")
            blk = t._ft_block  # noqa: SLF001
            dt = _DTYPES[msg["dtype"]]
            out = t[:math.prod(msg["shape"]) * dt.itemsize].view(dt).view(msg["shape"])
            out._ft_block = blk  # noqa: SLF001 - still the pool block: a zero-copy store
            try:
                tube.store(int(msg["id"]), out, response=bool(msg.get("response")),
                           producer=msg.get("producer", "func"), consumers=int(msg.get("consumers", 1)))
            except BaseException:
                del out
                self._free(t)                  # not published (e.g. DuplicateStore): back to the pool
                raise
            self._reply(conn, {})
        elif op == "store_host":
            fd, _ = ch.recv_fd()
            try:
                host = _from_memfd(fd, int(msg["nbytes"]))
            finally:
                os.close(fd)
            dt = _DTYPES[msg["dtype"]]
            host = host.view(dt).view(msg["shape"]) if host.numel() else torch.empty(msg["shape"], dtype=dt)
            tube.store(int(msg["id"]), host, producer=msg.get("producer", "func"),
                       consumers=int(msg.get("consumers", 1)))
            self._reply(conn, {})
        elif op == "fetch":
            g, did = int(msg["gpu"]), int(msg["id"])
            # zero-copy or not is decided atomically with the fetch (a concurrent store
            # could otherwise migrate the object to host memory between a check and the
            # fetch); the view pins the block, so it cannot move after
            res = tube.fetch_resident(did, g, consumer=msg.get("consumer", "func"))
            if res is not None:
                t, blk = res
            else:
                obj = tube._objs.get(did)  # noqa: SLF001
                nbytes = obj.nbytes if obj is not None else 0
                dst = tube.empty((max(1, nbytes),), torch.uint8, device=g)
                try:
                    t = tube.fetch(did, out=dst[:nbytes].view(obj.dtype).view(obj.shape) if obj is not None else dst,
                                   consumer=msg.get("consumer", "func"), slo_ms=msg.get("slo_ms"),
                                   infer_ms=msg.get("infer_ms"))
                except BaseException:
                    tube.pools[g].free(dst._ft_block)  # noqa: SLF001
                    raise
                t._ft_keep = dst  # noqa: SLF001
                blk = dst._ft_block  # noqa: SLF001
            # the consumer stream is ordered after the bytes (a host->GPU stage's last
            # batch is issued before fetch returns; the stream waits on its join events)
            tube.sync_stream(g)
            self._reply_block(conn, g, blk, {"token": self._hold(conn, t), "nbytes": t.nbytes,
                                             "dtype": str(t.dtype), "shape": list(t.shape)})
        elif op == "fetch_host":
            t = tube.fetch(int(msg["id"]), device=None, consumer=msg.get("consumer", "func"))
            fd = _memfd(t.reshape(-1).view(torch.uint8))
            try:
                self._reply(conn, {"nbytes": t.nbytes, "dtype": str(t.dtype), "shape": list(t.shape)}, fd)
            finally:
                os.close(fd)
        elif op == "done":                     # no reply (the client does not wait for it)
            self._unhold(conn, int(msg["token"]))
        elif op == "release":
            tube.release(int(msg["id"]))
            self._reply(conn, {})
        else:
            raise ValueError(f"unknown op {op!r}")

    def close(self):
        """Stop accepting, drop every connection (their loans go back to the pool)."""
        self._closing = True
        try:
            self.server.shutdown(2)            # wakes the acceptor blocked in accept()
        except OSError:
            pass
        self._acceptor.join(timeout=5)
        with self._lock:
            conns = list(self._conns)
        for conn in conns:
            try:
                conn.ch.sock.shutdown(2)
            except OSError:
                pass
        for th in self._threads:
            th.join(timeout=5)
        try:
            self.server.close()
        finally:
            if os.path.exists(self.path):
                os.unlink(self.path)


class DaemonError(RuntimeError):
    pass


class TubeClient:
    """Listing 1 in a function process: ``unique_id`` / ``store`` / ``fetch``
    through the daemon at ``path``, for a function running on ``device``."""

    def __init__(self, path: str, device: int = 0):
        self.ch = Channel.connect(path)
        self.device = device
        self._imports = {}           # daemon block id -> ImportedBlock (until the daemon drops it)
        self._stream = dev.new_stream(device)

    def _call(self, msg: dict):
        self.ch.send_msg(msg)
        return self._recv()

    def _recv(self):
        rep = self.ch.recv_msg()
        if not rep.get("ok"):
            raise DaemonError(f"{rep.get('error')}: {rep.get('msg')}")
        for bid in rep.get("drop", ()):
            imp = self._imports.pop(bid, None)
            if imp is not None:
                imp.close()
        if rep.get("fd"):
            rep["_fd"] = self.ch.recv_fd()[0]
        return rep

    def _mapped(self, rep: dict) -> dev.ImportedBlock:
        bid, fd = rep["block"], rep.get("_fd")
        if fd is None:
            return self._imports[bid]
        try:
            imp = self._imports.get(bid)
            if imp is None:
                imp = self._imports[bid] = dev.ImportedBlock(self.device, fd, rep["block_bytes"])
            return imp
        finally:
            os.close(fd)

    def unique_id(self) -> int:
        return self._call({"op": "unique_id"})["id"]

    def store(self, data_id: int, output: torch.Tensor, response: bool = False, producer: str = "func",
              consumers: int = 1):
        """FaaSTube.store(index, output, response) from a function process."""
        if not output.is_cuda:
            fd = _memfd(output)
            try:
                self.ch.send_msg({"op": "store_host", "id": data_id, "nbytes": output.nbytes,
                                  "dtype": str(output.dtype), "shape": list(output.shape), "producer": producer,
                                  "consumers": consumers})
                self.ch.send_fd(fd, {})
            finally:
                os.close(fd)
            self._recv()
            return
        t = output.contiguous()
        rep = self._call({"op": "alloc", "gpu": self.device, "nbytes": t.nbytes})
        imp = self._mapped(rep)
        self._stream.wait_stream(torch.cuda.current_stream(self.device))
        dev.copy(imp.ptr, t.data_ptr(), t.nbytes, self.device, self._stream)
        self._stream.synchronize()                     # written before the daemon publishes it
        self._call({"op": "commit", "token": rep["token"], "id": data_id, "dtype": str(t.dtype),
                    "shape": list(t.shape), "producer": producer, "consumers": consumers, "response": response})

    def fetch(self, data_id: int, out: torch.Tensor | None = None, host: bool = False, consumer: str = "func",
              slo_ms: float | None = None, infer_ms: float | None = None) -> torch.Tensor:
        """FaaSTube.fetch(index, input): the bytes land in ``out`` (or a new
        tensor on this function's GPU; in host memory with ``host=True`` or a
        host ``out``)."""
        if host or (out is not None and not out.is_cuda):
            rep = self._call({"op": "fetch_host", "id": data_id, "consumer": consumer})
            try:
                buf = _from_memfd(rep["_fd"], rep["nbytes"])
            finally:
                os.close(rep["_fd"])
            res = buf.clone().view(_DTYPES[rep["dtype"]]).view(rep["shape"])
            if out is not None:
                out.view(-1).view(torch.uint8).copy_(res.view(-1).view(torch.uint8))
                return out
            return res
        rep = self._call({"op": "fetch", "id": data_id, "gpu": self.device, "consumer": consumer,
                          "slo_ms": slo_ms, "infer_ms": infer_ms})
        imp = self._mapped(rep)
        if out is None:
            out = torch.empty(rep["shape"], dtype=_DTYPES[rep["dtype"]], device=f"cuda:{self.device}")
        elif not out.is_contiguous() or out.nbytes != rep["nbytes"]:
            self.ch.send_msg({"op": "done", "token": rep["token"]})
            raise ValueError("out must be contiguous with exactly the stored byte count")
        cur = torch.cuda.current_stream(self.device)
        self._stream.wait_stream(cur)
        dev.copy(out.data_ptr(), imp.ptr, rep["nbytes"], self.device, self._stream)
        self._stream.synchronize()                     # read before the daemon may reuse the block
        self.ch.send_msg({"op": "done", "token": rep["token"]})   # no reply: served before the next request
        cur.wait_stream(self._stream)
        return out

    def release(self, data_id: int):
        self._call({"op": "release", "id": data_id})

    def close(self):
        for imp in self._imports.values():
            imp.close()
        self._imports.clear()
        dev.destroy_stream(self._stream)
        self.ch.close()

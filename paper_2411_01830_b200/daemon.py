"""Function <-> daemon put/get over the local channel — the paper's unified
interface: function processes call ``TubeClient.store`` /
``fetch`` (Listing 1); the per-box daemon (``TubeDaemon``) owns the FaaSTube
(index, pools, pacer). GPU payloads never cross the socket: pool blocks are
exported as POSIX fds (``cuMemExportToShareableHandle``, SCM_RIGHTS over
AF_UNIX, ``channel.py``) and mapped by the function process; host payloads
travel as a sealed memfd. The socket carries small messages (msgpack) and the
descriptors; with the native lane (below) messages move to shared memory.

Protocol (msgpack frames): every request gets one reply message; a reply
with ``"fd": true`` is followed by one descriptor (SCM_RIGHTS). Replies also
carry ``"drop"``: block ids the daemon's pool has unmapped since, which the
client unmaps too (its mappings would otherwise keep the physical memory
alive), and ``"acked"``: how many of the client's messages were served.

Ordering across processes is stream-ordered, not host-synchronised, once the
client has said ``hello`` with its interprocess events: each side owns a ring
of CUDA IPC events (``ft_ipc_event_create``) whose handles were exchanged at
``hello``. A message may name one of the sender's events (``"ev"``): the
receiver's stream waits on it before touching the block. So a store is: the
client's stream waits the daemon's "block free" event, copies into the
mapped block, records its event; ``commit`` makes the daemon's stream wait
on it before publishing. A fetch reply names the daemon's "bytes ready"
event; ``done`` names the client's "read finished" event, which fences the
block's reuse. A connection without ``hello`` gets host synchronisation
instead (the daemon syncs its stream before replying).

  {"op": "hello", "gpu", "ev": [64-byte handles]}     -> {"ev": [handles]}

  {"op": "unique_id"}                                -> {"id"}
  {"op": "alloc", "gpu", "nbytes"}                   -> {"token", "block", "fd"} [+ fd]
      a pool block for the producer's output; the client writes it and commits
  {"op": "commit", "token", "id", "dtype", "shape", "producer", "consumers", "response", "ev", "next"}
      -> {} or {"loan": <alloc reply>} (tube.store of the pool-backed block: zero copy; "next":
         the byte count of the producer's next output — its block is lent in the reply, so a
         steady producer pays one round trip per store)
  {"op": "store_host", "id", "nbytes", ...} + memfd  -> {}
  {"op": "fetch", "id", "gpu", "consumer", "slo_ms", "infer_ms"}
      -> {"token", "block", "nbytes", "dtype", "shape", "fd"} [+ fd]: a block
         holding the bytes on the consumer's GPU (the stored block itself for a
         same-GPU object — zero copy — else a pool block the daemon fetched into)
  {"op": "fetch_host", "id", ...}                    -> {"nbytes", "dtype", "shape"} + memfd
  {"op": "done", "token", "ev"}                      -> no reply (the client has read it)
  {"op": "release", "id"}                            -> {}

A block's fd is exported and sent once per connection
(``cuMemExportToShareableHandle`` costs ~1 ms): pool blocks are reused by
size class, so a steady stream of requests maps and exports nothing new.

The native lane (the default, csrc/lane.cc + client.cc). A client that sends
``{"op": "chan"}`` + a memfd moves its messages to shared-memory rings
(chan.cc); the daemon attaches a C++ worker to them. With ``hello`` +
``"memops"`` the daemon hands back a 256-byte slot of a pool block (two sync
words: the client's marks, the daemon's) instead of IPC event rings — a mark
is a stream write of the sender's next sequence number, a wait is the
receiver's stream waiting for it (``"ev"`` is that number; 0 / -1 = none).
The hot requests are then binary (little-endian, packed):

  unique_id  u8 op=4                                         -> i64 id
  commit     u8 op=1, dtype, ndim, response; i32 ev, consumers; u32 name_len;
             u64 token; i64 id; u64 next; i64 shape[ndim]; name
                                                             -> BlockRep (loan=1: the next block)
  fetch      u8 op=2; i32 gpu; i64 id; f64 slo_ms, infer_ms  -> BlockRep + i64 shape[ndim]
  done       u8 op=3; i32 ev; u64 token                      -> no reply

A binary reply is RepHdr (u8 0xB1, ok, has_fd; u32 acked, n_drop) + payload +
u64 drop[n_drop]; BlockRep = u64 token, arena, off, arena_bytes, nbytes; i32
ev; u8 dtype, ndim, loan. An error reply (ok=0) carries the exception's name
and message. The worker answers these itself and hands everything else
(msgpack, misses, responses, objects on another GPU) to the connection's
Python thread, which replies in the request's own format.
"""

from __future__ import annotations

import contextlib
import functools
import ctypes as C
import itertools
import math
import mmap
import os
import struct
import threading
import weakref

import torch

from . import device as dev
import msgpack

from .channel import Channel

_DTYPES = {str(t): t for t in (torch.uint8, torch.int8, torch.int16, torch.int32, torch.int64, torch.float16,
                               torch.bfloat16, torch.float32, torch.float64, torch.bool)}
# binary messages of the native lane (csrc/lane.cc): dtype codes and packed structs
_CODES = (torch.uint8, torch.int8, torch.int16, torch.int32, torch.int64, torch.float16, torch.bfloat16,
          torch.float32, torch.float64, torch.bool)
_CODE = {t: i for i, t in enumerate(_CODES)}
OP_COMMIT, OP_FETCH, OP_DONE, OP_UID = 1, 2, 3, 4
_COMMIT = struct.Struct("<BBBBiiIQqQ")
_FETCH = struct.Struct("<B3xiqdd")
_DONE = struct.Struct("<B3xiQ")
_REPHDR = struct.Struct("<BBBxIII")
_BLOCKREP = struct.Struct("<QQQQQiBBBx")
_REP_KIND = 0xB1
_NATIVE_TOKENS = 1 << 62       # tokens at or above are the lane's


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


class _Pin:
    """A daemon-side loan of a stored block to a client's zero-copy read: looks
    like the tensor it stands for (nbytes / dtype / shape) and unpins the block
    when the daemon drops it (client ``done`` or a dead connection)."""

    __slots__ = ("release", "nbytes", "dtype", "shape")

    def __init__(self, release, nbytes, dtype, shape):
        self.release, self.nbytes, self.dtype, self.shape = release, nbytes, dtype, shape

    def __del__(self):
        rel, self.release = self.release, None
        if rel is not None:
            rel()


class _Lend:
    """A pool block lent to a client for its next output (``alloc`` / a commit's
    ``loan``) until the client commits it; returned to the pool otherwise."""

    __slots__ = ("blk",)

    def __init__(self, blk):
        self.blk = blk


class _Conn:
    __slots__ = ("ch", "tokens", "mapped", "drop", "gpu", "stream", "mine", "peer", "served", "seen", "lc",
                 "chan", "bin", "buf", "stocked", "slot")

    def __init__(self, ch):
        self.ch = ch
        self.lc = None           # ft_lane_conn: a native worker reads this connection's requests
        self.chan = None         # its ft_chan (closed after the worker)
        self.bin = False         # the request being served arrived as a binary message
        self.buf = None
        self.stocked = set()     # (gpu, size class) whose lane stock this connection filled
        self.slot = None         # (gpu, index) of the connection's sync words (lane connections)
        self.tokens = set()      # loans of this connection (dropped if the client dies)
        self.mapped = set()      # (gpu, block id) the client has mapped
        self.drop = []           # block ids to unmap, sent with the next reply
        self.gpu = None          # after hello: the client's GPU, a private stream, both event rings
        self.stream = None
        self.mine = None         # dev.IpcEventRing (the daemon's events, exported to the client)
        self.peer = None         # dev.PeerEvents (the client's events)
        self.served = 0          # messages handled (acknowledged in every reply)
        self.seen = 0            # messages received

    def ctx(self):
        """Request handling runs on the connection's private stream (after hello)."""
        if self.stream is None:
            return contextlib.nullcontext()
        return torch.cuda.stream(self.stream)

    def mark(self) -> int:
        """Mark the connection stream for the client (-1 / 0: no ordering — host sync)."""
        if self.lc is not None and self.slot is not None:   # the daemon's sync word (shared with the worker)
            i = C.c_int()
            dev.LIB.ft_lane_conn_mark(self.lc, C.byref(i))
            return i.value
        if self.mine is None:
            return -1
        i = self.mine.take()
        self.mine.record(i, self.stream)
        return i

    def wait_peer(self, i):
        if self.lc is not None and self.slot is not None:
            if i is not None and i not in (0, -1):      # a mark of the client's sync word
                dev.LIB.ft_lane_conn_wait(self.lc, int(i) & 0xFFFFFFFF)
            return
        if self.peer is not None and i is not None and i >= 0:
            self.peer.wait(int(i), self.stream)

    def close(self):
        for x in (self.mine, self.peer):
            if x is not None:
                x.close()
        if self.stream is not None:
            dev.destroy_stream(self.stream)


class TubeDaemon:
    """Serves the put/get API of ``tube`` to function processes on ``path``."""

    def __init__(self, tube, path: str, lane: bool = True):
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
        # the native lane serves the hot requests of upgraded connections (csrc/lane.cc);
        # its events are applied to the tube by the service thread
        self._lane = None
        self._sync = {}            # gpu -> (pool block of 256-byte sync slots, free slot indices)
        if lane and hasattr(tube, "attach_lane") and tube.pools:
            h = C.c_void_p()
            dev.LIB.ft_lane_create(tube.index._h, int(tube.node), float(tube._t0), C.byref(h))  # noqa: SLF001
            for g, pool in tube.pools.items():
                dev.LIB.ft_lane_set_pool(h, int(g), pool._h)  # noqa: SLF001
            tube.attach_lane(h)
            self._lane = h
            for g in tube.pools:
                # each connection's two sync words live in a 256-byte slot of this block
                # (mapped by the client like any pool block); held for the daemon's life
                blk = tube.lend_block(g, 2 * 10**6)
                for e in blk.take_fences():
                    e.synchronize()
                self._sync[g] = (blk, list(range(blk.nbytes // 256 - 1, -1, -1)))
            self._service = threading.Thread(target=self._service_loop, name="faastube-lane", daemon=True)
            self._service.start()
        self._acceptor = threading.Thread(target=self._accept_loop, name="faastube-daemon", daemon=True)
        self._acceptor.start()

    def _service_loop(self):
        import traceback
        while not self._closing:
            try:
                if not self.tube.lane_service(50.0):
                    return
            except Exception:  # noqa: BLE001 - keep serving; the failure is visible in the log
                traceback.print_exc()

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
        if self._lane is not None:
            dev.LIB.ft_lane_dropped(self._lane, int(g), int(vid))
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
        # died between alloc and commit), goes back to the pool — fenced on the
        # connection's stream, which waited for the client's last access
        if isinstance(t, _Lend):
            self._free(t.blk, conn)
        elif isinstance(t, _Pin):              # a zero-copy read: unpin, fenced on the connection's stream
            rel, t.release = t.release, None
            if rel is not None:
                rel(conn.stream)
        elif t is not None:
            keep = getattr(t, "_ft_keep", None)
            del t
            if keep is not None:
                self._free(keep._ft_block, conn)  # noqa: SLF001

    def _free(self, blk, conn=None):
        """Back to the pool; with stream-ordered connections fenced on the connection's
        stream (it waited for the client's last access), else the client synchronised."""
        g = blk.device
        fences = [dev.Ev(g).record(conn.stream)] if conn is not None and conn.stream is not None else []
        self.tube.pools[g].free(blk, fences)

    def _serve(self, ch: Channel):
        conn = _Conn(ch)
        with self._lock:
            self._conns.append(conn)
        try:
            while True:
                msg = ch.recv_msg() if conn.lc is None else self._lane_recv(conn)
                conn.seen += 1
                try:
                    self._handle(conn, msg)
                except Exception as exc:  # noqa: BLE001 - the error travels back to the caller
                    if msg.get("op") == "done":        # fire-and-forget: nobody waits for a reply
                        if conn.lc is not None:
                            dev.LIB.ft_lane_conn_finish(conn.lc)
                        conn.served = max(conn.served, conn.seen)
                        continue
                    self._reply_error(conn, msg, exc)
        except (ConnectionError, OSError):
            pass
        finally:
            with self._lock:
                self._conns.remove(conn)
            if conn.lc is not None:
                # the worker stops (its native loans and views are released on the
                # connection stream) before anything it uses is torn down
                dev.LIB.ft_lane_conn_close(conn.lc)
                conn.lc = None
            with conn.ctx():
                for tok in list(conn.tokens):      # a client that died drops its loans
                    self._unhold(conn, tok)
            if conn.stream is not None:
                conn.stream.synchronize()
            if conn.slot is not None:
                g, i = conn.slot
                with self._lock:
                    self._sync[g][1].append(i)
                conn.slot = None
            conn.close()
            if conn.chan is not None:
                dev.LIB.ft_chan_close(conn.chan)
                conn.chan = None
            ch.close()

    # ---- the native lane's connections
    def _lane_recv(self, conn) -> dict:
        """The next request the connection's worker handed over (binary or msgpack)."""
        n = C.c_uint32()
        rc = dev.LIB.raw("ft_lane_conn_next")(conn.lc, conn.buf, len(conn.buf), C.byref(n), -1)
        if rc == 13:
            raise ConnectionError("client gone")
        if rc:
            from ._lib import raise_status
            raise_status(rc)
        raw = conn.buf.raw[:n.value]
        conn.bin = raw[:1] in (b"\x01", b"\x02", b"\x03", b"\x04")
        return _decode_bin(raw) if conn.bin else msgpack.unpackb(raw)

    def _reply_error(self, conn, msg, exc):
        name, text = type(exc).__name__, str(exc)
        if conn.lc is None:
            conn.served += 1
            conn.ch.send_msg({"ok": False, "error": name, "msg": text, "acked": conn.served})
        elif conn.bin:
            nb, tb = name.encode(), text.encode()
            p = struct.pack("<I", len(nb)) + nb + struct.pack("<I", len(tb)) + tb
            dev.LIB.ft_lane_conn_reply_bin(conn.lc, p, len(p), 0, -1)
        else:
            acked = C.c_uint32()
            dev.LIB.ft_lane_conn_served(conn.lc, C.byref(acked))
            body = msgpack.packb({"ok": False, "error": name, "msg": text, "acked": acked.value})
            dev.LIB.ft_lane_conn_reply(conn.lc, body, len(body))

    def _reply(self, conn, meta, fd=None):
        if conn.lc is not None:
            self._lane_reply(conn, meta, fd)
            return
        with self._lock:
            drop, conn.drop = conn.drop, []
        conn.served += 1
        conn.ch.send_msg(dict(meta, ok=True, fd=fd is not None, drop=drop, acked=conn.served))
        if fd is not None:
            conn.ch.send_fd(fd, {})

    def _lane_reply(self, conn, meta, fd):
        """A reply to a request the worker handed over: binary for a binary request
        (the lane adds the header: acked, unmap notices, the fd), else msgpack."""
        if conn.bin:
            p = _encode_bin_reply(meta)
            dev.LIB.ft_lane_conn_reply_bin(conn.lc, p, len(p), 1, -1 if fd is None else int(fd))
            return
        ids, n = (C.c_uint64 * 256)(), C.c_int()
        dev.LIB.ft_lane_conn_take_drops(conn.lc, ids, 256, C.byref(n))
        acked = C.c_uint32()
        dev.LIB.ft_lane_conn_served(conn.lc, C.byref(acked))
        body = msgpack.packb(dict(meta, ok=True, fd=fd is not None, drop=list(ids[:n.value]), acked=acked.value))
        if fd is not None:
            conn.ch.send_fd(fd, {})            # ahead of the reply: the client reads it right after
        dev.LIB.ft_lane_conn_reply(conn.lc, body, len(body))

    def _reply_block(self, conn, g, blk, meta):
        # the client maps the block's arena once (the unit of physical memory) and
        # finds the block at its offset
        arena, off, abytes = self.tube.pools[g].locate(blk)
        key = (g, int(arena))
        meta = dict(meta, block=key[1], off=int(off), block_bytes=int(abytes))
        if conn.lc is not None:
            k = C.c_int()
            dev.LIB.ft_lane_conn_known(conn.lc, g, key[1], C.byref(k))
            known = bool(k.value)
        else:
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

    def _lend(self, conn, g: int, n: int) -> dict:
        """A pool block for a producer's output: its previous users are fenced on
        the connection's stream, then marked (the client's stream waits on the
        mark before writing; without events the stream is synchronised)."""
        blk = self.tube.lend_block(g, max(1, n))
        # the block's previous users are done before the client writes: the connection's
        # stream waits on them and is marked, or (no events) the device's default stream
        # waits and is synchronised
        blk.wait_fences(conn.stream if conn.stream is not None else 0)
        ev = conn.mark()
        if ev < 0:
            self.tube.sync_stream(g)
        if conn.lc is not None and conn.gpu == g:
            tok = self.tube.lane_lend(conn.lc, blk)    # its commit is served by the worker
            cls = int(blk.policy_block.class_bytes)
            if (g, cls) not in conn.stocked:
                # the first output of this size on this connection: stock the class now, so
                # the commit that follows lends the next block (no second alloc round trip)
                conn.stocked.add((g, cls))
                cid = C.c_uint64()
                dev.LIB.ft_lane_conn_id(conn.lc, C.byref(cid))
                for _ in range(3):                     # lane.cc kStockDepth
                    self.tube._lane_stock(cid.value, g, cls)  # noqa: SLF001
        else:
            tok = self._hold(conn, _Lend(blk))
        return {"token": tok, "nbytes": n, "ev": ev, "_blk": blk}

    def _handle(self, conn, msg: dict):
        tube, op, ch = self.tube, msg["op"], conn.ch
        if op == "unique_id":
            self._reply(conn, {"id": tube.unique_id()})
        elif op == "chan":                     # messages move to the client's shared-memory rings
            if self._lane is None:
                ch.attach()
                self._reply(conn, {"lane": False})
                return
            fd, _ = dev.recv_fd(ch.sock)
            h, lc = C.c_void_p(), C.c_void_p()
            try:
                dev.LIB.ft_chan_attach(fd, C.byref(h))
            finally:
                os.close(fd)
            conn.chan = h
            conn.buf = C.create_string_buffer(1 << 16)
            dev.LIB.ft_lane_attach(self._lane, h, ch.sock.fileno(), C.byref(lc))
            conn.lc = lc                       # a native worker reads the rings from here on
            self._reply(conn, {"lane": True})
        elif op == "hello":
            g = int(msg["gpu"])
            conn.gpu = g
            conn.stream = dev.new_stream(g)
            if conn.lc is not None and msg.get("memops"):
                # ordering through two words of pool memory the client maps: a 256-byte
                # slot of the lane's sync block on this GPU, zeroed before first use
                blk, ptr = self._sync_slot(conn, g)
                dev.LIB.ft_lane_conn_set_gpu(conn.lc, g, C.c_void_p(conn.stream.cuda_stream), C.c_void_p(ptr),
                                             C.c_void_p(ptr + 128))
                meta = {"sync_off": ptr - blk.ptr}
                self._reply_block(conn, g, blk, meta)
                return
            conn.peer = dev.PeerEvents(g, msg.get("ev", []))
            conn.mine = dev.IpcEventRing(g)
            self._reply(conn, {"ev": conn.mine.handles})
        elif op == "alloc":
            g, n = int(msg["gpu"]), int(msg["nbytes"])
            meta = self._lend(conn, g, n)
            self._reply_block(conn, g, meta.pop("_blk"), meta)
        elif op == "commit":
            tok = int(msg["token"])
            t = self._take(conn, tok)
            if t is None and conn.lc is not None and tok >= _NATIVE_TOKENS:
                pbid = C.c_int64()                 # a lane loan this request needs served here
                dev.LIB.ft_lane_take_lend(conn.lc, tok, C.byref(pbid))
                t = _Lend(tube.lane_block(pbid.value))
            if not isinstance(t, _Lend):
                raise KeyError(f"unknown token {msg['token']}")
            conn.wait_peer(msg.get("ev"))      # the client's copy into the block is done (stream-ordered)
            dt, shape = _DTYPES[msg["dtype"]], msg["shape"]
            nbytes = math.prod(shape) * dt.itemsize
            if nbytes > t.blk.nbytes or any(d < 0 for d in shape):
                self._free(t.blk, conn)
                raise ValueError(f"commit of shape {shape} ({nbytes} B) into a {t.blk.nbytes} B block")
            stream = conn.stream if conn.stream is not None else 0     # 0: the legacy default stream
            try:                               # the pool block itself is published: a zero-copy store
                tube.store_block(int(msg["id"]), t.blk, nbytes, dt, shape, stream,
                                 response=bool(msg.get("response")), producer=msg.get("producer", "func"),
                                 consumers=int(msg.get("consumers", 1)))
            except BaseException:
                self._free(t.blk, conn)        # not published (e.g. DuplicateStore): back to the pool
                raise
            nxt = msg.get("next")
            if nxt is not None and conn.gpu is not None:
                # lend the block of the producer's next output now: its next store is one round trip
                meta = self._lend(conn, conn.gpu, int(nxt))
                self._reply_block(conn, conn.gpu, meta.pop("_blk"), dict(meta, loan=True))
            else:
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
            res = tube.fetch_resident(did, g, consumer=msg.get("consumer", "func"), stream=conn.stream)
            if res is not None:
                blk, nbytes, dtype, shape, release = res
                t = _Pin(release, nbytes, dtype, shape)   # the loan: unpins the block when dropped
            else:
                with conn.ctx():
                    t, blk = self._fetch_into_block(conn, g, did, msg)
            # the consumer stream is ordered after the bytes (a host->GPU stage's last
            # batch is issued before fetch returns; the stream waits on its join events):
            # the client's stream waits on a mark of it, or the stream is synchronised
            ev = conn.mark()
            if ev < 0:
                tube.sync_stream(g)
            self._reply_block(conn, g, blk, {"token": self._hold(conn, t), "nbytes": t.nbytes, "ev": ev,
                                             "dtype": str(t.dtype), "shape": list(t.shape)})
        elif op == "fetch_host":
            with conn.ctx():
                t = tube.fetch(int(msg["id"]), device=None, consumer=msg.get("consumer", "func"))
            fd = _memfd(t.reshape(-1).view(torch.uint8))
            try:
                self._reply(conn, {"nbytes": t.nbytes, "dtype": str(t.dtype), "shape": list(t.shape)}, fd)
            finally:
                os.close(fd)
        elif op == "done":                     # no reply (the client does not wait for it)
            conn.wait_peer(msg.get("ev"))      # the client's last read of the block (stream-ordered)
            tok = int(msg["token"])
            if conn.lc is not None:
                if tok >= _NATIVE_TOKENS:
                    dev.LIB.ft_lane_conn_release(conn.lc, tok)
                else:
                    self._unhold(conn, tok)
                dev.LIB.ft_lane_conn_finish(conn.lc)
                return
            conn.served += 1
            self._unhold(conn, tok)
        elif op == "release":
            with conn.ctx():
                tube.release(int(msg["id"]))
            self._reply(conn, {})
        else:
            raise ValueError(f"unknown op {op!r}")

    def _sync_slot(self, conn, g):
        """A zeroed 256-byte slot of the lane's sync block on GPU g for this connection
        (c2d word at +0, d2c word at +128). Returns (block, slot pointer)."""
        with self._lock:
            blk, free = self._sync[g]
            if not free:
                raise MemoryError("no free sync slot (too many function connections on this GPU)")
            i = free.pop()
        conn.slot = (g, i)
        ptr = blk.ptr + 256 * i
        z = dev.as_tensor(ptr, 256, g)
        with torch.cuda.stream(conn.stream):
            z.zero_()
        conn.stream.synchronize()
        return blk, ptr

    def _fetch_into_block(self, conn, g, did, msg):
        """A fetch that is not a same-GPU zero-copy read: into a pool block the
        client maps (on the connection's stream)."""
        tube = self.tube
        obj = tube.peek(did)
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
        return t, blk

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
        if self._lane is not None:
            self._service.join(timeout=5)
            for g, (blk, _free) in self._sync.items():
                self.tube.pools[g].free(blk, [])
            self._sync = {}
            self.tube.detach_lane()            # its objects into the tube's table, stocked blocks back
            dev.LIB.ft_lane_destroy(self._lane)
            self._lane = None
        try:
            self.server.close()
        finally:
            if os.path.exists(self.path):
                os.unlink(self.path)


_SPIN = int(os.environ.get("FT_CHAN_SPIN_US", 2000))
_KEPT_IMPORTS = []   # mappings of closed clients whose zero-copy views were still alive (kept until exit)
_PyCapsule_New = C.pythonapi.PyCapsule_New
_PyCapsule_New.restype = C.py_object
_PyCapsule_New.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]


@functools.lru_cache(maxsize=4096)
def _class_of(n: int) -> int:
    """The pool's size class of an n-byte output (datastore.py:24-29)."""
    from .datastore import size_class
    return size_class(max(1, n))


def _capsule(dlmanaged: int):
    """A "dltensor" capsule over a DLManagedTensor the native client made (torch's
    from_dlpack consumes it and calls its deleter when the storage is freed)."""
    return _PyCapsule_New(dlmanaged, b"dltensor", None)


def _decode_bin(raw: bytes) -> dict:
    """A binary request of the lane protocol (csrc/lane.cc) as the dict the handlers take."""
    op = raw[0]
    if op == OP_COMMIT:
        _, dt, nd, resp, ev, cons, nl, tok, did, nxt = _COMMIT.unpack_from(raw)
        shape = list(struct.unpack_from(f"<{nd}q", raw, _COMMIT.size))
        name = raw[_COMMIT.size + 8 * nd:_COMMIT.size + 8 * nd + nl].decode()
        return {"op": "commit", "token": tok, "id": did, "dtype": str(_CODES[dt]), "shape": shape,
                "producer": name, "consumers": cons, "response": bool(resp), "ev": ev, "next": nxt or None}
    if op == OP_FETCH:
        _, g, did, slo, infer = _FETCH.unpack_from(raw)
        return {"op": "fetch", "gpu": g, "id": did, "consumer": "func", "slo_ms": None if slo != slo else slo,
                "infer_ms": None if infer != infer else infer}
    if op == OP_DONE:
        _, ev, tok = _DONE.unpack_from(raw)
        return {"op": "done", "token": tok, "ev": ev}
    return {"op": "unique_id"}


def _encode_bin_reply(meta: dict) -> bytes:
    """The payload of a binary reply (the lane prepends the header): a block
    (fetch / alloc / a commit's loan), a bare commit, or an id."""
    if "id" in meta and len(meta) == 1:
        return struct.pack("<q", meta["id"])
    if "block" not in meta:
        return bytes(_BLOCKREP.size)                  # a commit without a loan
    shape = meta.get("shape", [])
    dt = _CODE[_DTYPES[meta["dtype"]]] if "dtype" in meta else 0
    return _BLOCKREP.pack(meta["token"], meta["block"], meta["off"], meta["block_bytes"], meta["nbytes"],
                          meta.get("ev", -1), dt, len(shape), int(bool(meta.get("loan")))) + \
        struct.pack(f"<{len(shape)}q", *shape)


def _parse_block_reply(p: bytes) -> dict:
    tok, arena, off, abytes, nbytes, ev, dt, nd, loan = _BLOCKREP.unpack_from(p)
    shape = list(struct.unpack_from(f"<{nd}q", p, _BLOCKREP.size))
    return {"token": tok, "block": arena, "off": off, "block_bytes": abytes, "nbytes": nbytes, "ev": ev,
            "dtype": str(_CODES[dt]), "shape": shape, "loan": bool(loan)}


class DaemonError(RuntimeError):
    pass


class _Release:
    """Owner of a zero-copy view's mapping: when the last tensor over it dies,
    the client tells the daemon (``done``) so the loan's block can be reused."""

    __slots__ = ("__weakref__",)


class TubeClient:
    """Listing 1 in a function process: ``unique_id`` / ``store`` / ``fetch``
    through the daemon at ``path``, for a function running on ``device``.

    With ``events`` (default) the client and the daemon order each other's
    GPU work with interprocess events instead of host synchronisation (see the
    module doc): ``store`` returns once the copy into the lent block is
    enqueued and committed; ``fetch()`` without ``out`` returns a zero-copy
    view of the stored block itself (same GPU), released back to the daemon
    when the last tensor over it dies; ``fetch(out=)`` copies on the caller's
    current stream. Consumer kernels issued afterwards on the caller's current
    stream see the bytes."""

    def __init__(self, path: str, device: int = 0, events: bool = True, shm: bool = True):
        self.ch = Channel.connect(path)
        self.device = device
        self._imports = {}           # daemon block id -> ImportedBlock (until the daemon drops it)
        self._loans = {}             # size class -> a lent block for the producer's next output of that class
        self._io = threading.RLock()  # one frame at a time on the socket (releases come from finalizers)
        self._sent_py = 0            # messages sent from Python (the native client counts its own)
        self._cl = None              # ft_client: the lane's hot requests in one native call each
        self._acked = 0              # messages the daemon has served (from its replies)
        self._mine = self._peer = None
        self._sync = None            # lane connections: (c2d, d2c) word pointers in the mapped sync slot
        self._seq = 0                # our last mark (c2d)
        self._events = events
        self._closed = False
        self._views = 0              # zero-copy views handed out and not yet released
        self._lane = False           # the daemon's native lane serves the hot requests (binary messages)
        if shm:                      # messages over shared-memory rings from here on (channel.py)
            with self._io:
                self.ch.upgrade()
                self._sent_py += 1
                self._lane = bool(self._recv().get("lane"))
        if events and self._lane:
            # the lane orders both sides through two words of a pool slot mapped here
            rep = self._call({"op": "hello", "gpu": device, "memops": True})
            p = self._mapped(rep).ptr + rep["off"] + rep["sync_off"]
            self._sync = (p, p + 128)
            cl = C.c_void_p()
            dev.LIB.ft_client_create(self.ch._chan, self.ch.sock.fileno(), C.c_void_p(p), C.c_void_p(p + 128),
                                     device, C.byref(cl))  # noqa: SLF001
            self.ch.adopt_client(cl)
            self._cl = cl
            self._rbuf, self._rn = C.create_string_buffer(8192), C.c_uint32()
            self._rn_ref = C.byref(self._rn)
        elif events:
            self._mine = dev.IpcEventRing(device)
            self._used = [0] * self._mine.k        # message number that carried each event's last record
            rep = self._call({"op": "hello", "gpu": device, "ev": self._mine.handles})
            self._peer = dev.PeerEvents(device, rep["ev"])
        else:
            self._stream = dev.new_stream(device)
        self._bin = self._lane and events      # binary requests need the stream-ordered protocol

    # ---- framing
    @property
    def _sent(self) -> int:
        """Messages sent (Python's and the native client's)."""
        if self._cl is None:
            return self._sent_py
        n = C.c_uint64()
        dev.LIB.ft_client_sent(self._cl, C.byref(n))
        return self._sent_py + n.value

    def _send(self, msg: dict):
        with self._io:
            self.ch.send_msg(msg)
            if self._cl is None:
                self._sent_py += 1

    def _call(self, msg: dict):
        with self._io:
            self._send(msg)
            return self._recv()

    def _call_bin(self, body: bytes) -> bytes:
        """A binary request / reply of the native lane (csrc/lane.cc): header (acked,
        unmap notices, an fd after the message), payload."""
        with self._io:
            if self._cl is not None:
                rep = self.ch.client_reply(dev.LIB.raw("ft_client_call")(
                    self._cl, body, len(body), self._rbuf, len(self._rbuf), C.byref(self._rn), _SPIN),
                    self._rbuf, self._rn)
            else:
                self.ch.send_raw(body)
                self._sent_py += 1
                rep = self.ch.recv_raw()
            return self._bin_reply(rep)

    def _bin_reply(self, rep: bytes):
        """(payload, fd) of a binary reply: acked, unmap notices, typed errors, the fd."""
        kind, ok, has_fd, acked, n_drop, _ = _REPHDR.unpack_from(rep)
        if kind != _REP_KIND:
            raise DaemonError(f"unexpected reply kind {kind:#x}")
        self._acked = max(self._acked, acked)
        end = len(rep) - 8 * n_drop
        for bid in struct.unpack_from(f"<{n_drop}Q", rep, end):
            imp = self._imports.pop(bid, None)
            if imp is not None:
                imp.close()
        p = rep[_REPHDR.size:end]
        if not ok:
            n = struct.unpack_from("<I", p)[0]
            name = p[4:4 + n].decode()
            m = struct.unpack_from("<I", p, 4 + n)[0]
            raise DaemonError(f"{name}: {p[8 + n:8 + n + m].decode()}")
        fd = dev.recv_fd(self.ch.sock)[0] if has_fd else None
        return p, fd

    def _block_bin(self, body: bytes) -> dict:
        p, fd = self._call_bin(body)
        rep = _parse_block_reply(p)
        if fd is not None:
            rep["_fd"] = fd
        return rep

    def _recv(self):
        rep = self.ch.recv_msg()
        self._acked = max(self._acked, rep.get("acked", 0))
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
        bid, fd = rep["block"], rep.pop("_fd", None)
        if fd is None:
            return self._imports[bid]
        try:
            imp = self._imports.get(bid)
            if imp is None:
                imp = self._imports[bid] = dev.ImportedBlock(self.device, fd, rep["block_bytes"])   # the arena
            return imp
        finally:
            os.close(fd)

    # ---- stream ordering
    def _mark(self, stream) -> int:
        """Record one of our events on ``stream`` for the next message (-1: the
        daemon may still have a wait on that event's previous record to enqueue —
        synchronise ``stream`` instead)."""
        if self._cl is not None:
            ev = C.c_int32()
            dev.LIB.ft_client_mark(self._cl, C.c_void_p(dev.stream_ptr(stream)), C.byref(ev))
            return ev.value
        if self._mine is None:
            stream.synchronize()
            return -1
        with self._io:
            i = self._mine.take()
            if self._used[i] > self._acked:
                stream.synchronize()
                return -1
            self._mine.record(i, stream)
            self._used[i] = self._sent + 1
            return i

    def _after_daemon(self, rep: dict, stream):
        """``stream`` waits for the daemon's mark in ``rep`` (host-synced connections: nothing)."""
        ev = rep.get("ev", -1)
        if self._cl is not None:
            if ev is not None and ev not in (0, -1):
                dev.LIB.ft_client_wait(self._cl, C.c_void_p(dev.stream_ptr(stream)), int(ev))
            return
        if self._peer is not None and ev is not None and ev >= 0:
            self._peer.wait(int(ev), stream)

    def unique_id(self) -> int:
        if self._bin:
            return struct.unpack("<q", self._call_bin(b"\x04")[0])[0]
        return self._call({"op": "unique_id"})["id"]

    def store(self, data_id: int, output: torch.Tensor, response: bool = False, producer: str = "func",
              consumers: int = 1):
        """FaaSTube.store(index, output, response) from a function process."""
        if not output.is_cuda:
            fd = _memfd(output)
            try:
                with self._io:
                    self._send({"op": "store_host", "id": data_id, "nbytes": output.nbytes,
                                "dtype": str(output.dtype), "shape": list(output.shape), "producer": producer,
                                "consumers": consumers})
                    self.ch.send_fd(fd, {})
                    self._recv()
            finally:
                os.close(fd)
            return
        t = output.contiguous()
        n = t.nbytes
        cls = _class_of(n)                            # a lent block holds any output of its size class
        rep = self._loans.pop(cls, None)
        if rep is None:
            rep = self._call({"op": "alloc", "gpu": self.device, "nbytes": n})
            imp = self._mapped(rep)
        else:
            imp = self._imports[rep["block"]]
        ptr = imp.ptr + rep.get("off", 0)
        if self._cl is not None and not response and t.dtype in _CODE and t.dim() <= 8:
            # wait for the loan's mark, copy, mark, commit, reply: one native call
            name = producer.encode()
            body = _COMMIT.pack(OP_COMMIT, _CODE[t.dtype], t.dim(), 0, 0, consumers, len(name), rep["token"],
                                data_id, n) + struct.pack(f"<{t.dim()}q", *t.shape) + name
            cur = dev.current_stream(self.device)
            with self._io:
                rc = dev.LIB.raw("ft_client_store")(self._cl, cur, rep.get("ev") or 0, ptr, t.data_ptr(), n,
                                                    self._engine(t), body, len(body), self._rbuf, len(self._rbuf),
                                                    self._rn_ref, _SPIN)
                if rc not in (0, 12, 13):
                    from ._lib import raise_status
                    raise_status(rc)
                p, fd = self._bin_reply(self.ch.client_reply(rc, self._rbuf, self._rn))
            if t is not output:
                t.record_stream(torch.cuda.current_stream(self.device))
            rep = _parse_block_reply(p)
            if fd is not None:
                rep["_fd"] = fd
            if rep.get("loan"):
                self._mapped(rep)
                self._loans[cls] = rep
            return
        if not self._events:
            cur = self._stream
            cur.wait_stream(torch.cuda.current_stream(self.device))
        else:
            cur = torch.cuda.current_stream(self.device)
        self._after_daemon(rep, cur)                  # the block's previous users are done
        # the engine is known (the mapped block is memory of this GPU): no pointer queries
        dev.copy(ptr, t.data_ptr(), n, self.device, cur, self._engine(t))
        if t is not output or not self._events:
            t.record_stream(cur)
        if self._bin and not response and t.dtype in _CODE and t.dim() <= 8:
            name = producer.encode()
            with self._io:                            # the mark rides on the very next message
                ev = self._mark(cur)
                body = _COMMIT.pack(OP_COMMIT, _CODE[t.dtype], t.dim(), 0, ev, consumers, len(name), rep["token"],
                                    data_id, n) + struct.pack(f"<{t.dim()}q", *t.shape) + name
                rep = self._block_bin(body)
        else:
            with self._io:                            # the mark rides on the very next message
                ev = self._mark(cur)                  # written (or synchronised) before the daemon publishes it
                rep = self._call({"op": "commit", "token": rep["token"], "id": data_id, "dtype": str(t.dtype),
                                  "shape": list(t.shape), "producer": producer, "consumers": consumers,
                                  "response": response, "ev": ev,
                                  **({"next": n} if self._events else {})})
        if rep.get("loan"):
            self._mapped(rep)
            self._loans[cls] = rep

    def fetch(self, data_id: int, out: torch.Tensor | None = None, host: bool = False, consumer: str = "func",
              slo_ms: float | None = None, infer_ms: float | None = None) -> torch.Tensor:
        """FaaSTube.fetch(index, input): the bytes land in ``out`` (or, without
        ``out``, a zero-copy view of the block on this function's GPU; in host
        memory with ``host=True`` or a host ``out``)."""
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
        if self._cl is not None:
            # request, reply and the stream's wait for the daemon's mark: one native call
            nan = float("nan")
            req = _FETCH.pack(OP_FETCH, self.device, data_id, nan if slo_ms is None else slo_ms,
                              nan if infer_ms is None else infer_ms)
            cur = dev.current_stream(self.device)
            with self._io:
                rc = dev.LIB.raw("ft_client_fetch")(self._cl, cur, req, len(req), self._rbuf, len(self._rbuf),
                                                    self._rn_ref, _SPIN)
                if rc not in (0, 12, 13):
                    from ._lib import raise_status
                    raise_status(rc)
                raw = self.ch.client_reply(rc, self._rbuf, self._rn)
                if rc == 12 and raw[1]:                 # (the reply came late: wait for its mark here)
                    self._after_daemon({"ev": struct.unpack_from("<i", raw, 56)[0]}, cur)
                p, fd = self._bin_reply(raw)
            rep = _parse_block_reply(p)
            ptr = self._mapped(dict(rep, _fd=fd) if fd is not None else rep).ptr + rep["off"]
            n = rep["nbytes"]
            if out is None:
                # zero copy: a DLPack view of the stored block itself; freeing it releases
                # the block (marked on the legacy default stream by the native deleter)
                shape = rep["shape"]
                dl = C.c_void_p()
                dev.LIB.ft_client_view(self._cl, C.c_void_p(ptr), _CODE[_DTYPES[rep["dtype"]]], len(shape),
                                       (C.c_int64 * max(1, len(shape)))(*shape), rep["token"], C.byref(dl))
                return torch.utils.dlpack.from_dlpack(_capsule(dl.value))
            if not out.is_contiguous() or out.nbytes != n:
                dev.LIB.ft_client_done(self._cl, None, rep["token"], 0)
                raise ValueError("out must be contiguous with exactly the stored byte count")
            dev.LIB.ft_client_copy_done(self._cl, C.c_void_p(cur), C.c_void_p(out.data_ptr()), C.c_void_p(ptr), n,
                                        self._engine(out), rep["token"])
            return out
        if self._bin:
            nan = float("nan")
            rep = self._block_bin(_FETCH.pack(OP_FETCH, self.device, data_id, nan if slo_ms is None else slo_ms,
                                              nan if infer_ms is None else infer_ms))
        else:
            rep = self._call({"op": "fetch", "id": data_id, "gpu": self.device, "consumer": consumer,
                              "slo_ms": slo_ms, "infer_ms": infer_ms})
        imp = self._mapped(rep)
        ptr = imp.ptr + rep.get("off", 0)
        dt, shape, n = _DTYPES[rep["dtype"]], rep["shape"], rep["nbytes"]
        if out is not None and (not out.is_contiguous() or out.nbytes != n):
            self._done(rep["token"], -1)
            raise ValueError("out must be contiguous with exactly the stored byte count")
        if self._events:
            cur = torch.cuda.current_stream(self.device)
            self._after_daemon(rep, cur)               # the bytes are in place
            if out is None:
                # zero copy: a view of the stored block itself, released to the daemon
                # (with a mark of the releasing thread's stream) when the last tensor
                # over it dies
                owner = _Release()
                self._views += 1
                weakref.finalize(owner, self._release, rep["token"])
                return dev.as_tensor(ptr, n, self.device, dt, tuple(shape), owner=owner)
            dev.copy(out.data_ptr(), ptr, n, self.device, cur, self._engine(out))
            with self._io:
                self._done(rep["token"], self._mark(cur))
            return out
        # host-synced connection: copy on the private stream, synchronise, release
        if out is None:
            out = torch.empty(shape, dtype=dt, device=f"cuda:{self.device}")
        cur = torch.cuda.current_stream(self.device)
        self._stream.wait_stream(cur)
        dev.copy(out.data_ptr(), ptr, n, self.device, self._stream, self._engine(out))
        self._stream.synchronize()                     # read before the daemon may reuse the block
        self._send({"op": "done", "token": rep["token"]})
        cur.wait_stream(self._stream)
        return out

    def _release(self, token):
        self._views -= 1
        if self._closed:
            return
        try:
            cur = torch.cuda.current_stream(self.device)
            with self._io:
                self._done(token, self._mark(cur))
        except Exception:  # noqa: BLE001 - the daemon drops a dead connection's loans itself
            pass

    def _engine(self, t: torch.Tensor) -> int:
        """TMA bulk between this GPU's memory and a mapped block; the peer-safe vector
        engine when the tensor lives on another GPU."""
        return dev.ENGINE_BULK if t.get_device() == self.device else dev.ENGINE_VEC

    def _done(self, token: int, ev: int):
        """Release a read block (no reply): binary to the lane, else msgpack."""
        if self._bin:
            with self._io:
                self.ch.send_raw(_DONE.pack(OP_DONE, ev, token))
                if self._cl is None:
                    self._sent_py += 1
        else:
            self._send({"op": "done", "token": token, "ev": ev})

    def release(self, data_id: int):
        self._call({"op": "release", "id": data_id})

    def close(self):
        import gc
        gc.collect()                                   # views dropped by the caller send their done now
        self._closed = True
        views = self._views
        if self._cl is not None:
            nv = C.c_int()
            dev.LIB.ft_client_views(self._cl, C.byref(nv))
            views += nv.value
        if not views:                                  # a live view keeps its mapping (until exit)
            # copies into / out of the mapped blocks may still be queued: unmapping under
            # them faults (an illegal address in this process)
            torch.cuda.synchronize(self.device)
            for imp in self._imports.values():
                imp.close()
        else:
            _KEPT_IMPORTS.extend(self._imports.values())   # dropping them would unmap under the views
        self._imports.clear()
        self._loans.clear()
        if not self._events:
            dev.destroy_stream(self._stream)
        else:
            torch.cuda.synchronize(self.device)
            if self._mine is not None:
                self._peer.close()
                self._mine.close()
        self.ch.close()

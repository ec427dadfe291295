"""Function <-> daemon channel: an AF_UNIX stream socket carrying pool-block
file descriptors (SCM_RIGHTS, ``ft_fd_send``/``ft_fd_recv``), and binary
(msgpack) messages over a shared-memory ring pair (``ft_chan_*``, csrc/chan.cc)
once the client upgraded the connection. This is the paper's fast local
channel (a Linux pipe there) and the CUDA-IPC handoff of GPU
buffers: bytes never cross the channel — the receiver maps
the exported VMM block.
"""

from __future__ import annotations

import ctypes as C
import os
import socket
import struct

import msgpack

from . import device as dev
from ._lib import LIB, raise_status

_HDR = struct.Struct("<I")


_SLOT = 8192            # bytes per ring slot (the largest message: hello's 16 x 64-byte event handles)
_SLOTS = 16
# a receiver spins this long for the next message before it sleeps on a futex (a
# futex wake-up measured ~75 us in a VM, a spinning receiver ~7 us round trip)
SPIN_US = int(os.environ.get("FT_CHAN_SPIN_US", 2000))
_POLL_US = 200_000      # how often a blocked receiver checks that the peer is alive


class Channel:
    """Messages go over a shared-memory ring pair once ``upgrade`` (client) /
    ``attach`` (daemon) ran (``ft_chan_*``); before that, and for descriptors
    always, over the socket."""

    def __init__(self, sock: socket.socket):
        self.sock = sock
        self._client = None     # ft_client (the lane's function side) once it owns the rings
        self._chan = None
        self._dir = 0           # ring this side sends on (0: client requests, 1: daemon replies)
        self._buf = None
        self._n = None

    def _use(self, h, send_dir):
        self._chan, self._dir = h, send_dir
        self._buf = C.create_string_buffer(_SLOT)
        self._n = C.c_uint32()

    def upgrade(self):
        """Client: create the ring pair and hand it to the daemon (which attaches on ``chan``)."""
        fd, h = C.c_int(), C.c_void_p()
        LIB.ft_chan_create(_SLOT, _SLOTS, C.byref(fd), C.byref(h))
        self.send_msg({"op": "chan"})
        dev.send_fd(self.sock, fd.value, 0)
        self._use(h, 0)

    def attach(self):
        """Daemon: map the client's ring pair (its memfd follows the ``chan`` message)."""
        fd, _ = dev.recv_fd(self.sock)
        h = C.c_void_p()
        try:
            LIB.ft_chan_attach(fd, C.byref(h))
        finally:
            os.close(fd)
        self._use(h, 1)

    @classmethod
    def connect(cls, path: str, timeout: float = 60.0) -> "Channel":
        import time
        s = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        t_end = time.time() + timeout
        while True:
            try:
                s.connect(path)
                return cls(s)
            except (FileNotFoundError, ConnectionRefusedError):
                if time.time() > t_end:
                    raise
                time.sleep(0.01)

    @staticmethod
    def listen(path: str) -> socket.socket:
        if os.path.exists(path):
            os.unlink(path)
        s = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        s.bind(path)
        s.listen(16)
        return s

    @classmethod
    def accept(cls, server: socket.socket) -> "Channel":
        c, _ = server.accept()
        return cls(c)

    def send_fd(self, fd: int, meta: dict):
        """One descriptor + its metadata (size, dtype, shape, data id ...)."""
        body = msgpack.packb(meta)
        dev.send_fd(self.sock, fd, len(body))
        self.sock.sendall(body)

    def recv_fd(self):
        fd, n = dev.recv_fd(self.sock)
        return fd, msgpack.unpackb(self._recv_exact(n))

    def adopt_client(self, client):
        """The native lane client takes the rings over (every send through its mutex)."""
        self._client, self._chan = client, None

    def send_msg(self, meta: dict):
        body = msgpack.packb(meta)
        if self._client is not None:
            self._client_send(body)
            return
        if self._chan is not None:
            self._chan_send(body)
            return
        self.sock.sendall(_HDR.pack(len(body)) + body)

    def _chan_send(self, body: bytes):
        # a full ring waits for the peer to drain it while the peer lives
        while True:
            rc = LIB.raw("ft_chan_send")(self._chan, self._dir, body, len(body), _POLL_US)
            if rc == 0:
                return
            if rc == 13:
                raise ConnectionError("channel closed")
            if rc != 12:
                raise_status(rc)
            self._check_peer()

    def _client_send(self, body: bytes):
        rc = LIB.raw("ft_client_send")(self._client, body, len(body))
        if rc == 13:
            self._daemon_gone("channel closed")
        if rc:
            raise_status(rc)

    def _daemon_gone(self, why: str):
        # our streams may wait on marks the daemon will never write: release them, so
        # a later synchronise (or close) does not hang
        LIB.ft_client_abandon(self._client)
        raise ConnectionError(why)

    def client_reply(self, rc: int, buf=None, n=None, spin_us: int = SPIN_US) -> bytes:
        """The reply a native client call left in ``buf`` (``n`` bytes) with status
        ``rc``; on a timeout, wait longer while the daemon is alive."""
        buf = self._buf if buf is None else buf
        n = self._n if n is None else n
        while rc == 12:
            try:
                self._check_peer()
            except ConnectionError as e:
                self._daemon_gone(str(e))
            rc = LIB.raw("ft_client_recv")(self._client, buf, len(buf), C.byref(n), spin_us)
        if rc == 13:
            self._daemon_gone("channel closed")
        if rc:
            raise_status(rc)
        return buf.raw[:n.value]

    def send_raw(self, body: bytes):
        """One binary message on the rings (the native lane's protocol)."""
        if self._client is not None:
            self._client_send(body)
            return
        self._chan_send(body)

    def recv_raw(self, spin_us: int = SPIN_US) -> bytes:
        if self._client is not None:
            return self.client_reply(12, spin_us=spin_us)
        while True:
            rc = LIB.raw("ft_chan_recv")(self._chan, 1 - self._dir, self._buf, _SLOT, self._n, spin_us, _POLL_US)
            if rc == 0:
                return self._buf.raw[:self._n.value]
            if rc == 13:
                raise ConnectionError("channel closed")
            if rc != 12:
                raise_status(rc)
            self._check_peer()

    def recv_msg(self, spin_us: int = SPIN_US) -> dict:
        if self._client is not None:
            return msgpack.unpackb(self.client_reply(12, spin_us=spin_us))
        if self._chan is None:
            n = _HDR.unpack(self._recv_exact(4))[0]
            return msgpack.unpackb(self._recv_exact(n))
        while True:
            rc = LIB.raw("ft_chan_recv")(self._chan, 1 - self._dir, self._buf, _SLOT, self._n, spin_us, _POLL_US)
            if rc == 0:
                return msgpack.unpackb(self._buf.raw[:self._n.value])
            if rc == 13:
                raise ConnectionError("channel closed")
            if rc != 12:
                raise_status(rc)
            self._check_peer()                        # timeout: is the peer still there?

    def _check_peer(self):
        try:
            if self.sock.recv(1, socket.MSG_PEEK | socket.MSG_DONTWAIT) == b"":
                raise ConnectionError("peer went away")
        except (BlockingIOError, InterruptedError):
            pass

    def _recv_exact(self, n):
        buf = self.sock.recv(n)
        if len(buf) == n:
            return buf
        parts = [buf]
        got = len(buf)
        while got < n:
            if not buf:
                raise ConnectionError("channel closed")
            buf = self.sock.recv(n - got)
            parts.append(buf)
            got += len(buf)
        return b"".join(parts)

    def close(self):
        h, self._chan = self._chan, None
        if h is not None:
            LIB.ft_chan_close(h)
        cl, self._client = self._client, None
        if cl is not None:                   # the rings close with the client's last view
            LIB.ft_client_destroy(cl)
        self.sock.close()

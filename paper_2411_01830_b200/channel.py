"""Function <-> daemon channel: AF_UNIX stream sockets carrying pool-block
file descriptors (SCM_RIGHTS, ``ft_fd_send``/``ft_fd_recv``) plus binary
(msgpack) messages, length-prefixed. This is the paper's fast local channel (a Linux
pipe there) and the CUDA-IPC handoff of GPU buffers:
bytes never cross the socket — the receiver maps the exported VMM block.
"""

from __future__ import annotations

import os
import socket
import struct

import msgpack

from . import device as dev

_HDR = struct.Struct("<I")


class Channel:
    def __init__(self, sock: socket.socket):
        self.sock = sock

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

    def send_msg(self, meta: dict):
        body = msgpack.packb(meta)
        self.sock.sendall(_HDR.pack(len(body)) + body)

    def recv_msg(self) -> dict:
        n = _HDR.unpack(self._recv_exact(4))[0]
        return msgpack.unpackb(self._recv_exact(n))

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
        self.sock.close()

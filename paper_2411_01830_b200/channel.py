"""Function <-> daemon channel: AF_UNIX stream sockets carrying pool-block
file descriptors (SCM_RIGHTS, ``ft_fd_send``/``ft_fd_recv``) plus a JSON
descriptor. This is the paper's fast local channel (a Linux
pipe there) and the CUDA-IPC handoff of GPU buffers:
bytes never cross the socket — the receiver maps the exported VMM block.
"""

from __future__ import annotations

import json
import os
import socket
import struct

from . import device as dev


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
        body = json.dumps(meta).encode()
        dev.send_fd(self.sock, fd, len(body))
        self.sock.sendall(body)

    def recv_fd(self):
        fd, n = dev.recv_fd(self.sock)
        body = b""
        while len(body) < n:
            chunk = self.sock.recv(n - len(body))
            if not chunk:
                raise ConnectionError("channel closed mid-message")
            body += chunk
        return fd, json.loads(body.decode())

    def send_msg(self, meta: dict):
        body = json.dumps(meta).encode()
        self.sock.sendall(struct.pack("<Q", len(body)) + body)

    def recv_msg(self) -> dict:
        hdr = self._recv_exact(8)
        return json.loads(self._recv_exact(struct.unpack("<Q", hdr)[0]).decode())

    def _recv_exact(self, n):
        buf = b""
        while len(buf) < n:
            chunk = self.sock.recv(n - len(buf))
            if not chunk:
                raise ConnectionError("channel closed")
            buf += chunk
        return buf

    def close(self):
        self.sock.close()

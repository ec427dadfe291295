"""Cross-process gFunc->gFunc handoff over NVLink (one process per GPU).

Rank r's producer stores into a pool block B_r that is exported (VMM POSIX fd,
``channel.py``) to rank r+1; rank r+1's consumer pulls it over the peer
mapping with the vector copy engine. Ordering uses doorbells in device
memory instead of host round trips (``ft_signal`` / ``ft_wait``):

    producer r : wait ACK_r >= k-1 ; store x -> B_r ; signal RDY_{r+1} = k
    consumer c : wait RDY_c >= k   ; pull B_{c-1} -> input ; signal ACK_{c-1} = k

RDY_c lives on GPU c (written remotely by the producer), ACK_r on GPU r
(written remotely by the consumer), so every wait spins on local memory.
Each rank is a producer (to r+1) and a consumer (of r-1) on separate streams.
Waits are bounded (``ft_wait_timeout``): a peer that never rings cannot park a
stream forever; the expired wait leaves its value in the error word that
``check()`` reports.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import device as dev
from .channel import Channel

FLAG_BYTES = 4096
WAIT_TIMEOUT_NS = 20 * 10**9


class CrossPair:
    def __init__(self, tube, device: int, rank: int, world: int, sock_dir: str, nbytes: int, barrier):
        self.tube, self.g, self.rank, self.world, self.n = tube, device, rank, world, int(nbytes)
        pool = tube.pools[device]
        self.payload = pool.allocate(self.n)                 # B_r (my producer's stored output)
        self.flags = pool.allocate(FLAG_BYTES)               # [0] RDY (I consume), [1] ACK (I produce)
        dev.as_tensor(self.flags.ptr, FLAG_BYTES, device).zero_()
        torch.cuda.synchronize(device)
        self.prod_stream = dev.new_stream(device)
        self.cons_stream = dev.new_stream(device)
        nxt, prv = (rank + 1) % world, (rank - 1) % world
        srv = Channel.listen(os.path.join(sock_dir, f"r{rank}.sock"))
        barrier()
        # to the next rank (my consumer): payload + my flags (for its ACK writes)
        out = Channel.connect(os.path.join(sock_dir, f"r{nxt}.sock"))
        exp = [pool.export(self.payload), pool.export(self.flags), pool.export(self.flags)]
        mine = [e[0] for e in exp]

        def meta(kind, blk, e):
            return {"kind": kind, "nbytes": blk.nbytes, "arena_bytes": e[1], "off": e[2]}

        def imp(fd, m):
            return dev.ImportedBlock(device, fd, m["arena_bytes"], m["off"], m["nbytes"])

        out.send_fd(mine[0], meta("payload", self.payload, exp[0]))
        out.send_fd(mine[1], meta("flags", self.flags, exp[1]))
        # from the previous rank (my producer): its payload + flags; reply with mine
        inc = Channel.accept(srv)
        fd_p, meta_p = inc.recv_fd()
        fd_f, meta_f = inc.recv_fd()
        self.peer_payload = imp(fd_p, meta_p)
        self.peer_flags = imp(fd_f, meta_f)                                   # previous rank's flags
        inc.send_fd(mine[2], meta("flags", self.flags, exp[2]))
        fd_n, meta_n = out.recv_fd()
        self.next_flags = imp(fd_n, meta_n)                                   # next rank's flags
        for fd in (fd_p, fd_f, fd_n, *mine):
            os.close(fd)
        barrier()
        self._chans = (srv, out, inc)
        self.step = 0

    # flag words
    def _rdy_local(self):
        return self.flags.ptr               # RDY_me, written by my producer peer
    def _ack_local(self):
        return self.flags.ptr + 4           # ACK_me, written by my consumer peer
    def _rdy_next(self):
        return self.next_flags.ptr          # RDY of rank r+1 (peer)
    def _ack_prev(self):
        return self.peer_flags.ptr + 4      # ACK of rank r-1 (peer)
    def _err(self):
        return self.flags.ptr + 8           # awaited value of an expired wait (0: none)

    def _wait(self, flag, value, stream):
        dev.LIB.ft_wait_timeout(C.c_void_p(flag), value & 0xFFFFFFFF, WAIT_TIMEOUT_NS, C.c_void_p(self._err()),
                                self.g, C.c_void_p(stream.cuda_stream))

    def check(self):
        """Raise if any doorbell wait expired (a peer stopped ringing)."""
        torch.cuda.synchronize(self.g)
        err = int(dev.as_tensor(self.flags.ptr + 8, 4, self.g, torch.int32)[0])
        if err:
            raise RuntimeError(f"rank {self.rank}: doorbell wait for step {err} expired")

    def produce(self, x: torch.Tensor):
        """store step k: wait until the consumer released B_r, snapshot x, ring RDY."""
        self.step += 1
        k = self.step
        s = self.prod_stream
        s.wait_stream(torch.cuda.current_stream(self.g))
        self._wait(self._ack_local(), k - 1, s)
        dev.copy(self.payload.ptr, x.data_ptr(), self.n, self.g, s, dev.ENGINE_BULK)
        dev.LIB.ft_signal(C.c_void_p(self._rdy_next()), k & 0xFFFFFFFF, self.g, C.c_void_p(s.cuda_stream))

    def consume(self, out: torch.Tensor):
        """fetch step k: wait for RDY, pull the peer's block over NVLink, ACK it."""
        k = self.step
        s = self.cons_stream
        self._wait(self._rdy_local(), k, s)
        dev.copy(out.data_ptr(), self.peer_payload.ptr, self.n, self.g, s, dev.ENGINE_VEC)
        dev.LIB.ft_signal(C.c_void_p(self._ack_prev()), k & 0xFFFFFFFF, self.g, C.c_void_p(s.cuda_stream))
        torch.cuda.current_stream(self.g).wait_stream(s)

    def close(self):
        torch.cuda.synchronize(self.g)
        for b in (self.peer_payload, self.peer_flags, self.next_flags):
            b.close()
        for c in self._chans:
            c.close()

"""The function <-> daemon shared-memory rings (csrc/chan.cc) on CPU: request /
reply between two processes, ordering, a full ring, messages larger than a slot,
timeouts, and the peer closing — no GPU involved."""

import ctypes as C
import multiprocessing as mp

import pytest


def _echo(fd, n_msgs):
    from paper_2411_01830_b200._lib import LIB
    h = C.c_void_p()
    LIB.ft_chan_attach(fd, C.byref(h))
    buf, n = C.create_string_buffer(4096), C.c_uint32()
    for _ in range(n_msgs):
        LIB.ft_chan_recv(h, 0, buf, 4096, C.byref(n), 100, 5_000_000)
        LIB.ft_chan_send(h, 1, buf.raw[:n.value][::-1], n.value, 5_000_000)
    LIB.ft_chan_close(h)


def test_request_reply_across_processes():
    from paper_2411_01830_b200._lib import LIB
    fd, h = C.c_int(), C.c_void_p()
    LIB.ft_chan_create(4096, 4, C.byref(fd), C.byref(h))
    p = mp.get_context("fork").Process(target=_echo, args=(fd.value, 200))
    p.start()
    buf, n = C.create_string_buffer(4096), C.c_uint32()
    for i in range(200):
        msg = bytes([i % 251]) * (1 + (i * 37) % 4000)
        LIB.ft_chan_send(h, 0, msg, len(msg), 5_000_000)
        LIB.ft_chan_recv(h, 1, buf, 4096, C.byref(n), 100, 5_000_000)
        assert buf.raw[:n.value] == msg[::-1]
    p.join(10)
    assert p.exitcode == 0
    # the peer closed: a receive reports it (ConnectionError), not a timeout
    with pytest.raises(ConnectionError):
        LIB.ft_chan_recv(h, 1, buf, 4096, C.byref(n), 10, 1_000_000)
    LIB.ft_chan_close(h)


def test_full_ring_oversize_and_timeouts():
    from paper_2411_01830_b200._lib import LIB, WaitTimeout
    fd, h = C.c_int(), C.c_void_p()
    LIB.ft_chan_create(256, 2, C.byref(fd), C.byref(h))
    buf, n = C.create_string_buffer(256), C.c_uint32()
    with pytest.raises(WaitTimeout):                       # nothing sent yet
        LIB.ft_chan_recv(h, 0, buf, 256, C.byref(n), 10, 20_000)
    LIB.ft_chan_send(h, 0, b"a", 1, 1000)
    LIB.ft_chan_send(h, 0, b"bb", 2, 1000)
    with pytest.raises(WaitTimeout):                       # two slots: the third waits for room
        LIB.ft_chan_send(h, 0, b"ccc", 3, 20_000)
    with pytest.raises(ValueError):                        # larger than a slot (256 - 8 header bytes)
        LIB.ft_chan_send(h, 1, b"x" * 249, 249, 1000)
    small = C.create_string_buffer(1)
    LIB.ft_chan_recv(h, 0, small, 1, C.byref(n), 10, 1000)
    assert small.raw[:n.value] == b"a"                     # in order
    rc = LIB.raw("ft_chan_recv")(h, 0, small, 1, C.byref(n), 10, 1000)
    assert rc == 9 and n.value == 2                        # FT_E_TRUNCATED: the message stays queued
    LIB.ft_chan_recv(h, 0, buf, 256, C.byref(n), 10, 1000)
    assert buf.raw[:n.value] == b"bb"
    LIB.ft_chan_send(h, 0, b"ccc", 3, 1000)                # room again
    LIB.ft_chan_close(h)

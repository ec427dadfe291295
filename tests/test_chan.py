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


def test_peer_written_geometry_and_lengths_are_not_trusted():
    """The daemon maps a ring pair its client created and the client can keep
    writing the header: attach checks the geometry against the file's real size,
    the mapped side indexes by the geometry it attached with, and a slot length no
    sender could have written is an error, not an out-of-bounds copy."""
    import mmap
    import struct
    from paper_2411_01830_b200._lib import LIB
    fd, h = C.c_int(), C.c_void_p()
    LIB.ft_chan_create(256, 4, C.byref(fd), C.byref(h))
    m = mmap.mmap(fd.value, 640 + 2 * 256 * 4)
    slot_bytes, slots = struct.unpack_from("<II", m, 4)
    assert (slot_bytes, slots) == (256, 4)
    struct.pack_into("<I", m, 8, 1 << 15)                  # more slots than the file holds
    h2 = C.c_void_p()
    with pytest.raises(ValueError, match="geometry"):
        LIB.ft_chan_attach(fd.value, C.byref(h2))
    struct.pack_into("<I", m, 8, 4)
    LIB.ft_chan_attach(fd.value, C.byref(h2))
    struct.pack_into("<II", m, 4, 1 << 20, 1 << 10)        # rewritten after attach: ignored
    with pytest.raises(ValueError):                        # still 256-byte slots
        LIB.ft_chan_send(h2, 1, b"x" * 300, 300, 1000)
    LIB.ft_chan_send(h2, 1, b"ok", 2, 1000)
    buf, n = C.create_string_buffer(256), C.c_uint32()
    LIB.ft_chan_recv(h, 1, buf, 256, C.byref(n), 10, 1000)
    assert buf.raw[:n.value] == b"ok"
    # a forged message: ring 0's slot 0 claims 4 GiB, head bumped by hand
    struct.pack_into("<I", m, 640, 0xFFFFFFFF)
    struct.pack_into("<I", m, 128, 1)
    with pytest.raises(ValueError, match="corrupt"):
        LIB.ft_chan_recv(h2, 0, C.create_string_buffer(1 << 16), 1 << 16, C.byref(n), 10, 1000)
    m.close()
    LIB.ft_chan_close(h2)
    LIB.ft_chan_close(h)


def test_counters_wrap_around_2_32():
    """The ring's head / tail are free-running 32-bit counters: a channel that has
    carried ~2^32 messages keeps its order and its full / empty tests across the wrap."""
    import mmap
    import struct
    from paper_2411_01830_b200._lib import LIB, WaitTimeout
    fd, h = C.c_int(), C.c_void_p()
    LIB.ft_chan_create(256, 4, C.byref(fd), C.byref(h))
    m = mmap.mmap(fd.value, 640 + 2 * 256 * 4)
    start = 0xFFFFFFFE
    struct.pack_into("<I", m, 128, start)                  # ring 0 head
    struct.pack_into("<I", m, 192, start)                  # ring 0 tail
    buf, n = C.create_string_buffer(256), C.c_uint32()
    sent = 0
    for i in range(10):
        while sent < i + 4:                                # keep the ring full (4 slots)
            msg = b"m%d" % sent
            LIB.ft_chan_send(h, 0, msg, len(msg), 1000)
            sent += 1
        with pytest.raises(WaitTimeout):                   # full across the wrap
            LIB.ft_chan_send(h, 0, b"x", 1, 2000)
        LIB.ft_chan_recv(h, 0, buf, 256, C.byref(n), 10, 1000)
        assert buf.raw[:n.value] == b"m%d" % i
    head, tail = struct.unpack_from("<I", m, 128)[0], struct.unpack_from("<I", m, 192)[0]
    assert head == (start + sent) & 0xFFFFFFFF and tail == (start + 10) & 0xFFFFFFFF
    m.close()
    LIB.ft_chan_close(h)

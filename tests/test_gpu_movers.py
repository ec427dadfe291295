"""GPU parity of the byte movers through the C ABI: every mover must deliver
exactly the source bytes (uint8 equality — the reference's byte semantics are
identity), at edge sizes/alignments and at BASELINE sizes."""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SIZES = [1, 15, 16, 17, 255, 4096, 4097, 65536 + 3, 2 * 10**6, (2 << 20) + 16, 64 << 20]


def rnd(n, seed, device="cuda:0"):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g).to(device)


@pytest.fixture(scope="module")
def dev():
    from paper_2411_01830_b200 import device
    device.require_cuda()
    return device


@pytest.mark.parametrize("engine", [1, 2])
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("shift", [0, 3])
def test_copy_bit_exact(dev, engine, n, shift):
    src = rnd(n + 64, n)
    dst = torch.zeros(n + 64, dtype=torch.uint8, device="cuda:0")
    dev.copy(dst.data_ptr() + shift, src.data_ptr() + shift, n, 0, None, engine)
    torch.cuda.synchronize()
    assert torch.equal(dst[shift:shift + n], src[shift:shift + n])
    assert int(dst[:shift].sum()) == 0 and int(dst[shift + n:].sum()) == 0   # no overrun


def test_copy_misaligned_pair(dev):
    src = rnd(1 << 20, 5)
    dst = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda:0")
    dev.copy(dst.data_ptr() + 1, src.data_ptr() + 2, 100000, 0)
    torch.cuda.synchronize()
    assert torch.equal(dst[1:100001], src[2:100002])


def test_copy_1gib(dev):
    n = 1 << 30
    src = rnd(n, 2)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    dev.copy(dst.data_ptr(), src.data_ptr(), n, 0)
    torch.cuda.synchronize()
    assert torch.equal(dst, src)


@pytest.mark.parametrize("shift", [0, 3, 8])
def test_fingerprint_any_alignment(dev, shift):
    n = (1 << 20) + 13
    src = rnd(n + 16, 77)
    fp = dev.Fingerprint(0)
    fp.launch(src.data_ptr() + shift, n)
    assert fp.value() == dev.fingerprint_host(src[shift:shift + n].cpu())


@pytest.mark.parametrize("n", [1, 7, 8, 9, 4096, 12345677, 64 << 20])
def test_fingerprint_matches_host(dev, n):
    src = rnd(n, n + 1)
    fp = dev.Fingerprint(0)
    fp.launch(src.data_ptr(), n)
    assert fp.value() == dev.fingerprint_host(src.cpu())
    # single byte flip changes it
    flip = src.clone()
    flip[n // 2] ^= 1
    fp.launch(flip.data_ptr(), n)
    assert fp.value() != dev.fingerprint_host(src.cpu())


@pytest.mark.parametrize("batch", [0, 2 * 10**6, 10 * 10**6])
def test_pcie_legs(dev, batch):
    n = (64 << 20) + 12345
    host = torch.from_numpy(np.random.default_rng(3).integers(0, 256, n, dtype=np.uint8)).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    dev.pcie_copy(d.data_ptr(), host.data_ptr(), n, True, 0, None, batch)
    back = torch.empty(n, dtype=torch.uint8).pin_memory()
    dev.pcie_copy(back.data_ptr(), d.data_ptr(), n, False, 0, None, batch)
    torch.cuda.synchronize()
    assert torch.equal(back, host)


def test_h2g_striped_staging_route(dev):
    """The staging + NVLink-forward route, exercised on one GPU (staging GPU ==
    target): CE into a chunk ring, forward kernel into the destination."""
    from paper_2411_01830_b200._lib import LIB
    n = (32 << 20) + 777
    host = torch.from_numpy(np.random.default_rng(4).integers(0, 256, n, dtype=np.uint8)).pin_memory()
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    chunk, ring = 2 * 10**6, 3
    stg = torch.empty(chunk * ring, dtype=torch.uint8, device="cuda:0")
    s = [torch.cuda.Stream(0) for _ in range(4)]
    half = n // 2 // 256 * 256
    offs = (C.c_uint64 * 2)(0, half)
    lens = (C.c_uint64 * 2)(half, n - half)
    sd = (C.c_int32 * 2)(0, 0)
    stgp = (C.c_void_p * 2)(None, stg.data_ptr())       # route 0 direct, route 1 staged
    streams = (C.c_void_p * 4)(*[x.cuda_stream for x in s])
    LIB.ft_h2g_striped(C.c_void_p(dst.data_ptr()), 0, C.c_void_p(host.data_ptr()), n, 2, sd, offs, lens, stgp,
                       chunk, ring, streams)
    torch.cuda.synchronize()
    assert torch.equal(dst.cpu(), host)


def test_vmm_pool_map_unmap(dev):
    pool = dev.DevicePool(0, "autoscale", floor_bytes=0.0, spare_cap_bytes=0)   # exact physical accounting
    blocks = [pool.allocate(n) for n in (1, 2 * 10**6, 64 << 20, 3 * 10**6)]
    for i, b in enumerate(blocks):
        t = dev.as_tensor(b.ptr, b.nbytes, 0)
        t.fill_(i + 1)
    torch.cuda.synchronize()
    for i, b in enumerate(blocks):
        assert int(dev.as_tensor(b.ptr, b.nbytes, 0).float().mean()) == i + 1
    st = pool.stats()
    assert st["blocks"] == 4 and st["mapped_bytes"] >= sum(b.nbytes for b in blocks)
    # exact-class reuse: freeing then allocating the same class maps nothing new
    pool.free(blocks[2])
    again = pool.allocate(64 << 20)
    assert again.ptr == blocks[2].ptr and pool.stats()["blocks"] == 4
    for b in (blocks[0], blocks[1], blocks[3], again):
        pool.free(b)
    released = pool.shrink(1e9)          # no active window, floor 0 -> everything idle goes
    assert released > 0 and pool.stats()["blocks"] < 4
    pool.close()


def test_spin_ns_is_wall_time(dev):
    """The runtime's synthetic compute: duration follows the global timer,
    not the SM clock (an idle GPU idles at ~120 MHz)."""
    import time
    from paper_2411_01830_b200._lib import LIB
    s = torch.cuda.current_stream(0)
    LIB.ft_spin_ns(1000, 0, C.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    for ms in (2.0, 10.0):
        t0 = time.perf_counter()
        LIB.ft_spin_ns(int(ms * 1e6), 0, C.c_void_p(s.cuda_stream))
        torch.cuda.synchronize()
        got = (time.perf_counter() - t0) * 1e3
        assert ms <= got < ms + 1.5, (ms, got)


def test_doorbell_wait_is_bounded(dev):
    """A doorbell that never rings: the wait gives up after its timeout and
    leaves the awaited value in the error word (no stream parked forever)."""
    import time
    from paper_2411_01830_b200._lib import LIB
    words = torch.zeros(4, dtype=torch.int32, device="cuda:0")
    s = torch.cuda.current_stream(0)
    t0 = time.perf_counter()
    LIB.ft_wait_timeout(C.c_void_p(words.data_ptr()), 7, 50_000_000, C.c_void_p(words.data_ptr() + 8), 0,
                        C.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    assert 45.0 <= ms < 1000.0, ms
    assert int(words[2]) == 7
    # a rung doorbell passes at once and leaves the error word alone
    words.zero_()
    LIB.ft_signal(C.c_void_p(words.data_ptr()), 9, 0, C.c_void_p(s.cuda_stream))
    LIB.ft_wait_timeout(C.c_void_p(words.data_ptr()), 9, 50_000_000, C.c_void_p(words.data_ptr() + 8), 0,
                        C.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    assert int(words[0]) == 9 and int(words[2]) == 0


def test_copy_batch_segments(dev):
    """ft_copy_batch: >64 segments (several launches), ragged sizes, misaligned
    and empty segments — every byte lands."""
    rng = np.random.default_rng(3)
    sizes = [0, 1, 15, 16, 17, 4096, 4097, 32768, 32769, 65536 + 3, (1 << 20) + 5] * 7
    srcs = [rnd(max(n, 1) + 8, 100 + i) for i, n in enumerate(sizes)]
    dsts = [torch.zeros(max(n, 1) + 8, dtype=torch.uint8, device="cuda:0") for n in sizes]
    shifts = [int(rng.integers(0, 4)) for _ in sizes]
    segs = [(d.data_ptr() + sh, x.data_ptr() + sh2, n)
            for d, x, n, sh, sh2 in zip(dsts, srcs, sizes, shifts, reversed(shifts))]
    dev.copy_batch(segs, 0, None)
    torch.cuda.synchronize()
    for d, x, n, sh, sh2 in zip(dsts, srcs, sizes, shifts, reversed(shifts)):
        assert torch.equal(d[sh:sh + n], x[sh2:sh2 + n])
        assert not d[:sh].any() and not d[sh + n:].any()


def test_pool_spares_serve_growth(dev):
    """After a growth of a class, a background thread maps one spare of it; the
    next growth of that class (the policy's new block) is served by the spare,
    and the bytes are the new holder's (fenced, writable)."""
    import time
    pool = dev.DevicePool(0, "autoscale", floor_bytes=0.0, spare_cap_bytes=4 << 30)
    a = pool.allocate(32 << 20)
    deadline = time.time() + 5
    while pool.spares_mapped < 1 and time.time() < deadline:
        time.sleep(0.01)
    assert pool.spares_mapped == 1 and pool.released_bytes >= 32 << 20
    blocks_before = pool.stats()["blocks"]
    b = pool.allocate(32 << 20)                     # growth: a second live block of the class
    assert b.ptr != a.ptr and pool.stats()["blocks"] in (blocks_before, blocks_before + 1)
    t = dev.as_tensor(b.ptr, 32 << 20, 0)
    t.fill_(9)
    torch.cuda.synchronize()
    assert int(t.float().mean()) == 9
    pool.free(a)
    pool.free(b)
    pool.close()


def test_pool_spare_is_rounded_up_and_serves_nearby_classes(dev):
    """A growth of a 40 MB class maps a 64 MB spare (a power of two of the 2 MiB
    granule); a later growth of any class in (32, 64] MB takes it instead of
    mapping on the request path."""
    import time
    pool = dev.DevicePool(0, "autoscale", floor_bytes=0.0, spare_cap_bytes=4 << 30)
    a = pool.allocate(40 << 20)
    deadline = time.time() + 5
    while pool.spares_mapped < 1 and time.time() < deadline:
        time.sleep(0.01)
    assert pool.spares_mapped == 1 and pool.released_bytes == 64 << 20
    b = pool.allocate(60 << 20)                     # a class never seen: served by the spare
    assert pool.released_bytes < 64 << 20 or pool.spares_mapped > 1
    t = dev.as_tensor(b.ptr, 60 << 20, 0)
    t.fill_(5)
    torch.cuda.synchronize()
    assert int(t.float().mean()) == 5
    pool.free(a)
    pool.free(b)
    pool.close()


def test_pool_arenas_map_rarely_and_trim_when_idle(dev, monkeypatch):
    """Blocks are ranges of arenas: growth inside the reservation maps nothing,
    growth past it maps one arena (not one per block), a freed range is reused,
    and only an unused, unreserved arena is unmapped by the idle trim — its id
    reported to the unmap listeners (daemon clients drop their import)."""
    monkeypatch.setenv("FT_POOL_ARENA_BYTES", str(256 << 20))
    pool = dev.DevicePool(0, "autoscale", floor_bytes=0.0, reserve_bytes=128 << 20)
    dropped = []
    pool.on_unmap.append(dropped.append)
    assert pool.stats()["mapped_bytes"] == 128 << 20
    small = [pool.allocate(2 * 10**6) for _ in range(32)]            # 32 x 2 MiB inside the reservation
    assert pool.stats()["mapped_bytes"] == 128 << 20
    big = [pool.allocate(64 * 10**6) for _ in range(3)]              # past it: ONE 256 MiB arena
    assert pool.stats()["mapped_bytes"] == (128 << 20) + (256 << 20)
    for i, b in enumerate(small + big):
        dev.as_tensor(b.ptr, b.nbytes, 0).fill_(i % 251)
    torch.cuda.synchronize()
    for i, b in enumerate(small + big):
        assert int(dev.as_tensor(b.ptr, b.nbytes, 0)[:4096].float().mean()) == i % 251
    a, off, abytes = pool.locate(big[-1])              # (big[0] still fit in the reservation)
    assert abytes == 256 << 20 and off % (2 << 20) == 0
    for b in big:
        pool.free(b)
    pool.shrink(1e9)                                                 # policy drops the idle blocks, reclaim trims
    assert pool.stats()["mapped_bytes"] == 128 << 20 and a in dropped
    for b in small:
        pool.free(b)
    pool.shrink(1e9)
    assert pool.stats()["mapped_bytes"] == 128 << 20                 # the reservation stays
    pool.close()

"""GPU parity of the put/get API (tube.FaaSTube) against the oracle's CPU
host-memory path: for every transfer method the consumer must receive
exactly the bytes the reference path (store into host memory, fetch out of
it — oracle/host_path.py) delivers, compared as uint8."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MB = 1 << 20


@pytest.fixture(scope="module")
def tube():
    from paper_2411_01830_b200.tube import FaaSTube
    t = FaaSTube("faastube", pool_floor_bytes=0.0)
    yield t
    assert t._accounts_consistent()
    t.close()


def payload(seed=0, shape=(32, 1024, 1024), dtype=torch.float16, device="cuda:0"):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randn(shape, generator=g).to(dtype).to(device)


def oracle_bytes(t: torch.Tensor) -> np.ndarray:
    from oracle.host_path import HostMemoryStore
    hs = HostMemoryStore(threads=4)
    did = hs.unique_id()
    hs.store(did, t.detach().cpu().contiguous().view(torch.uint8).numpy())
    out = hs.fetch(did)
    hs.close()
    return out


def as_u8(t):
    return t.detach().contiguous().view(torch.uint8).reshape(-1).cpu().numpy()


def test_config1_same_gpu_copy_into_input(tube):
    x = payload(0)                                   # 64 MiB fp16, seed 0
    did = tube.unique_id()
    tube.store(did, x, producer="producer")
    inp = torch.empty_like(x)
    got = tube.fetch(did, device=0, out=inp, consumer="consumer")
    torch.cuda.synchronize()
    assert got.data_ptr() == inp.data_ptr()
    assert np.array_equal(as_u8(got), oracle_bytes(x))


def test_config1_zero_copy_view(tube):
    x = payload(1)
    did = tube.unique_id()
    tube.store(did, x)
    v = tube.fetch(did, device=0)
    assert v.shape == x.shape and v.dtype == x.dtype
    assert torch.equal(v.view(torch.uint8), x.view(torch.uint8))
    assert tube.stats["zero_copy"] >= 1


def test_zero_copy_store_from_pool_output(tube):
    out = tube.empty((1024, 1024), torch.float16, device=0)
    out.copy_(payload(2, (1024, 1024)))
    did = tube.unique_id()
    before = tube.stats["bytes_local"]
    tube.store(did, out)
    assert tube.stats["bytes_local"] == before               # no copy on store
    got = tube.fetch(did, device=0, out=torch.empty_like(out))
    assert torch.equal(got.view(torch.uint8), out.view(torch.uint8))


@pytest.mark.parametrize("n", [1, 4095, 4096, 2 * 10**6 + 1, 64 * MB])
def test_host_to_gpu(tube, n):
    rng = np.random.default_rng(n)
    host = torch.from_numpy(rng.integers(0, 256, n, dtype=np.uint8))
    did = tube.unique_id()
    tube.store(did, host, producer="decode")                  # cFunc output: host resident
    got = tube.fetch(did, device=0, consumer="preproc")
    torch.cuda.synchronize()
    assert np.array_equal(as_u8(got), oracle_bytes(host))


def test_gpu_to_host_and_response(tube):
    x = payload(3, (4, 1024, 1024))
    did = tube.unique_id()
    tube.store(did, x, response=True, consumers=2)
    assert np.array_equal(as_u8(tube.response(did)), oracle_bytes(x))
    h = tube.fetch(did, device=None)
    assert not h.is_cuda and np.array_equal(as_u8(h), oracle_bytes(x))
    tube.fetch(did, device=0, out=torch.empty_like(x))        # second consumer retires it
    from paper_2411_01830_b200 import MissingData
    with pytest.raises(MissingData):
        tube.fetch(did, device=0)


def test_multiple_consumers_and_retire(tube):
    x = payload(4, (2, 1024, 1024))
    did = tube.unique_id()
    tube.store(did, x, consumers=3)
    outs = [tube.fetch(did, device=0, out=torch.empty_like(x)) for _ in range(3)]
    for o in outs:
        assert torch.equal(o.view(torch.uint8), x.view(torch.uint8))
    from paper_2411_01830_b200 import MissingData
    with pytest.raises(MissingData):
        tube.fetch(did, device=0)


def test_duplicate_store(tube):
    from paper_2411_01830_b200 import DuplicateStore
    x = payload(5, (16,))
    did = tube.unique_id()
    tube.store(did, x, consumers=2)
    with pytest.raises(DuplicateStore):
        tube.store(did, x)
    tube.release(did)


def test_pool_reuse_no_growth(tube):
    x = payload(6, (8, 1024, 1024))
    pool = tube.pools[0]
    did = tube.unique_id()
    tube.store(did, x)
    tube.fetch(did, device=0, out=torch.empty_like(x))
    grown = pool.grow_events
    for _ in range(5):
        did = tube.unique_id()
        tube.store(did, x)
        tube.fetch(did, device=0, out=torch.empty_like(x))
    assert pool.grow_events == grown                           # same class served from the cache


def test_view_pins_block(tube):
    """A zero-copy view keeps its block from being reused by later stores."""
    x = payload(7, (1024, 1024))
    did = tube.unique_id()
    tube.store(did, x)
    v = tube.fetch(did, device=0)
    y = payload(8, (1024, 1024))
    for _ in range(3):
        d2 = tube.unique_id()
        tube.store(d2, y)
        tube.fetch(d2, device=0, out=torch.empty_like(y))
    torch.cuda.synchronize()
    assert torch.equal(v.view(torch.uint8), x.view(torch.uint8))
    del v


@pytest.mark.parametrize("strategy", ["infless_plus", "faastube_star", "deepplan_plus"])
def test_baseline_strategies_bit_exact(strategy):
    from paper_2411_01830_b200.tube import FaaSTube
    t = FaaSTube(strategy)
    x = payload(9, (8, 1024, 1024))
    did = t.unique_id()
    t.store(did, x)
    got = t.fetch(did, device=0, out=torch.empty_like(x))
    torch.cuda.synchronize()
    assert np.array_equal(as_u8(got), oracle_bytes(x))
    t.close()


def test_multi_hop_relay_chain(tube):
    """The store-and-forward relay of non-uniform fabrics (each hop pulled by
    its receiving GPU on its own stream, chained by events, private buffers
    kept alive until the last hop lands) — driven on one GPU with 3 hops."""
    n = (24 << 20) + 333
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    dst = torch.zeros_like(src)
    s = torch.cuda.current_stream(0)
    tube._relay([(0, 0), (0, 0), (0, 0)], src.data_ptr(), dst.data_ptr(), n, s)
    assert len(tube._keepalive) >= 1
    digest = dst.to(torch.int64).sum()          # ordered after the last hop on the consumer stream
    torch.cuda.synchronize()
    assert torch.equal(dst, src)
    assert int(digest) == int(src.to(torch.int64).sum())
    tube.maintain()
    assert not tube._keepalive


def test_fetch_many_batched_handoff(tube):
    """fetch_many: same-GPU objects in one batched copy, others (a host object)
    through fetch — all bytes exact, objects retired."""
    xs = [torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0") for n in (1, 4097, 1 << 20, 3 << 20)]
    ids = []
    for x in xs:
        d = tube.unique_id()
        tube.store(d, x, producer="p")
        ids.append(d)
    h = torch.randint(0, 256, (12345,), dtype=torch.uint8).pin_memory()
    hd = tube.unique_id()
    tube.store(hd, h, producer="gw")
    outs = [torch.empty_like(x) for x in xs] + [torch.empty(12345, dtype=torch.uint8, device="cuda:0")]
    got = tube.fetch_many(list(zip(ids + [hd], outs)), consumer="c")
    torch.cuda.synchronize()
    for x, o in zip(xs, got):
        assert torch.equal(x, o)
    assert torch.equal(got[-1].cpu(), h)
    for d in ids + [hd]:
        assert d not in tube._objs


def test_fetch_many_repeated_and_pinned_objects():
    """fetch_many with an object listed twice (its two consumers in one batch) and a
    last consumer of an object a zero-copy view still pins: bytes exact, each block
    returned to the pool exactly once (the view's release frees the pinned one)."""
    from paper_2411_01830_b200.tube import FaaSTube
    t = FaaSTube("faastube", pool_floor_bytes=0.0, gpus=[0])
    x = torch.randint(0, 256, (3 << 20,), dtype=torch.uint8, device="cuda:0")
    y = torch.randint(0, 256, (5 << 20,), dtype=torch.uint8, device="cuda:0")
    torch.cuda.synchronize()
    in_use0 = t.pools[0].policy.in_use_bytes
    dx, dy = t.unique_id(), t.unique_id()
    t.store(dx, x, consumers=2)
    t.store(dy, y, consumers=2)
    view = t.fetch(dy, device=0)                       # first consumer of y: a view (pins it)
    o1, o2, o3 = torch.empty_like(x), torch.empty_like(x), torch.empty_like(y)
    t.fetch_many([(dx, o1), (dx, o2), (dy, o3)])
    torch.cuda.synchronize()
    assert torch.equal(o1, x) and torch.equal(o2, x) and torch.equal(o3, y) and torch.equal(view, y)
    assert dx not in t._objs and dy not in t._objs
    del view
    import gc
    gc.collect()
    torch.cuda.synchronize()
    assert t.pools[0].policy.in_use_bytes == in_use0
    assert t._accounts_consistent()
    t.close()


def test_managed_response_and_host_fetch():
    """With the PCIe scheduler, responses and GPU->host fetches are managed
    GPU->host stages (engine.py:414-423, 537-575) — bytes exact, caller's
    pinned or pageable output."""
    from paper_2411_01830_b200.tube import FaaSTube
    t = FaaSTube("faastube", pool_floor_bytes=0.0)
    x = torch.randint(0, 256, ((12 << 20) + 5,), dtype=torch.uint8, device="cuda:0")
    before = t.pacer.stats()["managed_stages"]
    d = t.unique_id()
    t.store(d, x, producer="sink", response=True)
    assert torch.equal(t.response(d), x.cpu())
    t.release(d)
    for out in (None, torch.empty(x.numel(), dtype=torch.uint8).pin_memory(), torch.empty(x.numel(), dtype=torch.uint8)):
        d = t.unique_id()
        t.store(d, x, producer="p")
        got = t.fetch(d, device=None, out=out)
        assert torch.equal(got.reshape(-1).view(torch.uint8), x.cpu())
    assert t.pacer.stats()["managed_stages"] == before + 4
    t.close()


def test_inter_gpu_paths_on_one_gpu(tube):
    """The cross-GPU fetch executor driven on one GPU with hand-built plans
    (src == dst GPU): a striped GPU-oriented plan (a direct NVLink-pull branch
    and a 2-hop relay branch, fractional shares) and the host-oriented
    two-stage plan (D2H then H2D, dataplane.py:265-272) — bytes exact, source
    block fenced by its readers."""
    from types import SimpleNamespace
    from paper_2411_01830_b200.dataplane import Branch, Location, Stage
    n = (20 << 20) + 123
    x = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    for stages in ([Stage([Branch([("nv", 0, 0)], n * 0.37), Branch([("nv", 0, 0), ("nv", 0, 0)], n * 0.63)])],
                   [Stage([Branch([("d2h", 0, 0)], float(n))]), Stage([Branch([("h2d", 0, 0)], float(n))])]):
        d = tube.unique_id()
        tube.store(d, x, producer="p")
        obj = tube._objs[d]
        plan = SimpleNamespace(method="inter_gpu", stages=stages, claimed_func=None)
        out = torch.zeros_like(x)
        with tube._lock:
            res = tube._inter_gpu(obj, plan, Location(0, 0), Location(0, 0), out)
        digest = res.to(torch.int64).sum()        # ordered after the transfer on the consumer stream
        torch.cuda.synchronize()
        assert torch.equal(res, x) and int(digest) == int(x.to(torch.int64).sum())
        assert obj.readers                        # the source block is fenced by the pull / D2H
        tube.release(d)
    tube.maintain()


def test_full_size_round_trips():
    """BASELINE sizes through the public API: a 1 GiB host payload (config 2)
    host -> GPU (managed pacer stage) -> store -> GPU -> host (managed d2h stage)
    comes back bit-identical, and the device digest of the GPU copy equals the
    host digest of the payload; the 64 MiB config-1 pass copy-fetch and
    zero-copy view carry the same digest."""
    from paper_2411_01830_b200 import device as dev
    from paper_2411_01830_b200.tube import FaaSTube
    t = FaaSTube("faastube", pool_floor_bytes=0.0, capacity_limit_bytes=64e9)
    n = 1 << 30
    host = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0").cpu().pin_memory()
    d = t.unique_id()
    t.store(d, host, producer="gateway")
    g = t.fetch(d, device=0, consumer="f")                        # H2G
    fp = dev.Fingerprint(0)
    fp.launch(g.data_ptr(), n, torch.cuda.current_stream(0))
    assert fp.value() == dev.fingerprint_host(host)
    d2 = t.unique_id()
    t.store(d2, g, producer="f")
    back = torch.empty(n, dtype=torch.uint8).pin_memory()
    t.fetch(d2, device=None, out=back, consumer="sink")           # D2H
    assert torch.equal(back, host)
    x = payload(3)                                                # config 1: 64 MiB fp16
    want = dev.fingerprint_host(x.cpu())
    for zero_copy in (False, True):
        d3 = t.unique_id()
        t.store(d3, x, producer="p")
        y = t.fetch(d3, device=0) if zero_copy else t.fetch(d3, out=torch.empty_like(x))
        fp.launch(y.data_ptr(), y.nbytes, torch.cuda.current_stream(0))
        assert fp.value() == want
        del y
    assert t._accounts_consistent()
    t.close()


def _edge_payloads():
    g = torch.Generator(device="cpu").manual_seed(11)
    special = torch.tensor([float("nan"), float("inf"), -float("inf"), -0.0, 0.0, 65504.0, 6e-8, 1.0],
                           dtype=torch.float16)
    nan_payloads = torch.cat([special, torch.randn(4093, generator=g).half()])
    nan_bits = torch.randint(0, 1 << 16, (4097,), generator=g, dtype=torch.int32).to(torch.int16).view(torch.float16)
    return {
        "empty": torch.empty(0, dtype=torch.float16),
        "empty_3d": torch.empty(3, 0, 5, dtype=torch.int32),
        "fp16_specials": nan_payloads,
        "fp16_any_bits": nan_bits,                   # signalling/quiet NaNs of every payload
        "bool_odd": torch.rand(1001, generator=g) > 0.5,
        "int8_ragged": torch.randint(-128, 128, (7, 13, 3), generator=g, dtype=torch.int8),
        "transposed": torch.randn(64, 48, generator=g).t(),     # non-contiguous producer output
    }


@pytest.mark.parametrize("name", list(_edge_payloads()))
def test_edge_payloads_every_path(tube, name):
    """Empty, ragged, non-contiguous and NaN-carrying payloads through every
    path (GPU copy-fetch, zero-copy view, GPU -> host, host -> GPU): the bytes
    equal the oracle host path's as uint8 (so NaN bit patterns count)."""
    src = _edge_payloads()[name]
    want = oracle_bytes(src.contiguous()) if src.numel() else np.empty(0, dtype=np.uint8)
    x = src.to("cuda:0")
    # GPU producer: copy-fetch, zero-copy view and host fetch of one object
    did = tube.unique_id()
    tube.store(did, x, producer="p", consumers=3)
    a = tube.fetch(did, device=0, out=torch.empty(x.shape, dtype=x.dtype, device="cuda:0"), consumer="c")
    b = tube.fetch(did, device=0, consumer="c")
    h = tube.fetch(did, device=None, consumer="c")
    torch.cuda.synchronize()
    for got in (a, b, h):
        assert got.shape == src.shape and got.dtype == src.dtype
        assert np.array_equal(as_u8(got), want), name
    del b
    # host producer (cFunc output) -> GPU consumer
    hid = tube.unique_id()
    tube.store(hid, src.contiguous(), producer="decode")
    g = tube.fetch(hid, device=0, consumer="c")
    torch.cuda.synchronize()
    assert g.shape == src.shape and np.array_equal(as_u8(g), want), name


def test_object_larger_than_4gib_same_gpu():
    """5 GiB + 4097 B through store (snapshot copy) and fetch (copy into the input
    buffer): byte offsets past 2^32 in the copy kernels, digest-checked against
    the producer tensor and spot-checked at the tail."""
    from paper_2411_01830_b200 import device as dev
    from paper_2411_01830_b200.tube import FaaSTube
    t = FaaSTube("faastube", pool_floor_bytes=0.0, capacity_limit_bytes=64e9)
    n = (5 << 30) + 4097
    x = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    x.view(-1)[: n // 8 * 8].view(torch.int64).copy_(torch.arange(n // 8, device="cuda:0") * 0x9E3779B97F4A7C15)
    x[n // 8 * 8:] = 0xA5
    fp = dev.Fingerprint(0)
    fp.launch(x.data_ptr(), n, torch.cuda.current_stream(0))
    want = fp.value()
    did = t.unique_id()
    t.store(did, x, producer="p")
    y = t.fetch(did, device=0, out=torch.empty_like(x), consumer="c")
    fp.launch(y.data_ptr(), n, torch.cuda.current_stream(0))
    assert fp.value() == want
    assert torch.equal(y[-(1 << 20):], x[-(1 << 20):])
    del x, y
    assert t._accounts_consistent()
    t.close()


def _spin(ms, stream):
    import ctypes as C
    from paper_2411_01830_b200 import device as dev
    dev.LIB.ft_spin_ns(int(ms * 1e6), 0, C.c_void_p(stream.cuda_stream))


@pytest.mark.parametrize("batched", [False, True])
def test_early_consumer_read_fences_block_reuse(batched):
    """Two consumers copy the same object into their inputs on different
    streams. The first one's copy is still queued (its stream is busy) when the
    second, last consumer retires the object and a new store reuses the block:
    the reuse must wait for the first consumer's read (the read of a
    consumer that is not the last one is a fence of the block)."""
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube("faastube", pool_floor_bytes=0.0, gpus=[0])
    x = torch.randint(0, 256, (8 * MB,), dtype=torch.uint8, device="cuda:0")
    y = torch.randint(0, 256, (8 * MB,), dtype=torch.uint8, device="cuda:0")
    a, b = torch.cuda.Stream(0), torch.cuda.Stream(0)
    out_a, out_b = torch.empty_like(x), torch.empty_like(x)
    torch.cuda.synchronize()
    did = tube.unique_id()
    tube.store(did, x, consumers=2)
    with torch.cuda.stream(a):
        _spin(50, a)                                  # consumer A's stream is busy for 50 ms
        if batched:
            tube.fetch_many([(did, out_a)])
        else:
            tube.fetch(did, device=0, out=out_a)
    with torch.cuda.stream(b):
        tube.fetch(did, device=0, out=out_b)          # last consumer: retires, the block is free
        did2 = tube.unique_id()
        tube.store(did2, y)                           # same size class: reuses (overwrites) the block
    torch.cuda.synchronize()
    assert torch.equal(out_a, x) and torch.equal(out_b, x)
    got = tube.fetch(did2, device=0, out=torch.empty_like(y))
    torch.cuda.synchronize()
    assert torch.equal(got, y)
    assert tube._accounts_consistent()
    tube.close()


def test_event_unrecorded_is_refused():
    """A pooled event handle carries its previous record: an Ev that was never
    recorded must not be waited on (it would report unrelated work done)."""
    from paper_2411_01830_b200 import device as dev
    e = dev.Ev(0)
    with pytest.raises(RuntimeError):
        e.wait(torch.cuda.current_stream(0))
    with pytest.raises(RuntimeError):
        e.query()
    e.record(torch.cuda.current_stream(0))
    e.synchronize()
    assert e.query()

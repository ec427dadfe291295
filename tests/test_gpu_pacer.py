"""GPU parity of the native PCIe mover / bandwidth-share scheduler (ft_pacer,
include/faastube.h) through the C ABI: every stage delivers exactly the host
bytes — direct and staged routes (the staging + NVLink-forward path is forced
on one GPU), pinned and pageable sources (shared pinned ring), managed and
unmanaged, ragged and empty routes — with host-non-blocking stream semantics,
and its live arbiter calls replay through the oracle to the same decisions
(engine.py:537-646)."""

import json
import threading
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
MB = 10**6


@pytest.fixture(scope="module")
def dev():
    from paper_2411_01830_b200 import device
    device.require_cuda()
    return device


def host_bytes(n, seed, pinned=True):
    t = torch.from_numpy(np.random.default_rng(seed).integers(0, 256, n, dtype=np.uint8))
    return t.pin_memory() if pinned else t


def routes_for(n, kinds, streams, align=256):
    """kinds: per route 'd' (direct) or 's' (forced staging); equal shares."""
    k = len(kinds)
    bounds = [0] + [min(n, (n * (i + 1) // k) // align * align) for i in range(k - 1)] + [n]
    out = []
    for i, kind in enumerate(kinds):
        ce, fw = streams[i]
        out.append((0, int(kind == "s"), bounds[i], bounds[i + 1] - bounds[i], ce.cuda_stream, fw.cuda_stream))
    return out


@pytest.mark.parametrize("managed", [False, True])
@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("n,kinds", [(1, "d"), (4097, "ds"), ((32 << 20) + 777, "dss"), (3 * MB, "s"),
                                     (25 * MB + 5, "sd"), (0, "d")])
def test_stage_bit_exact(dev, managed, pinned, n, kinds):
    p = dev.Pacer(55.0, 5, 2 * MB, staging_slots=3, host_ring_bytes=8 * MB)
    streams = [(torch.cuda.Stream(0), torch.cuda.Stream(0)) for _ in kinds]
    host = host_bytes(n, n % 97, pinned)
    dst = torch.zeros(max(n, 1), dtype=torch.uint8, device="cuda:0")
    s = torch.cuda.current_stream(0)
    t = p.submit("", managed, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, pinned,
                 routes_for(n, kinds, streams), s.cuda_stream)
    # stream semantics: a kernel issued after submit on the consumer stream sees the bytes
    digest = dst[:n].to(torch.int64).sum() if n else None
    torch.cuda.synchronize()
    p.wait(t, 5000.0)                        # landing is reported by the host callback
    assert torch.equal(dst[:n].cpu(), host)
    if n:
        assert int(digest) == int(host.to(torch.int64).sum())
    st = p.stats()
    assert st["failed"] == 0 and st["active"] == 0 and st["managed_stages"] == int(managed)
    p.close()


@pytest.mark.parametrize("k2", ["0", "1"])
def test_concurrent_stages_share_staging_ring(dev, k2, monkeypatch):
    """Several tenants' staged routes through one staging GPU ring, each on its
    own stream pair: slots are reused only after their forward drained them
    (event chain and K2)."""
    monkeypatch.setenv("FT_K2", k2)
    p = dev.Pacer(55.0, 5, 2 * MB, staging_slots=2, host_ring_bytes=8 * MB)
    n = 24 * MB + 333
    payload = [host_bytes(n, 100 + i, pinned=i % 2 == 0) for i in range(6)]
    outs = [torch.zeros(n, dtype=torch.uint8, device="cuda:0") for _ in payload]
    errs = []

    def run(i):
        try:
            s = torch.cuda.Stream(0)
            pairs = [(torch.cuda.Stream(0), torch.cuda.Stream(0)) for _ in range(2)]
            p.submit("", i % 3 != 0, 1e9, 0.0, 55.0, outs[i].data_ptr(), 0, payload[i].data_ptr(), n,
                     payload[i].is_pinned(), routes_for(n, "ss", pairs), s.cuda_stream)
            s.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(payload))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not errs
    for i in range(len(payload)):
        assert torch.equal(outs[i].cpu(), payload[i]), i
    p.close()


def test_submit_returns_before_landing(dev):
    """A 512 MB managed stage (~10 ms on one PCIe link): submit returns once the
    last batch is issued — the tail is still in flight — and the consumer
    stream is ordered after the last byte."""
    p = dev.Pacer(55.0, 5, 2 * MB)
    n = 512 * MB
    host = host_bytes(n, 7)
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
    s = torch.cuda.current_stream(0)
    ce, fw = torch.cuda.Stream(0), torch.cuda.Stream(0)
    torch.cuda.synchronize()
    t = p.submit("m1", True, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True,
                 [(0, 0, 0, n, ce.cuda_stream, fw.cuda_stream)], s.cuda_stream)
    in_flight = not p.done(t)
    tail = dst[-4096:].clone()               # ordered after the stage on the consumer stream
    p.wait(t)
    torch.cuda.synchronize()
    assert in_flight
    assert torch.equal(tail.cpu(), host[-4096:])
    assert torch.equal(dst.cpu(), host)
    assert p.stats()["batches"] == -(-n // (10 * MB))
    p.close()


def test_live_decisions_replay_through_oracle(dev):
    """Every arbiter call the live pacer made (start / boundary / finish at its
    own clock) replayed through the oracle restatement gives the same decisions."""
    from oracle.stage_arbiter import Arbiter as Oracle
    p = dev.Pacer(55.0, 5, 2 * MB, logging=True)
    n = [200 * MB, 60 * MB, 120 * MB]
    slo = [(400.0, 5.0), (12.0, 2.0), (1e9, 0.0)]
    hosts = [host_bytes(x, 20 + i) for i, x in enumerate(n)]
    dsts = [torch.empty(x, dtype=torch.uint8, device="cuda:0") for x in n]
    for i in range(3):
        s = torch.cuda.Stream(0)
        ce, fw = torch.cuda.Stream(0), torch.cuda.Stream(0)
        p.submit(f"m{i}", True, slo[i][0], slo[i][1], 55.0, dsts[i].data_ptr(), 0, hosts[i].data_ptr(), n[i],
                 True, [(0, 0, 0, n[i], ce.cuda_stream, fw.cuda_stream)], s.cuda_stream)
        time.sleep(0.002)
    torch.cuda.synchronize()
    deadline = time.time() + 10
    while p.stats()["active"] and time.time() < deadline:
        time.sleep(0.01)
    log = p.log()
    calls = [e[1] for e in log]
    assert calls.count("start") == 3 and calls.count("finish") == 3
    o = Oracle(55.0, 5, 2 * MB)
    sizes = dict(zip(("m0", "m1", "m2"), n))
    slos = dict(zip(("m0", "m1", "m2"), slo))
    for t, call, key, want, arg in log:
        if call == "start":                      # arg: the per-branch cap the pacer used
            got = o.start(t, key, float(sizes[key]), slos[key][0], slos[key][1], t, arg, 1)
        elif call == "bw":                       # the live link estimator re-partitioned
            got = o.set_bw(t, arg, float(key))
        elif call == "boundary":
            got = o.boundary(t, key)
        else:
            got = o.finish(t, key)
        assert json.loads(json.dumps([list(d) for d in got])) == want, (t, call, key, got, want)
    for i in range(3):
        assert torch.equal(dsts[i].cpu(), hosts[i])
    p.close()


def test_back_to_back_loose_stages_do_not_starve(dev):
    """Reference defect A2: a stage admitted at its ~0 least
    rate while another drains re-arms its boundary hours away, so the idle
    bandwidth it is handed later never applies. The live guard applies the
    increase within two batches: back-to-back loose fetches (the bench's
    pattern) finish at link speed."""
    p = dev.Pacer(50.0, 5, 2 * MB, logging=True)
    n = 256 * MB
    hosts = [host_bytes(n, 40 + i) for i in range(3)]
    dsts = [torch.empty(n, dtype=torch.uint8, device="cuda:0") for _ in hosts]
    s = torch.cuda.current_stream(0)
    t0 = time.perf_counter()
    tickets = []
    for i in range(3):
        ce, fw = torch.cuda.Stream(0), torch.cuda.Stream(0)
        tickets.append(p.submit(f"b{i}", True, 1e9, 0.0, 50.0, dsts[i].data_ptr(), 0, hosts[i].data_ptr(), n,
                                True, [(0, 0, 0, n, ce.cuda_stream, fw.cuda_stream)], s.cuda_stream))
    for t in tickets:
        p.wait(t, 20000.0)
    elapsed = time.perf_counter() - t0
    torch.cuda.synchronize()
    for i in range(3):
        assert torch.equal(dsts[i].cpu(), hosts[i])
    assert elapsed < 3 * n * 3 / 10e9 + 1.0, elapsed     # >= 10 GB/s on any box (link 20-57 GB/s seen)
    p.close()


@pytest.mark.parametrize("adapt", [True, False])
def test_link_estimator_corrects_a_low_calibration(dev, adapt):
    """Created believing the link does 8 GB/s, the pacer measures the service
    rate of its uncontended batches and re-partitions at the real rate (a
    logged "bw" call); with the estimator off it paces at 8 GB/s."""
    p = dev.Pacer(8.0, 5, 2 * MB, logging=True, adapt=adapt)
    n = 512 * MB
    host = host_bytes(n, 9)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    s = torch.cuda.current_stream(0)
    ce, fw = torch.cuda.Stream(0), torch.cuda.Stream(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = p.submit("m1", True, 1e9, 0.0, 1e9, dst.data_ptr(), 0, host.data_ptr(), n, True,
                 [(0, 0, 0, n, ce.cuda_stream, fw.cuda_stream)], s.cuda_stream)
    p.wait(t, 20000.0)
    ms = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    assert torch.equal(dst.cpu(), host)
    bws = [e[4] for e in p.log() if e[1] == "bw"]
    if adapt:
        assert bws and bws[-1] > 15.0, bws
        assert ms < 0.7 * n / 8e6, (ms, bws)
    else:
        assert not bws and ms > 0.9 * n / 8e6, ms
    p.close()


@pytest.mark.parametrize("managed", [False, True])
@pytest.mark.parametrize("n,kinds", [(1, "d"), ((8 << 20) + 77, "ds"), (5 * MB + 3, "s")])
def test_d2h_stage_bit_exact(dev, managed, n, kinds):
    """GPU -> pinned host stages (responses, host fetches): direct routes out of the
    source GPU's root and staged routes (forward kernel into the staging ring, CE
    out of it — forced on one GPU), paced by the d2h arbiter."""
    p = dev.Pacer(55.0, 5, 2 * MB, staging_slots=3, logging=True)
    streams = [(torch.cuda.Stream(0), torch.cuda.Stream(0)) for _ in kinds]
    src = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda:0")
    host = torch.zeros(n, dtype=torch.uint8).pin_memory()
    s = torch.cuda.current_stream(0)
    t = p.submit_d2h("d1" if managed else "", managed, 1e9, 0.0, 55.0, host.data_ptr(), src.data_ptr(), 0, n,
                     routes_for(n, kinds, streams), s.cuda_stream)
    p.wait(t, 5000.0)
    assert torch.equal(host, src.cpu())
    calls = [e[1] for e in p.log()]
    assert (calls.count("d2h:start"), calls.count("d2h:finish")) == ((1, 1) if managed else (0, 0)), calls
    assert "start" not in calls
    p.close()


def test_startup_calibration_matches_the_link(dev):
    """measure_pcie_gbps (the pacer's start-up link rate) reads a buffer the CPU
    never wrote: within 10 % of a 1 GiB copy from a cold pinned buffer, run
    after a host write that would have dragged a dirty-buffer calibration to
    ~21 GB/s on these hosts (profiles/r01/diag_calib.txt)."""
    from paper_2411_01830_b200.tube import measure_pcie_gbps
    scratch = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
    scratch.fill_(3)                                   # the CPU just wrote pinned memory
    got = measure_pcie_gbps([0])
    n = 1 << 30
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    s = torch.cuda.Stream(0)
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, 0, s)
        b.record(s)
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    link = n / (best * 1e-3) / 1e9
    assert got > 0.9 * link, (got, link)


@pytest.mark.parametrize("k2", ["1", "0"])
@pytest.mark.parametrize("managed", [False, True])
def test_k2_forward_aliased_streams_and_misaligned_dst(dev, managed, k2, monkeypatch):
    """K2 (device flags between the CE legs and one forward kernel per batch):
    the route's CE and forward streams may be the SAME stream (torch's stream
    pool aliases), the destination may be misaligned, and a route longer than
    the ring cycles every slot several times — still bit-exact."""
    monkeypatch.setenv("FT_K2", k2)
    p = dev.Pacer(55.0, 5, 2 * MB, staging_slots=2, host_ring_bytes=8 * MB)
    n = 40 * MB + 13
    host = host_bytes(n, 7)
    buf = torch.zeros(n + 16, dtype=torch.uint8, device="cuda:0")
    dst = buf[3:3 + n]                                   # 3 bytes off the 16-byte grid
    one = torch.cuda.Stream(0)
    routes = [(0, 1, 0, n, one.cuda_stream, one.cuda_stream)]
    s = torch.cuda.current_stream(0)
    t = p.submit("", managed, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True, routes, s.cuda_stream)
    torch.cuda.synchronize()
    p.wait(t, 10000.0)
    assert torch.equal(dst.cpu(), host)
    assert int(buf[:3].sum()) == 0 and int(buf[3 + n:].sum()) == 0
    assert p.stats()["failed"] == 0
    p.close()


def test_k2_matches_event_chain(dev, monkeypatch):
    """The K2 forward and the previous per-piece event chain (FT_K2=0) deliver
    the same bytes for the same staged stage."""
    n = (24 << 20) + 4097
    host = host_bytes(n, 11)
    outs = []
    for k2 in ("1", "0"):
        monkeypatch.setenv("FT_K2", k2)
        p = dev.Pacer(55.0, 5, 2 * MB, staging_slots=3, host_ring_bytes=8 * MB)
        streams = [(torch.cuda.Stream(0), torch.cuda.Stream(0)) for _ in range(2)]
        dst = torch.zeros(n, dtype=torch.uint8, device="cuda:0")
        s = torch.cuda.current_stream(0)
        t = p.submit("", True, 1e9, 0.0, 55.0, dst.data_ptr(), 0, host.data_ptr(), n, True,
                     routes_for(n, "ss", streams), s.cuda_stream)
        torch.cuda.synchronize()
        p.wait(t, 10000.0)
        outs.append(dst.cpu())
        p.close()
    assert torch.equal(outs[0], host) and torch.equal(outs[1], host)

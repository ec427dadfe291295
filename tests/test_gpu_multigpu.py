"""Cross-device parity on real peers: every test
here needs >= 2 visible GPUs and skips with the reason on a 1-GPU box (the
single-GPU stand-ins of the same executors live in test_gpu_tube.py and
test_gpu_pacer.py). What runs for real here and nowhere else:

* cuMemSetAccess for a real peer at pool-block map time (device.cu grant_access)
  and cudaDeviceEnablePeerAccess (tube.py) — a block written on GPU 0 read by a
  kernel running on GPU 1;
* K1 peer pulls (k_copy_vec over the VMM peer mapping) through
  FaaSTube.store(GPU i) -> fetch(device=j, out=), every ordered pair, ragged sizes;
* config 2's striped host->GPU stage through a real staging GPU (CE into GPU 1's
  ring, NVLink forward into GPU 0), both forward implementations (event chain, K2);
* the staged GPU->host route (NVLink pull into the staging GPU's ring, out of its root);
* the multi-hop relay across 3 GPUs;
* concurrent disjoint pairs and fan-in into one GPU.

Bytes are compared as uint8 against the producer's tensor (byte parity is
identity)."""

import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2,
                                 reason=f"needs >= 2 GPUs with P2P (this box has {torch.cuda.device_count()})")]

MB = 1 << 20
SIZES = [1, 4095, 4096, (1 << 20) + 17, (64 << 20) + 3]


def _src(n, g, seed=0):
    gen = torch.Generator(device=f"cuda:{g}").manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, device=f"cuda:{g}", generator=gen)


def _tube(n_gpus=None, **kw):
    from paper_2411_01830_b200.topology import build_preset
    from paper_2411_01830_b200.tube import FaaSTube
    n = n_gpus or torch.cuda.device_count()
    return FaaSTube(kw.pop("strategy", "faastube"), topology=build_preset("b200", n_gpus=n, pcie_gbps=55.0),
                    gpus=list(range(n)), pool_floor_bytes=0.0, capacity_limit_bytes=64e9, **kw)


@pytest.mark.parametrize("n", SIZES)
def test_peer_pull_pair_0_1(n):
    """store on GPU 0, fetch into a buffer on GPU 1: Alg. 1 plans one direct
    NVLink path (inter_gpu), K1 pulls it; the claim is released after landing."""
    t = _tube()
    x = _src(n, 0, n % 97)
    d = t.unique_id()
    t.store(d, x)
    out = torch.zeros(n, dtype=torch.uint8, device="cuda:1")
    got = t.fetch(d, device=1, out=out)
    digest = got.to(torch.int64).sum()               # stream-ordered after the pull on GPU 1
    torch.cuda.synchronize(1)
    assert torch.equal(got.cpu(), x.cpu())
    assert int(digest) == int(x.to(torch.int64).sum().item())
    assert t.stats["bytes_nvlink"] >= n
    t.maintain()
    assert not t._pending_release                    # NVLink claim released once the copy landed
    t.close()


def test_every_ordered_pair_and_fresh_buffers():
    t = _tube()
    g = torch.cuda.device_count()
    for i in range(g):
        for j in range(g):
            if i == j:
                continue
            x = _src((3 << 20) + i * 7 + j, i, 10 * i + j)
            d = t.unique_id()
            t.store(d, x)
            y = t.fetch(d, device=j)                    # fresh buffer on GPU j
            torch.cuda.synchronize(j)
            assert y.device.index == j and torch.equal(y.cpu(), x.cpu()), (i, j)
    assert t._accounts_consistent()
    t.close()


def test_peer_write_visible_after_block_reuse():
    """A pool block of GPU 0 is read by GPU 1, retired, reused by a new store on
    GPU 0 and read by GPU 1 again: the second reader sees the new bytes (the
    reuse waited for the first pull; the peer mapping stays valid)."""
    t = _tube()
    out = torch.empty(8 * MB, dtype=torch.uint8, device="cuda:1")
    for k in range(3):
        x = _src(8 * MB, 0, 100 + k)
        d = t.unique_id()
        t.store(d, x)
        t.fetch(d, device=1, out=out)
        torch.cuda.synchronize(1)
        assert torch.equal(out.cpu(), x.cpu()), k
    assert t.pools[0].grow_events <= 2                 # the block is reused (no growth per store)
    t.close()


@pytest.mark.parametrize("k2", ["0", "1"])
@pytest.mark.parametrize("n", [(1 << 30), (24 << 20) + 5])
def test_striped_host_to_gpu_through_real_staging(n, k2, monkeypatch):
    """config 2: pinned host -> GPU 0 striped over every GPU's root; each
    non-target route lands on its staging GPU and is forwarded over NVLink."""
    monkeypatch.setenv("FT_K2", k2)
    t = _tube()
    host = _src(n, 0, 1).cpu().pin_memory()
    d = t.unique_id()
    t.store(d, host)
    before = t.stats["bytes_nvlink"]
    got = t.fetch(d, device=0, out=torch.zeros(n, dtype=torch.uint8, device="cuda:0"))
    torch.cuda.synchronize(0)
    assert torch.equal(got.cpu(), host)
    assert t.stats["bytes_nvlink"] - before > 0        # some bytes came through a staging GPU
    t.close()


def test_staged_gpu_to_host_route():
    """GPU -> host (response / host fetch) striped: the staging route pulls over
    NVLink into the staging GPU's ring and leaves by its own root."""
    t = _tube()
    x = _src((40 << 20) + 9, 0, 5)
    d = t.unique_id()
    t.store(d, x, response=True)
    assert torch.equal(t.response(d), x.cpu())
    t.close()


@pytest.mark.skipif(torch.cuda.device_count() < 3, reason="the relay chain needs >= 3 GPUs")
def test_relay_chain_across_three_gpus():
    t = _tube()
    n = (24 << 20) + 333
    src = _src(n, 0, 3)
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda:2")
    s = torch.cuda.current_stream(2)
    with t._lock:
        t._relay([(0, 1), (1, 2)], src.data_ptr(), dst.data_ptr(), n, s)
    torch.cuda.synchronize(2)
    assert torch.equal(dst.cpu(), src.cpu())
    t.close()


def test_concurrent_disjoint_pairs_and_fan_in():
    t = _tube()
    g = torch.cuda.device_count()
    plans = [[(i, i + 1) for i in range(0, g - 1, 2)], [(i, 0) for i in range(1, g)]]
    for plan in plans:
        xs = {src: _src(32 * MB + src, src, 7 + src) for src, _ in plan}
        ids = {}
        for src, _ in plan:
            ids[src] = t.unique_id()
            t.store(ids[src], xs[src])
        outs = []
        for src, dst in plan:
            st = torch.cuda.Stream(dst)
            with torch.cuda.device(dst), torch.cuda.stream(st):
                outs.append((src, dst, t.fetch(ids[src], device=dst)))
        for d in range(g):
            torch.cuda.synchronize(d)
        for src, dst, y in outs:
            assert torch.equal(y.cpu(), xs[src].cpu()), (src, dst)
    t.close()

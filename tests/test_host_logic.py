"""Host-side logic of the data path that needs no GPU: stripe byte ranges for
fractional plan shares, link-id parsing of plan branches, the CPU oracle's
byte path, and the put/get API's loud failure without a device."""

import numpy as np
import pytest


def test_stripes_cover_exactly():
    from paper_2411_01830_b200.tube import FaaSTube
    for n in (0, 1, 255, 256, 4097, 10**9 + 7, 1 << 30):
        for shares in ([1.0], [n / 3] * 3, [2.0, 1.0], [0.5, 0.25, 0.25], [1.0] * 8):
            r = FaaSTube._stripes(n, shares)
            assert len(r) == len(shares)
            assert r[0][0] == 0 and sum(m for _, m in r) == n
            for (a, m), (b, _) in zip(r, r[1:]):
                assert a + m == b and a % 256 == 0 and b % 256 == 0 or b == n


def test_branch_link_parsing():
    from paper_2411_01830_b200.tube import _hops, _staging_gpu
    assert _hops([("nvp_out", 3), ("nvp_in", 0)]) == [(3, 0)]
    assert _hops([("nv", 1, 2), ("nv", 2, 5)]) == [(1, 2), (2, 5)]
    assert _staging_gpu([("h2d", 0, 2), ("nvp_out", 2), ("nvp_in", 0)], 0) == 2
    assert _staging_gpu([("h2d", 0, 0)], 0) == 0


def test_host_path_identity_threads():
    from oracle.host_path import HostMemoryStore
    rng = np.random.default_rng(5)
    for threads in (1, 4):
        hs = HostMemoryStore(threads=threads)
        for n in (0, 1, 2 * 10**6 - 1, 2 * 10**6 + 1, 9 * 10**6):
            x = rng.integers(0, 256, n, dtype=np.uint8)
            d = hs.unique_id()
            hs.store(d, x)
            assert np.array_equal(hs.fetch(d), x)
            with pytest.raises(KeyError):
                hs.store(d, x)
        with pytest.raises(KeyError):
            hs.fetch(10**6)
        hs.close()


def test_tube_needs_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2411_01830_b200.tube import FaaSTube
    with pytest.raises(RuntimeError):
        FaaSTube()


def test_histogram_windows_match_oracle_with_eviction():
    """FuncHistogram keeps its windows sorted incrementally (one insert + one
    erase per record); p99s must equal sorted()-per-record nearest rank
    (datastore.py:32-62) through window eviction and heavy duplicates."""
    import random

    from oracle.decisions import Hist
    from paper_2411_01830_b200.datastore import FuncHistogram
    rnd = random.Random(5)
    for window in (1, 2, 7, 100, 1000):
        h, o = FuncHistogram("f", window), Hist("f", window)
        now = 0.0
        for i in range(2500 if window >= 100 else 300):
            now += rnd.choice([0.0, 0.5, 1.0, rnd.random() * 10])
            size = float(rnd.choice([0, 2e6, 4e6, rnd.randrange(0, 10**9)]))
            con = float(rnd.choice([0, 1, 2, 3, rnd.random() * 5]))
            h.record_execution(now, size, con)
            o.record(now, size, con)
            assert (h.r_window_ms, h.r_size_bytes, h.r_con) == (o.r_window, o.r_size, o.r_con), (window, i)


def test_plan_stage_accessors_match_json():
    """TransferPlan.stages (struct accessors, the request path) equals the
    stages of the plan's JSON form for every method on several topologies."""
    from paper_2411_01830_b200 import dataplane, strategies, topology
    for n in (1, 2, 8):
        topo = topology.build_preset("b200", n_gpus=n, pcie_gbps=55.0)
        for strat in ("faastube", "infless_plus"):
            m = topology.snapshot_matrix(topo)
            dp = dataplane.Dataplane(topo, strategies.strategy_preset(strat), m, 2e6)
            locs = [dataplane.Location(0, None)] + [dataplane.Location(0, g) for g in range(n)]
            for a in locs:
                for b in locs:
                    for size in (1.0, 4096.0, 64 * 2.0**20, 2.0**30):
                        fast = dp.fetch_plan(a, b, size)
                        fast.stages
                        dp.release_claim(fast)      # an inter-GPU plan claims its NVLink path
                        slow = dp.fetch_plan(a, b, size)
                        slow._full()
                        dp.release_claim(slow)
                        assert fast.stages == slow.stages, (n, strat, a, b, size)


def test_request_breakdown_accounts_every_millisecond():
    """Runtime.breakdown: dispatch delay + the reference's phases + cFunc host
    time + stores + the remainder add up to the request's latency."""
    from paper_2411_01830_b200.runtime import Record, Runtime
    r = Record(7, "traffic", arrival_ms=100.0, slo_ms=90.0, start_ms=100.4, end_ms=180.0)
    r.phases.update({"queuing": 10.0, "host_to_gfunc": 5.0, "gfunc_to_gfunc": 0.5, "compute": 40.0})
    r.extra.update({"cfunc": 12.0, "store": 3.0})
    b = Runtime.breakdown(r)
    assert b["latency_ms"] == 80.0 and b["dispatch_ms"] == 0.4
    total = b["dispatch_ms"] + sum(b["phases"].values()) + b["cfunc_ms"] + b["store_ms"] + b["unaccounted_ms"]
    assert abs(total - b["latency_ms"]) < 0.02, b
    assert b["unaccounted_ms"] == 9.1

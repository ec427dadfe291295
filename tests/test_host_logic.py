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
    from paper_2411_01830_b200.tube import _hops
    assert _hops([("nvp_out", 3), ("nvp_in", 0)]) == [(3, 0)]
    assert _hops([("nv", 1, 2), ("nv", 2, 5)]) == [(1, 2), (2, 5)]


def _staging_gpu(links, target):
    """tube.py's host->GPU staging GPU: the first GPU a branch lands on (its
    PCIe root's staging GPU), restated for the native planner's check."""
    for l in links:
        if l[0] in ("nvp_out", "nv"):
            return l[1]
    return target


@pytest.mark.parametrize("preset,strategy", [("b200", "faastube"), ("b200", "infless_plus"),
                                             ("dgx_v100", "faastube"), ("dgx_a100", "faastube"),
                                             ("quad_a10", "faastube"), ("b200", "deepplan_plus")])
def test_native_h2g_routes_match_the_plan(preset, strategy):
    """ft_h2g_routes (tube._host_to_gpu's planning step in one native call) gives
    the routes the Python restatement builds from the same plan: the plan's
    branches cut into byte ranges by FaaSTube._stripes, each route on its staging
    GPU's stream pair picked by the consumer stream's slot (no GPU needed: the
    streams are opaque handles here)."""
    import ctypes as C

    from paper_2411_01830_b200._lib import LIB, RouteC
    from paper_2411_01830_b200.dataplane import Dataplane, Location
    from paper_2411_01830_b200.strategies import strategy_preset
    from paper_2411_01830_b200.topology import build_preset, snapshot_matrix
    from paper_2411_01830_b200.tube import FaaSTube
    topo = build_preset(preset) if preset != "b200" else build_preset("b200", n_gpus=8)
    strat = strategy_preset(strategy)
    plane = Dataplane(topo, strat, snapshot_matrix(topo), 2e6)
    ref = Dataplane(topo, strat, snapshot_matrix(topo), 2e6)
    pairs = {g: [(0x1000 * (g + 1) + 16 * i, 0x9000 * (g + 1) + 16 * i) for i in range(16)] for g in topo.gpus()}
    for g, prs in pairs.items():
        LIB.ft_plane_set_pairs(plane._h, g, len(prs), (C.c_void_p * len(prs))(*[a for a, _ in prs]),
                               (C.c_void_p * len(prs))(*[b for _, b in prs]))
    routes, k, managed, cap, nv = (RouteC * 16)(), C.c_int(), C.c_int(), C.c_double(), C.c_uint64()
    for dst in topo.gpus():
        for n in (0, 1, 4096, 3 * 10**6 + 5, 1 << 30):
            stream = 0x7F3A00000000 + 0x1230 * (dst + 1) + n % 977 * 16
            LIB.ft_h2g_routes(plane._h, 0, dst, n, C.c_void_p(stream), routes, 16, C.byref(k), C.byref(managed),
                              C.byref(cap), C.byref(nv))
            plan = ref.fetch_plan(Location(0, None), Location(0, dst), n)
            st = plan.stages[0]
            br = st.branches
            ranges = FaaSTube._stripes(n, [b.bytes_share for b in br])
            slot = (stream >> 4) * 0x9E3779B1 >> 16
            want, want_nv = [], 0
            for b, (off, m) in zip(br, ranges):
                sg = _staging_gpu(b.links, dst)
                ce, fw = pairs[sg][slot % len(pairs[sg])]
                want.append((sg, m, ce, fw) if m else (sg, 0, ce, fw))
                want_nv += m if sg != dst else 0
            got = [(routes[i].stage_dev, routes[i].len, routes[i].ce_stream, routes[i].fw_stream) for i in range(k.value)]
            assert got == want, (preset, strategy, dst, n)
            offs = [routes[i].off for i in range(k.value) if routes[i].len]
            assert offs == [o for o, m in ranges if m]
            assert nv.value == want_nv
            assert bool(managed.value) == bool(strat.pcie_sched and st.managed)
            assert cap.value == min(min(b.hop_caps) for b in br)


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

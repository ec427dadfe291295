"""Queue-aware migration and prefetch on a real GPU store (SURVEY §8f row 1,
datastore.py:192-238, engine.py:685-736): over the store cap, the object
whose consumer is farthest back in the queue moves to host memory; fetches
stay bit-exact; retiring frees room and the migrated object is reloaded."""

import pytest
import torch

pytestmark = pytest.mark.gpu
MB = 1 << 20


def test_migrate_then_prefetch_bit_exact():
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube("faastube", pool_floor_bytes=0.0, capacity_limit_bytes=100 * MB)
    xs = [torch.randint(0, 256, (40 * MB,), dtype=torch.uint8, device="cuda:0") for _ in range(3)]
    ids = []
    for i, x in enumerate(xs):
        d = tube.unique_id()
        tube.store(d, x, producer="p", queue_pos=10 * (i + 1))    # consumers at queue positions 10, 20, 30
        ids.append(d)
    # 120 MB > 100 MB: the farthest-back consumer's object (queue 30) is migrated
    assert tube.stats["migrated_bytes"] == 40 * MB
    assert tube.index.resolve(ids[2], 0, 0.0)[0].location.gpu is None
    assert tube.index.resolve(ids[0], 0, 0.0)[0].location.gpu == 0
    # first consumer fetches (retires object 0) -> room -> object 2 prefetched back
    got0 = tube.fetch(ids[0], device=0, out=torch.empty_like(xs[0]))
    assert tube.stats["reload_bytes"] == 40 * MB
    assert tube.index.resolve(ids[2], 0, 0.0)[0].location.gpu == 0
    got1 = tube.fetch(ids[1], device=0, out=torch.empty_like(xs[1]))
    got2 = tube.fetch(ids[2], device=0, out=torch.empty_like(xs[2]))
    torch.cuda.synchronize()
    for g, x in zip((got0, got1, got2), xs):
        assert torch.equal(g, x)
    assert tube._accounts_consistent()
    tube.close()


def test_lru_policy_evicts_oldest():
    from paper_2411_01830_b200.strategies import strategy_preset
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(strategy_preset("faastube", migration="lru"), pool_floor_bytes=0.0,
                    capacity_limit_bytes=100 * MB)
    xs = [torch.randint(0, 256, (40 * MB,), dtype=torch.uint8, device="cuda:0") for _ in range(3)]
    ids = []
    for i, x in enumerate(xs):
        d = tube.unique_id()
        tube.store(d, x, producer="p", queue_pos=10 * (i + 1))
        ids.append(d)
    assert tube.index.resolve(ids[0], 0, 0.0)[0].location.gpu is None     # oldest stored goes first
    got = tube.fetch(ids[0], device=0, out=torch.empty_like(xs[0]))        # served from host memory
    torch.cuda.synchronize()
    assert torch.equal(got, xs[0])
    assert tube._accounts_consistent()
    tube.close()


def test_concurrent_stores_under_pressure():
    """Four tenants store 40 MB objects at once against a 100 MB store cap: the
    migration planned under the tube lock and executed outside it keeps every
    object fetchable and bit-exact, and the store accounting consistent."""
    import threading
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube("faastube", pool_floor_bytes=0.0, capacity_limit_bytes=100 * MB)
    xs = [torch.randint(0, 256, (40 * MB,), dtype=torch.uint8, device="cuda:0") for _ in range(8)]
    torch.cuda.synchronize()
    ids = [None] * len(xs)
    errs = []

    def tenant(k):
        try:
            for i in range(k, len(xs), 4):
                d = tube.unique_id()
                tube.store(d, xs[i], producer=f"p{k}", queue_pos=i)
                torch.cuda.current_stream().synchronize()
                ids[i] = d
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=tenant, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert tube.stats["migrated_bytes"] >= 4 * 40 * MB        # 320 MB stored against a 100 MB cap
    assert tube._accounts_consistent()
    assert tube._stored_on(0) <= 100 * MB                      # no in-flight victim counted twice
    for i, d in enumerate(ids):
        got = tube.fetch(d, device=0, out=torch.empty_like(xs[i]))
        torch.cuda.synchronize()
        assert torch.equal(got, xs[i]), i
    assert tube._accounts_consistent()
    tube.close()


@pytest.mark.parametrize("order", ["rising", "falling"])
def test_concurrent_stores_respect_cap(order):
    """Concurrent tenants against a 100 MB cap, with the newest stores nearest
    the queue front ("falling") or farthest ("rising"): after every store has
    returned the GPU store holds at most the cap (a plan never re-picks a
    victim another migration is already moving out), bytes stay exact."""
    import threading
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube("faastube", pool_floor_bytes=0.0, capacity_limit_bytes=100 * MB)
    xs = [torch.randint(0, 256, (40 * MB,), dtype=torch.uint8, device="cuda:0") for _ in range(12)]
    torch.cuda.synchronize()
    ids = [None] * len(xs)
    errs = []

    def tenant(k):
        try:
            for i in range(k, len(xs), 4):
                d = tube.unique_id()
                pos = i if order == "rising" else len(xs) - i
                tube.store(d, xs[i], producer=f"p{k}", queue_pos=pos)
                ids[i] = d
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=tenant, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert tube._stored_on(0) <= 100 * MB, tube._stored_on(0)
    assert tube._accounts_consistent()
    for i, d in enumerate(ids):
        got = tube.fetch(d, device=0, out=torch.empty_like(xs[i]))
        torch.cuda.synchronize()
        assert torch.equal(got, xs[i]), i
    tube.close()

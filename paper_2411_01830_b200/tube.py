"""FaaSTube put/get API on B200 — the drop-in for the reference's
data-passing path (Listing 1):

    tube = FaaSTube()                       # one per box (the daemon)
    did = tube.unique_id()                  # FaaSTube.unique_id
    tube.store(did, output, response=0)     # FaaSTube.store(index, output, response)
    x = tube.fetch(did, device=1, out=buf)  # FaaSTube.fetch(index, input)

Control decisions (index, transfer method, NVLink paths, PCIe routes and
byte shares, pool reuse/growth/shrink, per-function PCIe rates) come from
libfaastube's restatement of the reference (bit-identical to tubesim);
bytes move on real links:

* same GPU      — zero-copy view of the pool block, or one TMA-bulk copy into
                  the caller's input buffer (``out=``);
* GPU -> GPU    — SM-driven copy over NVLink (peer-mapped pool memory);
* host -> GPU   — copy-engine DMA on the target's own PCIe link plus, per
                  extra PCIe root, CE into a staging GPU and an NVLink forward
                  kernel into the target, chunk-pipelined (dataplane.py:203-250),
                  issued by the native pacer (``device.Pacer``: managed stages
                  at their bandwidth share, engine.py:537-646);
* GPU -> host   — copy-engine DMA out of the source GPU's root (plus staging
                  routes), a managed d2h stage with the PCIe scheduler
                  (responses and host fetches, engine.py:414-423);
* host-oriented strategies (infless_plus, deepplan_plus) stage GPU->GPU
  through pinned host memory, as the reference's baselines do.

Stream semantics: ``store`` orders after the producer's current stream;
``fetch`` enqueues on the consumer device's current stream, so consumer
kernels issued afterwards see the data (a host->GPU fetch returns once its
stage's last batch is issued; the consumer stream waits on the routes' last
ops). No call synchronizes the host unless the caller asks for a host tensor;
``FaaSTube.wait`` blocks until every host->GPU stage has landed.
"""

from __future__ import annotations

import collections
import heapq
import itertools
import math
import os
import struct
import threading
import time
import weakref

import torch

from . import datastore, device as dev
from .dataplane import DataIndex, Dataplane, Location
from .pcie_sched import BATCH_CHUNKS, CHUNK_BYTES, default_ring_capacity
from .strategies import Strategy, strategy_preset
from .topology import Topology, build_preset, snapshot_matrix

__all__ = ["FaaSTube"]

_ALIGN = 256  # stripe boundaries (bytes)
_L2_KEEP = 96 << 20  # stored blocks up to this size stay L2-resident (126 MB L2) for the next fetch
SHRINK_MIN_GAP_MS = 2.0
# dropped pool blocks are unmapped only after this long without a store/fetch:
# cuMemUnmap while the GPU is busy stalls every CUDA call of the process (0.3-1 s
# measured; at 1 req/s a 1 s threshold fired between requests and stalled the next
# one for 0.7 s). Until then they stay mapped, reused by growth of their class, and a
# failed physical allocation reclaims them first (memory pressure)
RECLAIM_IDLE_MS = 10000.0


class _Obj:
    __slots__ = ("did", "nbytes", "dtype", "shape", "gpu", "block", "host", "producer", "remaining", "ready",
                 "pins", "retired", "response_host", "response_event", "response_ticket", "stored_at", "home",
                 "queue_pos",
                 "readers", "__weakref__")

    def __init__(self, did, nbytes, dtype, shape, gpu, producer, consumers, now):
        self.did, self.nbytes, self.dtype, self.shape, self.gpu = did, nbytes, dtype, shape, gpu
        self.home = None       # GPU whose store holds / held it (migration target for prefetch)
        self.queue_pos = 0     # request-queue position of its next consumer (datastore.py:177)
        self.block = None      # device.PoolBlock when on a GPU
        self.host = None       # pinned host tensor when in host memory
        self.producer = producer
        self.remaining = consumers
        self.ready = None      # cuda event: bytes in place
        self.pins = 0          # live zero-copy views
        self.retired = False
        self.response_host = None
        self.response_event = None
        self.response_ticket = None  # pacer ticket of a managed GPU->host response stage
        self.stored_at = now
        self.readers = []      # events of copies on other streams/GPUs that read the block


_LANE_EV = struct.Struct("<IIqiiqQdQ")   # ft_lane_event (include/faastube.h)
_LANE_DTYPES = (torch.uint8, torch.int8, torch.int16, torch.int32, torch.int64, torch.float16, torch.bfloat16,
                torch.float32, torch.float64, torch.bool)


class FaaSTube:
    _lane = None                 # the daemon's native lane (attach_lane), if one serves this tube

    def __init__(self, strategy: str | Strategy = "faastube", topology: Topology | None = None,
                 pcie_gbps: float | str = "measure", chunk_bytes: int = CHUNK_BYTES, batch_chunks: int = BATCH_CHUNKS,
                 pool_floor_bytes: float = datastore.POOL_FLOOR_BYTES, node: int = 0, map_ms: float = 0.05,
                 gpus: list | None = None, capacity_limit_bytes: float = datastore.CAPACITY_LIMIT_BYTES):
        n = dev.require_cuda()
        if topology is None and pcie_gbps == "measure":
            # the link share the pacer hands out must be the link this box really has
            # (the measured pinned-H2D rate is the PCIe roofline)
            pcie_gbps = measure_pcie_gbps(list(gpus) if gpus is not None else list(range(n)))
        self.topo = topology or build_preset("b200", n_gpus=n, pcie_gbps=float(pcie_gbps))
        if self.topo.gpu_count > n:
            raise ValueError(f"topology has {self.topo.gpu_count} GPUs but only {n} are visible")
        self.strategy = strategy_preset(strategy) if isinstance(strategy, str) else strategy
        self._gpu_store = bool(self.strategy.gpu_store())
        self._so_cache = {}          # (gpu, raw stream pointer) -> torch stream object
        self.node = node
        self.chunk_bytes, self.batch_chunks = int(chunk_bytes), int(batch_chunks)
        self.matrix = snapshot_matrix(self.topo)
        self.plane = Dataplane(self.topo, self.strategy, self.matrix, float(chunk_bytes), map_ms)
        self.index = DataIndex()
        self.gpus = list(gpus) if gpus is not None else self.topo.gpus()   # GPUs this process drives
        for a in self.gpus:
            for b in self.gpus:
                if a != b and self.topo.nvlink_gbps(a, b) > 0:
                    try:
                        dev.LIB.ft_peer_enable(a, b)
                    except Exception:  # noqa: BLE001 - fabric without P2P: plans avoid NVLink
                        pass
        self.pools = {}
        if self.strategy.gpu_store():
            for g in self.gpus:
                self.pools[g] = dev.DevicePool(g, self.strategy.pool, pool_floor_bytes)
        roots = self.topo.roots()
        bw_all = self.topo.pcie_gbps * len(roots)  # engine.py:186-190
        # every host->GPU leg goes through the native pacer (managed stages paced at
        # their share; pageable payloads staged through its warm pinned ring). The
        # physical ring is twice the reference's modelled warm capacity
        # (pcie_sched.py:155-162): at 1x the ring, not the 8 memcpy workers, capped a
        # pageable 1 GiB fetch at 28-42 GB/s; at 2x it runs at 44-47 GB/s
        # (profiles/r01/sweep_pageable.txt)
        self.pacer = dev.Pacer(bw_all, batch_chunks, chunk_bytes, staging_slots=4,
                               host_ring_bytes=int(os.environ.get("FT_HOST_RING_BYTES", 0)) or
                               2 * default_ring_capacity(len(roots), batch_chunks * chunk_bytes),
                               logging=bool(os.environ.get("FT_TRACE")), links=len(roots))
        self._tickets = []           # (ticket, keep-alive refs) until the stage has landed
        self.slow_stores = collections.deque(maxlen=64)   # stores over 10 ms: (alloc, locked, migrate ms, bytes)
        self._pending = set()        # ("pressure" | "prefetch", gpu): decided under the lock, run after it
        self._migrating = {}         # gpu -> bytes of migration victims being moved out
        self._off_gpu = collections.Counter()   # home gpu -> live objects migrated off it (prefetch candidates)
        self._t0 = time.perf_counter()
        self._objs: dict[int, _Obj] = {}
        self._lock = threading.RLock()
        self._ce = {g: [dev.new_stream(g) for _ in range(2)] for g in self.gpus}  # copy-engine streams
        # per-transfer CE stream pairs (PCIe leg, NVLink forward): concurrent tenants'
        # DMA must not queue FIFO behind each other on one stream
        self._ce_pairs = {g: [(dev.new_stream(g), dev.new_stream(g)) for _ in range(16)] for g in self.gpus}
        # GPU->host stages get their own pairs: a D2H op queued behind another
        # tenant's H2D batches on a shared stream would wait for them
        self._d2h_pairs = {g: [(dev.new_stream(g), dev.new_stream(g)) for _ in range(8)] for g in self.gpus}
        for g, prs in self._ce_pairs.items():        # the same pairs, for the native host->GPU planning call
            n = len(prs)
            dev.LIB.ft_plane_set_pairs(self.plane._h, g, n, (dev.C.c_void_p * n)(*[a.cuda_stream for a, _ in prs]),
                                       (dev.C.c_void_p * n)(*[b.cuda_stream for _, b in prs]))
        self._tls = threading.local()                # per-thread route arrays of that call
        self._ce_rr = itertools.count()
        self._keepalive = []         # (event, buffers) released once the event has completed
        self._last_op_ms = 0.0       # last store/fetch (idle detection for physical reclaim)
        self._live = collections.Counter()    # (producer, gpu) -> live objects (see _account)
        self._stored = collections.Counter()  # gpu -> bytes of live objects in its store
        self._pending_release = []   # (event, plan): NVLink claims held until the copy lands
        self._shrink_due = []        # heap of (due_ms, gpu)
        self._last_due = None        # the newest (due, gpu) pushed (a retire repeats its store's)
        self._managed_ids = itertools.count(1)
        self._queue = itertools.count(1)
        self._maint_cv = threading.Condition()
        self._closing = False
        self._maint = threading.Thread(target=self._maint_loop, name="faastube-shrink", daemon=True)
        self._maint.start()
        self.capacity_limit = float(capacity_limit_bytes)   # per-GPU store cap (datastore.py:19)
        self.stats = {"stores": 0, "fetches": 0, "bytes_h2d": 0, "bytes_d2h": 0, "bytes_nvlink": 0,
                      "bytes_local": 0, "zero_copy": 0, "migrated_bytes": 0, "reload_bytes": 0}

    # ------------------------------------------------------------ helpers
    def now_ms(self) -> float:
        return (time.perf_counter() - self._t0) * 1e3

    def _loc(self, gpu) -> Location:
        return Location(self.node, gpu)

    def _reap(self):
        """Release NVLink claims of transfers that have landed, and the
        keep-alive references of host->GPU stages that have landed."""
        if self._tickets:
            self._tickets = [t for t in self._tickets if not self.pacer.done(t[0])]
        if self._keepalive:
            self._keepalive = [k for k in self._keepalive if not k[0].query()]
        keep = []
        for ev, plan in self._pending_release:
            if ev.query():
                self.plane.release_claim(plan)
            else:
                keep.append((ev, plan))
        self._pending_release = keep

    def _maint_loop(self):
        """Pool shrink timer (engine.py:656-665): at last_request + R_window the
        policy drops idle blocks and their physical memory is unmapped — off the
        request path, fenced on each dropped block's own events. Live, due timers are
        coalesced to at most one shrink per GPU every SHRINK_MIN_GAP_MS: under
        a request every ~100 us, R_window is that small and a shrink per
        request would compete with the request path for the GIL."""
        last_run = -1e18
        while True:
            with self._maint_cv:
                if self._closing:
                    return
                now = self.now_ms()
                self._reclaim_if_idle(now)
                if now - last_run < SHRINK_MIN_GAP_MS:
                    self._maint_cv.wait((SHRINK_MIN_GAP_MS - (now - last_run)) / 1e3)
                    continue
                due = set()
                while self._shrink_due and self._shrink_due[0][0] <= now:
                    due.add(heapq.heappop(self._shrink_due)[1])
                if not due:
                    wait = (self._shrink_due[0][0] - now) / 1e3 if self._shrink_due else 0.1
                    if any(p.reclaimable for p in self.pools.values()):
                        wait = min(wait, RECLAIM_IDLE_MS / 1e3)
                    self._maint_cv.wait(min(0.1, max(0.001, wait)))
                    continue
            last_run = self.now_ms()
            for g in sorted(due):
                if g in self.pools:
                    # policy shrink now; physical unmap deferred to a quiet moment
                    self.pools[g].shrink(self.now_ms(), reclaim=False)

    def _reclaim_if_idle(self, now):
        """Give dropped blocks' physical memory back once no store/fetch has run
        for RECLAIM_IDLE_MS (cuMemUnmap stalls the process's CUDA calls while
        the GPU is busy; growth meanwhile reuses parked blocks of its class)."""
        if now - self._last_op_ms >= RECLAIM_IDLE_MS:
            for p in self.pools.values():
                if p.reclaimable or p.stats()["mapped_bytes"] > p.reserved_bytes:
                    p.reclaim()

    @staticmethod
    def _stream(g) -> int:
        """Raw pointer of the caller's current stream on GPU ``g``."""
        return dev.current_stream(g)

    def _torch_stream(self, g):
        """The caller's current stream on GPU ``g`` as a torch stream object (for
        ``record_stream``), cached by raw pointer (building one costs ~1.5 us)."""
        key = (g, dev.current_stream(g))
        st = self._so_cache.get(key)
        if st is None:
            st = self._so_cache[key] = torch.cuda.current_stream(g)
        return st

    @staticmethod
    def _stripes(nbytes, shares):
        """Integer byte ranges for fractional shares (dataplane.py:215/288)."""
        total = sum(shares)
        if total <= 0 or nbytes == 0:
            return [(0, nbytes if i == 0 else 0) for i in range(len(shares))]
        bounds = [0]
        acc = 0.0
        for s in shares[:-1]:
            acc += s
            b = int(nbytes * (acc / total)) // _ALIGN * _ALIGN
            bounds.append(max(bounds[-1], min(nbytes, b)))
        bounds.append(nbytes)
        return [(bounds[i], bounds[i + 1] - bounds[i]) for i in range(len(shares))]

    def _pinned(self, nbytes) -> torch.Tensor:
        return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)

    # ------------------------------------------------------------ API
    def unique_id(self) -> int:
        """FaaSTube.unique_id (dataplane.py:69-70)."""
        return self.index.unique_id()

    def empty(self, shape, dtype=torch.float16, device: int = 0) -> torch.Tensor:
        """An output buffer carved from the tube's pool: storing it is zero-copy."""
        nbytes = math.prod(shape) * torch.empty((), dtype=dtype).element_size()
        blk = self.pools[device].allocate(nbytes)
        blk.wait_fences(self._stream(device))      # the block's previous users are done
        t = dev.as_tensor(blk.ptr, nbytes, device, dtype, tuple(shape), owner=blk)
        t._ft_block = blk  # noqa: SLF001 - marks pool-backed outputs
        return t

    def lend_block(self, device: int, nbytes: int):
        """A pool block for an output another process writes (the daemon's
        ``alloc`` / loan): the caller waits on its ``fences`` before handing it
        out, then publishes it with ``store_block`` or gives it back with
        ``pools[device].free``."""
        return self.pools[device].allocate(nbytes)

    def store(self, data_id: int, output: torch.Tensor, response: bool = False, producer: str = "func",
              consumers: int = 1, queue_pos: int | None = None) -> None:
        """FaaSTube.store(index, output, response) — engine.py:342-423.

        ``queue_pos``: request-queue position of the object's next consumer
        (the runtime knows it; default: store order) — drives queue-aware
        migration under memory pressure (datastore.py:192-222)."""
        # pinned host buffers are allocated before taking the tube lock (cudaHostAlloc
        # can take milliseconds and must not stall other tenants' calls)
        t0 = time.perf_counter()
        pre_host = pre_blk = None
        if output.is_cuda and (response or not self._gpu_store):
            pre_host = self._pinned(output.nbytes)
        if output.is_cuda and self._gpu_store:
            fb = getattr(output, "_ft_block", None)
            if fb is None or fb.ptr != output.data_ptr():
                # the pool block for the snapshot: growth maps physical memory, which
                # must not happen under the tube lock
                pre_blk = self.pools[output.get_device()].allocate(output.nbytes)
        t1 = time.perf_counter()
        try:
            stage = self._store_locked(data_id, output, response, producer, consumers, queue_pos, pre_host, pre_blk)
        except BaseException:
            if pre_blk is not None:
                self.pools[output.get_device()].free(pre_blk, list(pre_blk.fences))
            raise
        t2 = time.perf_counter()
        self._after_store(stage)
        t3 = time.perf_counter()
        if t3 - t0 > 0.01:   # slow stores, for diagnosis: ms allocating / in the locked part / migrating, bytes
            self.slow_stores.append((round(1e3 * (t1 - t0), 2), round(1e3 * (t2 - t1), 2),
                                     round(1e3 * (t3 - t2), 2), output.nbytes))

    def _after_store(self, stage):
        """The part of a store after the tube lock: a managed GPU->host response
        stage (engine.py:414-423 -> 537-575) is paced by the d2h arbiter outside
        the lock (the object stays pinned until its block's readers include the
        stage), then the migration the store decided runs."""
        if stage is not None:
            obj, args = stage
            try:
                ticket = self.pacer.submit_d2h(*args)
                with self._lock:
                    obj.response_ticket = ticket
                    obj.readers.append(dev.Ev(obj.gpu).record(args[-1]))   # source stream waits on the routes
                    self._tickets.append((ticket, obj.response_host, None))
            finally:
                self._unpin(obj)
        if self._pending:
            self._drain_pending()                         # migration decided by this store

    def store_block(self, data_id: int, blk, nbytes: int, dtype, shape, stream, response: bool = False,
                    producer: str = "func", consumers: int = 1) -> None:
        """``store`` of a pool block another process wrote (the daemon's commit of
        a lent block): zero copy, the object's bytes ready after
        ``stream``'s current work — no tensor is built on this path."""
        pre_host = self._pinned(nbytes) if response else None
        with self._lock:
            self._reap()
            if data_id in self._objs:
                from ._lib import DuplicateStore
                raise DuplicateStore(f"data id {data_id} already stored")
            self._last_op_ms = now = self.now_ms()
            g = blk.device
            obj = _Obj(data_id, nbytes, dtype, tuple(shape), g, producer, consumers, now)
            obj.home = g
            obj.queue_pos = next(self._queue)
            stage = self._commit_block(obj, blk, dev.stream_ptr(stream), response, pre_host, now)
        self._after_store(stage)

    def _commit_block(self, obj, blk, stream: int, response, pre_host, now):
        """(lock held) Publish a pool-backed object: ``ready`` on ``stream``, index
        entry (dataplane.py:72-83) + histogram sample (datastore.py:51-62), the
        shrink timer, the response leg. Returns the response stage to submit."""
        g = obj.gpu
        obj.block = blk
        obj.ready = dev.Ev(g).record(stream)
        rw, last = self.pools[g].commit_store(self.index, obj.did, self.node, g, obj.nbytes, now, obj.producer,
                                              response, self._live[(obj.producer, g)] + 1)
        self._push_due(g, rw, last, now)
        stage = None
        if response:
            resp = self._respond(obj, pre_host)
            if resp is not None:
                obj.pins += 1                    # released once the stage is submitted
                stage = (obj, resp)
        self._objs[obj.did] = obj
        self._account(obj, 1)
        self.stats["stores"] += 1
        if self.strategy.migration != "none" and self._stored_on(g) > self.capacity_limit:
            self._pending.add(("pressure", g))          # engine.py:685-702, after the lock
        return stage

    def _store_locked(self, data_id, output, response, producer, consumers, queue_pos, pre_host, pre_blk):
        """Returns (obj, pacer.submit_d2h args) when a managed response stage must be submitted."""
        stage = None
        with self._lock:
            self._reap()
            if data_id in self._objs:
                from ._lib import DuplicateStore
                raise DuplicateStore(f"data id {data_id} already stored")
            t = output.contiguous() if not output.is_contiguous() else output
            nbytes = t.nbytes
            self._last_op_ms = now = self.now_ms()
            obj = _Obj(data_id, nbytes, t.dtype, tuple(t.shape), None, producer, consumers, now)
            obj.queue_pos = queue_pos if queue_pos is not None else next(self._queue)
            if t.is_cuda and self._gpu_store:
                g = t.get_device()
                obj.gpu = obj.home = g
                pool = self.pools[g]
                blk = getattr(t, "_ft_block", None)
                live_here = self._live[(producer, g)]     # this producer's live objects here
                if blk is not None and blk.ptr == t.data_ptr():
                    # zero-copy store of a pool-backed output
                    return self._commit_block(obj, blk, self._stream(g), response, pre_host, now)
                else:
                    blk = pre_blk                        # datastore.py:130-144 (allocated above)
                    obj.block = blk
                    # snapshot on the producer's stream: ordered after the kernels that
                    # wrote the output AND before any later kernel that overwrites it
                    so = self._torch_stream(g)
                    # stream the producer's output through L2 (evict_first); the block itself is
                    # written with the normal policy — pinning it (evict_last) for the fetch
                    # measured 5% slower per pass (tools/sweep_hints.py: 37.9 vs 35.8 us)
                    hints = dev.L2_EVICT_FIRST if nbytes <= _L2_KEEP else 0
                    obj.ready = dev.Ev(g)
                    # one native call: wait the block's previous users, copy, record `ready`,
                    # index entry (dataplane.py:72-83) + histogram sample (datastore.py:51-62)
                    rw, last = pool.store_local(self.index, data_id, self.node, nbytes, now, producer, response,
                                                live_here + 1, blk, t.data_ptr(), so.cuda_stream, hints, obj.ready)
                    t.record_stream(so)
                    self.stats["bytes_local"] += nbytes
                # the shrink timer at last_request + R_window (engine.py:656-659)
                self._push_due(g, rw, last, now)
                if response:
                    resp = self._respond(obj, pre_host)
                    if resp is not None:
                        obj.pins += 1                    # released once the stage is submitted
                        stage = (obj, resp)
            elif t.is_cuda:
                # host-oriented store: the output lands in host memory (engine.py:361-381)
                g = t.device.index
                host = pre_host
                s = self._ce[g][0]
                dev.Ev(g).record(self._stream(g)).wait(s)    # the producer's output is written
                dev.pcie_copy(host.data_ptr(), t.data_ptr(), nbytes, False, g, s)
                ev = dev.Ev(g).record(s)
                # the producer's tensor stays referenced until the D2H has read it (no
                # record_stream on a private stream: the allocator would keep its handle)
                self._keepalive.append((ev, [t]))
                obj.host, obj.ready = host, ev
                if response:                               # already in host memory
                    obj.response_host, obj.response_event = host, ev
                self.stats["bytes_d2h"] += nbytes
                self.index.store(data_id, self._loc(None), nbytes, now, producer, response)
            else:
                # cFunc output / request payload: host resident. With the PCIe scheduler
                # a pageable payload is kept as is (ownership passes to the tube) and
                # staged through the shared warm pinned ring at fetch time
                # (pcie_sched.py:122-162); other strategies pin a
                # private staging copy per object (their cold-pin behaviour).
                flat = t.reshape(-1).view(torch.uint8)
                if t.is_pinned() or self.strategy.pcie_sched:
                    host = flat
                else:
                    host = self._pinned(nbytes).copy_(flat)
                obj.host = host
                self.index.store(data_id, self._loc(None), nbytes, now, producer, response)
            self._objs[data_id] = obj
            self._account(obj, 1)
            self.stats["stores"] += 1
            if obj.block is not None and self.strategy.migration != "none" and \
                    self._stored_on(obj.gpu) > self.capacity_limit:
                self._pending.add(("pressure", obj.gpu))      # engine.py:685-702, after the lock
        return stage

    # ------------------------------------------------ queue-aware migration (§8f row 1)
    def _stored_on(self, g) -> int:
        """Bytes of live objects held in GPU g's store (kept as a running sum)."""
        return self._stored[g]

    def _accounts_consistent(self) -> bool:
        """The running counters equal a recount of the table (tests)."""
        if self._lane is not None:
            with self._lock:
                self._lane_adopt(-1)
        live, stored, off = collections.Counter(), collections.Counter(), collections.Counter()
        for o in self._objs.values():
            if o.gpu is not None:
                live[(o.producer, o.gpu)] += 1
                if o.block is not None:
                    stored[o.gpu] += o.nbytes
            if o.home is not None and o.block is None and o.host is not None:
                off[o.home] += 1
        return (+self._live == +live) and (+self._stored == +stored) and (+self._off_gpu == +off)

    def _account(self, o: _Obj, sign: int):
        """Running per-(producer, GPU) live counts and per-GPU stored bytes of the
        objects in the table (the policy's concurrency samples and the store cap
        check read them on every store instead of scanning the table)."""
        if o.gpu is not None:
            self._live[(o.producer, o.gpu)] += sign
            if o.block is not None:
                self._stored[o.gpu] += sign * o.nbytes

    def _policy_objs(self, g, movable_only=False):
        """The policy's view of GPU g's store. ``movable_only`` leaves out pinned
        objects (live zero-copy views, victims another migration is already
        moving out): their bytes are discounted by the caller, and a plan that
        picked them would be dropped by the pins filter and cover nothing."""
        from .datastore import StoredObject
        objs = sorted((o for o in self._objs.values() if o.home == g and not (movable_only and o.pins)),
                      key=lambda o: o.did)
        recs = [StoredObject(o.did, float(o.nbytes), o.producer, g, o.stored_at,
                             "gpu" if o.block is not None else "host",
                             {("c", i): o.queue_pos for i in range(max(1, o.remaining))}, not o.retired)
                for o in objs]
        return objs, recs

    def _drain_pending(self):
        """Migration (store cap exceeded) and prefetch (room freed) decided under
        the tube lock, executed after it: the victims / candidates are chosen
        and pinned under the lock, their pinned host buffers or pool blocks are
        allocated outside it (cudaHostAlloc of a 512 MB buffer or a VMM growth
        under the lock stalled every tenant's store and fetch for 40-110 ms in
        config 5), then the moves are issued under the lock again. Runs in
        the caller's thread before its store/fetch/release returns, so the
        reference's synchronous semantics hold for the caller."""
        while True:
            with self._lock:
                if not self._pending:
                    return
                kind, g = self._pending.pop()
                if kind == "pressure" and self._lane is not None:
                    self._lane_adopt(g)                   # the lane's objects on g are candidates too
                chosen = self._plan_migration(g) if kind == "pressure" else self._plan_prefetch(g)
                for o in chosen:
                    o.pins += 1
                moving = sum(o.nbytes for o in chosen) if kind == "pressure" else 0
                self._migrating[g] = self._migrating.get(g, 0) + moving   # a concurrent plan sees them gone
            if not chosen:
                continue
            bufs = []
            try:
                for o in chosen:
                    bufs.append(self._pinned(o.nbytes) if kind == "pressure" else self.pools[g].allocate(o.nbytes))
            finally:
                with self._lock:
                    self._migrating[g] -= moving
                    skipped = False
                    for i, o in enumerate(chosen):
                        o.pins -= 1
                        buf = bufs[i] if i < len(bufs) else None
                        if kind == "pressure":
                            if buf is not None and o.block is not None and o.pins == 0 and not o.retired:
                                self._migrate_out(o, buf)
                            else:
                                skipped = skipped or (o.block is not None and not o.retired)
                                self._maybe_free(o)
                        else:
                            if buf is not None and o.host is not None and o.block is None and not o.retired:
                                self._reload(o, g, buf)
                            elif buf is not None:
                                self.pools[g].free(buf, list(buf.fences))
                    if skipped and self._stored_on(g) - self._migrating.get(g, 0) > self.capacity_limit:
                        # a victim was pinned (zero-copy view) meanwhile: plan again without it
                        self._pending.add(("pressure", g))

    def _plan_migration(self, g) -> list:
        """Store cap exceeded -> the objects whose consumers sit farthest back in
        the queue go to host memory (datastore.py:192-222)."""
        stored = self._stored_on(g) - self._migrating.get(g, 0)    # minus moves already under way
        if stored <= self.capacity_limit:
            return []
        from .datastore import migration_plan
        objs, recs = self._policy_objs(g, movable_only=True)     # in-flight victims are discounted above
        try:
            plan = migration_plan(recs, stored - self.capacity_limit, self.strategy.migration)
        except Exception:  # noqa: BLE001 - HardPressure: nothing migratable (engine.py:696-697)
            return []
        by_id = {o.did: o for o in objs}
        return [by_id[rec.data_id] for action, rec in plan
                if action == "migrate" and by_id[rec.data_id].block is not None and by_id[rec.data_id].pins == 0]

    def _migrate_out(self, o: _Obj, host: torch.Tensor):
        """D2H on the GPU's own link, then the block goes back to the pool (engine.py:704-715)."""
        g = o.gpu
        ce = self._ce[g][1]
        o.ready.wait(ce)
        dev.pcie_copy(host.data_ptr(), o.block.ptr, o.nbytes, False, g, ce)
        ev = dev.Ev(g).record(ce)
        self._account(o, -1)
        blk, o.block = o.block, None
        self.pools[g].free(blk, [ev] + o.readers)            # later writers of the block wait for the D2H
        o.readers = []
        o.host, o.ready, o.gpu = host, ev, None
        self._account(o, 1)
        self._off_gpu[o.home] += 1
        self.index.relocate(o.did, self._loc(None))
        self.stats["migrated_bytes"] += o.nbytes
        self.stats["bytes_d2h"] += o.nbytes

    def _plan_prefetch(self, g) -> list:
        """Room freed -> reload migrated objects, nearest consumer first (datastore.py:225-238)."""
        if not self._off_gpu[g]:
            return []                                 # nothing migrated off this GPU
        free = self.capacity_limit - self._stored_on(g)
        if free <= 0:
            return []
        from .datastore import prefetch_back
        objs, recs = self._policy_objs(g)
        by_id = {o.did: o for o in objs}
        return [by_id[rec.data_id] for rec in prefetch_back(recs, free)
                if by_id[rec.data_id].host is not None and by_id[rec.data_id].block is None]

    def _reload(self, o: _Obj, g: int, blk):
        ce = self._ce[g][0]
        if o.ready is not None:
            o.ready.wait(ce)
        blk.wait_fences(ce)
        dev.pcie_copy(blk.ptr, o.host.data_ptr(), o.nbytes, True, g, ce)
        ev = dev.Ev(g).record(ce)
        self._account(o, -1)
        o.block, o.ready, o.gpu, o.host = blk, ev, g, None
        self._account(o, 1)
        self._off_gpu[o.home] -= 1
        self.index.relocate(o.did, self._loc(g))
        self.stats["reload_bytes"] += o.nbytes
        self.stats["bytes_h2d"] += o.nbytes

    def fetch(self, data_id: int, device: int | None = None, out: torch.Tensor | None = None,
              consumer: str = "func", slo_ms: float | None = None, infer_ms: float | None = None) -> torch.Tensor:
        """FaaSTube.fetch(index, input) — see ``_fetch``."""
        res = self._fetch(data_id, device, out, consumer, slo_ms, infer_ms)
        if self._pending:
            self._drain_pending()          # prefetch made possible by this consumer's retire
        return res

    def _fetch(self, data_id: int, device: int | None = None, out: torch.Tensor | None = None,
               consumer: str = "func", slo_ms: float | None = None, infer_ms: float | None = None) -> torch.Tensor:
        """FaaSTube.fetch(index, input) — dataplane.py:176-186 + engine.py:440-511.

        ``device=None`` fetches into host memory. With ``out`` the bytes land
        in the caller's buffer (Listing-1 semantics); without it a same-GPU
        fetch is a zero-copy view of the stored block."""
        if out is None and device is not None:
            o = self._objs.get(data_id)
            if o is not None and o.gpu != device:
                # a fresh input buffer (not a same-GPU view): allocated outside the tube
                # lock — the caching allocator can stall for milliseconds
                out = self._out(o, device, None)
        with self._lock:
            self._reap()
            obj = self._objs.get(data_id)
            if obj is None and self._lane is not None:
                obj = self._lane_take(data_id)
            self._last_op_ms = self.now_ms()
            if obj is None:
                # the index's own miss (dataplane.py:85-96): MissingData / unknown id
                self.index.resolve(data_id, self.node, self._last_op_ms)
                from ._lib import MissingData
                raise MissingData(f"data id {data_id} has no live payload")
            # where the payload lives: the index entry (dataplane.py:85-96), mirrored on
            # the object at every store / relocate, so the hot path skips the FFI lookup
            if out is not None:
                if not out.is_contiguous() or out.nbytes != obj.nbytes:
                    raise ValueError("out must be contiguous with exactly the stored byte count")
                device = out.device.index if out.is_cuda else None
            src = self._loc(obj.gpu)
            dst = self._loc(device)
            if src.node == dst.node and src.gpu is not None and src.gpu == dst.gpu:
                plan = _INTRA_GPU        # dataplane.py:184-185: same GPU -> map only (no plan object)
                if out is not None and obj.block is not None and not obj.retired:
                    self._fetch_local(obj, out)          # copy into the consumer's input: one native call
                    self.stats["fetches"] += 1
                    return out
            elif src.gpu is None and dst.gpu is not None and src.node == dst.node:
                plan = None                  # host -> GPU: planned in one native call (_host_to_gpu)
            else:
                plan = self.plane.fetch_plan(src, dst, obj.nbytes)
            h2g = plan is None or (plan.method == "host_gpu" and not dst.on_host)
            d2h = (plan is not None and plan.method == "host_gpu" and dst.on_host and obj.block is not None
                   and self.strategy.pcie_sched and plan.stages[0].managed)
            if h2g:
                res, stage = self._host_to_gpu(obj, plan, dst, out, slo_ms, infer_ms)
            elif d2h:
                # managed GPU->host fetch: into pinned memory (the caller's if pinned); the
                # object stays pinned until its block's readers include the stage
                res = out if out is not None and out.is_pinned() else self._pinned(obj.nbytes)
                stage = self._d2h_stage(obj, plan, res, consumer, slo_ms, infer_ms)
                self.stats["bytes_d2h"] += obj.nbytes
                obj.pins += 1
            else:
                res = self._execute(obj, plan, src, dst, out, slo_ms, infer_ms)
            self.stats["fetches"] += 1
            drop_after = False
            if h2g and obj.block is None:
                # the last consumer of a host object: out of the table now, its index entry
                # dropped once the stage is issued (the DMA goes out first)
                obj.remaining -= 1
                if obj.remaining <= 0:
                    drop_after = not obj.retired
                    self._retire(obj, drop=False)
            else:
                self._consumed(obj)
            if not (h2g or d2h):
                return res
        if d2h:
            # the pacer paces the stage outside the tube lock; a host result means waiting for it
            try:
                ticket = self.pacer.submit_d2h(*stage)
                with self._lock:
                    obj.readers.append(dev.Ev(obj.gpu).record(stage[-1]))  # source stream waits on the routes
            finally:
                self._unpin(obj)
            self.pacer.wait(ticket)
            if out is not None and res.data_ptr() != out.data_ptr():
                out.view(-1).view(torch.uint8).copy_(res.view(-1))
                return out
            return res.view(torch.uint8).view(obj.dtype).view(obj.shape)
        # host->GPU stage: the pacer returns once its last batch is issued — outside
        # the tube lock, so concurrent tenants' stages are paced side by side
        tl = self._tls
        rc = tl.submit(self.pacer._h, b"", *stage, tl.ticket)  # noqa: SLF001
        with self._lock:
            if rc == 0:
                self._tickets.append((tl.ticket.value, obj.host, res))
            if drop_after:
                self.index.drop(obj.did)
        if rc:
            from ._lib import raise_status
            raise_status(rc)
        return res

    def _fetch_local(self, obj: _Obj, out: torch.Tensor):
        """Same-GPU fetch into the consumer's input (dataplane.py:184-185 +
        engine.py:667-679), one native call: the consumer's stream waits for the
        stored bytes, copies them, records ``done``; the last consumer also
        drops the index entry and returns the block to the pool, fenced on
        ``done`` (its read) and every earlier reader. A consumer that is not
        the last one leaves ``done`` on the object for that retire."""
        g = obj.gpu
        blk = obj.block
        obj.remaining -= 1
        retire = obj.remaining <= 0 and obj.pins == 0
        done = dev.Ev(g)
        fences = tuple(obj.readers) + ((obj.ready,) if obj.ready is not None else ())
        rw, last = self.pools[g].fetch_local(
            self.index, obj.did, blk, obj.producer, retire, out.data_ptr(), obj.nbytes, dev.current_stream(g),
            dev.L2_EVICT_FIRST if obj.remaining <= 0 else dev.L2_NORMAL, (obj.ready,), done, fences)
        self.stats["bytes_local"] += obj.nbytes
        if not retire:
            self._hold_until(obj, done)
            if obj.remaining <= 0:
                self._retire(obj, done)                # pinned by a view: the view's release frees it
            return
        obj.retired = True
        obj.readers = []
        if self._objs.pop(obj.did, None) is not None:
            self._account(obj, -1)                     # (block still set: its bytes leave the store)
        obj.block = None
        self.index._meta.pop(obj.did, None)
        self._push_due(g, rw, last, self._last_op_ms)
        if self.strategy.migration != "none" and self._off_gpu[g]:
            self._pending.add(("prefetch", g))         # engine.py:678-679, 717-736

    def fetch_resident(self, data_id: int, device: int, consumer: str = "func", stream=None):
        """Zero-copy fetch for another process (the daemon's same-GPU path), if the
        object is stored in GPU ``device``'s pool right now: the caller's stream
        is ordered after the stored bytes, the block is pinned, and this counts
        as the consumer's fetch (dataplane.py:184-185). Decided under the tube
        lock, so a concurrent migration cannot move it in between. Returns
        (pool block, nbytes, dtype, shape, release) — ``release(stream)`` unpins
        the block once the reader is done (``stream``, default the caller's
        current one, must be ordered after the read by then). ``stream``: the
        reader's stream (default the current one). None if it lives elsewhere."""
        with self._lock:
            obj = self._objs.get(data_id)
            if obj is None and self._lane is not None:
                obj = self._lane_take(data_id)
            if obj is None or obj.gpu != device or obj.block is None:
                return None
            self._reap()
            self._last_op_ms = self.now_ms()
            s = dev.stream_ptr(stream) if stream is not None else self._stream(device)
            obj.ready.wait(s)
            obj.pins += 1
            self.stats["zero_copy"] += 1
            self.stats["fetches"] += 1
            self._consumed(obj, stream=s)
            res = (obj.block, obj.nbytes, obj.dtype, obj.shape, lambda st=None: self._unpin(obj, st))
        if self._pending:
            self._drain_pending()          # prefetch made possible by this consumer's retire
        return res

    def fetch_many(self, items, consumer: str = "func") -> list:
        """Batched fetch (an extension of Listing 1): ``[(data_id, out)]`` into
        the callers' input buffers. Every object stored on ``out``'s own GPU
        (the intra_gpu plan, dataplane.py:184-185) moves in ONE copy launch per
        64 objects, ordered after all of their stores — small handoffs pay the
        launch once; anything else goes through ``fetch``."""
        if not items:
            return []
        rest = []
        with self._lock:
            self._reap()
            self._last_op_ms = self.now_ms()
            objs = self._objs
            get = objs.get
            rest_add = rest.append
            # one pass: validate, order (newest ready record per stream), segment, and
            # count the consumer off — the last consumers' retires go after the launch
            by_gpu = {}
            last_g, grp = None, None
            for did, out in items:
                obj = get(did)
                if obj is None or obj.block is None:
                    rest_add((did, out))
                    continue
                og = obj.gpu
                if og != out.get_device() or out.nbytes != obj.nbytes or not out.is_contiguous():
                    rest_add((did, out))
                    continue
                if og != last_g:
                    grp = by_gpu.get(og)
                    if grp is None:            # keep, retire, newest ready per stream, segments, bytes
                        grp = by_gpu[og] = [[], [], {}, [], 0]
                    last_g = og
                r = obj.ready
                if r is not None:                              # (the newest record per stream covers the rest)
                    k = r.stream if r.stream is not None else id(r)
                    cur = grp[2].get(k)
                    if cur is None or r.seq > cur.seq:
                        grp[2][k] = r
                grp[3].extend((out.data_ptr(), obj.block.ptr, obj.nbytes))
                grp[4] += obj.nbytes
                obj.remaining -= 1
                if obj.remaining <= 0 and obj.pins == 0 and not obj.retired:
                    grp[1].append(obj)
                else:
                    grp[0].append(obj)
            for g, (keep, retiring, readies, flat, nb) in by_gpu.items():
                s = self._stream(g)
                dev.wait_events(s, readies.values())
                dev.copy_batch_flat(flat, g, s)
                done = dev.Ev(g).record(s)     # one fence for every block the batch read
                for o in keep:
                    o.readers.append(done)          # the last consumer's retire fences on this read
                    if o.remaining <= 0 and o.pins:
                        # a pinned last consumer (an object listed twice whose second entry
                        # retires is in `retiring`)
                        self._retire(o, done)
                self.stats["bytes_local"] += nb
                self.stats["fetches"] += len(keep) + len(retiring)
                if retiring:
                    # every last consumer's retire in one native call (dataplane.py:98-101,
                    # datastore.py:146-149), fenced on the batch's read (its stream waited on
                    # each object's `ready` before `done`) and any earlier readers
                    fence1 = (done,)
                    r_ids = [o.did for o in retiring]
                    rws, lasts = self.pools[g].retire_many(
                        self.index, r_ids, [o.block.policy_block for o in retiring],
                        [o.producer for o in retiring],
                        [fence1 + tuple(o.readers) if o.readers else fence1 for o in retiring])
                    live, freed, last_of = self._live, 0, {}
                    pop = objs.pop
                    for i, o in enumerate(retiring):
                        o.retired = True
                        if pop(o.did, None) is not None:
                            live[(o.producer, g)] -= 1
                            freed += o.nbytes
                        o.block = None
                        last_of[o.producer] = i           # one shrink timer per producer
                    meta = self.index._meta
                    if meta:
                        for did in r_ids:
                            meta.pop(did, None)
                    self._stored[g] -= freed
                    for i in last_of.values():
                        last = lasts[i]
                        self._push_due(g, rws[i], None if last != last else last, self._last_op_ms)
                    if self.strategy.migration != "none" and self._off_gpu[g]:
                        self._pending.add(("prefetch", g))
        for did, out in rest:
            self.fetch(did, out=out, consumer=consumer)
        if self._pending:
            self._drain_pending()
        return [out for _, out in items]

    def sync_stream(self, g: int):
        """Block the host until the caller's current stream on GPU ``g`` drained
        (another process is about to touch what it ordered)."""
        dev.Ev(g).record(self._stream(g)).synchronize()

    def wait(self, timeout_ms: float = -1.0):
        """Block the host until every host->GPU stage submitted so far has landed."""
        with self._lock:
            tickets = [t[0] for t in self._tickets]
        for t in tickets:
            self.pacer.wait(t, timeout_ms)
        with self._lock:
            self._reap()

    def release(self, data_id: int):
        """Drop a stored object regardless of remaining consumers."""
        with self._lock:
            obj = self._objs.get(data_id)
            if obj is None and self._lane is not None:
                obj = self._lane_take(data_id)
            if obj is not None:
                obj.remaining = 0
                self._retire(obj)
        if self._pending:
            self._drain_pending()

    def response(self, data_id: int) -> torch.Tensor:
        """Host copy of a ``store(..., response=True)`` output (waits for it)."""
        obj = self._objs.get(data_id)
        if obj is None or obj.response_host is None:
            from ._lib import MissingData
            raise MissingData(f"no response for data id {data_id}")
        if obj.response_ticket is not None:
            self.pacer.wait(obj.response_ticket)
        else:
            obj.response_event.synchronize()
        return obj.response_host.view(obj.dtype).view(obj.shape)

    def close(self):
        if self._lane is not None:
            self.detach_lane()
        self.pacer.close()                        # drains in-flight host->GPU stages
        self._tickets.clear()
        with self._maint_cv:
            self._closing = True
            self._maint_cv.notify()
        self._maint.join(timeout=5)
        for g in self.gpus:
            torch.cuda.synchronize(g)
        self._objs.clear()
        for p in self.pools.values():
            p.close()
        for g in self.gpus:
            for st in self._ce[g] + [x for pr in self._ce_pairs[g] + self._d2h_pairs[g] for x in pr]:
                dev.destroy_stream(st)
        dev.Ev.drain_free()

    # ------------------------------------------------ the daemon's native lane
    def attach_lane(self, lane):
        """The daemon's native lane (csrc/lane.cc, ``ft_lane``) serves function
        processes' hot requests — commits of lent blocks, same-GPU zero-copy fetches
        and their releases — with C++ workers. Objects it commits live in its table
        until their last view is released or this tube adopts them (``_lane_take``);
        its events (committed / retired / freed / stock / unpin) are applied here in
        order (``lane_service``)."""
        self._lane = lane
        self._lane_blocks = {}       # pool policy block id -> PoolBlock lent to / stocked in / stored by the lane
        self._lane_adopted = {}      # data id -> adopted object whose lane views are still alive
        self._lane_stock_todo = []   # (gpu, class bytes) the lane's stock asked for
        self._lane_buf = dev.C.create_string_buffer(1 << 20)
        self._lane_n = dev.C.c_uint64()

    def detach_lane(self):
        """Adopt every lane object and take the stocked blocks back (the daemon closed)."""
        with self._lock:
            self._lane_sync()                   # the closed connections' loans and stock came back
            self._lane_adopt(-1)
            for blk in self._lane_blocks.values():   # (none expected: only blocks of live connections)
                self.pools[blk.device].free(blk, list(blk.fences))
            self._lane_blocks = {}
            self._lane_stock_todo = []
            self._lane = None

    def lane_service(self, timeout_ms: float = 50.0) -> bool:
        """Wait for lane events, apply them, refill the stock it asked for (the
        daemon's service thread calls this in a loop). False once detached."""
        lane = self._lane
        if lane is None:
            return False
        n = dev.C.c_uint64()
        # cap 0: wait without consuming — events are consumed and applied under the tube
        # lock so that the service thread and an adopting request apply them in order
        dev.LIB.ft_lane_events(lane, None, 0, dev.C.byref(n), int(timeout_ms * 1e3))
        with self._lock:
            self._lane_sync()
            todo, self._lane_stock_todo = self._lane_stock_todo, []
        for conn_id, g, cls in todo:
            self._lane_stock(conn_id, g, cls)
        if self._pending:
            self._drain_pending()
        return True

    def _lane_stock(self, conn_id, g, cls):
        """A lendable block of class ``cls`` for connection ``conn_id``'s stock in the
        lane (allocated outside the tube lock: growth may map memory)."""
        lane = self._lane
        if lane is None or g not in self.pools:
            return
        blk = self.pools[g].allocate(int(cls))
        arena, off, abytes = self.pools[g].locate(blk)
        fences = [e._recorded() for e in blk.fences]
        with self._lock:
            rc = 1
            if self._lane is not None:
                self._lane_blocks[blk.policy_block.block_id] = blk
                rc = dev.LIB.raw("ft_lane_stock_put")(
                    lane, int(conn_id), g, blk.policy_block.block_id, blk.vmm_id, dev.C.c_void_p(blk.ptr),
                    int(blk.policy_block.class_bytes), arena, off, abytes,
                    (dev.C.c_void_p * max(1, len(fences)))(*fences), len(fences))
            if rc:                              # the connection (or the lane) is gone: the block goes back
                self._lane_blocks.pop(blk.policy_block.block_id, None)
                self.pools[g].free(blk, list(blk.fences))

    def lane_lend(self, conn_lane, blk) -> int:
        """Register a block lent through Python (the daemon's ``alloc``) with the lane:
        the client's commit of it is then served natively. Returns the token."""
        arena, off, abytes = self.pools[blk.device].locate(blk)
        tok = dev.C.c_uint64()
        with self._lock:
            self._lane_blocks[blk.policy_block.block_id] = blk
        dev.LIB.ft_lane_lend(conn_lane, blk.policy_block.block_id, blk.vmm_id, dev.C.c_void_p(blk.ptr),
                             int(blk.policy_block.class_bytes), arena, off, abytes, dev.C.byref(tok))
        return tok.value

    def lane_block(self, block_id: int):
        """(the daemon, serving a commit of a lane-lent block itself) the PoolBlock back."""
        with self._lock:
            return self._lane_blocks.pop(block_id)

    def peek(self, data_id: int):
        """The stored object's record (adopting it from the lane if it lives there), or None."""
        with self._lock:
            obj = self._objs.get(data_id)
            if obj is None and self._lane is not None:
                obj = self._lane_take(data_id)
            return obj

    def _lane_sync(self):
        """(lock held) Apply the lane's queued events now, in order."""
        n = self._lane_n
        while True:
            dev.LIB.ft_lane_events(self._lane, self._lane_buf, len(self._lane_buf), dev.C.byref(n), 0)
            if not n.value:
                return
            self._lane_apply(self._lane_buf.raw[:n.value])

    def _lane_apply(self, data: bytes):
        """(lock held) COMMITTED: the histogram sample, live/stored accounting, the
        shrink timer and the store cap check of a store (engine.py:342-360,
        datastore.py:51-62, 685-702) — the index entry was written by the lane;
        RETIRED: the accounting of a last consumer's retire (engine.py:667-679);
        FREED: the block back to the pool policy, fenced on its reader's release;
        STOCK: the lane wants a lendable block of a class; UNPIN: a lane view of an
        adopted object was released."""
        off, end, ev = 0, len(data), _LANE_EV
        while off < end:
            kind, nlen, did, g, cons, pbid, nbytes, now, evh = ev.unpack_from(data, off)
            off += ev.size
            name = data[off:off + nlen].decode() if nlen else ""
            off += nlen
            if kind == 1:
                live = self._live[(name, g)] + 1
                self.pools[g].record(name, now, float(nbytes), float(live))
                self._live[(name, g)] = live
                self._stored[g] += nbytes
                self.stats["stores"] += 1
                self._push_shrink(g, name, now)
                if self.strategy.migration != "none" and self._stored_on(g) > self.capacity_limit:
                    self._pending.add(("pressure", g))
            elif kind == 2:
                self._live[(name, g)] -= 1
                self._stored[g] -= nbytes
                self.stats["fetches"] += 1
                self.stats["zero_copy"] += 1
                if self.strategy.migration != "none" and self._off_gpu[g]:
                    self._pending.add(("prefetch", g))
            elif kind == 3:
                blk = self._lane_blocks.pop(pbid, None)
                # (no fence: a stocked block nobody wrote — its previous users' fences stay)
                fences = [dev.Ev.adopt(evh, g)] if evh else list(blk.fences if blk is not None else ())
                if blk is not None:
                    self.pools[g].free(blk, fences)
                    if name:
                        self._push_shrink(g, name, self.now_ms())
            elif kind == 4:
                self._lane_stock_todo.extend([(did, g, nbytes)] * max(1, cons))
            elif kind == 5:
                o = self._lane_adopted.get(did)
                if o is not None:
                    if o.block is not None and evh:
                        o.readers.append(dev.Ev.adopt(evh, g))
                    if o.pins <= 1:
                        self._lane_adopted.pop(did, None)
                    self._unpin(o)

    def _lane_take(self, did: int):
        """(lock held) Adopt lane object ``did`` into the table (its queued events
        applied first); None if the lane does not hold it (or it is already retired
        and only pinned by views)."""
        self._lane_sync()
        C = dev.C
        rec, shape, name = _lane_obj_t(), (C.c_int64 * 8)(), C.create_string_buffer(512)
        if dev.LIB.raw("ft_lane_take")(self._lane, int(did), C.byref(rec), shape, name, 512):
            return None
        g = rec.gpu
        obj = _Obj(did, rec.nbytes, _LANE_DTYPES[rec.dtype], tuple(shape[:rec.ndim]), g, name.value.decode(),
                   rec.remaining, rec.stored_at_ms)
        obj.home = g
        obj.queue_pos = next(self._queue)
        obj.block = self._lane_blocks.pop(rec.block_id)
        obj.ready = dev.Ev.adopt(rec.ready, g) if rec.ready else None
        obj.pins = rec.pins
        if rec.pins:
            self._lane_adopted[did] = obj
        if rec.remaining <= 0:                 # retired (accounted already), kept only by views
            obj.retired = True
            return None
        self._objs[did] = obj
        return obj

    def _lane_adopt(self, g: int):
        """(lock held) Adopt every lane object (on GPU ``g``; all with g < 0)."""
        C = dev.C
        ids, n = (C.c_int64 * 65536)(), C.c_int()
        dev.LIB.raw("ft_lane_ids")(self._lane, int(g), ids, 65536, C.byref(n))
        for i in range(min(n.value, 65536)):
            self._lane_take(ids[i])

    # ------------------------------------------------------------ internals
    def _push_shrink(self, g, func, now):
        """Shrink timer at last_request + R_window (engine.py:656-659)."""
        r_window, last = self.pools[g].hist_window(func)
        self._push_due(g, r_window, last, now)

    def _push_due(self, g, r_window, last, now):
        due = (last if last is not None else now) + r_window
        if self._last_due == (due, g):
            return                                    # the same deadline is queued already
        self._last_due = (due, g)
        with self._maint_cv:
            wake = not self._shrink_due or due < self._shrink_due[0][0]
            heapq.heappush(self._shrink_due, (due, g))
            if wake:                                  # only an earlier deadline needs the timer thread
                self._maint_cv.notify()

    def _respond(self, obj: _Obj, host=None):
        """Response D2H of a stored output (engine.py:414-423). With the PCIe
        scheduler it is a managed GPU->host stage over the plan's routes
        (returned for submission outside the tube lock); otherwise one CE copy."""
        g = obj.gpu
        host = host if host is not None else self._pinned(obj.nbytes)
        if self.strategy.pcie_sched:
            plan = self.plane.fetch_plan(self._loc(g), self._loc(None), obj.nbytes)
            obj.response_host = host
            self.stats["bytes_d2h"] += obj.nbytes
            return self._d2h_stage(obj, plan, host, obj.producer, None, None)
        s = self._ce[g][1]
        obj.ready.wait(s)
        dev.pcie_copy(host.data_ptr(), obj.block.ptr, obj.nbytes, False, g, s)
        ev = dev.Ev(g).record(s)
        obj.response_host, obj.response_event = host, ev
        obj.readers.append(ev)
        self.stats["bytes_d2h"] += obj.nbytes
        return None

    def _d2h_stage(self, obj, plan, host, consumer, slo_ms, infer_ms):
        """pacer.submit_d2h arguments for a GPU->host plan (dataplane.py:190-250
        with into=False): route i moves branch i's byte range out of the source
        GPU's own root, or over NVLink into a staging GPU's ring and out of its root."""
        g = obj.gpu
        st = plan.stages[0]
        br = st.branches
        ranges = self._stripes(obj.nbytes, [b.bytes_share for b in br])
        s = self._stream(g)
        obj.ready.wait(s)
        slot = (s >> 4) * 0x9E3779B1 >> 16
        routes = []
        for b, (off, n) in zip(br, ranges):
            sg = _staging_gpu_d2h(b.links, g)
            if sg not in self._d2h_pairs:
                from ._lib import NotSupported
                raise NotSupported(f"the plan routes through GPU {sg}, which this tube does not drive")
            ce, fw = self._d2h_pairs[sg][slot % len(self._d2h_pairs[sg])]
            routes.append((sg, 0, off, n, ce.cuda_stream, fw.cuda_stream))
            if sg != g:
                self.stats["bytes_nvlink"] += n
        managed = bool(self.strategy.pcie_sched and st.managed)
        self.stats["managed_stages"] = self.stats.get("managed_stages", 0) + int(managed)
        return (f"m{next(self._managed_ids)}" if managed else "", managed,
                slo_ms if slo_ms else 1e9, infer_ms if infer_ms is not None else 0.0,
                min(min(b.hop_caps) for b in br), host.data_ptr(), obj.block.ptr, g, obj.nbytes, routes, s)

    def _consumed(self, obj: _Obj, fence=None, stream=None):
        obj.remaining -= 1
        if obj.remaining <= 0:
            self._retire(obj, fence, stream)

    def _retire(self, obj: _Obj, fence=None, stream=None, drop: bool = True):
        """engine.py:667-679: last consumer done -> drop index entry, free block.
        ``drop=False`` (a block-less object): the caller drops the index entry itself
        once its transfer is issued."""
        if obj.retired:
            return
        obj.retired = True
        if self._objs.pop(obj.did, None) is not None:
            self._account(obj, -1)
            if obj.home is not None and obj.block is None and obj.host is not None:
                self._off_gpu[obj.home] -= 1          # a migrated object left the table
        blk = obj.block
        if blk is not None and obj.pins == 0:
            # drop the index entry, return the block (fenced on its last users) and re-arm
            # the shrink timer in one FFI call (dataplane.py:98-101, datastore.py:146-149)
            obj.block = None
            # the caller's last read of the block: an event on its stream (or the one
            # a batched fetch recorded after its copy)
            ev = fence if fence is not None else dev.Ev(blk.device).record(
                stream if stream is not None else self._stream(blk.device))
            fences = [ev] + obj.readers + ([obj.ready] if obj.ready is not None else [])
            obj.readers = []
            self.index._meta.pop(obj.did, None)
            rw, last = self.pools[blk.device].commit_retire(self.index, obj.did, blk, fences, obj.producer)
            self._push_due(blk.device, rw, last, self.now_ms())
            if self.strategy.migration != "none" and self._off_gpu[blk.device]:
                self._pending.add(("prefetch", blk.device))  # engine.py:678-679, 717-736
            return
        if drop:
            self.index.drop(obj.did)
        self._maybe_free(obj, stream)

    def _maybe_free(self, obj: _Obj, stream=None):
        if obj.block is not None and obj.pins == 0 and obj.retired:
            blk, obj.block = obj.block, None
            g = blk.device
            # later writers of this block must order after our readers
            ev = dev.Ev(g).record(stream if stream is not None else self._stream(g))
            fences = [ev] + obj.readers + ([obj.ready] if obj.ready is not None else [])
            obj.readers = []
            # the block back to the policy (fenced) and the producer's window in one
            # native call — the index entry went at retire (id -1 drops nothing)
            rw, last = self.pools[g].commit_retire(self.index, -1, blk, fences, obj.producer)
            self._push_due(g, rw, last, self.now_ms())
            if self.strategy.migration != "none" and self._off_gpu[g]:
                self._pending.add(("prefetch", g))  # engine.py:678-679, 717-736

    def _unpin(self, obj, stream=None):
        with self._lock:
            obj.pins -= 1
            self._maybe_free(obj, stream)

    def _view(self, obj: _Obj) -> torch.Tensor:
        obj.pins += 1
        t = obj.block.view(obj.nbytes, obj.dtype, obj.shape)
        weakref.finalize(t, self._unpin, obj)   # strong ref: the object may already be retired
        self.stats["zero_copy"] += 1
        return t

    def _execute(self, obj, plan, src, dst, out, slo_ms, infer_ms):
        m = plan.method
        if m == "intra_gpu":
            if src.on_host:  # host -> host shared memory
                if out is None:
                    return obj.host.view(obj.dtype).view(obj.shape)
                out.view(-1).view(torch.uint8).copy_(obj.host)
                return out
            s = self._stream(dst.gpu)
            if out is None:
                obj.ready.wait(s)
                return self._view(obj)
            last = obj.remaining <= 1
            # wait for the stored bytes and copy into the caller's input: one call. A
            # consumer that is not the last one leaves its read's event on the object:
            # the last consumer's retire (maybe on another stream) fences the block on it
            done = None if last else dev.Ev(dst.gpu)
            dev.copy_ordered(out.data_ptr(), obj.block.ptr, obj.nbytes, dst.gpu, s,
                             dev.L2_EVICT_FIRST if last else dev.L2_NORMAL, (obj.ready,), done)
            if done is not None:
                self._hold_until(obj, done)
            self.stats["bytes_local"] += obj.nbytes
            return out
        if m == "inter_gpu":
            return self._inter_gpu(obj, plan, src, dst, out)
        if m == "host_gpu":
            return self._gpu_to_host(obj, plan, out)
        from ._lib import NotSupported
        raise NotSupported("inter-node transfers need a multi-node deployment (SURVEY §8f row 4)")

    def _out(self, obj, gpu, out):
        if out is not None:
            return out
        return dev.empty_shared(obj.nbytes, gpu).view(obj.dtype).view(obj.shape)

    def _inter_gpu(self, obj, plan, src, dst, out):
        res = self._out(obj, dst.gpu, out)
        s = self._stream(dst.gpu)
        obj.ready.wait(s)
        if len(plan.stages) == 2:
            # host-oriented baseline: D2H to host, then H2D (dataplane.py:265-272)
            host = self._pinned(obj.nbytes)
            ce = self._ce[src.gpu][0]
            obj.ready.wait(ce)
            dev.pcie_copy(host.data_ptr(), obj.block.ptr if obj.block else obj.host.data_ptr(), obj.nbytes,
                          False, src.gpu, ce)
            ev = dev.Ev(src.gpu).record(ce)
            if obj.block is not None:
                obj.readers.append(ev)
            ev.wait(s)
            dev.pcie_copy(res.data_ptr(), host.data_ptr(), obj.nbytes, True, dst.gpu, s)
            self._keepalive.append((dev.Ev(dst.gpu).record(s), [host]))   # until the H2D has read it
            self.stats["bytes_d2h"] += obj.nbytes
            self.stats["bytes_h2d"] += obj.nbytes
            return res
        br = plan.stages[0].branches
        ranges = self._stripes(obj.nbytes, [b.bytes_share for b in br])
        for b, (off, n) in zip(br, ranges):
            if n == 0:
                continue
            hops = _hops(b.links)
            if len(hops) == 1:
                # direct NVLink: pull over the peer mapping on the consumer's stream
                dev.copy(res.data_ptr() + off, obj.block.ptr + off, n, dst.gpu, s, dev.ENGINE_VEC)
            else:
                self._relay(hops, obj.block.ptr + off, res.data_ptr() + off, n, s)
            self.stats["bytes_nvlink"] += n
        ev = dev.Ev(dst.gpu).record(s)
        if plan.claimed_func:
            self._pending_release.append((ev, plan))
        self._hold_until(obj, ev)
        return res

    def _relay(self, hops, src_ptr, dst_ptr, n, s):
        """Multi-hop NVLink branch (non-uniform fabrics): store-and-forward
        through each intermediate GPU into a private buffer. Each hop is pulled
        by its receiving GPU on a stream of that GPU, chained to the previous
        hop by an event; the last hop runs on the consumer's stream. Buffers
        stay referenced until the last hop has completed."""
        ev = dev.Ev(hops[-1][1]).record(s)            # source ready / destination free
        cur, keep = src_ptr, []
        for i, (u, v) in enumerate(hops):
            last = i == len(hops) - 1
            st = s if last else self._pair(v)[1].cuda_stream
            ev.wait(st)
            if last:
                out = dst_ptr
            else:
                buf = torch.empty(n, dtype=torch.uint8, device=f"cuda:{v}")
                keep.append(buf)
                out = buf.data_ptr()
            dev.copy(out, cur, n, v, st, dev.ENGINE_VEC)
            ev = dev.Ev(v).record(st)
            cur = out
        if keep:
            self._keepalive.append((ev, keep))

    def _hold_until(self, obj, ev):
        """Keep the source block alive until a reader's event completes."""
        if obj.block is not None:
            obj.readers.append(ev)

    def _pair(self, g, slot=None):
        pairs = self._ce_pairs.get(g)
        if pairs is None:
            from ._lib import NotSupported
            raise NotSupported(f"the plan routes through GPU {g}, which this tube does not drive (gpus={self.gpus})")
        return pairs[(next(self._ce_rr) if slot is None else slot) % len(pairs)]

    def _host_to_gpu(self, obj, plan, dst, out, slo_ms, infer_ms):
        """A host_gpu plan (dataplane.py:190-250) as one pacer stage: route i
        carries the contiguous byte range of branch i's share — CE straight in on
        the target's own root, or CE into the staging GPU's chunk ring + NVLink
        forward. Managed stages (strategy.pcie_sched) enter the SLO partition and
        are paced in batches at their rate (engine.py:537-646); the consumer's
        stream is ordered after the last byte. The plan, the byte ranges and the
        route streams come from one native call (``ft_h2g_routes``). Returns
        (result, ft_pacer_submit's arguments after the key); the caller submits outside the
        tube lock (the routes live in this thread's array until then)."""
        res = self._out(obj, dst.gpu, out)
        s = self._stream(dst.gpu)
        if obj.ready is not None:
            obj.ready.wait(s)
        tl = self._tls
        if not hasattr(tl, "routes"):
            from ._lib import RouteC
            tl.routes, tl.k, tl.managed = (RouteC * 16)(), dev.C.c_int(), dev.C.c_int()
            tl.cap, tl.nv, tl.ticket = dev.C.c_double(), dev.C.c_uint64(), dev.C.c_uint64()
            tl.plan = dev.LIB.raw("ft_h2g_routes")
            tl.submit = dev.LIB.raw("ft_pacer_submit")
        rc = tl.plan(self.plane._h, self.node, dst.gpu, obj.nbytes, s, tl.routes, 16, tl.k, tl.managed, tl.cap,
                     tl.nv)
        if rc:
            from ._lib import raise_status
            raise_status(rc)
        managed = tl.managed.value
        host = obj.host
        # (the pacer names a managed stage itself: "h<ticket>")
        stage = (managed, slo_ms if slo_ms else 1e9,                  # engine.py:546-547
                 infer_ms if infer_ms is not None else 0.0, tl.cap.value, res.data_ptr(), dst.gpu,
                 host.data_ptr(), obj.nbytes, host.is_pinned(), tl.k.value, tl.routes, s)
        self.stats["bytes_h2d"] += obj.nbytes
        self.stats["bytes_nvlink"] += tl.nv.value
        if managed:
            self.stats["managed_stages"] = self.stats.get("managed_stages", 0) + 1
        return res, stage

    def reclaim(self) -> int:
        """Unmap every parked pool block now (call when the GPU is quiet)."""
        with self._maint_cv:
            return sum(p.reclaim() for p in self.pools.values())

    def maintain(self):
        """Release landed NVLink claims; give parked pool blocks back when idle."""
        with self._lock:
            self._reap()
        with self._maint_cv:
            self._reclaim_if_idle(self.now_ms())

    def _gpu_to_host(self, obj, plan, out):
        res = out if out is not None else self._pinned(obj.nbytes).view(obj.dtype).view(obj.shape)
        g = obj.gpu
        ce = self._ce[g][0]
        obj.ready.wait(ce)
        dev.pcie_copy(res.data_ptr(), obj.block.ptr, obj.nbytes, False, g, ce)
        dev.Ev(g).record(ce).synchronize()
        self.stats["bytes_d2h"] += obj.nbytes
        return res


class _IntraPlan:
    method = "intra_gpu"
    claimed_func = None


_INTRA_GPU = _IntraPlan()


def measure_pcie_gbps(gpus, nbytes: int = 64 << 20, reps: int = 12, margin: float = 1.0) -> float:
    """Pinned host->GPU copy-engine rate (GB/s) of the slowest link among
    ``gpus``: best of ``reps`` back-to-back copies after a warm-up burst (an
    idle PCIe link trains down and needs traffic to come back to full speed),
    times ``margin``. The pacer must not hand out more than the link delivers
    (its shares would stop isolating tenants) nor much less (a lone stage
    would be throttled below the link)."""
    # a pinned buffer the CPU never wrote: DMA out of lines the CPU holds dirty in its
    # caches runs at ~21 GB/s on the B200 hosts (vs 55 from DRAM), and a calibration
    # from a just-written buffer read 20-38 GB/s (tools/diag_calib2.py)
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    rates = []
    for g in gpus:
        dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{g}")
        s = torch.cuda.Stream(g)
        for _ in range(4):                                   # wake the link up
            dev.pcie_copy(dst.data_ptr(), host.data_ptr(), nbytes, True, g, s)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        ev[0].record(s)
        for i in range(reps):
            dev.pcie_copy(dst.data_ptr(), host.data_ptr(), nbytes, True, g, s)
            ev[i + 1].record(s)
        ev[-1].synchronize()
        best = min(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
        rates.append(nbytes / (best * 1e-3) / 1e9)
        del dst
    return round(min(rates) * margin, 2)


def _hops(links):
    """GPU hops of an NVLink branch from its link ids (dataplane.py:128-133)."""
    hops = []
    pending = None
    for l in links:
        if l[0] == "nv":
            hops.append((l[1], l[2]))
        elif l[0] == "nvp_out":
            pending = l[1]
        elif l[0] == "nvp_in":
            hops.append((pending, l[1]))
    return hops


def _staging_gpu_d2h(links, source):
    """GPU whose PCIe root carries a GPU->host branch (the NVLink hop's far end)."""
    for l in links:
        if l[0] == "nvp_in":
            return l[1]
        if l[0] == "nv":
            return l[2]
    return source


class _lane_obj_t(dev.C.Structure):
    """ft_lane_obj (include/faastube.h)."""
    _fields_ = [("data_id", dev.C.c_int64), ("block_id", dev.C.c_int64), ("nbytes", dev.C.c_uint64),
                ("stored_at_ms", dev.C.c_double), ("ready", dev.C.c_void_p), ("gpu", dev.C.c_int32),
                ("dtype", dev.C.c_int32), ("ndim", dev.C.c_int32), ("remaining", dev.C.c_int32),
                ("pins", dev.C.c_int32), ("consumers", dev.C.c_int32)]

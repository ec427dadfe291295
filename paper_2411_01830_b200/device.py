"""Device side: elastic VMM pool per GPU + the sm_100a movers (libfaastube).

``DevicePool`` pairs the reference's pool POLICY (``datastore.MemoryPool``,
datastore.py:91-166: exact size-class reuse, growth, histogram-driven shrink)
with real memory: each policy block is backed by a ``cuMemCreate`` physical
allocation mapped into one reserved VA range per GPU, readable/writable from
every peer GPU and exportable to other processes as a POSIX fd
("auto-scaling memory pool"). When the policy drops a block
the physical memory is unmapped and returned to the driver — that is the
"shrink" the paper measures.

torch is used only for device selection, streams, events and to wrap pool
memory as tensors (``__cuda_array_interface__``); all bytes move in our
kernels or on the copy engines.
"""

from __future__ import annotations

import array
import ctypes as C
import itertools
import os
import threading
import weakref

import torch

from . import datastore
from ._lib import LIB, raise_status

GiB = 1 << 30
ENGINE_AUTO, ENGINE_BULK, ENGINE_VEC = 0, 1, 2

_TYPESTR = {torch.uint8: "|u1", torch.int8: "|i1", torch.float16: "<f2", torch.bfloat16: "<f2",
            torch.float32: "<f4", torch.float64: "<f8", torch.int16: "<i2", torch.int32: "<i4",
            torch.int64: "<i8", torch.bool: "|b1"}


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("FaaSTube device path needs a CUDA GPU (no CPU fallback exists)")
    n = C.c_int()
    LIB.ft_device_count(C.byref(n))
    return n.value


def stream_ptr(stream) -> int:
    """cudaStream_t of a torch stream, a raw pointer (int) or None (legacy default)."""
    if stream is None:
        return 0
    return stream if isinstance(stream, int) else stream.cuda_stream


def current_stream(device: int) -> int:
    """Raw pointer of the current stream on ``device`` (no torch.cuda.Stream object)."""
    return torch._C._cuda_getCurrentRawStream(device)


def empty_shared(nbytes: int, device: int) -> torch.Tensor:
    """A device buffer from torch's caching allocator that every stream can
    reuse: allocated on the device's default stream, then recorded on the
    caller's current stream. Allocated directly on per-tenant streams, freed
    blocks only serve the same stream again; with many tenant streams the
    allocator keeps growing (cudaMalloc under load: 10-100 ms stalls measured)."""
    cur = torch.cuda.current_stream(device)
    with torch.cuda.stream(torch.cuda.default_stream(device)):
        t = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", device))
    if cur.cuda_stream != 0:
        t.record_stream(cur)
    return t


def new_stream(device: int) -> torch.cuda.ExternalStream:
    """A private CUDA stream (``ft_stream_create``) as a torch stream object.
    torch.cuda.Stream() hands out a round-robin pool of 32 streams per device:
    two "new" torch streams can be the same CUDA stream, and a copy-engine
    route would then share a FIFO with another tenant's consumer stream."""
    h = C.c_void_p()
    LIB.ft_stream_create(int(device), C.byref(h))
    return torch.cuda.ExternalStream(h.value, device=torch.device("cuda", device))


def destroy_stream(stream: torch.cuda.ExternalStream):
    stream.synchronize()
    LIB.ft_stream_destroy(C.c_void_p(stream.cuda_stream))


# every event record (and the seq it gets) happens under this lock, so a later seq
# on a stream is a later record there — wait dedup relies on it (_needed)
REC_LOCK = threading.Lock()


class Ev:
    """A raw CUDA event (libfaastube ``ft_event_*``): request-path stream
    ordering without torch.cuda.Event objects. Destroyed with the object
    (CUDA defers the destruction of an event still pending)."""

    __slots__ = ("h", "device", "rec", "stream", "seq", "__weakref__")
    # handles of dropped events, per device, reused by new ones: a request makes
    # several (ready, fences) and create + destroy cost ~2 us of driver time each.
    # Reuse is safe: a wait already enqueued on a stream captured the old record.
    # A reused handle still carries its previous record, so an Ev refuses to be
    # waited on or queried until it has been recorded again (``rec``).
    _free: dict = {}
    _FREE_MAX = 1024

    _seq = itertools.count(1)        # record order (a later record on a stream covers earlier ones)

    def __init__(self, device: int):
        self.rec = False
        self.stream = None
        self.seq = 0
        free = Ev._free.get(device)
        if free:
            try:
                self.h, self.device = free.pop(), device
                return
            except IndexError:               # another thread took the last one
                pass
        h = C.c_void_p()
        LIB.ft_event_create(int(device), C.byref(h))
        self.h, self.device = h.value, device

    @classmethod
    def adopt(cls, handle: int, device: int) -> "Ev":
        """An event recorded elsewhere (the daemon's native lane) whose handle this
        process now owns: already recorded, on a stream unknown here."""
        e = cls.__new__(cls)
        e.h, e.device, e.rec, e.stream, e.seq = handle, device, True, None, next(Ev._seq)
        return e

    def _recorded(self):
        if not self.rec:
            raise RuntimeError("event used before it was recorded (its work was never enqueued)")
        return self.h

    def record(self, stream):
        sp = stream_ptr(stream)
        with REC_LOCK:
            LIB.ft_event_record(C.c_void_p(self.h), C.c_void_p(sp))
            self._recorded_on(sp)
        return self

    def _recorded_on(self, sp: int):
        """Mark recorded on stream ``sp``; callers hold REC_LOCK around the record
        call and this, so ``seq`` follows the order of the records."""
        self.rec, self.stream, self.seq = True, sp, next(Ev._seq)

    def wait(self, stream):
        """``stream`` waits for the work this event captured."""
        LIB.ft_stream_wait_events(C.c_void_p(stream_ptr(stream)), (C.c_void_p * 1)(self._recorded()), 1)

    def query(self) -> bool:
        d = C.c_int()
        LIB.ft_event_query(C.c_void_p(self._recorded()), C.byref(d))
        return bool(d.value)

    def synchronize(self):
        LIB.ft_event_synchronize(C.c_void_p(self._recorded()))

    @staticmethod
    def drain_free():
        """Destroy the pooled handles (teardown; none of them is in use)."""
        for free in list(Ev._free.values()):
            while free:
                try:
                    h = free.pop()
                except IndexError:
                    break
                LIB.raw("ft_event_destroy")(C.c_void_p(h))

    def __del__(self):
        # (hot: every retired object drops its events — kept to a dict lookup and an append)
        try:
            h = self.h
            if not h:
                return
            self.h = None
            free = Ev._free.get(self.device)
            if free is None:
                free = Ev._free.setdefault(self.device, [])
            if len(free) < 1024:                       # Ev._FREE_MAX
                free.append(h)
                return
            LIB.raw("ft_event_destroy")(C.c_void_p(h))
        except Exception:  # noqa: BLE001 - interpreter teardown / never initialised
            pass


def copy_batch(segments, device: int, stream=None):
    """[(dst_ptr, src_ptr, nbytes)] in one launch per 64 segments (ft_copy_batch).
    The segment array is built as one flat u64 array (ft_segment = 3 x 8 bytes)."""
    from ._lib import SegmentC
    flat = [v for seg in segments for v in seg]
    arr = (C.c_uint64 * len(flat))(*flat)
    LIB.ft_copy_batch(C.cast(arr, C.POINTER(SegmentC)), len(segments), int(device), C.c_void_p(stream_ptr(stream)))


def copy_batch_flat(flat, device: int, stream=None):
    """``copy_batch`` with the segments already flat: [dst, src, nbytes, dst, src, nbytes, ...]
    (packed by the array module: a ctypes array built element by element cost ~10 us at 64)."""
    arr = array.array("Q", flat)
    addr, _n = arr.buffer_info()
    LIB.ft_copy_batch(C.c_void_p(addr), len(flat) // 3, int(device), C.c_void_p(stream_ptr(stream)))


def _needed(stream: int, events) -> list:
    """The waits ``stream`` needs for ``events``: none for one recorded on the
    stream itself (stream order), and per other stream only the newest record
    (it covers that stream's earlier ones)."""
    last = {}
    for e in events:
        if e is None:
            continue
        e._recorded()
        if e.stream == stream and stream is not None:
            continue
        k = e.stream if e.stream is not None else id(e)
        cur = last.get(k)
        if cur is None or e.seq > cur.seq:
            last[k] = e
    return [e.h for e in last.values()]


def wait_events(stream, events):
    sp = stream_ptr(stream)
    evs = _needed(sp, events)
    if evs:
        LIB.ft_stream_wait_events(C.c_void_p(sp), (C.c_void_p * len(evs))(*evs), len(evs))


def copy_ordered(dst_ptr: int, src_ptr: int, nbytes: int, device: int, stream, hints: int = 0, waits=(),
                 done: "Ev | None" = None):
    """One call: ``stream`` waits on ``waits``, TMA-bulk copy with L2 ``hints``, record ``done``."""
    sp = stream_ptr(stream)
    evs = _needed(sp, waits)
    with REC_LOCK:
        LIB.ft_copy_ordered(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), int(nbytes), int(device),
                            C.c_void_p(sp), int(hints), (C.c_void_p * max(1, len(evs)))(*evs),
                            len(evs), C.c_void_p(done.h if done is not None else None))
        if done is not None:
            done._recorded_on(sp)


class _Mem:
    """__cuda_array_interface__ exporter over raw device memory. The owner
    reference keeps the backing pool block alive while any tensor view lives."""

    def __init__(self, ptr: int, nbytes: int, device: int, owner=None):
        self.ptr, self.nbytes, self.device, self.owner = ptr, nbytes, device, owner
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def as_tensor(ptr: int, nbytes: int, device: int, dtype=torch.uint8, shape=None, owner=None) -> torch.Tensor:
    """Zero-copy tensor over device memory at ``ptr`` (owner pinned by the view)."""
    with torch.cuda.device(device):
        t = torch.as_tensor(_Mem(ptr, nbytes, device, owner), device=f"cuda:{device}")
    if dtype != torch.uint8:
        t = t.view(dtype)
    if shape is not None:
        t = t.view(shape)
    return t


def copy(dst_ptr: int, src_ptr: int, nbytes: int, device: int, stream=None, engine=ENGINE_AUTO, grid=0):
    """K1/K3: SM-driven copy on ``device`` (TMA bulk locally, vector engine for peers)."""
    if engine == ENGINE_AUTO and grid == 0:
        LIB.ft_copy(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), int(nbytes), int(device), C.c_void_p(stream_ptr(stream)))
    else:
        LIB.ft_copy_ex(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), int(nbytes), int(device),
                       C.c_void_p(stream_ptr(stream)), int(engine), int(grid))


L2_NORMAL, L2_EVICT_FIRST, L2_EVICT_LAST = 0, 1, 2


def copy_hint(dst_ptr: int, src_ptr: int, nbytes: int, device: int, stream=None, src_policy=L2_NORMAL,
              dst_policy=L2_NORMAL):
    """TMA-bulk copy with L2 eviction policies on the source reads / destination writes."""
    LIB.ft_copy_hint(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), int(nbytes), int(device),
                     C.c_void_p(stream_ptr(stream)), int(src_policy | (dst_policy << 2)))


def copy_tensor(dst: torch.Tensor, src: torch.Tensor, stream=None, engine=ENGINE_AUTO):
    assert dst.is_contiguous() and src.is_contiguous() and dst.nbytes == src.nbytes
    dev = dst.device.index if dst.is_cuda else src.device.index
    copy(dst.data_ptr(), src.data_ptr(), dst.nbytes, dev, stream, engine)


def pcie_copy(dst_ptr: int, src_ptr: int, nbytes: int, to_device: bool, device: int, stream=None, batch_bytes=0):
    """One PCIe leg on the copy engine (pinned host <-> device)."""
    LIB.ft_pcie_copy(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), int(nbytes), int(bool(to_device)), int(device),
                     C.c_void_p(stream_ptr(stream)), int(batch_bytes))


class Fingerprint:
    """Fused integrity digest (u64 sum + xor of index-mixed words)."""

    def __init__(self, device: int):
        self.device = device
        self.buf = torch.zeros(2, dtype=torch.int64, device=f"cuda:{device}")

    def launch(self, ptr: int, nbytes: int, stream=None):
        LIB.ft_fingerprint(C.c_void_p(ptr), int(nbytes), C.c_void_p(self.buf.data_ptr()), int(self.device),
                           C.c_void_p(stream_ptr(stream)))
        return self.buf

    def value(self) -> tuple:
        v = self.buf.cpu().tolist()
        return tuple(x & 0xFFFFFFFFFFFFFFFF for x in v)


def fingerprint_host(buf) -> tuple:
    """Same digest on host memory (numpy array / bytes / pinned tensor)."""
    import numpy as np
    if isinstance(buf, torch.Tensor):
        buf = buf.contiguous().view(torch.uint8).numpy()
    a = np.ascontiguousarray(np.frombuffer(buf, dtype=np.uint8) if isinstance(buf, (bytes, bytearray)) else buf)
    out = (C.c_uint64 * 2)()
    LIB.ft_fingerprint_host(C.c_void_p(a.ctypes.data), int(a.nbytes), out)
    return out[0], out[1]


class PoolBlock:
    """A live pool block: policy block + mapped device memory. ``fences``:
    events of the previous holder's last readers/writers — a new writer's
    stream waits on them before touching the memory (``wait_fences``)."""

    __slots__ = ("policy_block", "vmm_id", "ptr", "nbytes", "device", "fences", "pool", "__weakref__")

    def __init__(self, policy_block, vmm_id, ptr, nbytes, device, fences=(), pool=None):
        self.policy_block, self.vmm_id, self.ptr, self.nbytes, self.device = (
            policy_block, vmm_id, ptr, nbytes, device)
        self.fences = fences
        self.pool = pool

    def view(self, nbytes: int, dtype=torch.uint8, shape=None) -> torch.Tensor:
        """Zero-copy tensor over the block's first ``nbytes``: a slice of a
        per-mapping uint8 tensor built once (``torch.as_tensor`` on an array
        interface costs ~10 us per call; a slice costs ~1 us)."""
        base = self.pool.base_tensor(self) if self.pool is not None else as_tensor(self.ptr, self.nbytes, self.device)
        t = base[:nbytes]
        if dtype != torch.uint8:
            t = t.view(dtype)
        # (a flat byte payload is the slice itself: each view costs ~1 us)
        return t.view(shape) if shape is not None and (dtype != torch.uint8 or len(shape) != 1) else t

    def wait_fences(self, stream):
        wait_events(stream, self.fences)
        self.fences = ()

    def take_fences(self) -> tuple:
        f, self.fences = self.fences, ()
        return f


class DevicePool:
    """Elastic VMM-backed store for one GPU, driven by the reference pool policy."""

    def __init__(self, device: int, mode: str = "autoscale", floor_bytes: float = datastore.POOL_FLOOR_BYTES,
                 native_alloc_ms: float = datastore.NATIVE_ALLOC_MS, va_bytes: int = 256 * GiB,
                 physical_bytes: float | None = None, spare_cap_bytes: int = 0, reserve_bytes: int | None = None):
        require_cuda()
        self.device = device
        self.on_unmap = []           # callbacks(arena id) after an arena is unmapped (daemon.py)
        if physical_bytes is None:
            physical_bytes = float(torch.cuda.get_device_properties(device).total_memory)
        self.policy = datastore.MemoryPool(device, mode, floor_bytes, native_alloc_ms, physical_bytes)
        h = C.c_void_p()
        LIB.ft_vmm_pool_create(int(device), int(va_bytes), C.byref(h))
        self._h = h
        # physical memory is mapped in arenas (csrc/device.cu): blocks are ranges of
        # them, so growth and shrink of the policy's blocks cost no driver call; an up-front
        # arena covers the common working set (a new one is mapped only when none has
        # room, and unused ones are unmapped only when the GPU is quiet — reclaim())
        if reserve_bytes is None:
            reserve_bytes = int(os.environ.get("FT_POOL_RESERVE_BYTES", 4 * GiB))
        self.reserved_bytes = 0
        if mode != "none" and reserve_bytes > 0:
            LIB.ft_vmm_pool_reserve(h, int(reserve_bytes))
            mapped = C.c_uint64()
            LIB.ft_vmm_pool_stats(h, C.byref(mapped), None, None)
            self.reserved_bytes = mapped.value
        self._mapped = {}  # policy block id -> (vmm id, ptr, bytes)
        self._fences = {}  # policy block id -> events the freed block's last users recorded
        self._bases = {}   # vmm id -> uint8 tensor over the whole mapping (zero-copy views slice it)
        # physical blocks the policy dropped, still mapped: reused by growth of the same
        # class, unmapped by reclaim() when the GPU is quiet (cuMemUnmap under load stalls
        # every CUDA call of the process for 100s of ms — measured)
        self._released = []  # [(vmm id, ptr, bytes, fences)]: spare mappings awaiting a holder
        self._range_fences = []  # [(lo, hi, fences)]: ranges given back to their arenas, last users
        self._lock = threading.Lock()
        self._names = {}             # producer name -> bytes (encoded once)
        self._addrs = {}             # producer name -> address of those bytes
        self._rw, self._last = C.c_double(), C.c_double()   # out-params of the hot calls (under _lock)
        self._noev = (C.c_void_p * 1)()
        self._store_fn, self._fetch_fn = LIB.raw("ft_store_local"), LIB.raw("ft_fetch_local")
        self._retire_fn = LIB.raw("ft_retire_commit")
        self.grow_events = 0
        # spares: after growth of a class, a background thread maps one more block of
        # that class into the parked list, so the next growth of the class is a reuse.
        # cuMemMap waits for the GPU's running kernels (measured 30-80 ms while tenants
        # compute) — a cost for this thread, not for the request that needs the block
        self.spare_cap_bytes = int(os.environ.get("FT_SPARE_CAP_BYTES", spare_cap_bytes))
        self._spare_q = []
        self._spare_cv = threading.Condition(self._lock)
        self._spare_thread = None
        self.spares_mapped = 0

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            th = self._spare_thread
            with self._lock:
                self._spare_q = None                   # stops the spare thread
                self._spare_cv.notify_all()
            if th is not None:
                th.join(timeout=10)
            torch.cuda.synchronize(self.device)
            LIB.ft_vmm_pool_destroy(h)
            self._h = None

    # ---- spare mappings (background growth)
    def _want_spare(self, class_bytes: int):
        """Called with the lock held after a growth of ``class_bytes``: map one
        spare of the class in the background (the next growth takes it instead
        of mapping on the request path). More spares per class were tried —
        as many as the class ever had in use at once — and did not remove the
        first-burst stalls (the concurrent tenants of a burst each grow before
        any spare exists) while doubling the mapped memory of bursty classes."""
        if self._spare_q is None or self.spare_cap_bytes <= 0:
            return
        # the spare is rounded up to a power of two of the 2 MiB granule: growth reuses a
        # parked block of up to twice its class, so one spare serves every class in
        # (P/2, P] — payload sizes drawn per request (config 4's detector outputs) land
        # in classes never seen before, and each new class otherwise mapped on the
        # request path (25 ms under load, one request over its SLO)
        gran = 2 << 20
        spare = gran << max(0, (int(class_bytes) - 1) // gran).bit_length()
        parked = sum(r[2] for r in self._released) + sum(self._spare_q)
        if parked + spare > self.spare_cap_bytes:
            return
        if any(class_bytes <= r[2] <= 2 * class_bytes for r in self._released) or \
                any(class_bytes <= q <= 2 * class_bytes for q in self._spare_q):
            return
        self._spare_q.append(spare)
        if self._spare_thread is None:
            self._spare_thread = threading.Thread(target=self._spare_loop, name=f"faastube-spares{self.device}",
                                                  daemon=True)
            self._spare_thread.start()
        self._spare_cv.notify()

    def _spare_loop(self):
        torch.cuda.set_device(self.device)
        while True:
            with self._lock:
                while self._spare_q is not None and not self._spare_q:
                    self._spare_cv.wait()
                if self._spare_q is None:
                    return
                cls = self._spare_q.pop(0)
            vid, ptr = C.c_uint64(), C.c_void_p()
            try:
                LIB.ft_vmm_block_map(self._h, int(cls), C.byref(vid), C.byref(ptr))
            except Exception:  # noqa: BLE001 - a spare is an optimisation; pressure wins
                continue
            with self._lock:
                if self._spare_q is None:            # closing: the pool unmaps everything
                    return
                self._released.append((vid.value, ptr.value, int(cls), ()))
                self.spares_mapped += 1

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass

    def allocate(self, nbytes: int) -> PoolBlock:
        """Policy decision (reuse exact class or grow) + physical mapping on growth.
        The mapping (cuMemCreate + cuMemMap + cuMemSetAccess, milliseconds for a
        large block) runs outside the pool lock: the policy already marked the
        block in use, so no other allocation or shrink can touch it."""
        with self._lock:
            b, _model_ms = self.policy.allocate(max(1, nbytes))
            m = self._mapped.get(b.block_id)
            fences = self._fences.pop(b.block_id, ())
        if m is None:
            with self._lock:
                # growth served by a dropped, still-mapped block: the smallest one that fits
                # (at most 2x — the policy still accounts the class it asked for)
                fits = [(r[2], i) for i, r in enumerate(self._released) if b.class_bytes <= r[2] <= 2 * b.class_bytes]
                reuse = min(fits)[1] if fits else None
                if reuse is not None:
                    vid, ptr, nb, rf = self._released.pop(reuse)
                    m = self._mapped[b.block_id] = (vid, ptr, nb)
                    fences = tuple(fences) + tuple(rf)
                    self.grow_events += 1
                    self._want_spare(int(b.class_bytes))
            if m is None:
                vid, ptr = C.c_uint64(), C.c_void_p()
                try:
                    LIB.ft_vmm_block_map(self._h, int(b.class_bytes), C.byref(vid), C.byref(ptr))
                except MemoryError:
                    # physical pressure: give parked blocks back, then try once more
                    if not self.reclaim():
                        with self._lock:
                            self.policy.free(b)
                        raise
                    LIB.ft_vmm_block_map(self._h, int(b.class_bytes), C.byref(vid), C.byref(ptr))
                with self._lock:
                    m = self._mapped[b.block_id] = (vid.value, ptr.value, b.class_bytes)
                    fences = tuple(fences) + self._fences_over(ptr.value, b.class_bytes)
                    self.grow_events += 1
                    self._want_spare(int(b.class_bytes))
        return PoolBlock(b, m[0], m[1], m[2], self.device, fences, self)

    def base_tensor(self, blk: PoolBlock) -> torch.Tensor:
        t = self._bases.get(blk.vmm_id)
        if t is None:
            t = self._bases[blk.vmm_id] = as_tensor(blk.ptr, blk.nbytes, self.device)
        return t

    def free(self, blk: PoolBlock, fences=()):
        """Return a block to the policy. ``fences``: events after which no
        kernel or copy of the old holder touches it any more."""
        with self._lock:
            self.policy.free(blk.policy_block)
            if fences:
                self._fences[blk.policy_block.block_id] = tuple(fences)
            if self.policy.mode == "none":           # temporary allocations: give it back now
                self._unmap(blk.policy_block.block_id)

    def commit_store(self, index, data_id: int, node: int, gpu: int, nbytes: int, now_ms: float, producer: str,
                     response: bool, concurrency: float):
        """Index entry + histogram sample + the producer's window in one call
        (``ft_store_commit``); returns (R_window, last_request_ms | None)."""
        rw, last = C.c_double(), C.c_double()
        with self._lock:
            LIB.ft_store_commit(index._h, self.policy._h, int(data_id), int(node), int(gpu), float(nbytes),
                                float(now_ms), producer.encode(), int(bool(response)), float(concurrency),
                                C.byref(rw), C.byref(last))
        return rw.value, (None if last.value != last.value else last.value)

    def _enc(self, func: str) -> bytes:
        b = self._names.get(func)
        if b is None:
            b = self._names[func] = func.encode()
        return b

    def _name_addr(self, func: str) -> int:
        """Address of the producer's NUL-terminated encoded name (the bytes object
        lives in ``_names`` for the pool's lifetime, so the address stays valid)."""
        a = self._addrs.get(func)
        if a is None:
            a = self._addrs[func] = C.cast(C.c_char_p(self._enc(func)), C.c_void_p).value
        return a

    def store_local(self, index, data_id: int, node: int, nbytes: int, now_ms: float, producer: str,
                    response: bool, concurrency: float, blk: "PoolBlock", src_ptr: int, stream: int, hints: int,
                    ready: "Ev"):
        """The same-GPU put in one native call (``ft_store_local``): the stream
        waits on the block's fences, copies the output into it, records
        ``ready``; index entry + histogram sample. Returns (R_window, last | None)."""
        evs = _needed(stream, blk.fences) if blk.fences else ()
        arr = (C.c_void_p * len(evs))(*evs) if evs else self._noev
        name = self._names.get(producer) or self._enc(producer)
        with self._lock, REC_LOCK:
            # (the raw entry point with plain ints / floats: ctypes converts them; the
            # wrapper objects cost ~2 us a call on this path)
            rc = self._store_fn(index._h, self.policy._h, data_id, node, self.device, nbytes, now_ms, name,
                                bool(response), concurrency, blk.ptr, src_ptr, stream, hints, arr, len(evs),
                                ready.h, self._rw, self._last)
            if rc:
                raise_status(rc)
            ready._recorded_on(stream)
            blk.fences = ()                  # the copy waited on them
            rw, last = self._rw.value, self._last.value
        return rw, (None if last != last else last)

    def fetch_local(self, index, data_id: int, blk: "PoolBlock", producer: str, retire: bool, dst_ptr: int,
                    nbytes: int, stream: int, hints: int, waits, done: "Ev", fences=()):
        """The same-GPU get into the consumer's input in one native call
        (``ft_fetch_local``): wait ``waits``, copy, record ``done``; with
        ``retire`` the index entry goes and the block returns to the policy,
        fenced on ``done`` + ``fences``. Returns (R_window, last | None)."""
        evs = _needed(stream, waits) if waits else ()
        arr = (C.c_void_p * len(evs))(*evs) if evs else self._noev
        name = self._names.get(producer) or self._enc(producer)
        with self._lock, REC_LOCK:
            rc = self._fetch_fn(index._h, self.policy._h, data_id, blk.policy_block.block_id if retire else -1,
                                name, bool(retire), dst_ptr, blk.ptr, nbytes, self.device, stream, hints, arr,
                                len(evs), done.h, self._rw, self._last)
            if rc:
                raise_status(rc)
            done._recorded_on(stream)
            if retire:
                blk.policy_block.in_use = False
                self._fences[blk.policy_block.block_id] = (done,) + tuple(fences)
                if self.policy.mode == "none":
                    self.policy._blocks.pop(blk.policy_block.block_id, None)
                    self._unmap(blk.policy_block.block_id)
            rw, last = self._rw.value, self._last.value
        return rw, (None if last != last else last)

    def retire_many(self, index, ids, pblocks, producers, fences):
        """Batched retire (``fetch_many``): parallel lists of data ids, policy blocks,
        producers and each block's fences -> (R_window, last_request) float arrays
        (NaN: no last request), one native call for the index drops, policy frees
        and windows (``ft_retire_many``)."""
        n = len(ids)
        addrs = self._addrs
        ids_a = array.array("q", ids)
        bid_list = [pb.block_id for pb in pblocks]
        bids = array.array("q", bid_list)
        # the char* array as addresses of the cached names (a ctypes c_char_p array
        # built element by element cost ~18 us at 64)
        names = array.array("Q", [addrs.get(f) or self._name_addr(f) for f in producers])
        rws, lasts = array.array("d", bytes(8 * n)), array.array("d", bytes(8 * n))
        with self._lock:
            LIB.ft_retire_many(index._h, self.policy._h, n, C.c_void_p(ids_a.buffer_info()[0]),
                               C.c_void_p(bids.buffer_info()[0]), C.c_void_p(names.buffer_info()[0]),
                               C.c_void_p(rws.buffer_info()[0]),
                               C.c_void_p(lasts.buffer_info()[0]))
            for pb in pblocks:
                pb.in_use = False
            self._fences.update(zip(bid_list, fences))
            if self.policy.mode == "none":
                for pb in pblocks:
                    self.policy._blocks.pop(pb.block_id, None)
                    self._unmap(pb.block_id)
        return rws, lasts

    def commit_retire(self, index, data_id: int, blk: "PoolBlock", fences, producer: str):
        """Index drop + block back to the policy (fenced) + the producer's window
        in one call (``ft_retire_commit``); returns (R_window, last | None)."""
        name = self._names.get(producer) or self._enc(producer)
        with self._lock:
            rc = self._retire_fn(index._h, self.policy._h, data_id, blk.policy_block.block_id, name, self._rw,
                                 self._last)
            if rc:
                raise_status(rc)
            blk.policy_block.in_use = False
            if fences:
                self._fences[blk.policy_block.block_id] = tuple(fences)
            if self.policy.mode == "none":
                self.policy._blocks.pop(blk.policy_block.block_id, None)
                self._unmap(blk.policy_block.block_id)
            rw, last = self._rw.value, self._last.value
        return rw, (None if last != last else last)

    def record(self, func: str, now_ms: float, size: float, concurrency: float):
        with self._lock:
            self.policy.histogram(func).record_execution(now_ms, size, concurrency)

    def shrink(self, now_ms: float, reclaim: bool = True) -> int:
        """Apply the policy's shrink (datastore.py:152-166); returns the bytes it
        dropped. With ``reclaim`` their physical memory is unmapped now,
        otherwise it is parked in the released list until ``reclaim()``."""
        with self._lock:
            dropped = self.policy.shrink(now_ms)
            for b in dropped:
                m = self._mapped.pop(b.block_id, None)
                if m is not None:
                    # the range goes back to its arena now (no driver call); its last
                    # users' fences stay with the range for whoever is carved there next
                    self._release_range(m, self._fences.pop(b.block_id, ()))
            n = sum(b.class_bytes for b in dropped)
        if reclaim:
            self.reclaim()
        return n

    def _release_range(self, m, fences):
        """(lock held) Give a mapped block's range back to its arena; remember its fences."""
        vid, ptr, nb = m
        self._bases.pop(vid, None)
        LIB.ft_vmm_block_unmap(self._h, vid)
        if fences:
            self._range_fences.append((ptr, ptr + nb, tuple(fences)))
            if len(self._range_fences) > 256:            # drop the ranges whose users are done
                self._range_fences = [r for r in self._range_fences if not all(e.query() for e in r[2])]

    def _fences_over(self, ptr, nb) -> tuple:
        """(lock held) Fences of released ranges a new block at [ptr, ptr+nb) overlaps."""
        out = ()
        for lo, hi, f in self._range_fences:
            if lo < ptr + nb and ptr < hi:
                out += f
        return out

    @property
    def reclaimable(self) -> bool:
        return bool(self._released or self._range_fences)

    def reclaim(self) -> int:
        """Give every released block back to its arena (after its last users'
        events), then unmap the arenas no block uses — the physical memory goes
        back to the driver. Returns the bytes of the released blocks."""
        with self._lock:
            gone, self._released = self._released, []
            ranges, self._range_fences = self._range_fences, []
        for _vid, _ptr, _n, fences in gone:
            for ev in fences:
                ev.synchronize()
        for _lo, _hi, fences in ranges:           # nothing may still touch a range of an arena to unmap
            for ev in fences:
                ev.synchronize()
        for vid, _ptr, _n, _f in gone:
            self._bases.pop(vid, None)
            LIB.ft_vmm_block_unmap(self._h, vid)
        self.trim()
        return sum(r[2] for r in gone)

    def trim(self) -> int:
        """Unmap the arenas no block uses (driver calls: only when the GPU is quiet)."""
        cap = 256
        ids, n = (C.c_uint64 * cap)(), C.c_int()
        LIB.ft_vmm_pool_trim(self._h, ids, cap, C.byref(n))
        for i in range(min(n.value, cap)):
            self._notify_unmap(ids[i])
        return n.value

    def locate(self, blk: "PoolBlock") -> tuple:
        """(arena id, offset of the block in it, arena bytes): what another process maps."""
        a, o, n = C.c_uint64(), C.c_uint64(), C.c_uint64()
        LIB.ft_vmm_block_locate(self._h, blk.vmm_id, C.byref(a), C.byref(o), C.byref(n))
        return a.value, o.value, n.value

    def _notify_unmap(self, vid):
        for fn in self.on_unmap:     # importers of an exported block drop their mapping
            fn(vid)

    @property
    def released_bytes(self) -> int:
        return sum(r[2] for r in self._released)

    def hist_window(self, func: str):
        with self._lock:
            return self.policy.hist_window(func)

    def _unmap(self, block_id) -> int:
        m = self._mapped.pop(block_id, None)
        if m is None:
            return 0
        self._release_range(m, self._fences.pop(block_id, ()))   # back to its arena (no driver call)
        return m[2]

    def export_fd(self, blk: PoolBlock) -> int:
        """POSIX fd of the block's arena (pair it with ``locate`` / use ``export``)."""
        fd = C.c_int()
        LIB.ft_vmm_block_export_fd(self._h, blk.vmm_id, C.byref(fd))
        return fd.value

    def export(self, blk: PoolBlock) -> tuple:
        """(fd, arena bytes, offset of the block): ImportedBlock(device, fd, arena_bytes, offset, n)."""
        _arena, off, abytes = self.locate(blk)
        return self.export_fd(blk), abytes, off

    def stats(self) -> dict:
        mapped, reserved, n = C.c_uint64(), C.c_uint64(), C.c_int()
        LIB.ft_vmm_pool_stats(self._h, C.byref(mapped), C.byref(reserved), C.byref(n))
        return {"mapped_bytes": mapped.value, "reserved_va": reserved.value, "blocks": n.value,
                "policy_pool_bytes": self.policy.pool_bytes, "in_use_bytes": self.policy.in_use_bytes,
                "released_bytes": self.released_bytes}


class ImportedBlock:
    """A pool arena exported by another process and mapped here whole (zero
    copy); ``ptr`` is the block at ``offset`` in it, ``nbytes`` long."""

    def __init__(self, device: int, fd: int, arena_bytes: int, offset: int = 0, nbytes: int | None = None):
        base, h = C.c_void_p(), C.c_uint64()
        LIB.ft_vmm_import_fd(int(device), int(fd), int(arena_bytes), C.byref(base), C.byref(h))
        self.device, self.base, self._h = device, base.value, h.value
        self.ptr = base.value + int(offset)
        self.nbytes = int(nbytes) if nbytes is not None else int(arena_bytes) - int(offset)
        self._fin = weakref.finalize(self, LIB.ft_vmm_unimport, h.value)

    def tensor(self, dtype=torch.uint8, shape=None) -> torch.Tensor:
        return as_tensor(self.ptr, self.nbytes, self.device, dtype, shape, owner=self)

    def close(self):
        self._fin()


class IpcEventRing:
    """``k`` interprocess CUDA events of this process on ``device``, handed out
    round-robin; ``handles`` (64 bytes each) let a peer process open them."""

    def __init__(self, device: int, k: int = 16):
        self.device, self.k = device, k
        self.h, self.handles = [], []
        for _ in range(k):
            ev, buf = C.c_void_p(), C.create_string_buffer(64)
            LIB.ft_ipc_event_create(int(device), C.byref(ev), buf)
            self.h.append(ev.value)
            self.handles.append(buf.raw)
        self._next = 0

    def take(self) -> int:
        i = self._next
        self._next = (i + 1) % self.k
        return i

    def record(self, i: int, stream):
        LIB.ft_event_record(C.c_void_p(self.h[i]), C.c_void_p(stream_ptr(stream)))

    def close(self):
        for h in self.h:
            LIB.raw("ft_event_destroy")(C.c_void_p(h))
        self.h = []


class PeerEvents:
    """A peer process's interprocess events, opened from their handles."""

    def __init__(self, device: int, handles):
        self.h = []
        for hd in handles:
            ev = C.c_void_p()
            LIB.ft_ipc_event_open(int(device), bytes(hd), C.byref(ev))
            self.h.append(ev.value)

    def wait(self, i: int, stream):
        """``stream`` waits for the peer's latest record of its event ``i``."""
        LIB.ft_stream_wait_events(C.c_void_p(stream_ptr(stream)), (C.c_void_p * 1)(self.h[i]), 1)

    def close(self):
        for h in self.h:
            LIB.raw("ft_event_destroy")(C.c_void_p(h))
        self.h = []


def send_fd(sock, fd: int, tag: int = 0):
    LIB.ft_fd_send(sock.fileno(), int(fd), int(tag))


def recv_fd(sock) -> tuple:
    fd, tag = C.c_int(), C.c_uint64()
    LIB.ft_fd_recv(sock.fileno(), C.byref(fd), C.byref(tag))
    return fd.value, tag.value


class Pacer:
    """Live PCIe mover + per-function bandwidth-share scheduler (``ft_pacer``).

    One per tube: every host->GPU leg is submitted as a stage of routes
    (dataplane.py:203-250); managed stages are paced at the arbiter's rate in
    5 x 2 MB batches by a native thread (engine.py:537-646), unmanaged ones are
    issued at once. ``submit`` returns at once; the consumer stream is parked
    on the stage's completion word, so later work on it sees the bytes."""

    def __init__(self, bw_all_gbps: float, batch_chunks: int, chunk_bytes: int, staging_slots: int = 4,
                 host_ring_bytes: int = 0, logging: bool = False, links: int = 1, adapt: bool = True):
        from ._lib import RouteC
        self._route_t = RouteC
        h = C.c_void_p()
        flags = int(bool(logging)) | (0 if adapt else 2)
        LIB.ft_pacer_create(float(bw_all_gbps), int(links), int(batch_chunks), int(chunk_bytes), int(staging_slots),
                            int(host_ring_bytes), flags, C.byref(h))
        self._h = h

    def submit(self, key: str, managed: bool, slo_ms: float, infer_ms: float, per_branch_cap_gbps: float,
               dst_ptr: int, dst_dev: int, host_ptr: int, nbytes: int, host_pinned: bool, routes: list,
               consumer_stream: int) -> int:
        """routes: [(stage_dev, force_staging, off, len, ce_stream, fw_stream)] -> ticket"""
        arr = (self._route_t * len(routes))(*[self._route_t(int(a), int(b), int(c), int(d), e, f)
                                               for a, b, c, d, e, f in routes])
        t = C.c_uint64()
        LIB.ft_pacer_submit(self._h, key.encode(), int(bool(managed)), float(slo_ms), float(infer_ms),
                            float(per_branch_cap_gbps), C.c_void_p(dst_ptr), int(dst_dev), C.c_void_p(host_ptr),
                            int(nbytes), int(bool(host_pinned)), len(routes), arr, C.c_void_p(consumer_stream),
                            C.byref(t))
        return t.value

    def submit_routes(self, key: str, managed: bool, slo_ms: float, infer_ms: float, per_branch_cap_gbps: float,
                      dst_ptr: int, dst_dev: int, host_ptr: int, nbytes: int, host_pinned: bool, k: int, routes,
                      consumer_stream: int) -> int:
        """``submit`` with the routes already in a ft_route array (``ft_h2g_routes``) -> ticket"""
        t = C.c_uint64()
        LIB.ft_pacer_submit(self._h, key.encode(), int(managed), float(slo_ms), float(infer_ms),
                            float(per_branch_cap_gbps), C.c_void_p(dst_ptr), int(dst_dev), C.c_void_p(host_ptr),
                            int(nbytes), int(host_pinned), int(k), routes, C.c_void_p(consumer_stream), C.byref(t))
        return t.value

    def submit_d2h(self, key: str, managed: bool, slo_ms: float, infer_ms: float, per_branch_cap_gbps: float,
                   host_ptr: int, src_ptr: int, src_dev: int, nbytes: int, routes: list, producer_stream: int) -> int:
        """GPU -> pinned host; routes as for submit (stage_dev == src_dev: direct) -> ticket"""
        arr = (self._route_t * len(routes))(*[self._route_t(int(a), int(b), int(c), int(d), e, f)
                                               for a, b, c, d, e, f in routes])
        t = C.c_uint64()
        LIB.ft_pacer_submit_d2h(self._h, key.encode(), int(bool(managed)), float(slo_ms), float(infer_ms),
                                float(per_branch_cap_gbps), C.c_void_p(host_ptr), C.c_void_p(src_ptr), int(src_dev),
                                int(nbytes), len(routes), arr, C.c_void_p(producer_stream), C.byref(t))
        return t.value

    def done(self, ticket: int) -> bool:
        d = C.c_int()
        LIB.ft_pacer_done(self._h, int(ticket), C.byref(d))
        return bool(d.value)

    def wait(self, ticket: int, timeout_ms: float = -1.0):
        LIB.ft_pacer_wait(self._h, int(ticket), float(timeout_ms))

    def stats(self) -> dict:
        out = (C.c_uint64 * 7)()
        LIB.ft_pacer_stats(self._h, out, 7)
        keys = ("stages", "managed_stages", "batches", "bytes", "active", "failed", "blocking")
        return dict(zip(keys, list(out)))

    def now_ms(self) -> float:
        t = C.c_double()
        LIB.ft_pacer_now_ms(self._h, C.byref(t))
        return t.value

    def trace(self) -> list:
        from ._lib import json_out
        return json_out("ft_pacer_trace_json", self._h)

    def log(self) -> list:
        from ._lib import json_out
        return json_out("ft_pacer_log_json", self._h)

    def state(self) -> dict:
        from ._lib import json_out
        return json_out("ft_pacer_state_json", self._h)

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            LIB.ft_pacer_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass

"""Live workflow runtime on B200: requests walk their
workflow DAG, gFuncs run on their placed GPU in FIFO order (temporal sharing,
engine.py:310-338), and every intermediate payload moves through the
FaaSTube put/get API — host->gFunc for request inputs, gFunc->gFunc between
stages, gFunc->host for responses (engine.py:284-298, 342-464).

The request trace, branch draws, payload sizes, placement and per-function
SLOs are the reference's (``workload.py``, golden-checked), so the same seed
replays the simulator's workload on real hardware; latency percentiles use the
reference's nearest-rank estimator (simcore.py:247-252).

Compute stand-ins: ``"sleep"`` occupies the function's stream for its
compute_latency_ms on the GPU's global timer (``ft_spin_ns``: a cycle-count
sleep would stretch 16x on an idle-clocked GPU) — the reference's compute
model; ``"model"`` runs random-init convolutional models on the
payload (config 4: decode -> detector -> recognizers on 1080p frames).
"""

from __future__ import annotations

import contextlib
import ctypes as C
import math
import os
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import torch

from . import device as dev
from .simcore import PHASES
from .workload import Request, Workflow

FRAME = (3, 1080, 1920)   # synthetic 1080p RGB uint8 frame = 6,220,800 B


def nearest_rank(vals, pct):
    vals = sorted(vals)
    return vals[max(1, math.ceil(pct / 100.0 * len(vals))) - 1] if vals else None


@dataclass
class Record:
    rid: int
    workflow: str
    arrival_ms: float
    slo_ms: float
    start_ms: float = 0.0
    end_ms: float | None = None
    phases: dict = field(default_factory=lambda: {p: 0.0 for p in PHASES})
    extra: dict = field(default_factory=dict)   # time outside the reference's phases (cFunc host compute)


class _Models:
    """Random-init conv stand-ins (bf16), one set per GPU; each call processes a
    fixed batch of BATCH 1080p frames taken from the payload."""

    BATCH = 4

    def __init__(self, device):
        g = torch.Generator(device="cpu").manual_seed(1234)
        mk = lambda co, ci, k: (torch.randn(co, ci, k, k, generator=g) * (ci * k * k) ** -0.5).to(
            device=device, dtype=torch.bfloat16)
        self.pre = mk(3, 3, 3)
        self.det = [mk(32, 3, 3), mk(64, 32, 3), mk(64, 64, 3)]
        self.rec = [mk(64, 3, 3), mk(128, 64, 3), mk(128, 128, 3)]

    def run(self, fid, x: torch.Tensor, out_bytes: int) -> torch.Tensor:
        import torch.nn.functional as F
        n = x.numel() * x.element_size()
        fb = FRAME[0] * FRAME[1] * FRAME[2]
        frames = self.BATCH                      # fixed shapes: no per-request kernel selection
        flat_in = x.reshape(-1).view(torch.uint8)
        if n < frames * fb:                      # short payload: zero-pad the frame batch
            pad = torch.zeros(frames * fb, dtype=torch.uint8, device=x.device)
            pad[:n] = flat_in
            flat_in = pad
        h = flat_in[: frames * fb].view(frames, *FRAME).to(torch.bfloat16)
        if "pre" in fid or "denoise" in fid:
            h = F.conv2d(h, self.pre, padding=1)
        elif "det" in fid or "yolo" in fid:
            h = F.avg_pool2d(h, 4)
            for w in self.det:
                h = F.relu(F.conv2d(h, w, padding=1, stride=2))
        else:
            h = F.avg_pool2d(h, 8)
            for w in self.rec:
                h = F.relu(F.conv2d(h, w, padding=1, stride=2))
        flat = h.reshape(-1).view(torch.uint8)
        out = dev.empty_shared(out_bytes, x.device.index)
        k = min(out_bytes, flat.numel())
        out[:k] = flat[:k]
        if k < out_bytes:
            out[k:] = 0
        return out


def build_requests_for(wf: Workflow, pattern: str, rate: float, duration_s: float, seed: int) -> list:
    from .workload import build_requests, gen_workload
    return build_requests(wf, gen_workload(pattern, rate, duration_s, seed), seed)


_MODELS = {}
_MODELS_LOCK = threading.Lock()


def _models(gpu: int) -> "_Models":
    """One set of random-init stand-in models per GPU for the process (fixed seed)."""
    with _MODELS_LOCK:
        m = _MODELS.get(gpu)
        if m is None:
            m = _MODELS[gpu] = _Models(f"cuda:{gpu}")
        return m


class Runtime:
    def __init__(self, tube, compute: str = "sleep", workers: int = 32):
        self.tube = tube
        self.compute = compute
        self.pool = ThreadPoolExecutor(workers)
        self.gpu_locks = {g: threading.Lock() for g in tube.gpus}
        self._host_bufs = {}
        self.records: list[Record] = []
        self._rec_lock = threading.Lock()
        self.pool_timeline = []
        self._tls = threading.local()

    # ------------------------------------------------------------ one request
    def _host_out(self, fid, nbytes):
        """Synthetic cFunc output / request payload: a prefix of one pinned buffer
        per function (content is not request specific). The buffers are sized
        before the trace starts (``_size_host_bufs``): a 512 MB cudaHostAlloc +
        fill inside a request cost it 350 ms that no phase accounted for."""
        with self._rec_lock:
            buf = self._host_bufs.get(fid)
            if buf is None or buf.numel() < nbytes:
                buf = self._host_bufs[fid] = torch.empty(max(1, nbytes), dtype=torch.uint8,
                                                         pin_memory=True).fill_(7)
        return buf[:nbytes]

    def _size_host_bufs(self, jobs):
        need = {}
        for wf, where, reqs in jobs:
            for r in reqs:
                need["gateway"] = max(need.get("gateway", 0), int(r.input_bytes))
                for fid, (kind, _) in where.items():
                    if kind == "gpu":
                        continue
                    outs = [e for e in wf.outs(fid) if (e.src, e.dst) in r.fired]
                    n = int(r.response_bytes if not outs else max(r.edge_bytes[(e.src, e.dst)] for e in outs))
                    need[fid] = max(need.get(fid, 0), n)
        for fid, n in need.items():
            self._host_out(fid, n)

    def _compute(self, fid, gpu, ms, x, out_bytes):
        if self.compute == "model":
            return _models(gpu).run(fid, x, out_bytes)
        dev.LIB.ft_spin_ns(int(ms * 1e6), int(gpu), C.c_void_p(torch.cuda.current_stream(gpu).cuda_stream))
        return dev.empty_shared(out_bytes, gpu).fill_(len(fid) & 0xFF)

    def _stream(self, gpu) -> torch.cuda.Stream:
        """This worker thread's own stream on ``gpu`` (a function's CUDA context):
        its fetches park only its own stream, never another tenant's."""
        d = getattr(self._tls, "streams", None)
        if d is None:
            d = self._tls.streams = {}
        if gpu not in d:
            # torch's pool stream: the caching allocator keeps per-stream free lists, and a
            # private stream per worker would fragment it (measured: seconds of cudaMalloc /
            # cudaFree stalls); the tube's own copy-engine streams are private
            d[gpu] = torch.cuda.Stream(gpu)
        return d[gpu]

    def _request(self, wf: Workflow, where: dict, req: Request, rec: Record, t0: float):
        with contextlib.ExitStack() as es:
            for g in self.tube.gpus:
                es.enter_context(torch.cuda.stream(self._stream(g)))
            self._request_on_streams(wf, where, req, rec, t0)

    def _request_on_streams(self, wf: Workflow, where: dict, req: Request, rec: Record, t0: float):
        tube = self.tube
        now = lambda: (time.perf_counter() - t0) * 1e3
        rec.start_ms = now()
        active = set(wf.entries())
        for fid in wf.order():
            if fid not in active and any(e.src in active and (e.src, e.dst) in req.fired for e in wf.ins(fid)):
                active.add(fid)
        # request payload arrives at the gateway (host memory)
        in_id = tube.unique_id()
        payload = self._host_out("gateway", int(req.input_bytes))
        entries = [f for f in wf.entries() if f in active]
        t_g = now()
        tube.store(in_id, payload, producer="gateway", consumers=max(1, len(entries)))
        rec.extra["store"] = now() - t_g
        outputs = {}
        for fid in wf.order():
            if fid not in active:
                continue
            f = wf.func(fid)
            kind, loc = where[fid]
            gpu = loc if kind == "gpu" else None
            ins = [e for e in wf.ins(fid) if (e.src, e.dst) in req.fired and e.src in active]
            t_in = now()
            if not ins:
                x = tube.fetch(in_id, device=gpu, consumer=fid, slo_ms=f.slo_ms, infer_ms=f.infer_ms)
                if gpu is not None:
                    torch.cuda.current_stream(gpu).synchronize()   # the paced H2G stage landed
                rec.phases["host_to_gfunc"] += now() - t_in
            else:
                xs = []
                for e in ins:
                    xs.append(tube.fetch(outputs[e.src], device=gpu, consumer=fid, slo_ms=f.slo_ms,
                                         infer_ms=f.infer_ms))
                if gpu is not None:
                    torch.cuda.current_stream(gpu).synchronize()   # inputs landed (phase accounting)
                phase = "gfunc_to_gfunc" if gpu is not None and where[ins[0].src][0] == "gpu" else "host_to_gfunc"
                rec.phases[phase] += now() - t_in
                x = xs[0]
            outs = [e for e in wf.outs(fid) if (e.src, e.dst) in req.fired and e.dst in active]
            sink = not outs
            out_bytes = int(req.response_bytes if sink else max(req.edge_bytes[(e.src, e.dst)] for e in outs))
            t_c = now()
            if gpu is None:
                time.sleep(f.compute_ms / 1e3)              # cFunc on a host core
                y = self._host_out(fid, out_bytes)
                rec.extra["cfunc"] = rec.extra.get("cfunc", 0.0) + now() - t_c
            else:
                with self.gpu_locks[gpu], torch.cuda.device(gpu):   # GPU FIFO (temporal sharing)
                    t_q = now()
                    rec.phases["queuing"] += t_q - t_c
                    y = self._compute(fid, gpu, f.compute_ms, x, out_bytes)
                    torch.cuda.current_stream(gpu).synchronize()
                    rec.phases["compute"] += now() - t_q
            did = tube.unique_id()
            t_s = now()
            tube.store(did, y, producer=fid, response=sink and gpu is not None, consumers=max(1, len(outs)))
            if sink:
                if gpu is not None:
                    tube.response(did)                      # D2H of the response lands on the host
                    tube.release(did)
                rec.phases["host_to_gfunc"] += now() - t_s
            else:
                rec.extra["store"] = rec.extra.get("store", 0.0) + now() - t_s
            outputs[fid] = did
        rec.end_ms = now()

    # ------------------------------------------------------------ driver
    @staticmethod
    def warm_daemon(tube, jobs: list, compute: str = "sleep", seconds: float = 0.5):
        """One untimed pass over the first ``seconds`` of the trace on ``tube``
        (pool blocks, pinned buffers, allocator segments, kernels): measured
        runs then see a warm daemon, as a long-running deployment does."""
        warm = [(wf, where, [r for r in reqs if r.arrival_ms < seconds * 1e3]) for wf, where, reqs in jobs]
        Runtime(tube, compute=compute).run(warm, seconds, drain_s=60)

    @staticmethod
    def max_throughput(tube, wf, where, pattern: str = "sporadic", duration_s: float = 1.0,
                       compute: str = "sleep", rate_lo: float = 1.0, rate_hi: float = 256.0,
                       iterations: int = 4, seed: int = 0, slo_ms: float | None = None) -> dict:
        """harness.max_throughput (harness.py:383-428) on the live runtime: the
        highest offered rate whose p99 stays within the workflow SLO with >= 95%
        of the offered requests completed — doubling from ``rate_lo``, then
        ``iterations`` bisection steps. Each trial replays the reference's trace
        for that rate on ``tube`` (a warm daemon)."""
        slo = slo_ms if slo_ms else (wf.slo_ms or 1e12)
        trials = []

        def trial(rate):
            reqs = build_requests_for(wf, pattern, rate, duration_s, seed)
            # a daemon that has been serving this traffic: the trial's own requests
            # replayed untimed first, 5x compressed in time. Payload sizes are drawn per
            # request, and the first store of a size class the pool never held maps a
            # block (a cuMemCreate of up to 192 MB: 25-95 ms) — one such store decided
            # whole trials (p99 of 15 requests is their maximum)
            warm = [Request(r.rid, r.workflow, r.arrival_ms / 5.0, r.edge_bytes, r.fired, r.input_bytes,
                            r.response_bytes) for r in reqs]
            Runtime(tube, compute=compute).run([(wf, where, warm)], duration_s / 5.0, drain_s=60, idle_s=0.0)
            rt = Runtime(tube, compute=compute)
            rep = rt.run([(wf, where, reqs)], duration_s, drain_s=30, idle_s=0.0)
            ok = not reqs or (rep["requests_completed"] >= 0.95 * len(reqs) and rep.get("p99_ms") is not None
                              and rep["p99_ms"] <= slo)       # no arrival drawn: vacuously met
            trials.append({"rate": round(rate, 3), "ok": ok, "p99_ms": rep.get("p99_ms"),
                           "completed": rep["requests_completed"], "offered": len(reqs),
                           **({"worst": rep["worst"]} if "worst" in rep and not ok else {})})
            return ok, rep

        lo, hi, last = 0.0, None, None
        rate = rate_lo
        while rate <= rate_hi:
            ok, rep = trial(rate)
            if not ok:
                hi = rate
                break
            lo, last = rate, rep
            rate *= 2
        if lo == 0.0:
            return {"max_rps": 0.0, "slo_ms": slo, "trials": trials, "diagnostic": "SLO unachievable at the lowest rate"}
        if hi is not None:
            for _ in range(iterations):
                mid = (lo + hi) / 2
                ok, rep = trial(mid)
                if ok:
                    lo, last = mid, rep
                else:
                    hi = mid
        return {"max_rps": round(lo, 3), "slo_ms": round(slo, 3), "p99_ms_at_max": last.get("p99_ms"),
                "trials": trials}

    def run(self, jobs: list, duration_s: float, drain_s: float = 30.0, sample_ms: float = 50.0,
            idle_s: float = 1.0) -> dict:
        """jobs: [(workflow, placement, [Request])]; arrivals replayed in real time.
        The interpreter's GIL switch interval is lowered for the run
        (FT_SWITCH_INTERVAL_S, default 1 ms): 32 function threads share one
        interpreter, and at the default 5 ms a thread ready to issue a
        transfer or a kernel can wait several switch intervals."""
        old = sys.getswitchinterval()
        sys.setswitchinterval(float(os.environ.get("FT_SWITCH_INTERVAL_S", "0.001")))
        try:
            return self._run(jobs, duration_s, drain_s, sample_ms, idle_s)
        finally:
            sys.setswitchinterval(old)

    def _run(self, jobs, duration_s, drain_s, sample_ms, idle_s) -> dict:
        events = sorted(((r.arrival_ms, i, wf, where, r) for i, (wf, where, reqs) in enumerate(jobs) for r in reqs),
                        key=lambda e: (e[0], e[1], e[4].rid))
        # warm-up outside the trace: every worker thread sets up its CUDA state — its
        # streams and, with model compute, its cuDNN/cuBLAS handles and workspaces (per
        # thread in torch: a worker's first conv otherwise costs 0.3-2 s inside the trace)
        n_workers = self.pool._max_workers  # noqa: SLF001
        barrier = threading.Barrier(n_workers)
        gfuncs = sorted({(fid, g) for _, where, _ in jobs for fid, (kind, g) in where.items() if kind == "gpu"})

        def warm_worker(_):
            barrier.wait(timeout=60)         # one task per worker thread
            for g in self.tube.gpus:
                with torch.cuda.stream(self._stream(g)):
                    if self.compute == "model":
                        for fid, fg in gfuncs:
                            if fg == g:
                                self._compute(fid, g, 0.0, torch.zeros(1 << 20, dtype=torch.uint8,
                                                                       device=f"cuda:{g}"), 1 << 20)
                    torch.cuda.current_stream(g).synchronize()

        list(self.pool.map(warm_worker, range(n_workers)))
        self._size_host_bufs(jobs)
        for wf, where, reqs in jobs:
            if reqs:
                r0 = reqs[0]
                warm = Request(-1, r0.workflow, 0.0, r0.edge_bytes, r0.fired, r0.input_bytes, r0.response_bytes)
                self.pool.submit(self._request, wf, where, warm, Record(-1, wf.name, 0.0, 0.0),
                                 time.perf_counter()).result()
        if self.compute == "model":              # build/warm the models outside the trace
            for wf, where, _ in jobs:
                for fid, (kind, g) in where.items():
                    if kind == "gpu":
                        with torch.cuda.device(g):
                            self._compute(fid, g, 0.0, torch.zeros(1 << 20, dtype=torch.uint8, device=f"cuda:{g}"),
                                          1 << 20)
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        futs = []
        stop = threading.Event()

        def sampler():
            while not stop.is_set():
                st = {g: p.stats() for g, p in self.tube.pools.items()}
                # (t, pool bytes the elastic policy holds, bytes in use, physically mapped)
                self.pool_timeline.append(((time.perf_counter() - t0) * 1e3,
                                           sum(s["policy_pool_bytes"] for s in st.values()),
                                           sum(s["in_use_bytes"] for s in st.values()),
                                           sum(s["mapped_bytes"] for s in st.values())))
                stop.wait(sample_ms / 1e3)

        smp = threading.Thread(target=sampler, daemon=True)
        smp.start()
        for t_ms, _, wf, where, r in events:
            dt = t_ms / 1e3 - (time.perf_counter() - t0)
            if dt > 0:
                time.sleep(dt)
            rec = Record(r.rid, wf.name, t_ms, wf.slo_ms or float("inf"))
            with self._rec_lock:
                self.records.append(rec)
            futs.append(self.pool.submit(self._request, wf, where, r, rec, t0))
        deadline = time.perf_counter() + drain_s
        errors = []
        for fu in futs:
            try:
                fu.result(timeout=max(0.1, deadline - time.perf_counter()))
            except Exception as exc:  # noqa: BLE001 - reported, not hidden
                errors.append(repr(exc))
        stop.set()
        smp.join()
        out = self.summary(duration_s, errors)
        # elasticity: after the trace, idle past the reservation windows and let
        # the pool policy shrink (engine.py:656-665)
        t_idle = time.perf_counter()
        while time.perf_counter() - t_idle < idle_s:
            self.tube.maintain()
            time.sleep(0.05)
        self.tube.maintain()
        if idle_s > 0:
            self.tube.reclaim()              # quiet now: physical memory of dropped blocks goes back
        out["pool_after_idle_bytes"] = sum(p.stats()["policy_pool_bytes"] for p in self.tube.pools.values())
        out["mapped_after_idle_bytes"] = sum(p.stats()["mapped_bytes"] for p in self.tube.pools.values())
        return out

    def summary(self, duration_s: float, errors=()) -> dict:
        done = [r for r in self.records if r.end_ms is not None]
        lat = [r.end_ms - r.arrival_ms for r in done]
        out = {"requests_seen": len(self.records), "requests_completed": len(done),
               "throughput_rps": round(len(done) / duration_s, 3), "errors": list(errors)[:5],
               "peak_pool_bytes": max((p[1] for p in self.pool_timeline), default=0),
               "final_pool_bytes": self.pool_timeline[-1][1] if self.pool_timeline else 0,
               "peak_mapped_bytes": max((p[3] for p in self.pool_timeline), default=0)}
        if done:
            out["p50_ms"] = round(nearest_rank(lat, 50), 4)
            out["p99_ms"] = round(nearest_rank(lat, 99), 4)
            out["slo_violation_rate"] = round(sum(1 for r in done if r.end_ms - r.arrival_ms > r.slo_ms + 1e-9)
                                              / len(done), 4)
            out["phase_p99_ms"] = {p: round(nearest_rank([r.phases[p] for r in done], 99), 4) for p in PHASES}
            per = {}
            for r in done:
                per.setdefault(r.workflow, []).append(r.end_ms - r.arrival_ms)
            out["per_workflow_p99_ms"] = {k: round(nearest_rank(v, 99), 4) for k, v in sorted(per.items())}
            out["worst"] = self.breakdown(max(done, key=lambda r: r.end_ms - r.arrival_ms))
            st = self.tube.stats
            out["tube"] = {"migrated_bytes": st.get("migrated_bytes", 0), "reload_bytes": st.get("reload_bytes", 0),
                           "grow_events": sum(p.grow_events for p in self.tube.pools.values()),
                           "spares_mapped": sum(p.spares_mapped for p in self.tube.pools.values()),
                           "slow_stores": [list(x) for x in list(self.tube.slow_stores)[-6:]]}
            out["_lat"] = lat                # raw latencies (callers pooling runs pop it)
            out["_slo_miss"] = [r.end_ms - r.arrival_ms > r.slo_ms + 1e-9 for r in done]
        return out

    @staticmethod
    def breakdown(r: Record) -> dict:
        """Where one request's latency went: dispatch delay, the reference's
        phases, cFunc host compute and what no phase covers."""
        return {"rid": r.rid, "workflow": r.workflow, "arrival_ms": round(r.arrival_ms, 1),
                "latency_ms": round(r.end_ms - r.arrival_ms, 2), "dispatch_ms": round(r.start_ms - r.arrival_ms, 2),
                "cfunc_ms": round(r.extra.get("cfunc", 0.0), 2), "store_ms": round(r.extra.get("store", 0.0), 2),
                "phases": {k: round(v, 2) for k, v in r.phases.items() if v},
                "unaccounted_ms": round(r.end_ms - r.start_ms - sum(r.phases.values()) - sum(r.extra.values()), 2)}

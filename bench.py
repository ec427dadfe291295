#!/usr/bin/env python
"""FaaSTube-on-B200 benchmark (BASELINE.json metric: "H2G/G2G pass GB/s &
p99 latency vs PCIe/NVLink peak; workflow req/s").

Headline workload (config 1): a 2-function pipeline — the
producer gFunc stores its 64 MiB fp16 output, the consumer gFunc fetches it
into its own input buffer, through the Listing-1 API (FaaSTube.store /
FaaSTube.fetch). One step = one such pass. At N=1 both functions share GPU 0;
under torchrun each rank runs its own pipeline on its GPU (weak scaling,
replicas — the data path has no collective).

  value  : payload bytes delivered / device time, inputs resident in HBM
  e2e    : same pass through the public API with the producer's input coming
           from pinned host memory (tube.fetch of a host object) and the
           consumer's digest read back to the host, wall-clocked
  roofline: the dominant kernel (k_copy_bulk, TMA bulk copy) vs measured HBM
  cpu_baseline / --impl reference: the reference's CPU host-memory path
           (oracle/host_path.py — infless_plus: store into host shared
           memory, fetch out of it) on the host cores

Extras: h2g (config 2 at k=1: 1 GiB pinned -> GPU over the copy engine, vs
the live-measured CE peak) and a same-GPU size sweep (config 3 at 1 GPU:
zero-copy handoff latency and copy-into-input bandwidth, p50/p99).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MIB = 1 << 20
PAYLOAD_SHAPE = (32, 1024, 1024)          # fp16 -> 64 MiB (config 1)
METRIC = "H2G/G2G pass GB/s & p99 latency vs PCIe/NVLink peak; workflow req/s"
L2_FLUSH_BYTES = 256 * MIB


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-s", type=float, default=10.0)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--max-throughput", action="store_true",
                    help="also search config 4's max req/s per strategy (harness.max_throughput; minutes)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def nearest_rank(sorted_vals, pct):
    import math
    return sorted_vals[max(1, math.ceil(pct / 100.0 * len(sorted_vals))) - 1]   # simcore.py:247-252


# ----------------------------------------------------------------- CPU path
def cpu_host_path(sample_s: float, nbytes: int, threads: int | None = None) -> dict:
    """The reference's CPU host-memory path (oracle port), bounded sample."""
    import numpy as np
    from oracle.host_path import HostMemoryStore
    hs = HostMemoryStore(threads=threads)
    rng = np.random.default_rng(0)
    payload = rng.integers(0, 256, nbytes, dtype=np.uint8)
    out = np.empty(nbytes, dtype=np.uint8)
    times = []
    t_end = time.perf_counter() + sample_s
    for i in range(3):  # warm-up
        did = hs.unique_id()
        hs.store(did, payload)
        hs.fetch(did, out)
        hs.drop(did)
    while time.perf_counter() < t_end or len(times) < 3:
        did = hs.unique_id()
        t0 = time.perf_counter()
        hs.store(did, payload)          # producer output -> host shared memory
        hs.fetch(did, out)              # host shared memory -> consumer input
        times.append(time.perf_counter() - t0)
        hs.drop(did)
    assert np.array_equal(out, payload)
    hs.close()
    times.sort()
    return {"pass_ms_p50": nearest_rank(times, 50) * 1e3, "pass_ms_p99": nearest_rank(times, 99) * 1e3,
            "gbps": nbytes / statistics.mean(times) / 1e9, "passes": len(times), "threads": hs.threads}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    nbytes = 2 * PAYLOAD_SHAPE[0] * PAYLOAD_SHAPE[1] * PAYLOAD_SHAPE[2]
    threads = len(os.sched_getaffinity(0))
    per = []
    for _ in range(args.warmup):
        cpu_host_path(0.05, nbytes, threads)
    t_all = time.perf_counter()
    for _ in range(args.steps):
        r = cpu_host_path(max(0.2, args.cpu_sample_s / max(1, args.steps)), nbytes, threads)
        per.append(r)
    wall = time.perf_counter() - t_all
    gbps = statistics.mean(r["gbps"] for r in per)
    p99 = max(r["pass_ms_p99"] for r in per)
    line = {"metric": METRIC, "value": round(gbps, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "config1: 2-function pipeline, 64 MiB fp16 put/get (reference CPU host-memory path)",
                       "payload_bytes": nbytes, "path": "oracle/host_path.py infless_plus restatement"},
            "p99_pass_ms": round(p99, 4),
            "cpu_baseline": {"value": round(gbps, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                             "sample": f"{sum(r['passes'] for r in per)} store+fetch passes of 64 MiB"},
            "e2e": {"value": round(gbps, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU path
class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self) -> dict:
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.count(",") >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "MEASURED_PEAKS.json"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def profile_traffic():
    """dram bytes per launch of the copy kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_copy_summary.json")
    try:
        with open(p) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except OSError:
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    shared = world > ndev          # more ranks than GPUs (path smoke test): ranks share devices
    if world > 1:
        # only barriers and one max-reduction of timings go through the process group
        dist.init_process_group("gloo" if shared else "nccl")
    g = local % ndev
    torch.cuda.set_device(g)
    from paper_2411_01830_b200 import device as dev
    from paper_2411_01830_b200.tube import FaaSTube

    if world > 1:
        # one process per GPU, each driving only its own GPU: its host->GPU legs use its own
        # PCIe root (replicas; no striping through GPUs another rank drives)
        from paper_2411_01830_b200.strategies import strategy_preset
        tube = FaaSTube(strategy_preset("faastube", parallel_pcie=False), topology=_single_gpu_topology(g), gpus=[g])
    else:
        tube = FaaSTube("faastube")            # drives every visible GPU: H2G stripes over all their roots
    gen = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn(PAYLOAD_SHAPE, generator=gen).half().to(f"cuda:{g}")   # producer output (in HBM)
    nbytes = x.nbytes
    inp = torch.empty_like(x)                                                # consumer input buffer
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=f"cuda:{g}")
    s = torch.cuda.current_stream(g)
    pair, pair_error = None, None
    if world > 1:
        # N > 1: rank r's producer hands its output to rank r+1's consumer over
        # NVLink (exported pool block + device doorbells) — pairs.CrossPair
        try:
            from paper_2411_01830_b200.pairs import CrossPair
            sock_dir = f"/tmp/ft_bench_{os.environ.get('MASTER_PORT', '0')}"
            os.makedirs(sock_dir, exist_ok=True)
            pair = CrossPair(tube, g, rank, world, sock_dir, nbytes, dist.barrier)
        except Exception as exc:  # noqa: BLE001 - reported; falls back to same-GPU replicas
            pair_error = repr(exc)

    def one_pass():
        if pair is not None:
            pair.produce(x)
            pair.consume(inp)
            return
        did = tube.unique_id()
        tube.store(did, x, producer="producer")
        tube.fetch(did, device=g, out=inp, consumer="consumer")

    def flush_l2(i):
        # inputs < L2 (126 MB): evict between passes; the read leaves L2 clean
        # so no write-back of flush data lands inside the timed pass
        flush.fill_(i & 0xFF)
        flush.amax()

    # ---- warm-up (>= W passes and >= 0.5 s under the clock sampler), then K timed passes
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with Clocks(g) as clk:
        t_w = time.perf_counter()
        i = 0
        # N > 1: the producer->consumer ring counts steps on both ends, so every rank runs
        # the same number of warm-up passes (a time-based count differed by one between
        # ranks and left a doorbell waiting for a step its peer never ran)
        while i < max(3, args.warmup) or (world == 1 and time.perf_counter() - t_w < 0.5):
            flush_l2(i)
            one_pass()
            i += 1
        if world > 1:
            while time.perf_counter() - t_w < 0.5:   # same clock-sampling window, no extra passes
                time.sleep(0.01)
        torch.cuda.synchronize()
        assert torch.equal(inp.view(torch.uint8), x.view(torch.uint8)), "delivered bytes differ"
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = tube.stats["bytes_local"]
        t_timed = time.perf_counter()
        for i in range(args.steps):
            flush_l2(i)
            starts[i].record(s)
            one_pass()
            ends[i].record(s)
        torch.cuda.synchronize()
        timed_wall_s = time.perf_counter() - t_timed
    if world > 1:
        dist.barrier()
    per_ms = sorted(a.elapsed_time(b) for a, b in zip(starts, ends))
    total_ms = sum(per_ms)
    copies = (tube.stats["bytes_local"] - launches0) // nbytes
    gpu_launches = int(copies)                       # one k_copy_bulk per store + one per fetch
    if pair is not None:                             # wait+copy+signal on each side
        gpu_launches = 6 * args.steps
        pair.check()
    assert torch.equal(inp.view(torch.uint8), x.view(torch.uint8)), "delivered bytes differ"

    # ---- dominant kernel: k_copy_bulk on the same buffers, CUDA events on its stream
    kern = []
    for i in range(args.steps):
        flush_l2(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        dev.copy(inp.data_ptr(), x.data_ptr(), nbytes, g, s, dev.ENGINE_BULK)
        b.record(s)
        kern.append((a, b))
    torch.cuda.synchronize()
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in kern)

    # ---- variant: producer writes into a tube-allocated output (zero-copy store, 1 copy / pass)
    xo = tube.empty(PAYLOAD_SHAPE, torch.float16, device=g)
    xo.copy_(x)
    zc = []
    for i in range(max(3, args.warmup) + args.steps):
        flush_l2(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        did = tube.unique_id()
        tube.store(did, xo, producer="producer", consumers=1)
        tube.fetch(did, device=g, out=inp, consumer="consumer")
        b.record(s)
        zc.append((a, b))
        xo = tube.empty(PAYLOAD_SHAPE, torch.float16, device=g)   # next request's output buffer
        xo.copy_(x) if i < max(3, args.warmup) else None
    torch.cuda.synchronize()
    zc_ms = sorted(a.elapsed_time(b) for a, b in zc[max(3, args.warmup):])
    peaks, peak_src = measured_peaks()
    achieved = 2 * nbytes / (kern_ms * 1e-3) / 1e9   # read + write bytes per launch

    # ---- e2e through the public API with host buffers. Listing-1 usage: the request
    # payload is stored from (pinned) host memory; the producer fetches it into an
    # output buffer carved from the tube's pool (tube.empty — the next request's is
    # allocated while this one's H2D tail is in flight), stores it (zero copy), and
    # the consumer on the same GPU fetches a zero-copy view and reads it (digest ->
    # 16 B D2H). The copy-semantics variant (producer's own buffer, consumer's input
    # buffer: 2 HBM copies per step) is reported beside it.
    host_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    host_in.copy_(x.view(-1).view(torch.uint8).cpu())
    fp = dev.Fingerprint(g)
    ref_digest = dev.fingerprint_host(host_in)
    e2e = []
    nxt = tube.empty((nbytes,), torch.uint8, device=g)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        out = nxt
        d_in = tube.unique_id()
        tube.store(d_in, host_in, producer="decode")                 # request payload (host)
        tube.fetch(d_in, device=g, out=out, consumer="producer")      # H2G into the pool output
        nxt = tube.empty((nbytes,), torch.uint8, device=g)           # next request's output buffer
        did = tube.unique_id()
        tube.store(did, out, producer="producer")                    # G2G put (zero copy)
        del out
        view = tube.fetch(did, device=g, consumer="consumer")        # G2G get (same-GPU view)
        fp.launch(view.data_ptr(), nbytes, s)
        del view                                                     # block freed after the digest
        digest = fp.value()                                          # D2H of the result
        if i >= args.warmup:
            e2e.append(time.perf_counter() - t0)
    assert digest == ref_digest, "e2e digest mismatch"
    del nxt
    prod_out = torch.empty_like(x)
    e2e_copy = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        d_in = tube.unique_id()
        tube.store(d_in, host_in, producer="decode")
        tube.fetch(d_in, device=g, out=prod_out.view(-1).view(torch.uint8), consumer="producer")
        did = tube.unique_id()
        tube.store(did, prod_out, producer="producer")               # snapshot copy
        tube.fetch(did, device=g, out=inp, consumer="consumer")      # copy into the input buffer
        fp.launch(inp.data_ptr(), nbytes, s)
        digest = fp.value()
        if i >= args.warmup:
            e2e_copy.append(time.perf_counter() - t0)
    assert digest == ref_digest, "e2e (copy semantics) digest mismatch"

    # ---- aggregate over ranks (max time)
    t_tensor = torch.tensor([total_ms, statistics.mean(e2e)], dtype=torch.float64,
                            device="cpu" if shared else f"cuda:{g}")
    if world > 1:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
    total_ms_max, e2e_max = t_tensor.tolist()
    value = world * args.steps * nbytes / (total_ms_max * 1e-3) / 1e9

    extras = {} if args.no_extras or rank != 0 else run_extras(tube, g, dev, torch, args.max_throughput)

    if rank == 0:
        cpu = cpu_host_path(args.cpu_sample_s, nbytes) if world == 1 else None
        cpu1 = cpu_host_path(min(3.0, args.cpu_sample_s), nbytes, threads=1) if world == 1 else None
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms_max / args.steps, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "config1: 2-function pipeline, producer store(64 MiB fp16) -> consumer "
                                   + ("fetch(into its input buffer), same GPU" if pair is None else
                                      "on the next rank's GPU: pull over NVLink from the exported pool block, "
                                      "device doorbells (pairs.CrossPair)"),
                       "payload_bytes": nbytes, "strategy": "faastube", "l2": "flushed before each pass (256 MiB write + read, outside the timed pass)",
                       "parallelism": f"replicas x{world}" if pair is None else f"ring of {world} producer->consumer pairs",
                       **({"cross_gpu_setup_error": pair_error} if pair_error else {})},
            "p50_pass_ms": round(nearest_rank(per_ms, 50), 5), "p99_pass_ms": round(nearest_rank(per_ms, 99), 5),
            "e2e": {"value": round(world * nbytes / e2e_max / 1e9, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": 16,
                    "path": "store(pinned host payload) -> fetch H2G into a tube.empty output -> store (zero "
                            "copy) -> fetch (same-GPU view) -> digest kernel -> 16 B D2H",
                    "step_ms_p50": round(nearest_rank(sorted(e2e), 50) * 1e3, 4),
                    "step_ms_p99": round(nearest_rank(sorted(e2e), 99) * 1e3, 4),
                    "pcie_gbps_pacer": tube.topo.pcie_gbps,
                    "copy_semantics": {"path": "same, producer's own output buffer and the consumer's input "
                                               "buffer (store snapshot + fetch copy: 2 HBM copies per step)",
                                       "value": round(nbytes / statistics.mean(e2e_copy) / 1e9, 3),
                                       "step_ms_p50": round(nearest_rank(sorted(e2e_copy), 50) * 1e3, 4),
                                       "step_ms_p99": round(nearest_rank(sorted(e2e_copy), 99) * 1e3, 4)}},
            "roofline": {"bound": "hbm", "kernel": "k_copy_bulk (TMA cp.async.bulk ring)",
                         "achieved": round(achieved, 1), "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                         "frac": round(achieved / peaks.get("hbm_gbs", 6650.0), 4), "traffic": profile_traffic(),
                         "algorithmic_bytes_per_launch": 2 * nbytes, "kernel_ms": round(kern_ms, 5),
                         "peak_source": peak_src},
            "gpu_launches": gpu_launches,
            "clocks": dict(clk.summary(), window=f"warm-up + timed region ({timed_wall_s:.3f} s timed)"),
            "variant_pool_output": {"desc": "producer output allocated from the tube pool (zero-copy store): "
                                            "1 copy per pass", "p50_pass_ms": round(nearest_rank(zc_ms, 50), 5),
                                    "value": round(nbytes / (statistics.mean(zc_ms) * 1e-3) / 1e9, 3),
                                    "unit": "GB/s"},
        }
        if cpu:
            line["cpu_baseline"] = {"value": round(cpu["gbps"], 3), "unit": "GB/s", "cores": cpu["threads"],
                                    "kind": "port", "sample": f"{cpu['passes']} store+fetch passes of 64 MiB "
                                                              f"through host memory ({args.cpu_sample_s:.0f} s)",
                                    "p99_pass_ms": round(cpu["pass_ms_p99"], 3),
                                    "single_thread": {"value": round(cpu1["gbps"], 3), "cores": 1,
                                                      "p99_pass_ms": round(cpu1["pass_ms_p99"], 3),
                                                      "sample": f"{cpu1['passes']} passes"}}
        line.update(extras)
        print(json.dumps(line), flush=True)
    if pair is not None:
        pair.close()
    tube.close()
    if world > 1:
        dist.destroy_process_group()


def _single_gpu_topology(g):
    """Under torchrun each rank drives only its own GPU (CUDA_VISIBLE_DEVICES
    is not narrowed), so the tube's topology covers devices 0..g."""
    from paper_2411_01830_b200.topology import build_preset
    return build_preset("b200", n_gpus=g + 1)


def _daemon_client(path, g, q):
    """A function process: Listing 1 through the daemon (daemon.TubeClient)."""
    sys.path.insert(0, ROOT)
    try:
        import torch
        from paper_2411_01830_b200.daemon import TubeClient
        c = TubeClient(path, g)
        res = {}
        for n in (4096, 1 << 20, 64 << 20):
            x = torch.randint(0, 256, (n,), dtype=torch.uint8, device=f"cuda:{g}")
            out = torch.empty_like(x)
            st, ft = [], []
            for i in range(30):
                did = c.unique_id()
                t0 = time.perf_counter()
                c.store(did, x)
                t1 = time.perf_counter()
                c.fetch(did, out=out)
                t2 = time.perf_counter()
                if i >= 5:
                    st.append(t1 - t0)
                    ft.append(t2 - t1)
            assert torch.equal(out, x)
            res[str(n)] = {"store_us_p50": round(1e6 * statistics.median(st), 1),
                           "fetch_us_p50": round(1e6 * statistics.median(ft), 1)}
        c.close()
        q.put(("ok", res))
    except Exception as exc:  # noqa: BLE001
        q.put(("err", repr(exc)))


def run_daemon(tube, g):
    """Function process -> per-box daemon (daemon.py): store + fetch latency of a
    spawned client against a TubeDaemon on this tube (same GPU, bit-checked)."""
    import multiprocessing as mp
    import tempfile
    from paper_2411_01830_b200.daemon import TubeDaemon
    path = os.path.join(tempfile.mkdtemp(), "faastube.sock")
    d = TubeDaemon(tube, path)
    try:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        p = ctx.Process(target=_daemon_client, args=(path, g, q))
        p.start()
        status, res = q.get(timeout=180)
        p.join(timeout=30)
    finally:
        d.close()
    if status != "ok":
        return {"error": res}
    return {"workload": "spawned function process: TubeClient.store then fetch(out=) through the daemon, "
                        "GPU payloads as exported VMM pool blocks (same GPU)", "sizes": res}


def run_extras(tube, g, dev, torch, max_throughput=False):
    out = {}
    # config 2 at k = 1: 1 GiB pinned -> GPU through tube.fetch vs the live CE peak
    n = 1 << 30
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    host.fill_(7)
    dst = torch.empty(n, dtype=torch.uint8, device=f"cuda:{g}")
    s = torch.cuda.current_stream(g)
    ce = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        dev.pcie_copy(dst.data_ptr(), host.data_ptr(), n, True, g, s)
        b.record(s)
        b.synchronize()
        ce.append(a.elapsed_time(b))
    ce_peak = n / (min(ce) * 1e-3) / 1e9
    h2g = []
    for i in range(4):
        did = tube.unique_id()
        tube.store(did, host, producer="decode")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        tube.fetch(did, device=g, out=dst, consumer="preproc")
        b.record(s)
        b.synchronize()
        if i:
            h2g.append(a.elapsed_time(b))
    h2g_gbps = n / (statistics.mean(h2g) * 1e-3) / 1e9
    k = len(tube.topo.roots()) if tube.strategy.parallel_pcie else 1     # PCIe links the plan stripes over
    out["h2g"] = {"workload": f"config2 at k={k} ({k} PCIe link{'s' if k > 1 else ''}"
                              f"{', NVLink forwarding into the target' if k > 1 else ''}): 1 GiB pinned -> "
                              "GPU via FaaSTube.fetch",
                  "links": k, "value": round(h2g_gbps, 3), "unit": "GB/s", "peak": round(k * ce_peak, 3),
                  "peak_source": f"live: best-of-3 cudaMemcpyAsync 1 GiB pinned H2D on the target's link x {k}",
                  "frac": round(h2g_gbps / (k * ce_peak), 4)}
    # config 2 at k=1 across sizes: p50/p99 of one pinned host -> GPU fetch (device events)
    sweep = []
    for sz in (4096, 65536, 1 << 20, 16 << 20, 256 << 20, 1 << 30):
        reps = 60 if sz <= (1 << 20) else (20 if sz <= (256 << 20) else 6)
        ts = []
        for i in range(reps + 2):
            did = tube.unique_id()
            tube.store(did, host[:sz], producer="decode")
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            tube.fetch(did, device=g, out=dst[:sz], consumer="preproc")
            b.record(s)
            b.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        ts.sort()
        p50 = nearest_rank(ts, 50)
        sweep.append({"bytes": sz, "ms_p50": round(p50, 4), "ms_p99": round(nearest_rank(ts, 99), 4),
                      "gbps_p50": round(sz / (p50 * 1e-3) / 1e9, 2), "frac_p50": round(sz / (p50 * 1e-3) / 1e9 / ce_peak, 4)})
    out["h2g_sweep"] = {"workload": "config2 at k=1: pinned host -> GPU via FaaSTube.fetch (managed stage), "
                                    "device-event time per fetch", "peak_gbps": round(ce_peak, 3), "points": sweep}
    # config 2's striping machinery on one GPU: the same 1 GiB split over a direct route and a
    # staged route (CE into the staging chunk ring + forward kernel, here staging GPU == target,
    # so both routes share one PCIe link): the ring/forward pipeline must not cost link rate
    strm = [(torch.cuda.Stream(g), torch.cuda.Stream(g)) for _ in range(2)]
    half = n // 2
    routes = [(g, 0, 0, half, strm[0][0].cuda_stream, strm[0][1].cuda_stream),
              (g, 1, half, n - half, strm[1][0].cuda_stream, strm[1][1].cuda_stream)]
    host[::4093] = torch.arange(host[::4093].numel(), dtype=torch.int64).to(torch.uint8)  # not constant
    dst.zero_()
    st_ms = []
    for i in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        tube.pacer.submit("", False, 1e9, 0.0, 1e9, dst.data_ptr(), g, host.data_ptr(), n, True, routes, s.cuda_stream)
        b.record(s)
        b.synchronize()
        if i:
            st_ms.append(a.elapsed_time(b))
    for o in (0, half - 8192, half, n - 8192):
        assert torch.equal(dst[o:o + 8192].cpu(), host[o:o + 8192]), "striped delivery differs"
    st_gbps = n / (statistics.mean(st_ms) * 1e-3) / 1e9
    out["h2g_striped_machinery"] = {
        "workload": "config2 machinery at k=2 on one GPU: 1 GiB = direct route + staged route (CE -> 4-slot "
                    "chunk ring -> forward kernel), both on the one PCIe link",
        "value": round(st_gbps, 3), "unit": "GB/s", "peak": round(ce_peak, 3), "frac": round(st_gbps / ce_peak, 4)}
    # the NVLink mover (K1, vector engine) on local HBM: it must feed far more than a
    # 900 GB/s/direction link, so cross-GPU passes are link-bound by construction
    vec = []
    for lg in (20, 24, 26, 30):
        m = 1 << lg
        xa = torch.empty(m, dtype=torch.uint8, device=f"cuda:{g}")
        xb = torch.empty_like(xa)
        ts = []
        for i in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            dev.copy(xb.data_ptr(), xa.data_ptr(), m, g, s, dev.ENGINE_VEC)
            b.record(s)
            b.synchronize()
            if i:
                ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        vec.append({"bytes": m, "kernel_ms": round(ms, 5), "payload_gbps": round(m / (ms * 1e-3) / 1e9, 1)})
        del xa, xb
    out["nvlink_mover_local"] = {"kernel": "k_copy_vec (peer-safe 128-bit ld/st, the K1 NVLink engine)",
                                 "note": "local HBM copy on one GPU; NVLink peak 900 GB/s/dir nominal, 770 measured",
                                 "sweep": vec}
    # config 3 at 1 GPU: zero-copy handoff latency and copy-into-input bandwidth, 4 KiB .. 1 GiB.
    # The reference's 1 GB per-GPU store cap (datastore.py:19, sized for 16-32 GB GPUs)
    # would migrate the 1 GiB point to host memory; a B200 store holds it (180 GB HBM).
    cap0, tube.capacity_limit = tube.capacity_limit, 64e9
    sweep = []
    for lg in range(12, 31, 2):
        n = 1 << lg
        xs = torch.empty(n, dtype=torch.uint8, device=f"cuda:{g}").fill_(3)
        ys = torch.empty_like(xs)
        reps = 30 if n <= (64 << 20) else 6
        zc, cp = [], []
        for r in range(reps + 2):
            did = tube.unique_id()
            tube.store(did, xs)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            v = tube.fetch(did, device=g)              # zero-copy view (map only)
            t1 = time.perf_counter()
            del v
            did = tube.unique_id()
            tube.store(did, xs)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            tube.fetch(did, device=g, out=ys)
            b.record(s)
            b.synchronize()
            if r >= 2:
                zc.append((t1 - t0) * 1e3)
                cp.append(a.elapsed_time(b))
        zc.sort()
        cp.sort()
        sweep.append({"bytes": n, "zero_copy_ms_p50": round(nearest_rank(zc, 50), 4),
                      "zero_copy_ms_p99": round(nearest_rank(zc, 99), 4),
                      "copy_ms_p50": round(nearest_rank(cp, 50), 5), "copy_ms_p99": round(nearest_rank(cp, 99), 5),
                      "copy_gbps": round(n / (nearest_rank(cp, 50) * 1e-3) / 1e9, 2)})
    # small handoffs: 64 objects fetched one call each vs one fetch_many (one batched launch)
    batched = []
    for lg in (16, 20, 22):
        m, k = 1 << lg, 64
        xs = torch.empty(k, m, dtype=torch.uint8, device=f"cuda:{g}").fill_(5)
        ys = torch.empty_like(xs)
        row = {"bytes": m, "objects": k}
        for mode in ("one_by_one", "fetch_many"):
            ts = []
            for r in range(4):
                ids = []
                for j in range(k):
                    d = tube.unique_id()
                    tube.store(d, xs[j], producer="p")
                    ids.append(d)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                if mode == "fetch_many":
                    tube.fetch_many([(d, ys[j]) for j, d in enumerate(ids)])
                else:
                    for j, d in enumerate(ids):
                        tube.fetch(d, device=g, out=ys[j])
                b.record(s)
                b.synchronize()
                if r:
                    ts.append(a.elapsed_time(b))
            ms = statistics.median(ts)
            row[mode + "_ms"] = round(ms, 4)
            row[mode + "_gbps"] = round(k * m / (ms * 1e-3) / 1e9, 1)
        assert torch.equal(ys, xs)
        batched.append(row)
        del xs, ys
    tube.capacity_limit = cap0
    out["g2g_same_gpu_batched"] = batched
    out["g2g_same_gpu_sweep"] = sweep
    out["g2g_same_gpu_sweep_store_cap_bytes"] = 64e9
    try:
        out["daemon_put_get"] = run_daemon(tube, g)
    except Exception as exc:  # noqa: BLE001 - extras never hide the headline line
        out["daemon_put_get"] = {"error": repr(exc)}
    try:
        out.update(run_workflows(max_throughput=max_throughput))
    except Exception as exc:  # noqa: BLE001 - extras never hide the headline line
        out["workflows_error"] = repr(exc)
    return out


def run_workflows(dur_s=2.0, max_throughput=False, trial_s=10.0):
    """Configs 4 and 5 on the live runtime (one GPU): the reference's traces,
    placement and SLOs; FaaSTube vs the INFless+ host-memory baseline."""
    from paper_2411_01830_b200 import workload
    from paper_2411_01830_b200.runtime import Runtime
    from paper_2411_01830_b200.tube import FaaSTube

    def one(strategy, jobs_fn, compute):
        tube = FaaSTube(strategy)
        jobs = jobs_fn(tube)
        # a warm daemon: one untimed pass over the first 0.5 s of the same trace
        # (pool blocks, pinned buffers, allocator segments), then the measured run
        Runtime.warm_daemon(tube, jobs, compute, 0.5)
        rt = Runtime(tube, compute=compute)
        t0 = time.perf_counter()
        res = rt.run(jobs, dur_s, drain_s=60)
        res["wall_s"] = round(time.perf_counter() - t0, 3)
        res["pool_timeline_points"] = len(rt.pool_timeline)
        tube.close()
        return res

    def traffic(tube):
        wf = workload.preset_workflow("traffic")
        where = workload.place(wf, tube.topo, {}, colocate=tube.topo.gpu_count < len(wf.gfuncs()))
        workload.calibrate_slo(wf, tube.topo, where, 1.5)
        reqs = workload.build_requests(wf, workload.gen_workload("bursty", 10.0, dur_s, 0), 0)
        return [(wf, where, reqs)]

    def pairs(tube):
        jobs, occ = [], {}
        for i, mb in enumerate((1, 4, 16, 32, 64, 128, 256, 512)):
            wf = workload.Workflow.parse({
                "name": f"pair{mb}", "functions": [
                    {"id": f"prod{mb}", "kind": "gFunc", "compute_latency_ms": 2.0},
                    {"id": f"cons{mb}", "kind": "gFunc", "compute_latency_ms": 2.0}],
                "edges": [{"src": f"prod{mb}", "dst": f"cons{mb}", "size": {"const_mb": mb}}],
                "input_size": {"const_mb": 1}, "response_size": {"const_mb": 1}})
            where = workload.place(wf, tube.topo, occ, limit=2, colocate=tube.topo.gpu_count < 16)
            for k, (kind, g) in where.items():
                if kind == "gpu":
                    occ[g] = occ.get(g, 0) + 1
            workload.calibrate_slo(wf, tube.topo, where, 1.5)
            reqs = workload.build_requests(wf, workload.gen_workload("bursty", 5.0, dur_s, i), i, rid_start=1000 * i)
            jobs.append((wf, where, reqs))
        return jobs

    out = {}
    t4 = {s: one(s, traffic, "model") for s in ("faastube", "infless_plus")}
    out["config4_traffic"] = {"workload": "traffic DAG (decode->preproc->yolo_det->resnet_ped/veh, p=0.6), "
                                          "bursty 10 rps, random-init conv models on synthetic 1080p frames; "
                                          "warm daemon (0.5 s untimed warm-up trace per strategy)",
                              "faastube": t4["faastube"], "infless_plus": t4["infless_plus"]}
    def max_rps(strategy):
        # harness.max_throughput (harness.py:383-428) on the live runtime: highest Poisson
        # rate whose p99 meets the workflow SLO (harness.calibrate_slo: 1.5 x the modelled
        # unloaded runtime, the same for both strategies) with >= 95% completed; the
        # reference compute model (each gFunc occupies its GPU for compute_latency_ms)
        tube = FaaSTube(strategy)
        wf = workload.preset_workflow("traffic")
        where = workload.place(wf, tube.topo, {}, colocate=tube.topo.gpu_count < len(wf.gfuncs()))
        workload.calibrate_slo(wf, tube.topo, where, 1.5)
        t0 = time.perf_counter()
        res = Runtime.max_throughput(tube, wf, where, "sporadic", trial_s, "sleep", rate_lo=1.0, rate_hi=512.0)
        res["wall_s"] = round(time.perf_counter() - t0, 2)
        tube.close()
        return res

    mt = {s: max_rps(s) for s in ("faastube", "infless_plus")} if max_throughput else None
    if mt:
        out["config4_max_throughput"] = {
            "workload": "traffic DAG, Poisson arrivals, reference compute model (compute_latency_ms per gFunc), "
                        "SLO = 1.5 x modelled unloaded runtime (harness.calibrate_slo); binary search as "
                        "harness.max_throughput; each trial after an untimed warm-up at its rate",
            "faastube": mt["faastube"], "infless_plus": mt["infless_plus"],
            "gain": round(mt["faastube"]["max_rps"] / mt["infless_plus"]["max_rps"], 3)
            if mt["infless_plus"]["max_rps"] else None}
    t5 = {s: one(s, pairs, "sleep") for s in ("faastube", "infless_plus")}
    out["config5_multitenant"] = {"workload": "16 functions = 8 producer->consumer pairs, edges 1..512 MB, bursty "
                                              "5 rps each, elastic VMM pool (floor 300 MB)",
                                  "faastube": t5["faastube"], "infless_plus": t5["infless_plus"]}
    return out


def main():
    import faulthandler
    import signal
    faulthandler.register(signal.SIGUSR1, all_threads=True)   # `timeout -s USR1` dumps a hung run
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

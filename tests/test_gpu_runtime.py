"""Live workflow runtime on one B200: the reference's
trace, placement and SLOs replayed with real data passing; FaaSTube vs the
host-oriented INFless+ baseline on the same trace."""

import pytest

pytestmark = pytest.mark.gpu


def _run(strategy, preset="yelp", rate=20.0, dur=1.0, compute="sleep", seed=0):
    from paper_2411_01830_b200 import workload
    from paper_2411_01830_b200.runtime import Runtime
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube(strategy)
    wf = workload.preset_workflow(preset)
    where = workload.place(wf, tube.topo, {}, colocate=tube.topo.gpu_count < len(wf.gfuncs()))
    workload.calibrate_slo(wf, tube.topo, where, 1.5)
    reqs = workload.build_requests(wf, workload.gen_workload("sporadic", rate, dur, seed), seed)
    Runtime.warm_daemon(tube, [(wf, where, reqs)], compute, 0.5)
    rt = Runtime(tube, compute=compute)
    out = rt.run([(wf, where, reqs)], dur, drain_s=60)
    tube.close()
    return out, len(reqs)


def test_yelp_runs_and_beats_host_oriented():
    ft, n = _run("faastube")
    base, _ = _run("infless_plus")
    assert ft["errors"] == [] and base["errors"] == []
    assert ft["requests_completed"] == n and base["requests_completed"] == n
    keys = ("p50_ms", "p99_ms", "phase_p99_ms")
    assert ft["p50_ms"] < base["p50_ms"], ({k: ft[k] for k in keys}, {k: base[k] for k in keys})


def test_traffic_with_models():
    out, n = _run("faastube", preset="traffic", rate=5.0, dur=1.0, compute="model")
    assert out["errors"] == [] and out["requests_completed"] == n, out


def test_max_throughput_search_live():
    """harness.max_throughput (harness.py:383-428) on the live runtime: doubling
    then bisection; the answer is a rate whose trial met the SLO."""
    from paper_2411_01830_b200 import workload
    from paper_2411_01830_b200.runtime import Runtime
    from paper_2411_01830_b200.tube import FaaSTube
    tube = FaaSTube("faastube")
    wf = workload.preset_workflow("yelp")
    where = workload.place(wf, tube.topo, {}, colocate=tube.topo.gpu_count < len(wf.gfuncs()))
    workload.calibrate_slo(wf, tube.topo, where, 1.5)
    res = Runtime.max_throughput(tube, wf, where, "sporadic", 1.0, "sleep", rate_lo=1.0, rate_hi=8.0,
                                 iterations=1, slo_ms=10_000.0)
    tube.close()
    assert res["max_rps"] >= 1.0, res
    ok_rates = [t["rate"] for t in res["trials"] if t["ok"]]
    assert res["max_rps"] in ok_rates and all(t["ok"] == (t["p99_ms"] is None or t["p99_ms"] <= 10_000.0)
                                              or t["completed"] < 0.95 * t["offered"] for t in res["trials"])

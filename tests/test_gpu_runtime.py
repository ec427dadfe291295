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

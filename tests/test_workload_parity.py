"""The live runtime's inputs replay the reference exactly: arrival traces
(harness.py:45-88), per-request draws (harness.py:130-149), placement
(workflow.py:375-438) and SLO calibration (harness.py:154-208), against
tests/golden/harness.json recorded from the reference."""

import golden_replay as G


def test_traces():
    from paper_2411_01830_b200 import workload
    for c in G.load("harness")["traces"]:
        got = workload.gen_workload(c["pattern"], c["rate"], c["duration"], c["seed"])
        assert got == c["times"], (c["pattern"], c["rate"], c["duration"], c["seed"])


def test_requests():
    from paper_2411_01830_b200 import workload
    for case in G.load("harness")["requests"]:
        wf = workload.preset_workflow(case["workflow"])
        arr = workload.gen_workload("bursty", 20.0, 2.0, 3)
        reqs = workload.build_requests(wf, arr, 3, rid_start=100)
        assert len(reqs) == len(case["requests"])
        for r, e in zip(reqs, case["requests"]):
            assert r.rid == e["rid"] and r.arrival_ms == e["arrival"]
            assert sorted(map(list, r.fired)) == e["fired"]
            assert sorted([[a, b, v] for (a, b), v in r.edge_bytes.items()]) == e["edge_bytes"]
            assert r.input_bytes == e["input"] and r.response_bytes == e["response"]


def test_placement_and_slo_calibration():
    from paper_2411_01830_b200 import topology, workload
    docs = {c["name"]: c["doc"] for c in G.load("topology")["cases"]}
    for c in G.load("harness")["calibration"]:
        t = topology.from_dict(docs[c["topology"]])
        wf = workload.preset_workflow(c["workflow"])
        try:
            where = workload.place(wf, t, {}, c["limit"])
        except RuntimeError:
            assert c.get("error") == "PlacementError", c
            continue
        assert "error" not in c, c
        assert {k: list(v) for k, v in where.items()} == c["placement"], c["workflow"]
        rt = workload.calibrate_slo(wf, t, where, 1.5)
        assert rt == c["runtime"] and wf.slo_ms == c["slo"], (c["topology"], c["workflow"], rt, c["runtime"])
        assert {f.id: [f.slo_ms, f.infer_ms] for f in wf.funcs} == c["funcs"]

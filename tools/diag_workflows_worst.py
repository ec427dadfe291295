"""Configs 4-5 as the bench runs them; prints each strategy's worst request."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
out = bench.run_workflows()
for k in ("config4_traffic", "config5_multitenant"):
    for s in ("faastube", "infless_plus"):
        v = out[k][s]
        print(k, s, "p50", v.get("p50_ms"), "p99", v.get("p99_ms"), json.dumps(v.get("worst")))

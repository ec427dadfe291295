"""Config 4/5 tails on the live runtime, one strategy and seed at a time, with
the tube's diagnostics (slow stores: alloc / locked / migration ms; growth)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

seeds = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1").split(","))
out = bench.run_workflows(dur4_s=20.0, dur5_s=10.0, seeds=seeds)
for cfg in ("config4_traffic", "config5_multitenant"):
    for s in ("faastube", "infless_plus"):
        c = out[cfg][s]
        print(cfg, s, {k: c.get(k) for k in ("requests", "p50_ms", "p99_ms", "slo_violation_rate", "p99_ms_per_seed")})
        for r in c["runs"]:
            print("   worst", json.dumps(r.get("worst")))
            print("   tube", json.dumps(r.get("tube")))

"""Configs 4-5 as the bench runs them; prints each strategy's worst request."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2411_01830_b200.tube as T
_orig_close = T.FaaSTube.close
def _close(self):
    print("slow stores", self.strategy.name if hasattr(self.strategy, "name") else "", list(self.slow_stores)[:12])
    _orig_close(self)
T.FaaSTube.close = _close
out = bench.run_workflows()
for k in ("config4_traffic", "config5_multitenant"):
    for s in ("faastube", "infless_plus"):
        v = out[k][s]
        print(k, s, "p50", v.get("p50_ms"), "p99", v.get("p99_ms"), json.dumps(v.get("worst")))

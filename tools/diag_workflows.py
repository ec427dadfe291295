"""Configs 4/5 on the live runtime with per-request phases and pacer stats."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2411_01830_b200 import tube as tube_mod
orig = tube_mod.FaaSTube.close
def close(self):
    print("  pcie_gbps", self.topo.pcie_gbps, "pacer", self.pacer.stats(), "stats", self.stats, flush=True)
    if os.environ.get("FT_TRACE"):
        log = self.pacer.log()
        print("  log calls", len(log), "guards", sum(1 for x in self.pacer.trace() if x[2] == "guard"))
        st = {}
        for t, tk, kind, v in self.pacer.trace():
            if kind in ("start", "land"):
                st.setdefault(tk, {})[kind] = t
        durs = sorted((v["land"] - v["start"], tk) for tk, v in st.items() if "land" in v)
        print("  slowest stages ms", [(round(d, 2), tk) for d, tk in durs[-8:]])
    return orig(self)
tube_mod.FaaSTube.close = close
out = bench.run_workflows()
for c in ("config4_traffic", "config5_multitenant"):
    for s in ("faastube", "infless_plus"):
        x = out[c][s]
        print(c, s, json.dumps({k: x[k] for k in ("p50_ms", "p99_ms", "slo_violation_rate", "phase_p99_ms", "wall_s")}))

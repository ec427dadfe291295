import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
t0 = time.time()
out = bench.run_workflows(max_throughput=True, trial_s=float(sys.argv[1]) if len(sys.argv) > 1 else 10.0)
print(json.dumps(out["config4_max_throughput"]))
print("wall", time.time() - t0)

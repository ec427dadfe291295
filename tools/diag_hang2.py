"""Run bench.run_ours with a watchdog that dumps pacer state of every live tube."""
import os, sys, threading, time, json, faulthandler, gc
os.environ["FT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2411_01830_b200.tube import FaaSTube

def watchdog(limit):
    time.sleep(limit)
    print("WATCHDOG", flush=True)
    tubes = [o for o in gc.get_objects() if isinstance(o, FaaSTube)]
    for tube in tubes:
        res = {}
        def grab():
            res["stats"] = tube.pacer.stats()
            res["state"] = tube.pacer.state()
            res["trace"] = tube.pacer.trace()[-30:]
            res["log"] = tube.pacer.log()[-12:]
        t = threading.Thread(target=grab, daemon=True); t.start(); t.join(5)
        print(json.dumps(res, default=str)[:12000] if res else "pacer calls hung (mu held)", flush=True)
    faulthandler.dump_traceback(all_threads=True)
    os._exit(3)

threading.Thread(target=watchdog, args=(float(sys.argv[1]),), daemon=True).start()
sys.argv = ["bench.py", "--cpu-sample-s", "1"]
bench.main()
os._exit(0)

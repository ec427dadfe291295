"""The isolation scenario of tests/test_gpu_sched.py repeated: the tight tenant's
completion time under the managed pacer and under native sharing, per run.
python tools/probe_isolation.py [runs]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_sched import _contend  # noqa: E402

from paper_2411_01830_b200.tube import measure_pcie_gbps  # noqa: E402

link = measure_pcie_gbps([0])
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    m, w = _contend("faastube", link)
    print(f"link {link:.1f} window {w:.1f} managed T {m['T']:.1f} loose {max(v for k, v in m.items() if k != 'T'):.1f}",
          flush=True)

"""measure_pcie_gbps at process start, repeated; then with a 100 ms warm-up burst."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01830_b200.tube import measure_pcie_gbps
from paper_2411_01830_b200 import device as dev
t0 = time.perf_counter()
print("first", measure_pcie_gbps([0]), "in", round(time.perf_counter() - t0, 3), "s", flush=True)
for i in range(4):
    print("again", measure_pcie_gbps([0]), flush=True)
time.sleep(2.0)
print("after 2 s idle", measure_pcie_gbps([0]), flush=True)

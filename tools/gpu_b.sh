mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu --timeout 120 > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log
timeout -k 10 1200 python tools/diag_maxrps.py 10 > gpurun_out/diag_maxrps10.txt 2>&1

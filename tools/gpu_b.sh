mkdir -p gpurun_out
timeout -k 10 400 python tools/diag_cfg5.py > gpurun_out/diag_cfg5.txt 2>&1
timeout -k 10 400 python tools/diag_cfg5.py > gpurun_out/diag_cfg5b.txt 2>&1

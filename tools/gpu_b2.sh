for i in 1 2 3; do timeout -k 10 200 python tools/diag_slow1.py trial > gpurun_out/diag_slow1_$i.txt 2>&1; done

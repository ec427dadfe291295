timeout -k 10 300 python tools/diag_cfg5.py c4 > gpurun_out/diag_c4_spares.txt 2>&1
FT_SPARE_CAP_BYTES=0 timeout -k 10 300 python tools/diag_cfg5.py c4 > gpurun_out/diag_c4_nospares.txt 2>&1

mkdir -p gpurun_out
FT_TRACE=1 timeout 120 python tools/diag_e2e.py > gpurun_out/diag_e2e_d.txt 2>&1
timeout -s USR1 -k 30 400 python bench.py --no-extras > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; echo "bench rc=$?" >> gpurun_out/bench_d.err

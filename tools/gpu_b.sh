mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pacer.py tests/test_gpu_sched.py -q -m gpu --timeout 120 > gpurun_out/pytest_c.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c.log
timeout -s USR1 -k 30 400 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "bench rc=$?" >> gpurun_out/bench_c.err

mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_movers.py tests/test_gpu_tube.py -q -m gpu --timeout 120 > gpurun_out/pytest_n.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_n.log
timeout -s USR1 -k 30 600 python bench.py --cpu-sample-s 2 > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err

mkdir -p gpurun_out
timeout -s USR1 -k 30 600 python bench.py --cpu-sample-s 2 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 600 python -m pytest tests -q -m gpu --timeout 120 > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log

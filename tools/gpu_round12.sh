#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sched.py tests/test_gpu_runtime.py -q -m gpu > gpurun_out/pytest_gpu12.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu12.log
timeout 600 python -c "import bench, json; print(json.dumps(bench.run_workflows()))" > gpurun_out/workflows12.json 2> gpurun_out/workflows12.err
FT_TRACE=1 timeout 600 python tools/diag_traffic.py > gpurun_out/diag_traffic12.txt 2>&1
ls gpurun_out

#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python tools/sweep_copy.py > gpurun_out/sweep_copy3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sched.py tests/test_gpu_movers.py -x -q -m gpu > gpurun_out/pytest_gpu3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu3.log
ls gpurun_out

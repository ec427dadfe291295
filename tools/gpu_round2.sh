#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sched.py tests/test_gpu_tube.py -x -q -m gpu > gpurun_out/pytest_gpu2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 900 python tools/sweep_copy.py > gpurun_out/sweep_copy.log 2>&1
timeout 600 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err
ls gpurun_out

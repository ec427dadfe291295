#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_migration.py -x -q -m gpu > gpurun_out/pytest_gpu5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu5.log
timeout 600 python -c "import bench, json; print(json.dumps(bench.run_workflows()))" > gpurun_out/workflows5.json 2> gpurun_out/workflows5.err
ls gpurun_out

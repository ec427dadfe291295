#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu6.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu6.log
timeout 600 python -c "import bench, json; print(json.dumps(bench.run_workflows()))" > gpurun_out/workflows6.json 2> gpurun_out/workflows6.err
ls gpurun_out

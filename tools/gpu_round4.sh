#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 900 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "rc=$?" >> gpurun_out/bench4.err
ls gpurun_out

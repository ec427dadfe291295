#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu7.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu7.log
timeout 300 python tools/prof_api.py > gpurun_out/prof_api7.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "rc=$?" >> gpurun_out/bench7.err
ls gpurun_out

#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu9.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu9.log
timeout 300 python tools/prof_api.py > gpurun_out/prof_api9.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo "rc=$?" >> gpurun_out/bench9.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches9.csv python bench.py --steps 3 --warmup 3 --no-extras --cpu-sample-s 1 > gpurun_out/ncu_bench9.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_bulk -s 2 -c 2 -o gpurun_out/prof_copy9 python tools/prof_copy.py > gpurun_out/ncu_copy9.log 2>&1
ls gpurun_out

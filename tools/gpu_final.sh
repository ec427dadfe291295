#!/bin/bash
# Measurement session: sanitizer runs, full bench (both arms), ncu over the bench.
#   TAG=<name> bash tools/gpu_final.sh
set -x
mkdir -p gpurun_out/sanitizer_$TAG
T=${TAG:-final}
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool python tools/sanitize_kernels.py > gpurun_out/sanitizer_$T/sanitize_$tool.txt 2>&1
done
timeout -s USR1 -k 30 1800 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?" >> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo "ref rc=$?" >> gpurun_out/bench_ref_$T.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 3 --warmup 3 --no-extras --no-ncu --cpu-sample-s 1 > gpurun_out/ncu_bench_$T.log 2>&1
ls -la gpurun_out

#!/bin/bash
# Round-2 measurement session: tests, smoke, kernel ncu captures, bench launch list,
# full bench (both arms).   TAG=<name> bash tools/gpu_r02.sh
set -x
mkdir -p gpurun_out
T=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_copy_vec|k_copy_multi|k_forward|k_copy_bulk" -c 40 -o gpurun_out/prof_kernels_$T python tools/prof_kernels.py > gpurun_out/ncu_kernels_$T.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 3 --warmup 3 --no-extras --no-ncu --cpu-sample-s 1 > gpurun_out/ncu_bench_$T.log 2>&1
timeout -s USR1 -k 30 1800 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?" >> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo "ref rc=$?" >> gpurun_out/bench_ref_$T.err
ls -la gpurun_out

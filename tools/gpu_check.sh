#!/bin/bash
# One GPU session: full gpu tests, smoke, default bench (both arms).
set -x
mkdir -p gpurun_out
T=${TAG:-chk}
nvidia-smi topo -m > gpurun_out/topo_$T.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?" >> gpurun_out/bench_$T.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
ls -la gpurun_out

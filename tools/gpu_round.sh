#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), the N=2 path on one GPU,
# the ncu launch list of the bench and one full capture of the copy kernel.
#   TAG=<name> STAGES="tests smoke bench ref n2 ncu" bash tools/gpu_round.sh
set -x
mkdir -p gpurun_out
T=${TAG:-r}
S=${STAGES:-"tests smoke bench ref n2 ncu"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current --format=csv > gpurun_out/gpu_$T.txt 2>&1
has() { [[ " $S " == *" $1 "* ]]; }
if has tests; then timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log; fi
if has smoke; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log; fi
if has bench; then timeout -s USR1 -k 30 1500 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?" >> gpurun_out/bench_$T.err; fi
if has ref; then timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo "ref rc=$?" >> gpurun_out/bench_ref_$T.err; fi
if has n2; then timeout -k 10 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 50 --warmup 5 --no-extras > gpurun_out/bench_n2_$T.json 2> gpurun_out/bench_n2_$T.err; echo "n2 rc=$?" >> gpurun_out/bench_n2_$T.err; fi
if has ncu; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 3 --warmup 3 --no-extras --no-ncu --cpu-sample-s 1 > gpurun_out/ncu_bench_$T.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy_bulk -s 2 -c 2 -o gpurun_out/prof_copy_$T python tools/prof_copy.py > gpurun_out/ncu_copy_$T.log 2>&1
fi
ls -la gpurun_out

mkdir -p gpurun_out
timeout 200 python tools/prof_ffi.py > gpurun_out/prof_ffi.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu --timeout 120 -x > gpurun_out/pytest_m.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_m.log

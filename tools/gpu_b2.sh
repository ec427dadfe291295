mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/sanitize_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/sanitize_racecheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_kernels.py > gpurun_out/sanitize_synccheck.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitize_synccheck.txt

# correctness (virtual + multi-process) then traced N=4 bench of nvls/auto and the size table
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/gpu_tests.txt 2>&1; tail -3 gpurun_out/gpu_tests.txt
./tools/runs/trace_nvls.sh 2>&1 | grep -v Broken
./tools/runs/run_nvls_sizes.sh 2>&1 | grep "^N"

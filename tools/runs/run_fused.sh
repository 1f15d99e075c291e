timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "fused" > gpurun_out/fused_tests.txt 2>&1; tail -30 gpurun_out/fused_tests.txt

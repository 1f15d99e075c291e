timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x --timeout 600 -k "bn or batch_norm" > gpurun_out/bn_tests.txt 2>&1; tail -2 gpurun_out/bn_tests.txt
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 -k "bn or graph" > gpurun_out/bn_tests_mp.txt 2>&1; tail -2 gpurun_out/bn_tests_mp.txt
for dt in f32 bf16; do timeout 300 python tools/bench_bn.py --dtype $dt 2>&1 | grep -v "^{" ; done

timeout 900 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_multiproc.py -q -x --timeout 600 -k "bn or batch_norm or graph" > gpurun_out/bn_tests.txt 2>&1; tail -2 gpurun_out/bn_tests.txt
timeout 300 python tools/bench_bn.py --dtype f32 2>&1 | grep -v "^{" > gpurun_out/bn_f32.txt; cat gpurun_out/bn_f32.txt
timeout 300 python tools/bench_bn.py --dtype bf16 2>&1 | grep -v "^{" > gpurun_out/bn_bf16.txt; cat gpurun_out/bn_bf16.txt
timeout 600 python tools/train_sngan.py 2>/dev/null | tail -1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 tools/train_sngan.py 2>/dev/null | tail -1

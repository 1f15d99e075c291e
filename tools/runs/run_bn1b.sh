# 2 GPUs: BN with one barrier per call (double-buffered records): tests, bench N=1/N=2 (aligned ranks), SN-GAN N=2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x --timeout 600 > gpurun_out/b1_vtests.txt 2>&1; tail -1 gpurun_out/b1_vtests.txt
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 -k "bn or graph or fused or wrap" > gpurun_out/b1_tests.txt 2>&1; tail -1 gpurun_out/b1_tests.txt
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/bench_bn.py --dtype f32 2>&1 | grep bn_ > gpurun_out/b1_bn_n1.txt; cat gpurun_out/b1_bn_n1.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 tools/bench_bn.py --dtype f32 2>&1 | grep bn_ > gpurun_out/b1_bn_n2.txt; cat gpurun_out/b1_bn_n2.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 tools/train_sngan.py 2>/dev/null | tail -1

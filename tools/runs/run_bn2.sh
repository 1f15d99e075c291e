# 2 GPUs: full GPU test suite (multi-process at world 2), BN latency after the hierarchical exchange barrier
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/b2_tests.txt 2>&1; tail -3 gpurun_out/b2_tests.txt
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/bench_bn.py --dtype f32 > gpurun_out/bn2_f32_n1.txt 2>&1; head -12 gpurun_out/bn2_f32_n1.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 tools/bench_bn.py --dtype f32 > gpurun_out/bn2_f32_n2.txt 2>&1; grep bn_ gpurun_out/bn2_f32_n2.txt | head -21
RP_BN_UNFUSED=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 tools/bench_bn.py --dtype f32 --only 1024x4 2>&1 | grep bn_ | sed "s/^/unfused /"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 tools/train_sngan.py 2>/dev/null | tail -1

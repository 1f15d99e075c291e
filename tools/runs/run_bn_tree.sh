# 2 GPUs: BN split fold as a shuffle tree -- parity tests, bench N=1, SN-GAN N=2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_virtual.py -q -x --timeout 600 -k "bn or batch_norm or smoke" > gpurun_out/bt_vtests.txt 2>&1; tail -1 gpurun_out/bt_vtests.txt
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 -k "bn or graph" > gpurun_out/bt_tests.txt 2>&1; tail -1 gpurun_out/bt_tests.txt
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/bench_bn.py --dtype f32 2>&1 | grep bn_stats
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 tools/train_sngan.py 2>/dev/null | tail -1 | cut -c1-200

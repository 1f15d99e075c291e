# 8-GPU check: NVLS probe + bench (auto -> nvls) + bench P2P only + GPU multiproc tests
nvidia-smi -L | head -8
timeout 120 ./tools/nvls_probe 64 2>&1 | head -12
timeout 120 ./tools/barrier_probe 2>&1 | grep "world 8"
for nv in auto off; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 8 --steps 50 --warmup 5 --nvls $nv > gpurun_out/bench_n8_$nv.json 2> gpurun_out/bench_n8_$nv.err
python -c "import json; d=json.loads(open('gpurun_out/bench_n8_$nv.json').read().strip().splitlines()[-1]); print('N8', d['config']['algo'], round(d['ms_per_step']*1e3,1), 'us per_gpu_bus', round(d['per_gpu_busbw_gbs'],1), 'link/dir', round(d['roofline']['link_gbs_per_direction'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'])" || tail -5 gpurun_out/bench_n8_$nv.err
done
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 > gpurun_out/gpu_tests_mp8.txt 2>&1; tail -3 gpurun_out/gpu_tests_mp8.txt

timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 > gpurun_out/gpu_tests_mp.txt 2>&1; tail -3 gpurun_out/gpu_tests_mp.txt
for n in 4 2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $n --steps 50 --warmup 5 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err
python -c "import json; d=json.loads(open('gpurun_out/bench_n$n.json').read().strip().splitlines()[-1]); print('N$n', d['config']['algo'], round(d['ms_per_step']*1e3,1), 'us per_gpu_bus', round(d['per_gpu_busbw_gbs'],1), 'link/dir', round(d['roofline']['link_gbs_per_direction'],1), 'e2e', round(d['e2e']['value'],1), d['clocks'])" || tail -5 gpurun_out/bench_n$n.err
done

timeout 600 python -m pytest tests/test_gpu_virtual.py tests/test_gpu_multiproc.py -q -x --timeout 400 > gpurun_out/tests_n2.txt 2>&1; tail -3 gpurun_out/tests_n2.txt
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b_n1.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/b_n1.json').read().strip().splitlines()[-1]); print('N1', round(d['ms_per_step'],4), round(d['value'],1), round(d['roofline']['frac'],3), d['step_ms_min'])"
for impl in pull push; do for b in 67108864 268435456; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --ar-impl $impl --bytes $b --e2e-steps 2 --no-cpu-baseline > gpurun_out/ab_${impl}_${b}.json 2> /dev/null
python -c "import json,sys; d=json.loads(open('gpurun_out/ab_${impl}_${b}.json').read().strip().splitlines()[-1]); print('$impl', $b, round(d['ms_per_step'],4), round(d['per_gpu_busbw_gbs'],1), round(d['step_ms_min'],4), 'e2e', round(d['e2e']['value']/2,1))"
done; done
for impl in pull push; do
rm -f gpurun_out/tr_${impl}.jsonl*
RP_TRACE=gpurun_out/tr_${impl}.jsonl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 --ar-impl $impl --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/tr_${impl}.jsonl 16000000
done

for impl in pull push; do for b in 67108864 268435456; do
rm -f gpurun_out/tr_${impl}_${b}.jsonl*
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --ar-impl $impl --bytes $b --e2e-steps 2 --no-cpu-baseline > gpurun_out/ab_${impl}_${b}.json 2> /dev/null
python -c "import json,sys; d=json.loads(open('gpurun_out/ab_${impl}_${b}.json').read().strip().splitlines()[-1]); print('$impl', $b, round(d['ms_per_step'],4), round(d['per_gpu_busbw_gbs'],1), round(d['step_ms_min'],4), 'e2e', round(d['e2e']['value']/2,1))"
done; done
RP_TRACE=gpurun_out/tr_push.jsonl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 --ar-impl push --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
python tools/trace_summary.py gpurun_out/tr_push.jsonl 16000000
timeout 300 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 250 > gpurun_out/mp_tests.txt 2>&1; tail -3 gpurun_out/mp_tests.txt

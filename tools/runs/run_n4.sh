timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 > gpurun_out/tests_n4.txt 2>&1; tail -3 gpurun_out/tests_n4.txt
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 5 --e2e-steps 2 > gpurun_out/b_n$n.json 2> gpurun_out/b_n$n.err
python -c "import json; d=json.loads(open('gpurun_out/b_n$n.json').read().strip().splitlines()[-1]); print('N$n', round(d['ms_per_step'],4), 'value', round(d['value'],1), 'per_gpu', round(d['per_gpu_busbw_gbs'],1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'])"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py --out gpurun_out/sweep_n4.json --max-log2 30 --iters 10 > gpurun_out/sweep_n4.txt 2>&1; echo sweep_rc=$?
grep -E "auto" gpurun_out/sweep_n4.txt | awk '{printf "%s %s %s %s\n",$1,$3,$5,$8}'
